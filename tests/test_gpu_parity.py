"""GPU parity: the sm_100a path through the C-ABI against the CPU oracle.

Bars: kNN edge set, order and squared distances bit-exact;
weights within 1 ulp; B / Bᵀ / labels bit-exact; objectives and AL pieces at
rounding level; solver iterates within 1e-6 relative Frobenius of the oracle
and labels identical.  Reference test cases are cited per test.
"""
import numpy as np
import pytest

pytestmark = pytest.mark.gpu

ULP = 2.3e-16


def mixture(orc, n_per, d, m=4, seed=42, spread=None, cseed=1001):
    rng_c = orc.normals(cseed, m * d).reshape(m, d)
    centers = (3.0 / np.sqrt(d)) * rng_c
    return orc.gaussian_mixture(centers, spread if spread is not None else 1.0 / np.sqrt(d), n_per, seed)


def circle(orc, n_per, m=10, seed=42):
    ang = 2 * np.pi * np.arange(m) / m
    centers = np.stack([4 * np.cos(ang), 4 * np.sin(ang)], axis=1)
    return orc.gaussian_mixture(centers, 0.5, n_per, seed)


def check_graph(cp, orc, A, k, phi):
    g = cp.compute_knn_weights(cp.DataMatrix(A), k, phi)
    og = orc.knn_weights(A, k, phi)
    gi, gj, gw, gd2 = g.arrays()
    oi, oj, ow, od2 = og.arrays()
    assert np.array_equal(gi, oi) and np.array_equal(gj, oj)
    assert np.array_equal(gd2, od2)
    if len(ow):
        assert np.max(np.abs(gw - ow) / ow) <= 2 * ULP
    return g, og


# ---- kNN (graph.cpp:75-114; test_graph.cpp:91-138) ------------------------------

@pytest.mark.parametrize("n_per,d,k", [(25, 2, 10), (40, 3, 5), (30, 5, 7), (30, 7, 4), (20, 1, 3), (30, 64, 10),
                                       (40, 784, 10), (25, 97, 15), (10, 4, 1)])
def test_knn_bit_exact(cp, orc, n_per, d, k):
    A = mixture(orc, n_per, d)
    check_graph(cp, orc, A, k, 0.5)


def test_knn_c1_shape(cp, orc):
    check_graph(cp, orc, circle(orc, 100), 10, 0.5)


def test_knn_large_k_fallback(cp, orc):
    check_graph(cp, orc, mixture(orc, 30, 6), 40, 0.5)


def test_knn_kats(cp, orc):
    line = np.array([[0.0], [1.0], [3.0]])
    g = cp.compute_knn_weights(cp.DataMatrix(line), 1, 0.0)
    assert g.edges() == [(0, 1, 1.0), (1, 2, 1.0)]
    g = cp.compute_knn_weights(cp.DataMatrix(line), 1, 0.5)
    assert g.weights()[0] == pytest.approx(0.6065306597126334, rel=1e-14)
    assert g.weights()[1] == pytest.approx(0.1353352832366127, rel=1e-14)
    ties = np.array([[0.0, 0.0], [5.0, 0.0], [-5.0, 0.0], [5.1, 0.0], [-5.1, 0.0]])
    g = cp.compute_knn_weights(cp.DataMatrix(ties), 1, 0.0)
    assert g.find_edge(0, 1) is not None and g.find_edge(0, 2) is None and g.edge_count() == 3
    for k in (0, 3):
        with pytest.raises(ValueError):
            cp.compute_knn_weights(cp.DataMatrix(line), k, 0.5)
    assert cp.compute_knn_weights(cp.DataMatrix(line), 2, 0.5).edge_count() == 3
    assert cp.compute_knn_weights(cp.DataMatrix(line[:2]), 1, 1e10).edge_count() == 0
    with pytest.raises(ValueError):
        cp.compute_knn_weights(cp.DataMatrix(line), 1, -1.0)


def test_knn_duplicates_and_ties(cp, orc):
    rng = np.random.default_rng(0)
    A = np.round(rng.standard_normal((120, 3)), 1)  # many exact ties and duplicate points
    A[10] = A[11] = A[12]
    check_graph(cp, orc, A, 6, 0.5)


# ---- tensor-core kNN candidates + exact re-check (knn_tc.cu) ----------------------

def _knn_arrays(cp, A, k, tc):
    import os
    old = os.environ.get("CPB_KNN_TC")
    os.environ["CPB_KNN_TC"] = "1" if tc else "0"
    try:
        g = cp.compute_knn_weights(cp.DataMatrix(A), k, 0.5)
        info = cp.default_context().knn_info()
    finally:
        if old is None:
            del os.environ["CPB_KNN_TC"]
        else:
            os.environ["CPB_KNN_TC"] = old
    return g.arrays(), info


@pytest.mark.parametrize("n_per,d,k", [(512, 64, 10), (530, 17, 7), (520, 784, 10), (700, 33, 15)])
def test_knn_tensor_core_matches_oracle(cp, orc, n_per, d, k):
    """3xTF32 tcgen05 candidates + FP64 Eigen-order re-check == the oracle, bitwise."""
    A = mixture(orc, n_per, d)
    (gi, gj, gw, gd2), info = _knn_arrays(cp, A, k, True)
    assert info["tensor_cores"] == 1 and 0.0 <= info["worst_ratio"] < 1.0
    oi, oj, ow, od2 = orc.knn_weights(A, k, 0.5).arrays()
    assert np.array_equal(gi, oi) and np.array_equal(gj, oj) and np.array_equal(gd2, od2)
    assert np.max(np.abs(gw - ow) / ow) <= 2 * ULP


@pytest.mark.parametrize("n,d,k", [(10000, 784, 10), (4099, 128, 24)])
def test_knn_tensor_core_matches_exact_kernel(cp, orc, n, d, k):
    """At C2 size the oracle is slow; the exact FP64 tile kernel (itself pinned
    to the oracle above) is the reference."""
    A = mixture(orc, n // 10, d, m=10)
    (ti, tj, tw, td2), info = _knn_arrays(cp, A, k, True)
    (ei, ej, ew, ed2), info0 = _knn_arrays(cp, A, k, False)
    assert info["tensor_cores"] == 1 and info0["tensor_cores"] == 0
    assert info["worst_ratio"] < 1.0 and info["exact_rows"] == 0
    assert np.array_equal(ti, ei) and np.array_equal(tj, ej) and np.array_equal(td2, ed2)
    assert np.array_equal(tw, ew)


def test_knn_tensor_core_overflow_rows(cp, orc):
    """Groups of 40 identical points: a row whose 39 duplicates share one column
    segment has a full list inside its band, so the threshold pass collects
    its whole band (groups split across segments are settled by the first
    re-check)."""
    base = mixture(orc, 60, 48, m=40)
    A = np.repeat(base[:60], 40, axis=0)  # 2400 rows, 60 groups of 40 duplicates
    A = np.concatenate([A, base[60:]], axis=0)
    (ti, tj, tw, td2), info = _knn_arrays(cp, A, 10, True)
    assert info["tensor_cores"] == 1 and info["band_rows"] >= 1000 and info["exact_rows"] == 0
    oi, oj, ow, od2 = orc.knn_weights(A, 10, 0.5).arrays()
    assert np.array_equal(ti, oi) and np.array_equal(tj, oj) and np.array_equal(td2, od2)


@pytest.mark.parametrize("n_per,d,k,tc", [(1000, 64, 10, True), (60, 5, 4, False), (700, 33, 40, False)])
def test_knn_rows_sharded_bitwise(cp, orc, n_per, d, k, tc):
    """Row blocks computed separately (as the ranks of the sharded kNN do) and
    assembled give the single-call graph bit for bit."""
    import torch
    A = mixture(orc, n_per, d)
    n = len(A)
    data = cp.DataMatrix(A)
    g1 = cp.compute_knn_weights(data, k, 0.5)
    assert cp.default_context().knn_info()["tensor_cores"] == int(tc)
    kd = torch.zeros((n, k), dtype=torch.float64, device="cuda")
    kj = torch.zeros((n, k), dtype=torch.int32, device="cuda")
    for r in range(3):
        r0, r1 = cp.shard_rows(n, 3, r)
        cp.knn_rows_into(data, k, r0, r1, kd, kj)
    od, oj = orc.knn_rows(A, k, 0, min(n, 64))
    assert np.array_equal(kd[:64].cpu().numpy(), od) and np.array_equal(kj[:64].cpu().numpy(), oj)
    g2 = cp.compute_knn_weights_sharded(data, k, 0.5)  # world 1: one block, same assembly path
    for g in (g2,):
        for a, b in zip(g.arrays(), g1.arrays()):
            assert np.array_equal(a, b)
    bad = kj.clone()
    bad[5, 0] = 5  # self loop
    import ctypes as C
    from paper_2501_15964_b200 import _lib as L
    h = C.c_void_p()
    rc = L.load().cp_graph_from_knn(cp.default_context()._h, n, k, 0.5, C.c_void_p(kd.data_ptr()),
                                    C.c_void_p(bad.data_ptr()), C.byref(h))
    assert rc == 1


def test_data_validation(cp):
    bad = np.ones((3, 2))
    bad[0, 0] = np.inf
    with pytest.raises(ValueError):
        cp.DataMatrix(bad)


# ---- WeightedGraph / B / Bᵀ / CC (test_graph.cpp:51-232) ----------------------------

def test_graph_from_edges(cp):
    g = cp.WeightedGraph(4, [(2, 3, 0.5), (0, 1, 1.0), (1, 3, 2.0)])
    assert g.edges() == [(0, 1, 1.0), (1, 3, 2.0), (2, 3, 0.5)]
    assert g.degree(3) == 2 and g.max_degree() == 2 and g.find_edge(3, 1) == 1
    for bad in ([(1, 1, 1.0)], [(3, 1, 1.0)], [(0, 4, 1.0)], [(0, 1, 0.0)], [(0, 1, -2.0)],
                [(0, 1, 1.0), (0, 1, 2.0)], [(0, 1, float("nan"))]):
        with pytest.raises(ValueError):
            cp.WeightedGraph(4, bad)


def test_incidence_bitwise(cp, orc):
    A = mixture(orc, 40, 13)
    g, og = check_graph(cp, orc, A, 6, 0.5)
    B = cp.IncidenceOperator(g)
    rng = np.random.default_rng(11)
    X = rng.standard_normal(A.shape)
    Z = rng.standard_normal((g.edge_count(), A.shape[1]))
    assert np.array_equal(B.apply(X), orc.B(og, X))
    assert np.array_equal(B.apply_transpose(Z), orc.Bt(og, Z))
    g3 = cp.WeightedGraph(3, [(0, 1, 1.0), (1, 2, 1.0)])
    assert cp.IncidenceOperator(g3).apply(np.array([[5.0], [2.0], [9.0]]))[:, 0].tolist() == [3.0, -7.0]
    with pytest.raises(ValueError):
        cp.IncidenceOperator(g3).apply(np.zeros((4, 1)))
    with pytest.raises(ValueError):
        cp.IncidenceOperator(g3).apply_transpose(np.zeros((3, 1)))


def test_laplacian_csc(cp, orc):  # test_graph.cpp:173-210
    p3 = cp.IncidenceOperator(cp.WeightedGraph(3, [(0, 1, 0.7), (1, 2, 0.2)])).laplacian().toarray()
    assert np.array_equal(p3, [[1, -1, 0], [-1, 2, -1], [0, -1, 1]])
    rng = np.random.default_rng(3)
    n = 40
    edges = sorted({(i, j) for i in range(n) for j in range(i + 1, n) if rng.random() < 0.15} | {(0, 1)})
    g = cp.WeightedGraph(n + 2, [(i, j, 0.5 + rng.random()) for i, j in edges])  # two isolated nodes
    L = cp.IncidenceOperator(g).laplacian()
    B = np.zeros((n + 2, len(edges)))
    for l, (i, j) in enumerate(edges):
        B[i, l], B[j, l] = 1.0, -1.0
    assert np.array_equal(L.toarray(), B @ B.T)
    assert L.nnz == 2 * len(edges) + n and L.has_sorted_indices


def test_connected_components(cp, orc):
    assert cp.connected_components(cp.WeightedGraph(5, [(0, 1, 1.0), (2, 3, 1.0)])).tolist() == [0, 0, 1, 1, 2]
    assert cp.connected_components(cp.WeightedGraph(4, [(2, 3, 1.0)])).tolist() == [0, 1, 2, 2]
    rng = np.random.default_rng(5)
    n = 500
    edges = sorted({(min(a, b), max(a, b)) for a, b in rng.integers(0, n, (300, 2)) if a != b})
    g = cp.WeightedGraph(n, [(a, b, 1.0) for a, b in edges])
    og = orc.Graph(n, [(a, b, 1.0) for a, b in edges])
    assert np.array_equal(cp.connected_components(g), orc.connected_components(og)[0])


def test_laplacian_lambda_max(cp, orc):
    g = cp.WeightedGraph(3, [(0, 1, 1.0), (1, 2, 1.0)])
    assert cp.IncidenceOperator(g).laplacian_lambda_max() == pytest.approx(3.0, rel=1e-8)
    # the device reproduces the reference's CSC product order and Eigen's reduction order, so
    # lambda_max is bitwise the oracle's (small graphs in shared memory, large ones in HBM)
    for A in (circle(orc, 30), circle(orc, 100), mixture(orc, 4000, 3)):
        g, og = check_graph(cp, orc, A, 10, 0.5)
        assert cp.IncidenceOperator(g).laplacian_lambda_max() == orc.power_laplacian(og)


# ---- prox (test_prox.cpp) ------------------------------------------------------------

@pytest.mark.parametrize("q", [1, 2])
def test_prox_project_jacobian(cp, orc, q):
    rng = np.random.default_rng(42 + q)
    for d in (1, 2, 3, 33, 784):
        V = rng.normal(0, 2.0, (50, d))
        t = rng.uniform(0, 3.0 * np.sqrt(d), 50)
        t[0] = 0.0
        t[1] = np.linalg.norm(V[1])  # kink
        # The column norm is a tree sum on the GPU and an Eigen-order sum in the
        # reference: they agree to a few ulp of ||v||, so compare absolutely at
        # that scale (the kink column t = ||v|| may land on either side).
        scale = 8 * ULP * np.linalg.norm(V, axis=1, keepdims=True) * np.sqrt(d)
        p = cp.prox_columns(V, t, q)
        op = orc.prox_columns(q, V, t)
        assert np.all(np.abs(p - op) <= scale)
        z = cp.project_columns(V, t, q)
        oz = orc.project_columns(q, V, t)
        assert np.all(np.abs(z - oz) <= scale)
        if q == 1:
            assert np.array_equal(p, op) and np.array_equal(z, oz)
        # Moreau identity prox + projection = v (test_prox.cpp:78-87)
        assert np.max(np.abs(p + z - V)) <= 1e-12 * max(1.0, np.max(np.abs(V)))
        jd = cp.prox_jacobian_diag(V, t, q)
        ojd = np.stack([orc.prox_jacobian_diag(q, V[l], t[l]) for l in range(50)])
        assert np.allclose(jd, ojd, rtol=1e-13, atol=1e-15)
    with pytest.raises(ValueError):
        cp.prox_columns(np.ones((1, 2)), [-0.5], q)
    with pytest.raises(ValueError):
        cp.prox_columns(np.ones((1, 2)), [0.5], 3)


@pytest.mark.parametrize("q", [1, 2, 0])
def test_prox_jacobian_apply(cp, orc, q):  # test_prox.cpp:124-188 (q = 0: infinity)
    rng = np.random.default_rng(70 + q)
    for d in (1, 3, 33, 300):
        V = rng.normal(0, 2.0, (40, d))
        base = np.abs(V).sum(axis=1) if q == 0 else (np.linalg.norm(V, axis=1) if q == 2 else np.abs(V).max(axis=1))
        t = rng.uniform(0.05, 1.2, 40) * base
        t[0] = 0.0
        W = rng.normal(0, 1.0, (40, d))
        out = cp.prox_jacobian_apply(V, t, W, q)
        for l in range(40):
            J, _, _ = orc.prox_jacobian(q, V[l], t[l])
            assert np.allclose(out[l], J @ W[l], rtol=1e-12, atol=1e-12)
    J = cp.prox_jacobian([3.0, 4.0], 1.0)  # test_prox.cpp:146-170
    assert J.diag(0) == pytest.approx(0.8 + 9.0 / 125.0)
    assert np.allclose(J.apply([1.0, 0.0]), [0.8 + 9.0 / 125.0, 12.0 / 125.0])
    assert np.all(cp.prox_jacobian([3.0, 4.0], 5.0).apply([1.0, 2.0]) == 0)  # kink -> zero map
    with pytest.raises(ValueError):
        cp.prox_jacobian([1.0], -1.0)


def test_prox_project_jacobian_linf(cp, orc):
    """q = infinity (code 0): no reference; parity against the oracle's sort-based
    l1-ball threshold (the GPU uses Michelot's fixed point)."""
    rng = np.random.default_rng(4242)
    for d in (1, 2, 3, 33, 784, 3072):
        V = rng.normal(0, 2.0, (50, d))
        l1 = np.abs(V).sum(axis=1)
        t = rng.uniform(0, 1.2, 50) * l1
        t[0] = 0.0
        t[1] = l1[1]  # boundary of the l1 ball
        t[2] = 2.0 * l1[2]  # inside
        tol = 1e-13 * (1.0 + l1[:, None])
        p = cp.prox_columns(V, t, float("inf"))
        op = orc.prox_columns(0, V, t)
        assert np.all(np.abs(p - op) <= tol)
        z = cp.project_columns(V, t, "inf")
        oz = orc.project_columns(0, V, t)
        assert np.all(np.abs(z - oz) <= tol)
        assert np.max(np.abs(p + z - V)) <= 1e-12 * max(1.0, np.max(np.abs(V)))  # Moreau
        assert np.array_equal(p[0], V[0]) and np.all(p[2] == 0) and np.array_equal(z[2], V[2])
        jd = cp.prox_jacobian_diag(V, t, cp.PenaltyNorm.linf)
        ojd = np.stack([orc.prox_jacobian_diag(0, V[l], t[l]) for l in range(50)])
        keep = np.arange(50) != 1
        assert np.allclose(jd[keep], ojd[keep], rtol=1e-13, atol=1e-15)


# ---- objectives and AL pieces (test_solvers.cpp:108-136, 367-397) ---------------------

FIVE_A = np.array([[0.0, 0.0], [1.0, 0.2], [-0.8, 0.6], [0.3, -0.9], [-0.2, 0.5]])
FIVE_E = [(0, 1, 1.0), (0, 2, 0.7), (0, 3, 0.9), (0, 4, 1.1), (1, 2, 0.6), (1, 3, 0.8), (1, 4, 1.2),
          (2, 3, 0.5), (2, 4, 0.95), (3, 4, 0.65)]


def test_objectives_two_point(cp):
    data = cp.DataMatrix([[0.0], [2.0]])
    g = cp.WeightedGraph(2, [(0, 1, 1.0)])
    inst = cp.ProblemInstance(data, g, 0.5)
    assert cp.primal_objective(inst, [[0.5], [1.5]]) == pytest.approx(0.75, rel=1e-14)
    assert cp.dual_objective(inst, [[-0.5]]) == pytest.approx(0.75, rel=1e-14)
    with pytest.raises(ValueError):
        cp.dual_objective(inst, [[-0.6]])
    with pytest.raises(ValueError):
        cp.ProblemInstance(data, cp.WeightedGraph(3, [(0, 1, 1.0)]), 0.5)
    with pytest.raises(ValueError):
        cp.ProblemInstance(data, g, -0.5)


@pytest.mark.parametrize("q", [1, 2, 0])
def test_objectives_and_al_match_oracle(cp, orc, q):
    A = mixture(orc, 30, 11)
    g, og = check_graph(cp, orc, A, 6, 0.5)
    rng = np.random.default_rng(7)
    E = g.edge_count()
    gamma, sigma = 0.3, 1.7
    inst = cp.ProblemInstance(cp.DataMatrix(A), g, gamma, q)
    X = A + 0.3 * rng.standard_normal(A.shape)
    Z = orc.project_columns(q, 0.2 * rng.standard_normal((E, A.shape[1])), gamma * og.arrays()[2])
    D = rng.standard_normal(A.shape)
    rel = lambda a, b: abs(a - b) / max(1.0, abs(b))
    assert rel(cp.primal_objective(inst, X), orc.primal_objective(A, og, gamma, q, X)) <= 1e-13
    assert rel(cp.dual_objective(inst, Z), orc.dual_objective(A, og, gamma, q, Z)) <= 1e-13
    assert rel(cp.kkt_residual(inst, X, Z), orc.kkt_residual(A, og, gamma, q, X, Z)) <= 1e-12
    assert rel(cp.ssnal_phi_value(inst, Z, sigma, X), orc.phi_value(A, og, gamma, q, Z, sigma, X)) <= 1e-13
    G, OG = cp.ssnal_phi_gradient(inst, Z, sigma, X), orc.phi_gradient(A, og, gamma, q, Z, sigma, X)
    assert np.linalg.norm(G - OG) <= 1e-13 * np.linalg.norm(OG)
    H, OH = cp.ssnal_hessian_apply(inst, Z, sigma, X, D), orc.hessian_apply(A, og, gamma, q, Z, sigma, X, D)
    assert np.linalg.norm(H - OH) <= 1e-13 * np.linalg.norm(OH)


# ---- solvers (test_solvers.cpp) ------------------------------------------------------------

ALGOS = ["admm", "ama", "ssnal"]


@pytest.mark.parametrize("algo", ALGOS)
def test_two_point_closed_form(cp, algo):
    rng = np.random.default_rng(77)
    for trial in range(6):
        d = 1 + trial % 3
        a1, a2 = rng.uniform(-2, 2, d), rng.uniform(-2, 2, d)
        w, gamma = rng.uniform(0.5, 2.0), rng.uniform(0.05, 1.5)
        inst = cp.ProblemInstance(cp.DataMatrix(np.stack([a1, a2])), cp.WeightedGraph(2, [(0, 1, w)]), gamma)
        sol = cp.solve(inst, cp.SolverConfig(algorithm=cp.algorithm_from_name(algo), epsilon=1e-8))
        x1, x2 = cp.two_point_closed_form(a1, a2, w, gamma)
        assert sol.termination.converged
        assert np.max(np.abs(sol.X[0] - x1)) <= 1e-6 and np.max(np.abs(sol.X[1] - x2)) <= 1e-6


@pytest.mark.parametrize("algo", ALGOS)
def test_trivial_and_warm(cp, algo):
    data = cp.DataMatrix([[1.0], [-3.0]])
    for g, gamma in ((cp.WeightedGraph(2, [(0, 1, 1.0)]), 0.0), (cp.WeightedGraph(2, []), 1.0)):
        sol = cp.solve(cp.ProblemInstance(data, g, gamma), cp.SolverConfig(algorithm=cp.algorithm_from_name(algo)))
        assert sol.termination.converged and sol.termination.iterations == 0 and np.array_equal(sol.X, data.values)
    five = cp.ProblemInstance(cp.DataMatrix(FIVE_A), cp.WeightedGraph(5, FIVE_E), 0.15)
    cfg = cp.SolverConfig(algorithm=cp.algorithm_from_name(algo), epsilon=1e-7)
    cold = cp.solve(five, cfg)
    warm = cp.solve(five, cfg, warm=cold)
    assert cold.termination.converged and warm.termination.iterations == 0 and np.array_equal(warm.X, cold.X)
    with pytest.raises(ValueError):
        cp.solve(five, cfg, warm=cp.Solution(np.zeros((4, 2)), np.zeros((10, 2))))


@pytest.mark.parametrize("algo", ALGOS)
@pytest.mark.parametrize("q", [2, 1, 0])
def test_solver_parity_with_oracle(cp, orc, algo, q):
    """Same instance, same algorithm: X within 1e-6 relative Frobenius, labels equal."""
    A = mixture(orc, 25, 4, m=3, seed=9)
    g, og = check_graph(cp, orc, A, 5, 0.5)
    for gamma in (0.05, 0.3):
        inst = cp.ProblemInstance(cp.DataMatrix(A), g, gamma, q)
        sol = cp.solve(inst, cp.SolverConfig(algorithm=cp.algorithm_from_name(algo)))
        osol = orc.solve(A, og, gamma, q, orc.config(algo))
        assert sol.termination.converged == bool(osol.term["converged"])
        assert np.linalg.norm(sol.X - osol.X) <= 1e-6 * np.linalg.norm(osol.X)
        assert np.array_equal(cp.extract_clusters(sol.X, g).labels, orc.extract_clusters(osol.X, og)[0])


@pytest.mark.parametrize("d", [2, 33, 34, 64, 100, 130, 192, 194, 256, 784, 1000])
def test_hessian_tma_path_matches_oracle(cp, orc, d):
    """Even d >= 256 takes the TMA-staged single-pass Hessian (hess_tma.cu),
    including hub nodes split into segments (k = 30 makes degrees > 64); even
    d <= 192 the single-pass warp Hessian (k_hess_warp, 1/2/3 double2 pairs per
    lane: d = 2..64 / 100 / 130..192); odd d and 194 the two-pass path."""
    A = mixture(orc, 40, d, m=3, seed=5)
    for k in (6, 30):
        g, og = check_graph(cp, orc, A, k, 0.5)
        rng = np.random.default_rng(d + k)
        inst = cp.ProblemInstance(cp.DataMatrix(A), g, 0.2)
        X = A + 0.05 * rng.standard_normal(A.shape)
        Z = orc.project_columns(2, 0.1 * rng.standard_normal((g.edge_count(), d)), 0.2 * og.arrays()[2])
        D = rng.standard_normal(A.shape)
        for sigma in (0.7, 5.0):
            H = cp.ssnal_hessian_apply(inst, Z, sigma, X, D)
            OH = orc.hessian_apply(A, og, 0.2, 2, Z, sigma, X, D)
            assert np.linalg.norm(H - OH) <= 1e-13 * np.linalg.norm(OH)


@pytest.mark.parametrize("q", [1, 0])
@pytest.mark.parametrize("d", [33, 64, 300, 520, 1000, 3072])
def test_hessian_mask_path_matches_oracle(cp, orc, q, d):
    """q = 1 / inf Hessian (ssnal.cpp:56-64) through the per-edge Jacobian bit masks
    (gather.cu edge_masks: [|v_f| > t] or [|v_f| > theta] and sign(v_f)), which replace the V
    reads of the gathers: equal to the oracle's dense-Jacobian apply at rounding level
    (d = 3072 is C4's row length)."""
    A = mixture(orc, 30, d, m=3, seed=11)
    g, og = check_graph(cp, orc, A, 8, 0.5)
    rng = np.random.default_rng(d + 7 * q)
    gamma = 0.2
    inst = cp.ProblemInstance(cp.DataMatrix(A), g, gamma, q)
    X = A + 0.05 * rng.standard_normal(A.shape)
    Z = orc.project_columns(q, 0.05 * rng.standard_normal((g.edge_count(), d)), gamma * og.arrays()[2])
    D = rng.standard_normal(A.shape)
    for sigma in (0.7, 5.0):
        H = cp.ssnal_hessian_apply(inst, Z, sigma, X, D)
        OH = orc.hessian_apply(A, og, gamma, q, Z, sigma, X, D)
        assert np.linalg.norm(H - OH) <= 1e-13 * np.linalg.norm(OH)


@pytest.mark.parametrize("q", [0, 1])
@pytest.mark.parametrize("d", [40, 300, 600])
def test_ssnal_linf_l1_wide_rows_match_oracle(cp, orc, q, d):
    """SSNAL with q = inf / 1 at d > 32: the shared-memory-staged q = inf edge passes
    (k_phi_edge_linf_s, k_mult_inf_s, k_gap_edge_linf_s) and the bit-mask Hessian keep the
    oracle's Newton / CG / Armijo counts, X at rounding level."""
    A = mixture(orc, 20, d, m=3, seed=13)
    g, og = check_graph(cp, orc, A, 6, 0.5)
    gi, gj, gw, _ = g.arrays()
    og = orc.Graph.from_arrays(len(A), gi, gj, gw)  # identical weights (see the AMA block test)
    for gamma in (0.05, 0.2):
        inst = cp.ProblemInstance(cp.DataMatrix(A), g, gamma, q)
        sol = cp.solve(inst)
        osol = orc.solve(A, og, gamma, q)
        t, ot = sol.termination, osol.term
        if q == 1:  # no reduction enters the Jacobian: the iteration paths coincide
            assert (t.iterations, t.newton, t.cg, t.armijo) == (ot["iterations"], ot["newton"], ot["cg"], ot["armijo"])
        else:  # q = inf: the Hessian's <s_S, w> / |S| dots round differently over ~2000 CG steps
            assert (t.iterations, t.newton, t.armijo) == (ot["iterations"], ot["newton"], ot["armijo"])
            assert abs(t.cg - ot["cg"]) <= 2 + 0.002 * ot["cg"]
        assert np.linalg.norm(sol.X - osol.X) <= 1e-9 * np.linalg.norm(osol.X)
        assert cp.kkt_residual(inst, sol.X, sol.Z) == pytest.approx(orc.kkt_residual(A, og, gamma, q, sol.X, sol.Z),
                                                                    rel=1e-9, abs=1e-15)
        assert cp.primal_objective(inst, sol.X) == pytest.approx(orc.primal_objective(A, og, gamma, q, sol.X), rel=1e-12)


def test_ssnal_iteration_path_matches_tma(cp, orc):
    A = mixture(orc, 30, 40, m=3, seed=4)
    g, og = check_graph(cp, orc, A, 6, 0.5)
    sol = cp.solve(cp.ProblemInstance(cp.DataMatrix(A), g, 0.15))
    osol = orc.solve(A, og, 0.15, 2)
    t, ot = sol.termination, osol.term
    assert (t.iterations, t.newton, t.cg, t.armijo) == (ot["iterations"], ot["newton"], ot["cg"], ot["armijo"])
    assert np.linalg.norm(sol.X - osol.X) <= 1e-10 * np.linalg.norm(osol.X)


def test_ssnal_iteration_path_matches(cp, orc):
    A = mixture(orc, 30, 16, m=3, seed=3)
    g, og = check_graph(cp, orc, A, 6, 0.5)
    inst = cp.ProblemInstance(cp.DataMatrix(A), g, 0.2)
    sol = cp.solve(inst)
    osol = orc.solve(A, og, 0.2, 2)
    t, ot = sol.termination, osol.term
    assert (t.iterations, t.newton, t.cg, t.armijo) == (ot["iterations"], ot["newton"], ot["cg"], ot["armijo"])
    assert np.linalg.norm(sol.X - osol.X) <= 1e-10 * np.linalg.norm(osol.X)


@pytest.mark.parametrize("algo", ALGOS)
def test_deterministic(cp, algo):
    inst = cp.ProblemInstance(cp.DataMatrix(FIVE_A), cp.WeightedGraph(5, FIVE_E), 0.12)
    cfg = cp.SolverConfig(algorithm=cp.algorithm_from_name(algo))
    s1, s2 = cp.solve(inst, cfg), cp.solve(inst, cfg)
    assert np.array_equal(s1.X, s2.X) and np.array_equal(s1.Z, s2.Z)
    assert s1.termination.iterations == s2.termination.iterations and s1.termination.gap == s2.termination.gap


def test_iteration_cap(cp):
    inst = cp.ProblemInstance(cp.DataMatrix(FIVE_A), cp.WeightedGraph(5, FIVE_E), 0.2)
    sol = cp.solve(inst, cp.SolverConfig(algorithm=cp.Algorithm.ADMM, epsilon=1e-12, max_iter=3))
    assert not sol.termination.converged and sol.termination.iterations == 3 and sol.termination.gap > 0


@pytest.mark.parametrize("d", [16, 300])
def test_ssnal_best_iterate_when_capped(cp, orc, d):
    """A capped, non-converged SSNAL solve returns the best-gap iterate
    (solver_util.hpp:70-100): X and Z equal the oracle's."""
    A = mixture(orc, 25, d, m=3, seed=6)
    g, og = check_graph(cp, orc, A, 6, 0.5)
    inst = cp.ProblemInstance(cp.DataMatrix(A), g, 0.3)
    for cap in (1, 2, 3):
        sol = cp.solve(inst, cp.SolverConfig(epsilon=1e-14, max_iter=cap))
        osol = orc.solve(A, og, 0.3, 2, orc.config("ssnal", epsilon=1e-14, max_iter=cap))
        assert not sol.termination.converged and not osol.term["converged"]
        assert sol.termination.iterations == osol.term["iterations"] == cap
        assert np.linalg.norm(sol.X - osol.X) <= 1e-10 * np.linalg.norm(osol.X)
        assert np.linalg.norm(sol.Z - osol.Z) <= 1e-10 * max(np.linalg.norm(osol.Z), 1e-300)
        assert sol.termination.gap == pytest.approx(osol.term["gap"], rel=1e-8)


# ---- path (test_path.cpp) ------------------------------------------------------------------

def test_schedule_and_clusters(cp):
    s = cp.make_schedule(1.0, 100.0, 3)
    assert s.values == pytest.approx([1.0, 10.0, 100.0], rel=1e-14)
    with pytest.raises(ValueError):
        cp.make_schedule(0.5, 0.5, 2, cp.Spacing.linear)
    chain = cp.WeightedGraph(4, [(0, 1, 1.0), (1, 2, 1.0), (2, 3, 1.0)])
    c = cp.extract_clusters(np.array([[0.0], [1.0], [1.0], [3.0]]), chain)
    assert c.K == 3 and c.labels.tolist() == [0, 1, 1, 2] and c.centroids[1, 0] == 1.0
    assert cp.extract_clusters(np.array([[0.0], [1.0], [2.0], [0.0]]), chain).K == 4
    pair = cp.WeightedGraph(2, [(0, 1, 1.0)])
    assert cp.extract_clusters(np.array([[1000.0], [1000.5]]), pair).K == 1
    assert cp.extract_clusters(np.array([[1000.0], [1000.5]]), pair, 1e-5).K == 2
    with pytest.raises(ValueError):
        cp.extract_clusters(np.zeros((3, 1)), chain)


def test_centroids_bitwise(cp, orc):
    A = mixture(orc, 40, 9)
    g, og = check_graph(cp, orc, A, 6, 0.5)
    X = np.repeat(A[::4], 4, axis=0)  # exact fusions in groups of four
    c = cp.extract_clusters(X, g)
    ol, oK, oc = orc.extract_clusters(X, og)
    assert c.K == oK and np.array_equal(c.labels, ol) and np.array_equal(c.centroids, oc)


@pytest.mark.parametrize("algo", ["ssnal", "ama"])
def test_path_parity(cp, orc, algo):
    A = circle(orc, 12)
    g, og = check_graph(cp, orc, A, 10, 0.5)
    sched = cp.make_schedule(0.01, 10.0, 8)
    res = cp.run_path(cp.DataMatrix(A), g, 2, sched, cp.SolverConfig(algorithm=cp.algorithm_from_name(algo)))
    ores = orc.run_path(A, og, 2, sched.values, orc.config(algo))
    for t in range(len(sched.values)):
        assert res.stats[t].converged == bool(ores["terms"][t]["converged"])
        assert np.linalg.norm(res.solutions[t].X - ores["X"][t]) <= 1e-6 * np.linalg.norm(ores["X"][t])
        assert np.array_equal(res.assignments[t].labels, ores["labels"][t])
        assert res.assignments[t].K == ores["K"][t]


@pytest.mark.parametrize("pinned", [True, False])
def test_path_outputs_of_unchanged_gammas(cp, orc, monkeypatch, pinned):
    """run_path does not ship a gamma's X / Z again when its warm start was accepted as is and
    the dual projection moved nothing (the blocks are host copies of the last shipped gamma's):
    every gamma's X and Z must still equal, bit for bit, a chain of warm-started solve() calls."""
    if not pinned:  # pageable outputs: synchronous copies, the host copy right away
        import paper_2501_15964_b200.cluspath as cpm
        monkeypatch.setattr(cpm, "pinned_empty", lambda shape, dtype=np.float64: np.empty(shape, dtype))
    A = mixture(orc, 30, 16, m=3, seed=3)  # the oracle's path: gammas 9-12 take 0 iterations
    g, _ = check_graph(cp, orc, A, 10, 0.5)
    sched = cp.make_schedule(0.01, 10.0, 12)
    cfg = cp.SolverConfig()
    res = cp.run_path(cp.DataMatrix(A), g, 2, sched, cfg, keep_solutions=True, keep_z=True)
    data, prev = cp.DataMatrix(A), None
    zero_iter = 0
    for t, gamma in enumerate(sched.values):
        sol = cp.solve(cp.ProblemInstance(data, g, gamma, 2), cfg, prev)
        prev = sol
        zero_iter += int(t > 0 and res.stats[t].iterations == 0)
        assert res.stats[t].iterations == sol.termination.iterations
        assert np.array_equal(res.solutions[t].X, sol.X)
        assert np.array_equal(res.solutions[t].Z, sol.Z)
    assert zero_iter >= 1  # the path exercises the host-copied outputs


# q = inf: the device and the oracle compute the l1-ball threshold with the same Michelot
# passes and the same 32-lane summation order (linf.cuh, oracle l1_theta), so the projected
# iterates agree bit for bit and the d = 40 case holds the same 1e-10 bar as q = 1, 2.
# circle: 300 nodes, one node per warp (register-resident adjacency); circle1500: more nodes
# than warps in the grid, the grid-stride gather; d40: the CUDA-graph path.
@pytest.mark.parametrize("q,shape", [(2, "circle"), (1, "circle"), (0, "circle"), (2, "circle1500"), (2, "d40"),
                                     (1, "d40"), (0, "d40")])
def test_ama_graph_blocks_match_oracle(cp, orc, q, shape):
    """Fast AMA runs the iterations between gap checks as one cooperative kernel (d <= 32:
    k_ama_block) or as one CUDA graph per 10-iteration block with the Nesterov momenta computed
    on the device (d = 40): long solves (hundreds of blocks) must keep the oracle's iteration
    counts and X to near round-off."""
    A = {"circle": lambda: circle(orc, 30), "circle1500": lambda: circle(orc, 150),
         "d40": lambda: mixture(orc, 60, 40, m=5, seed=3)}[shape]()
    g, _ = check_graph(cp, orc, A, 10, 0.5)
    # both sides solve on the device's graph: its weights are pinned to the oracle's at <= 1 ulp
    # by check_graph (CUDA exp vs glibc exp), and AMA's thousands of iterations turn a 1-ulp radius
    # difference into a stop one gap check apart; with identical inputs the iterates agree bitwise
    gi, gj, gw, _ = g.arrays()
    og = orc.Graph.from_arrays(len(A), gi, gj, gw)
    sched = cp.make_schedule(0.01, 10.0, 6)
    cfg = cp.SolverConfig(algorithm=cp.Algorithm.FastAMA)
    res = cp.run_path(cp.DataMatrix(A), g, q, sched, cfg)
    ores = orc.run_path(A, og, q, sched.values, orc.config("ama"))
    assert sum(res.stats[t].iterations for t in range(len(sched.values))) > 200
    for t in range(len(sched.values)):
        assert res.stats[t].iterations == ores["terms"][t]["iterations"]
        assert res.stats[t].converged == bool(ores["terms"][t]["converged"])
        assert np.linalg.norm(res.solutions[t].X - ores["X"][t]) <= 1e-10 * np.linalg.norm(ores["X"][t])
        if q != 2:  # q = 1 clamps, q = inf thresholds in the oracle's order: iterates bit for bit
            assert np.array_equal(res.solutions[t].Z, ores["Z"][t])  # (q = 2 divides by a reduced norm)
        assert np.array_equal(res.assignments[t].labels, ores["labels"][t])


def test_c1_exact_config_matches_oracle(cp, orc):
    """BASELINE.json configs[0] as bench.py runs it: n = 1000 on the 10-centre circle (spread
    0.5), kNN k = 10, phi = 0.5, q = 2, fast AMA over the 20 geometric gammas in [0.01, 10]
    (path.cpp:110-142, ama.cpp:17-89): identical iteration counts and labels, X within 1e-10."""
    A = circle(orc, 100)
    g, og = check_graph(cp, orc, A, 10, 0.5)
    sched = cp.make_schedule(0.01, 10.0, 20)
    res = cp.run_path(cp.DataMatrix(A), g, 2, sched, cp.SolverConfig(algorithm=cp.Algorithm.FastAMA))
    ores = orc.run_path(A, og, 2, sched.values, orc.config("ama"))
    for t in range(20):
        assert res.stats[t].iterations == ores["terms"][t]["iterations"]
        assert res.stats[t].converged == bool(ores["terms"][t]["converged"])
        assert np.linalg.norm(res.solutions[t].X - ores["X"][t]) <= 1e-10 * np.linalg.norm(ores["X"][t])
        assert np.linalg.norm(res.solutions[t].Z - ores["Z"][t]) <= 1e-10 * max(1.0, np.linalg.norm(ores["Z"][t]))
        assert np.array_equal(res.assignments[t].labels, ores["labels"][t])
        assert res.assignments[t].K == ores["K"][t]


@pytest.mark.parametrize("shape", ["c1", "c2cap"])
def test_admm_matches_oracle_cholesky(cp, orc, shape):
    """ADMM's X-update (admm.cpp:38-62): the reference factors I + rho L once (SimplicialLLT,
    linalg.cpp:32-54) and the oracle with an exact envelope Cholesky; the device solves the
    same system by warm-started Laplacian PCG to 1e-13.  c1: BASELINE configs[0]'s data, the
    20-gamma ADMM path to convergence; c2cap: C2-shaped rows (d = 784) with every solve capped
    at 25 ADMM iterations (bench-sized systems, a bounded oracle run).  X within 1e-6, labels
    equal, the stopping iteration within one gap check."""
    if shape == "c1":
        A, T, cap = circle(orc, 100), 20, 0
    else:
        A, T, cap = mixture(orc, 100, 784, m=10, seed=42), 3, 25
    g, og = check_graph(cp, orc, A, 10, 0.5)
    sched = cp.make_schedule(0.01, 10.0, 20)
    sched.values = sched.values[:T]
    res = cp.run_path(cp.DataMatrix(A), g, 2, sched, cp.SolverConfig(algorithm=cp.Algorithm.ADMM, max_iter=cap))
    ores = orc.run_path(A, og, 2, sched.values, orc.config("admm", max_iter=cap))
    for t in range(T):
        assert abs(res.stats[t].iterations - ores["terms"][t]["iterations"]) <= 1
        assert res.stats[t].converged == bool(ores["terms"][t]["converged"])
        assert np.linalg.norm(res.solutions[t].X - ores["X"][t]) <= 1e-6 * np.linalg.norm(ores["X"][t])
        assert np.array_equal(res.assignments[t].labels, ores["labels"][t])


@pytest.mark.parametrize("d", [64, 96])
def test_edge_ring_wraps_match_oracle(cp, orc, d):
    """Short rows run the TMA edge kernels with an 8-deep per-warp ring; with
    ~20k edges every warp wraps its ring several times."""
    A = mixture(orc, 750, d, m=4, seed=21)
    g, og = check_graph(cp, orc, A, 10, 0.5)
    assert g.edge_count() > 15000
    gamma = 0.05
    sol = cp.solve(cp.ProblemInstance(cp.DataMatrix(A), g, gamma, 2), cp.SolverConfig())
    osol = orc.solve(A, og, gamma, 2, orc.config("ssnal"))
    assert sol.termination.converged == bool(osol.term["converged"])
    assert np.linalg.norm(sol.X - osol.X) <= 1e-6 * np.linalg.norm(osol.X)
    assert sol.termination.cg == osol.term["cg"] and sol.termination.newton == osol.term["newton"]


@pytest.mark.parametrize("d,k", [(64, 8), (300, 8)])
def test_partitioned_pcg_single_rank(cp, orc, d, k):
    """The node-partitioned PCG (NCCL communicator attached; one rank) through
    both Hessian paths (two-pass for d < 256, TMA for d >= 256): same solution
    as the oracle within 1e-6 and identical labels."""
    ctx = cp.Context(0)
    ctx.set_comm(1, 0, cp.nccl_unique_id())
    A = mixture(orc, 150, d, m=4, seed=31)
    data = cp.DataMatrix(A, ctx=ctx)
    g = cp.compute_knn_weights(data, k, 0.5)
    og = orc.knn_weights(A, k, 0.5)
    for gamma in (0.05, 0.2):
        sol = cp.solve(cp.ProblemInstance(data, g, gamma, 2), cp.SolverConfig())
        osol = orc.solve(A, og, gamma, 2, orc.config("ssnal"))
        assert sol.termination.converged and bool(osol.term["converged"])
        assert sol.termination.cg > 0
        assert np.linalg.norm(sol.X - osol.X) <= 1e-6 * np.linalg.norm(osol.X)
        assert np.array_equal(cp.extract_clusters(sol.X, g).labels, orc.extract_clusters(osol.X, og)[0])


@pytest.mark.parametrize("nranks,d", [(2, 64), (3, 300), (4, 784)])
def test_partitioned_path_multi_rank(cp, orc, nranks, d):
    """P ranks in one process (one host thread and context each, in-process
    group): the node-partitioned Newton PCG of a warm-started path matches the
    single-context path within 1e-6 at every gamma with identical labels, and
    every rank returns the same result bit for bit."""
    import threading
    A = mixture(orc, 90, d, m=4, seed=41)
    g0 = cp.compute_knn_weights(cp.DataMatrix(A), 8, 0.5)
    sched = cp.make_schedule(0.02, 2.0, 6)
    ref = cp.run_path(cp.DataMatrix(A), g0, 2, sched, cp.SolverConfig())
    group = cp.LocalGroup(nranks)
    ctxs = [cp.Context(0) for _ in range(nranks)]
    for r, c in enumerate(ctxs):
        c.set_local_comm(group, r)
    datas = [cp.DataMatrix(A, ctx=c) for c in ctxs]
    out, errs, graphs = [None] * nranks, [], [None] * nranks

    def work(r):
        try:  # the kNN is row-sharded across the group too (cp_knn_graph with a communicator)
            graphs[r] = cp.compute_knn_weights(datas[r], 8, 0.5)
            out[r] = cp.run_path(datas[r], graphs[r], 2, sched, cp.SolverConfig())
        except Exception as e:  # noqa: BLE001
            errs.append(e)

    th = [threading.Thread(target=work, args=(r,)) for r in range(nranks)]
    for t in th:
        t.start()
    for t in th:
        t.join(300)
    assert not errs, errs
    for r in range(nranks):
        for a_, b_ in zip(graphs[r].arrays(), g0.arrays()):
            assert np.array_equal(a_, b_)
    for t in range(len(sched.values)):
        X0 = ref.solutions[t].X
        for r in range(nranks):
            assert np.linalg.norm(out[r].solutions[t].X - X0) <= 1e-6 * np.linalg.norm(X0)
            assert np.array_equal(out[r].assignments[t].labels, ref.assignments[t].labels)
            assert np.array_equal(out[r].solutions[t].X, out[0].solutions[t].X)
        assert out[0].stats[t].converged
    assert sum(s.cg for s in out[0].stats) > 0


def test_path_parity_linf(cp, orc):
    """Warm-started SSNAL path with q = infinity (C4's prox variant): every X
    within 1e-6 relative Frobenius of the oracle path and identical labels."""
    A = mixture(orc, 20, 8, m=4, seed=5)
    g, og = check_graph(cp, orc, A, 6, 0.5)
    sched = cp.make_schedule(0.01, 3.0, 8)
    res = cp.run_path(cp.DataMatrix(A), g, float("inf"), sched, cp.SolverConfig())
    ores = orc.run_path(A, og, 0, sched.values, orc.config("ssnal"))
    for t in range(len(sched.values)):
        assert res.stats[t].converged == bool(ores["terms"][t]["converged"])
        assert np.linalg.norm(res.solutions[t].X - ores["X"][t]) <= 1e-6 * np.linalg.norm(ores["X"][t])
        assert np.array_equal(res.assignments[t].labels, ores["labels"][t])


def test_path_validation(cp):
    data = cp.DataMatrix([[0.0], [1.0], [10.0], [11.0]])
    g = cp.WeightedGraph(4, [(0, 1, 1.0), (2, 3, 1.0)])
    sched = cp.make_schedule(0.5, 1.0, 2)
    with pytest.raises(RuntimeError):
        cp.run_path(data, g, 2, sched, options=cp.PathOptions(require_connected=True))
    res = cp.run_path(data, g, 2, sched)
    assert res.all_converged() and res.assignments[-1].K >= 2
    with pytest.raises(ValueError):
        cp.run_path(data, cp.WeightedGraph(3, [(0, 1, 1.0)]), 2, sched)
