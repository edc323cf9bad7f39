"""Pins the CPU oracle against the reference's own known-answer tests.

Each test restates one reference test case (cited as test_*.cpp:line) and runs
it against oracle/ (the C++ restatement).  These run on CPU only.
"""
import math

import numpy as np
import pytest


def line(xs):
    return np.asarray(xs, dtype=np.float64).reshape(-1, 1)


# ---- graph (test_graph.cpp) -------------------------------------------------

def test_data_validation(orc):  # test_graph.cpp:35-49
    orc.validate_data(np.arange(6.0).reshape(3, 2))
    with pytest.raises(ValueError):
        orc.validate_data(np.zeros((0, 2)))
    bad = np.ones((3, 2))
    bad[0, 0] = np.nan
    with pytest.raises(ValueError):
        orc.validate_data(bad)


def test_graph_sorts_and_validates(orc):  # test_graph.cpp:51-77
    g = orc.Graph(4, [(2, 3, 0.5), (0, 1, 1.0), (1, 3, 2.0)])
    i, j, w, _ = g.arrays()
    assert list(zip(i, j)) == [(0, 1), (1, 3), (2, 3)]
    assert list(w) == [1.0, 2.0, 0.5]
    assert g.degree()[3] == 2 and g.degree().max() == 2
    assert g.find_edge(3, 1) == 1 and g.find_edge(0, 2) is None
    for bad in ([(1, 1, 1.0)], [(3, 1, 1.0)], [(0, 4, 1.0)], [(0, 1, 0.0)], [(0, 1, -2.0)],
                [(0, 1, 1.0), (0, 1, 2.0)]):
        with pytest.raises(ValueError):
            orc.Graph(4, bad)


def test_knn_line(orc):  # test_graph.cpp:91-102
    g = orc.knn_weights(line([0.0, 1.0, 3.0]), 1, 0.0)
    i, j, w, d2 = g.arrays()
    assert list(zip(i, j)) == [(0, 1), (1, 2)]
    assert list(w) == [1.0, 1.0]
    assert list(d2) == [1.0, 4.0]


def test_knn_weights(orc):  # test_graph.cpp:104-110
    g = orc.knn_weights(line([0.0, 1.0, 3.0]), 1, 0.5)
    _, _, w, _ = g.arrays()
    assert w[0] == pytest.approx(0.6065306597126334, rel=1e-14)
    assert w[1] == pytest.approx(0.1353352832366127, rel=1e-14)


def test_knn_tie_breaks_to_smaller_index(orc):  # test_graph.cpp:112-124
    A = np.array([[0.0, 0.0], [5.0, 0.0], [-5.0, 0.0], [5.1, 0.0], [-5.1, 0.0]])
    g = orc.knn_weights(A, 1, 0.0)
    assert g.find_edge(0, 1) is not None and g.find_edge(0, 2) is None
    assert g.find_edge(1, 3) is not None and g.find_edge(2, 4) is not None
    assert g.E == 3


def test_knn_k_range_and_underflow(orc):  # test_graph.cpp:126-138
    data = line([0.0, 1.0, 3.0])
    for k in (0, 3):
        with pytest.raises(ValueError):
            orc.knn_weights(data, k, 0.5)
    assert orc.knn_weights(data, 2, 0.5).E == 3
    assert orc.knn_weights(line([0.0, 1.0]), 1, 1.0).E == 1
    assert orc.knn_weights(line([0.0, 1.0]), 1, 1e10).E == 0


def test_incidence_differences(orc):  # test_graph.cpp:140-150
    g = orc.Graph(3, [(0, 1, 1.0), (1, 2, 1.0)])
    XB = orc.B(g, line([5.0, 2.0, 9.0]))
    assert XB[:, 0].tolist() == [3.0, -7.0]


def dense_incidence(n, edges):
    Bd = np.zeros((n, len(edges)))
    for l, (i, j, _) in enumerate(edges):
        Bd[i, l] = 1.0
        Bd[j, l] = -1.0
    return Bd


def test_incidence_transpose_dense_and_adjoint(orc):  # test_graph.cpp:152-171
    edges = [(0, 1, 1.0), (0, 3, 1.0), (1, 2, 1.0), (2, 4, 1.0), (3, 4, 1.0)]
    g = orc.Graph(5, edges)
    rng = np.random.default_rng(11)
    X = rng.standard_normal((5, 3))
    Z = rng.standard_normal((5, 3))
    Bd = dense_incidence(5, edges)
    assert np.array_equal(orc.B(g, X), (X.T @ Bd).T)
    assert np.array_equal(orc.Bt(g, Z), (Z.T @ Bd.T).T)
    lhs = np.sum(orc.B(g, X) * Z)
    rhs = np.sum(X * orc.Bt(g, Z))
    assert lhs == pytest.approx(rhs, rel=1e-12)


def test_laplacian(orc):  # test_graph.cpp:173-212
    L = orc.laplacian_dense(orc.Graph(3, [(0, 1, 0.7), (1, 2, 0.2)]))
    assert np.array_equal(L, np.array([[1, -1, 0], [-1, 2, -1], [0, -1, 1.0]]))
    L = orc.laplacian_dense(orc.Graph(3, [(0, 1, 1.0), (0, 2, 1.0), (1, 2, 1.0)]))
    assert np.array_equal(L, np.array([[2, -1, -1], [-1, 2, -1], [-1, -1, 2.0]]))
    rng = np.random.default_rng(3)
    edges = {(0, 1, 0.5)}
    for i in range(8):
        for j in range(i + 1, 8):
            if rng.integers(4) == 0:
                edges.add((i, j, float(rng.uniform(0.1, 2.0))))
    uniq = {}
    for i, j, w in sorted(edges):
        uniq.setdefault((i, j), w)
    edges = [(i, j, w) for (i, j), w in sorted(uniq.items())]
    g = orc.Graph(8, edges)
    Bd = dense_incidence(8, edges)
    L = orc.laplacian_dense(g)
    assert np.max(np.abs(L - Bd @ Bd.T)) <= 1e-14
    assert np.linalg.eigvalsh(L).max() <= 2.0 * g.degree().max() + 1e-12


def test_connected_components(orc):  # test_graph.cpp:214-232
    lab, K = orc.connected_components(orc.Graph(5, [(0, 1, 1.0), (2, 3, 1.0)]))
    assert lab.tolist() == [0, 0, 1, 1, 2] and K == 3
    lab, K = orc.connected_components(orc.Graph(4, [(2, 3, 1.0)]))
    assert lab.tolist() == [0, 1, 2, 2] and K == 3
    assert orc.connected_components(orc.Graph(3, [(0, 1, 1.0), (1, 2, 1.0)]))[1] == 1


# ---- prox (test_prox.cpp) ---------------------------------------------------

def test_norms(orc):  # test_prox.cpp:38-43
    assert orc.norms(2, [3, 4]) == (5.0, 5.0)
    assert orc.norms(1, [3, -4]) == (7.0, 4.0)


def test_group_soft_threshold(orc):  # test_prox.cpp:45-54
    p = orc.prox_columns(2, [[3.0, 4.0]], [1.0])[0]
    assert p[0] == pytest.approx(2.4, rel=1e-14) and p[1] == pytest.approx(3.2, rel=1e-14)
    assert np.all(orc.prox_columns(2, [[3.0, 4.0]], [5.0]) == 0)
    assert np.all(orc.prox_columns(2, [[3.0, 4.0]], [9.0]) == 0)
    assert orc.prox_columns(2, [[3.0, 4.0]], [0.0])[0].tolist() == [3.0, 4.0]
    with pytest.raises(ValueError):
        orc.prox_columns(2, [[1.0, 1.0]], [-0.5])


def test_componentwise_soft_threshold(orc):  # test_prox.cpp:56-64
    assert orc.prox_columns(1, [[3.0, -4.0]], [1.0])[0].tolist() == [2.0, -3.0]
    q = orc.prox_columns(1, [[0.5, -4.0]], [1.0])[0]
    assert q[0] == 0.0 and q[1] == -3.0


def test_projection(orc):  # test_prox.cpp:66-76
    p = orc.project_columns(2, [[6.0, 8.0]], [5.0])[0]
    assert p[0] == pytest.approx(3.0, rel=1e-14) and p[1] == pytest.approx(4.0, rel=1e-14)
    assert orc.project_columns(2, [[1.0, 2.0]], [5.0])[0].tolist() == [1.0, 2.0]
    assert orc.project_columns(1, [[3.0, -4.0]], [2.0])[0].tolist() == [2.0, -2.0]
    assert orc.project_columns(1, [[1.0, -1.5]], [2.0])[0].tolist() == [1.0, -1.5]
    assert np.all(orc.project_columns(2, [[3.0, -4.0]], [0.0]) == 0)


@pytest.mark.parametrize("q", [1, 2])
def test_moreau_identity(orc, q):  # test_prox.cpp:78-87
    rng = np.random.default_rng(42)
    for _ in range(1000):
        v = rng.normal(0.0, 2.0, size=1 + rng.integers(6))
        assert orc.moreau_check(q, v, rng.uniform(0.0, 3.0)) <= 1e-12


@pytest.mark.parametrize("q", [1, 2])
def test_jacobian_matches_fd(orc, q):  # test_prox.cpp:124-144
    rng = np.random.default_rng(5)
    h = 1e-6
    acc = 0
    while acc < 100:
        v = rng.normal(0, 2.0, 3)
        t = rng.uniform(0.1, 2.0)
        if abs(np.linalg.norm(v) - t) < 0.05 or np.min(np.abs(np.abs(v) - t)) < 0.05:
            continue
        acc += 1
        J, _, _ = orc.prox_jacobian(q, v, t)
        w = rng.normal(0, 1.0, 3)
        fd = (orc.prox_columns(q, [v + h * w], [t])[0] - orc.prox_columns(q, [v - h * w], [t])[0]) / (2 * h)
        assert np.linalg.norm(J @ w - fd) <= 1e-5 * (1.0 + np.linalg.norm(fd))


def test_jacobian_structure_l2(orc):  # test_prox.cpp:146-170
    J, a, b = orc.prox_jacobian(2, [3.0, 4.0], 1.0)
    assert a == pytest.approx(0.8)
    diag = orc.prox_jacobian_diag(2, [3.0, 4.0], 1.0)
    assert diag[0] == pytest.approx(0.8 + 9.0 / 125.0)
    assert J[0, 0] == pytest.approx(diag[0], rel=1e-14)
    assert np.all(orc.prox_jacobian(2, [1.0, 1.0], 5.0)[0] == 0)
    assert np.all(orc.prox_jacobian(2, [3.0, 4.0], 5.0)[0] == 0)  # kink -> zero map
    J, _, _ = orc.prox_jacobian(2, [3.0, 4.0], 0.0)
    assert np.array_equal(J, np.eye(2))


def test_jacobian_structure_l1(orc):  # test_prox.cpp:172-188
    assert orc.prox_jacobian_diag(1, [3.0, 0.5], 1.0).tolist() == [1.0, 0.0]
    assert orc.prox_jacobian_diag(1, [1.0, -3.0], 1.0).tolist() == [0.0, 1.0]
    assert orc.prox_jacobian_diag(1, [1.0, -3.0], 0.0).tolist() == [1.0, 1.0]


# ---- linalg (test_linalg.cpp) -----------------------------------------------

def test_cholesky_path3(orc):  # test_linalg.cpp:34-45
    g = orc.Graph(3, [(0, 1, 1.0), (1, 2, 1.0)])
    x = orc.cholesky_solve(g, 1.0, np.array([1.0, 0.0, 0.0]))
    assert x == pytest.approx([0.625, 0.25, 0.125], rel=1e-14)


def test_cholesky_random_laplacians(orc):  # test_linalg.cpp:47-70
    rng = np.random.default_rng(17)
    for _ in range(10):
        n = 4 + int(rng.integers(12))
        edges = [(i, i + 1, 1.0) for i in range(n - 1)]
        edges += [(i, j, 1.0) for i in range(n) for j in range(i + 2, n) if rng.integers(4) == 0]
        g = orc.Graph(n, edges)
        rho = rng.uniform(0.2, 3.0)
        M = rho * orc.laplacian_dense(g) + np.eye(n)
        rhs = rng.standard_normal((n, 3))
        x = orc.cholesky_solve(g, rho, rhs)
        assert np.max(np.abs(M @ x - rhs)) <= 1e-10 * (1.0 + np.max(np.abs(rhs)))
    with pytest.raises(ValueError):
        orc.cholesky_solve(orc.Graph(3, [(0, 1, 1.0)]), -1.0, np.zeros(3))


def test_pcg_frozen_2x2(orc):  # test_linalg.cpp:109-119
    x, it, res, conv = orc.pcg_dense(np.array([[4.0, 1.0], [1.0, 3.0]]), np.array([1.0, 2.0]), 1e-12, 50)
    assert conv and res <= 1e-12
    assert x == pytest.approx([1 / 11, 7 / 11], rel=1e-10)


def test_pcg_identity_one_iteration(orc):  # test_linalg.cpp:121-128
    b = np.array([1.0, -2.0, 3.0, -4.0])
    x, it, res, conv = orc.pcg_dense(np.eye(4), b, 1e-10, 10)
    assert conv and it == 1 and np.linalg.norm(x - b) <= 1e-14


def random_spd(rng, n):
    G = rng.standard_normal((n, n))
    return G @ G.T + 0.5 * np.eye(n)


def test_pcg_dense_and_block(orc):  # test_linalg.cpp:130-161
    rng = np.random.default_rng(29)
    for _ in range(8):
        M = random_spd(rng, 20)
        b = rng.standard_normal(20)
        x, it, res, conv = orc.pcg_dense(M, b, 1e-12, 400, pdiag=np.diag(M))
        ex = np.linalg.solve(M, b)
        assert conv and np.linalg.norm(x - ex) <= 1e-8 * (1 + np.linalg.norm(ex))
    M = random_spd(rng, 12)
    Bm = rng.standard_normal((12, 3))
    X, it, res, conv = orc.pcg_dense(M, Bm, 1e-11, 600)
    ex = np.linalg.solve(M, Bm)
    assert conv and np.max(np.abs(X - ex)) <= 1e-7 * (1 + np.max(np.abs(ex)))


def test_pcg_indefinite_and_zero_rhs(orc):  # test_linalg.cpp:163-173
    with pytest.raises(RuntimeError):
        orc.pcg_dense(-np.eye(3), np.ones(3), 1e-10, 10)
    x, it, res, conv = orc.pcg_dense(np.eye(3), np.zeros(3), 1e-10, 10)
    assert conv and it == 0 and np.all(x == 0)


def test_power_iteration(orc):  # test_linalg.cpp:175-210
    assert orc.power_dense(np.diag([1.0, 5.0])) == pytest.approx(5.0, rel=1e-8)
    assert orc.power_laplacian(orc.Graph(2, [(0, 1, 1.0)])) == pytest.approx(2.0, rel=1e-8)
    assert orc.power_dense(np.zeros((3, 3))) == 0.0
    g = orc.Graph(3, [(0, 1, 1.0), (1, 2, 1.0)])
    assert orc.power_laplacian(g) == pytest.approx(np.linalg.eigvalsh(orc.laplacian_dense(g)).max(), rel=1e-8)
    rng = np.random.default_rng(41)
    for _ in range(6):
        n = 5 + int(rng.integers(10))
        edges = [(i, i + 1, 1.0) for i in range(n - 1)]
        edges += [(i, j, 1.0) for i in range(n) for j in range(i + 2, n) if rng.integers(2) == 0]
        g = orc.Graph(n, edges)
        lm = orc.power_laplacian(g, 1e-12, 20000)
        assert lm == pytest.approx(np.linalg.eigvalsh(orc.laplacian_dense(g)).max(), rel=1e-6)


# ---- solvers (test_solvers.cpp) ---------------------------------------------

FIVE_A = np.array([[0.0, 0.0], [1.0, 0.2], [-0.8, 0.6], [0.3, -0.9], [-0.2, 0.5]])
FIVE_E = [(0, 1, 1.0), (0, 2, 0.7), (0, 3, 0.9), (0, 4, 1.1), (1, 2, 0.6), (1, 3, 0.8), (1, 4, 1.2),
          (2, 3, 0.5), (2, 4, 0.95), (3, 4, 0.65)]


def two_point(a1, a2, w, gamma):  # path.cpp:91-103
    a1, a2 = np.asarray(a1, float), np.asarray(a2, float)
    c = a1 - a2
    nc = np.linalg.norm(c)
    if nc == 0:
        return a1, a2
    s = min(2 * gamma * w / nc, 1.0)
    return a1 - 0.5 * s * c, a2 + 0.5 * s * c


def check_contract(orc, A, g, gamma, q, sol, eps):  # test_solvers.cpp:32-45
    check_contract_q(orc, A, g, gamma, q, sol, eps)


def check_contract_q(orc, A, g, gamma, q, sol, eps):
    """q in {1, 2} as the reference; q = 0 encodes infinity (dual norm l1)."""
    i, j, w, _ = g.arrays()
    r = gamma * w
    for l in range(g.E):
        z = sol.Z[l]
        dn = np.linalg.norm(z) if q == 2 else (np.max(np.abs(z)) if q == 1 else np.sum(np.abs(z)))
        assert dn <= r[l] + (1e-12 if q else 1e-10) * (1 + r[l])  # l1 sums round at d ulp
    fp = orc.primal_objective(A, g, gamma, q, sol.X)
    fd = orc.dual_objective(A, g, gamma, q, sol.Z)
    assert fd <= fp + 1e-10 * (1 + abs(fp))
    if sol.term["converged"]:
        assert abs(fp - fd) / (1 + abs(fp) + abs(fd)) <= eps * (1 + 1e-9)
        assert orc.kkt_residual(A, g, gamma, q, sol.X, sol.Z) <= 10 * eps * (1 + 1e-9)


def test_objectives_two_point(orc):  # test_solvers.cpp:108-136
    A = line([0.0, 2.0])
    g = orc.Graph(2, [(0, 1, 1.0)])
    assert orc.primal_objective(A, g, 0.5, 2, line([0.5, 1.5])) == pytest.approx(0.75, rel=1e-14)
    assert orc.dual_objective(A, g, 0.5, 2, line([-0.5])) == pytest.approx(0.75, rel=1e-14)
    assert orc.dual_objective(A, g, 1.0, 2, line([-1.0])) == pytest.approx(1.0, rel=1e-14)
    with pytest.raises(ValueError):
        orc.dual_objective(A, g, 0.5, 2, line([-0.6]))


@pytest.mark.parametrize("algo", ["admm", "ama", "ssnal"])
def test_two_point_closed_form(orc, algo):  # test_solvers.cpp:164-197
    rng = np.random.default_rng(77)
    for trial in range(12):
        d = 1 + trial % 3
        a1, a2 = rng.uniform(-2, 2, d), rng.uniform(-2, 2, d)
        w, gamma = rng.uniform(0.5, 2.0), rng.uniform(0.05, 1.5)
        A = np.stack([a1, a2])
        g = orc.Graph(2, [(0, 1, w)])
        sol = orc.solve(A, g, gamma, 2, orc.config(algo, epsilon=1e-8))
        x1, x2 = two_point(a1, a2, w, gamma)
        assert sol.term["converged"]
        assert np.max(np.abs(sol.X[0] - x1)) <= 1e-6 and np.max(np.abs(sol.X[1] - x2)) <= 1e-6
        check_contract(orc, A, g, gamma, 2, sol, 1e-8)


@pytest.mark.parametrize("algo", ["admm", "ama", "ssnal"])
def test_trivial_short_circuit(orc, algo):  # test_solvers.cpp:199-215
    A = line([1.0, -3.0])
    for g, gamma in ((orc.Graph(2, [(0, 1, 1.0)]), 0.0), (orc.Graph(2, []), 1.0)):
        sol = orc.solve(A, g, gamma, 2, orc.config(algo))
        assert sol.term["converged"] and sol.term["iterations"] == 0 and sol.term["gap"] == 0.0
        assert np.array_equal(sol.X, A)


@pytest.mark.parametrize("algo", ["admm", "ama", "ssnal"])
def test_warm_start_at_optimum(orc, algo):  # test_solvers.cpp:217-231
    g = orc.Graph(5, FIVE_E)
    cfg = orc.config(algo, epsilon=1e-7)
    cold = orc.solve(FIVE_A, g, 0.15, 2, cfg)
    warm = orc.solve(FIVE_A, g, 0.15, 2, cfg, warm=cold)
    assert warm.term["converged"] and warm.term["iterations"] == 0
    assert np.array_equal(warm.X, cold.X)


def test_warm_start_shape_mismatch(orc):  # test_solvers.cpp:233-242
    g = orc.Graph(5, FIVE_E)
    bogus = orc.Solution(np.zeros((4, 2)), np.zeros((10, 2)), {})
    with pytest.raises(ValueError):
        orc.solve(FIVE_A, g, 0.15, 2, orc.config(), warm=bogus)


def dense_dual_oracle(A, edges, n, gamma, q, steps):  # test_solvers.cpp:69-96
    Bd = dense_incidence(n, edges)
    r = gamma * np.array([e[2] for e in edges])
    step = 1.0 / np.linalg.eigvalsh(Bd @ Bd.T).max()
    At = A.T
    Z = np.zeros((A.shape[1], len(edges)))
    BBt = Bd.T
    for _ in range(steps):
        Z += step * ((At - Z @ BBt) @ Bd)
        if q == 2:
            nz = np.linalg.norm(Z, axis=0)
            s = np.where(nz > r, r / np.where(nz > 0, nz, 1), 1.0)
            Z *= s
        else:
            np.clip(Z, -r, r, out=Z)
    ZBt = Z @ Bd.T
    return -0.5 * np.sum(ZBt * ZBt) + np.sum(ZBt * At)


@pytest.mark.parametrize("q", [2, 1])
def test_solvers_match_dense_dual_oracle(orc, q):  # test_solvers.cpp:244-263
    g = orc.Graph(5, FIVE_E)
    for gamma in (0.05, 0.15):
        oracle = dense_dual_oracle(FIVE_A, FIVE_E, 5, gamma, q, 200000)
        for algo in ("admm", "ama", "ssnal"):
            sol = orc.solve(FIVE_A, g, gamma, q, orc.config(algo, epsilon=1e-9))
            assert sol.term["converged"]
            assert abs(orc.primal_objective(FIVE_A, g, gamma, q, sol.X) - oracle) <= 1e-5
            check_contract(orc, FIVE_A, g, gamma, q, sol, 1e-9)


def test_cross_solver_agreement_mixture(orc):  # test_solvers.cpp:265-294
    A = orc.gaussian_mixture([[-2.0, 0.0], [2.0, 0.0]], 0.5, 25, 93)
    g = orc.knn_weights(A, 5, 0.5)
    for gamma in (0.1, 0.6, 3.0):
        sols = [orc.solve(A, g, gamma, 2, orc.config(a)) for a in ("admm", "ama", "ssnal")]
        for s in sols:
            assert s.term["converged"]
            check_contract(orc, A, g, gamma, 2, s, 1e-6)
        f0 = orc.primal_objective(A, g, gamma, 2, sols[0].X)
        l0 = orc.extract_clusters(sols[0].X, g)[0]
        for s in sols[1:]:
            assert abs(orc.primal_objective(A, g, gamma, 2, s.X) - f0) <= 1e-5 * (1 + abs(f0))
            assert np.array_equal(orc.extract_clusters(s.X, g)[0], l0)


def test_iteration_cap(orc):  # test_solvers.cpp:318-335
    g = orc.Graph(5, FIVE_E)
    sol = orc.solve(FIVE_A, g, 0.2, 2, orc.config("admm", epsilon=1e-12, max_iter=3))
    assert not sol.term["converged"] and sol.term["iterations"] == 3 and sol.term["gap"] > 0
    assert np.all(np.isfinite(sol.X))


@pytest.mark.parametrize("algo", ["admm", "ama", "ssnal"])
def test_deterministic(orc, algo):  # test_solvers.cpp:352-365
    g = orc.Graph(5, FIVE_E)
    s1 = orc.solve(FIVE_A, g, 0.12, 2, orc.config(algo))
    s2 = orc.solve(FIVE_A, g, 0.12, 2, orc.config(algo))
    assert np.array_equal(s1.X, s2.X) and np.array_equal(s1.Z, s2.Z)
    assert s1.term["iterations"] == s2.term["iterations"] and s1.term["gap"] == s2.term["gap"]


def test_al_derivatives_fd(orc):  # test_solvers.cpp:367-397
    g = orc.Graph(5, FIVE_E)
    sigma = 1.7
    rng = np.random.default_rng(55)
    Z = 0.1 * rng.standard_normal((10, 2))
    X = FIVE_A + 0.3 * rng.standard_normal((5, 2))
    Dm = rng.standard_normal((5, 2))
    Dm /= np.linalg.norm(Dm)
    h = 1e-6
    fp = orc.phi_value(FIVE_A, g, 0.3, 2, Z, sigma, X + h * Dm)
    fm = orc.phi_value(FIVE_A, g, 0.3, 2, Z, sigma, X - h * Dm)
    G = orc.phi_gradient(FIVE_A, g, 0.3, 2, Z, sigma, X)
    assert (fp - fm) / (2 * h) == pytest.approx(np.sum(G * Dm), rel=1e-5)
    Gp = orc.phi_gradient(FIVE_A, g, 0.3, 2, Z, sigma, X + h * Dm)
    Gm = orc.phi_gradient(FIVE_A, g, 0.3, 2, Z, sigma, X - h * Dm)
    HD = orc.hessian_apply(FIVE_A, g, 0.3, 2, Z, sigma, X, Dm)
    assert np.linalg.norm(HD - (Gp - Gm) / (2 * h)) <= 1e-5 * (1 + np.linalg.norm(HD))


def test_q1_cross_solver(orc):  # test_solvers.cpp:399-414
    g = orc.Graph(5, FIVE_E)
    vals = []
    for algo in ("admm", "ama", "ssnal"):
        sol = orc.solve(FIVE_A, g, 0.25, 1, orc.config(algo, epsilon=1e-8))
        assert sol.term["converged"]
        check_contract(orc, FIVE_A, g, 0.25, 1, sol, 1e-8)
        vals.append(orc.primal_objective(FIVE_A, g, 0.25, 1, sol.X))
    assert vals[1] == pytest.approx(vals[0], rel=1e-7) and vals[2] == pytest.approx(vals[0], rel=1e-7)


# ---- path (test_path.cpp) ---------------------------------------------------

def test_schedules(orc):  # test_path.cpp:32-59
    s = orc.make_schedule(1.0, 100.0, 3, True)
    assert s == pytest.approx([1.0, 10.0, 100.0], rel=1e-14)
    s = orc.make_schedule(0.45, 0.09, 5, False)
    assert s == pytest.approx([0.09 * (i + 1) for i in range(5)], rel=1e-12)
    assert orc.make_schedule(0.7, 0.7, 1, True).tolist() == [0.7]
    for args in ((1.0, 2.0, 0, False), (0.0, 2.0, 3, True), (-1.0, 2.0, 3, False), (0.5, 0.5, 2, False)):
        with pytest.raises(ValueError):
            orc.make_schedule(*args)


def test_cluster_extraction(orc):  # test_path.cpp:99-146
    chain = orc.Graph(4, [(0, 1, 1.0), (1, 2, 1.0), (2, 3, 1.0)])
    lab, K, cent = orc.extract_clusters(line([0.0, 1.0, 2.0, 3.0]), chain)
    assert K == 4 and lab.tolist() == [0, 1, 2, 3] and cent[2, 0] == 2.0
    lab, K, cent = orc.extract_clusters(line([0.0, 1.0, 1.0, 3.0]), chain)
    assert K == 3 and lab.tolist() == [0, 1, 1, 2] and cent[1, 0] == pytest.approx(1.0)
    lab, K, cent = orc.extract_clusters(np.full((4, 1), 2.5), chain)
    assert K == 1 and cent[0, 0] == pytest.approx(2.5)
    assert orc.extract_clusters(line([0.0, 1.0, 2.0, 0.0]), chain)[1] == 4
    pair = orc.Graph(2, [(0, 1, 1.0)])
    assert orc.extract_clusters(line([1000.0, 1000.5]), pair)[1] == 1
    assert orc.extract_clusters(line([1000.0, 1002.0]), pair)[1] == 2
    assert orc.extract_clusters(line([1000.0, 1000.5]), pair, 1e-5)[1] == 2
    with pytest.raises(ValueError):
        orc.extract_clusters(line([0.0, 1.0, 2.0]), chain)


def test_two_point_path(orc):  # test_path.cpp:148-170
    A = line([0.0, 2.0])
    g = orc.Graph(2, [(0, 1, 1.0)])
    gam = orc.make_schedule(0.1, 10.0, 9, True)
    res = orc.run_path(A, g, 2, gam, orc.config(epsilon=1e-8))
    for t, gamma in enumerate(gam):
        assert res["terms"][t]["converged"]
        assert res["K"][t] == (2 if gamma < 1.0 else 1)
        x1, x2 = two_point(A[0], A[1], 1.0, gamma)
        assert np.max(np.abs(res["X"][t][0] - x1)) <= 1e-6 and np.max(np.abs(res["X"][t][1] - x2)) <= 1e-6


def test_warm_starts_save_iterations(orc):  # test_path.cpp:172-205
    A = orc.gaussian_mixture([[-2.0, 0.0], [2.0, 0.0]], 0.4, 15, 7)
    g = orc.knn_weights(A, 4, 0.5)
    gam = orc.make_schedule(0.05, 5.0, 12, True)
    w = orc.run_path(A, g, 2, gam, orc.config(epsilon=1e-6), warm_start=True)
    c = orc.run_path(A, g, 2, gam, orc.config(epsilon=1e-6), warm_start=False)
    assert all(t["converged"] for t in w["terms"]) and all(t["converged"] for t in c["terms"])
    assert sum(t["iterations"] for t in w["terms"]) <= sum(t["iterations"] for t in c["terms"])
    assert np.max(np.abs(w["X"] - c["X"])) <= 1e-3


def test_unconverged_path_continues(orc):  # test_path.cpp:207-229
    A = np.array([[0.0, 0.0], [1.0, 0.7], [5.0, -0.3]])
    g = orc.Graph(3, [(0, 1, 1.0), (1, 2, 1.0)])
    res = orc.run_path(A, g, 2, orc.make_schedule(0.2, 2.0, 4, True),
                       orc.config("admm", epsilon=1e-10, max_iter=2), warm_start=False)
    assert not any(t["converged"] for t in res["terms"]) and np.all(np.isfinite(res["X"]))


def test_disconnected_rejected_only_when_required(orc):  # test_path.cpp:231-245
    A = line([0.0, 1.0, 10.0, 11.0])
    g = orc.Graph(4, [(0, 1, 1.0), (2, 3, 1.0)])
    gam = orc.make_schedule(0.5, 1.0, 2, True)
    with pytest.raises(RuntimeError):
        orc.run_path(A, g, 2, gam, orc.config(), require_connected=True)
    res = orc.run_path(A, g, 2, gam, orc.config())
    assert all(t["converged"] for t in res["terms"]) and res["K"][-1] >= 2


def test_mixture_generator_deterministic(orc):  # test_io.cpp:157-183
    a = orc.gaussian_mixture([[0.0, 0.0], [3.0, 3.0]], 0.5, 10, 123)
    b = orc.gaussian_mixture([[0.0, 0.0], [3.0, 3.0]], 0.5, 10, 123)
    assert np.array_equal(a, b) and a.shape == (20, 2)
    z = orc.gaussian_mixture([[1.0, 2.0]], 0.0, 3, 1)
    assert np.array_equal(z, np.array([[1.0, 2.0]] * 3))
