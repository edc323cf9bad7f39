"""linalg.hpp:17-87 through the C-ABI (LinearOperator, pcg, power_iteration,
CholeskyFactor) and prox.hpp:14-26's norms / *_into forms, against the CPU
oracle's restatement of linalg.cpp and numpy.  Cases follow
test_linalg.cpp:35-212 (the same seeds and shapes)."""
import numpy as np
import pytest
import scipy.sparse as sp

pytestmark = pytest.mark.gpu


def random_spd(rng, n):
    G = rng.standard_normal((n, n))
    M = G @ G.T
    M[np.diag_indices(n)] += 0.5
    return M


def test_factories_agree_with_dense(cp):
    rng = np.random.default_rng(3)
    M = random_spd(rng, 5)
    dense = cp.LinearOperator.dense(M, True)
    assert dense.rows() == 5 and dense.symmetric() and dense.positive_definite()
    sparse = cp.LinearOperator.sparse(sp.csc_matrix(M), True)
    X = rng.standard_normal((5, 2))
    assert np.max(np.abs(dense.apply(X) - M @ X)) <= 1e-14
    assert np.max(np.abs(sparse.apply(X) - M @ X)) <= 1e-14
    assert np.array_equal(cp.LinearOperator.identity(5).apply(X), X)
    d = np.array([1.0, 2, 4, 8, 16])
    assert np.allclose(cp.LinearOperator.jacobi(d).apply(X), X / d[:, None], rtol=1e-15)
    with pytest.raises(ValueError):
        cp.LinearOperator.jacobi(np.zeros(3))
    with pytest.raises(ValueError):
        dense.apply(np.zeros((4, 1)))
    with pytest.raises(ValueError):
        cp.LinearOperator.dense(np.ones((2, 3)))
    assert not cp.LinearOperator.dense(np.array([[1.0, 2.0], [0.0, 1.0]])).symmetric()


def test_pcg_matches_oracle_and_dense_solves(cp, orc):
    rng = np.random.default_rng(29)
    for _ in range(6):
        M = random_spd(rng, 20)
        b = rng.standard_normal(20)
        res = cp.pcg(cp.LinearOperator.dense(M, True), b, cp.LinearOperator.jacobi(np.diag(M).copy()), 1e-12, 400)
        ox, oit, ores, oconv = orc.pcg_dense(M, b, 1e-12, 400, np.diag(M).copy())
        assert res.converged and oconv
        exact = np.linalg.solve(M, b)
        assert np.linalg.norm(res.x - exact) <= 1e-8 * (1 + np.linalg.norm(exact))
        assert abs(res.iterations - oit) <= 1  # same algorithm, different dot-product order
        assert res.residual <= 1e-12
    # block right-hand side: one Krylov sequence, worst relative row residual (linalg.cpp:128-139)
    M = random_spd(rng, 12)
    B = rng.standard_normal((12, 3))
    res = cp.pcg(cp.LinearOperator.dense(M, True), B, None, 1e-11, 600)
    assert res.converged and res.x.shape == (12, 3)
    assert np.max(np.abs(res.x - np.linalg.solve(M, B))) <= 1e-7 * (1 + np.max(np.abs(np.linalg.solve(M, B))))


def test_pcg_edge_cases(cp):
    res = cp.pcg(cp.LinearOperator.identity(4), np.array([1.0, -2, 3, -4]), None, 1e-10, 10)
    assert res.converged and res.iterations == 1
    with pytest.raises(RuntimeError):
        cp.pcg(cp.LinearOperator.dense(-np.eye(3)), np.ones(3), None, 1e-10, 10)
    res = cp.pcg(cp.LinearOperator.identity(3), np.zeros(3), None, 1e-10, 10)
    assert res.converged and res.iterations == 0 and not res.x.any()
    with pytest.raises(ValueError):
        cp.pcg(cp.LinearOperator.identity(3), np.ones(3), None, -1.0, 10)


def test_callback_operator(cp):
    M = np.array([[4.0, 1.0], [1.0, 3.0]])
    calls = []

    def fn(x):
        calls.append(1)
        return M @ x

    op = cp.LinearOperator(2, fn, True, True)
    res = cp.pcg(op, np.array([1.0, 2.0]), None, 1e-12, 50)
    assert res.converged and np.allclose(res.x, [1 / 11, 7 / 11], rtol=1e-10) and len(calls) >= 2
    assert cp.power_iteration(op) == pytest.approx(3.5 + np.sqrt(1.25), rel=1e-8)

    def bad(x):
        raise ValueError("functor says no")

    with pytest.raises(ValueError, match="functor says no"):
        cp.pcg(cp.LinearOperator(2, bad), np.ones(2), None, 1e-12, 5)


def test_power_iteration(cp, orc):
    assert cp.power_iteration(cp.LinearOperator.dense(np.diag([1.0, 5.0]), True)) == pytest.approx(5.0, rel=1e-8)
    assert cp.power_iteration(cp.LinearOperator.dense(np.zeros((3, 3)))) == 0.0
    rng = np.random.default_rng(41)
    for _ in range(4):
        n = 5 + int(rng.integers(10))
        edges = [(i, i + 1, 1.0) for i in range(n - 1)]
        edges += [(i, j, 1.0) for i in range(n) for j in range(i + 2, n) if rng.integers(2) == 0]
        g = cp.WeightedGraph(n, edges)
        L = cp.IncidenceOperator(g).laplacian()
        lm = cp.power_iteration(cp.LinearOperator.sparse(L), 1e-12, 20000)
        assert lm == pytest.approx(np.linalg.eigvalsh(L.toarray()).max(), rel=1e-6)
        assert lm == pytest.approx(orc.power_dense(L.toarray(), 1e-12, 20000), rel=1e-9)


def test_cholesky_factor(cp, orc):
    g = cp.WeightedGraph(3, [(0, 1, 1.0), (1, 2, 1.0)])
    f = cp.CholeskyFactor(cp.IncidenceOperator(g).laplacian(), 1.0)
    assert f.size() == 3 and f.rho() == 1.0
    x = f.solve(np.array([1.0, 0.0, 0.0]))
    assert np.allclose(x, [0.625, 0.25, 0.125], rtol=1e-14, atol=0)
    rng = np.random.default_rng(17)
    for _ in range(6):
        n = 4 + int(rng.integers(12))
        edges = [(i, i + 1, 1.0) for i in range(n - 1)]
        edges += [(i, j, 1.0) for i in range(n) for j in range(i + 2, n) if rng.integers(4) == 0]
        g = cp.WeightedGraph(n, edges)
        og = orc.Graph(n, edges)
        rho = float(rng.uniform(0.2, 3.0))
        L = cp.IncidenceOperator(g).laplacian()
        M = np.eye(n) + rho * L.toarray()
        rhs = rng.standard_normal((n, 3))
        X = cp.CholeskyFactor(L, rho).solve(rhs)
        assert np.max(np.abs(M @ X - rhs)) <= 1e-10 * (1 + np.max(np.abs(rhs)))
        assert np.max(np.abs(X - orc.cholesky_solve(og, rho, rhs))) <= 1e-12 * (1 + np.max(np.abs(X)))
    with pytest.raises(ValueError):
        cp.CholeskyFactor(cp.IncidenceOperator(g).laplacian(), -1.0)
    with pytest.raises(ValueError):
        cp.CholeskyFactor(sp.csc_matrix(np.array([[0.0, 1.0], [0.0, 0.0]])), 1.0)


def test_norms_and_into_forms(cp, orc):
    rng = np.random.default_rng(5)
    for q in (1, 2, 0):
        for _ in range(20):
            v = rng.standard_normal(1 + int(rng.integers(40)))
            a, b = orc.norms(q, v)
            assert cp.norm_value(v, q) == pytest.approx(a, rel=1e-14)
            assert cp.dual_norm_value(v, q) == pytest.approx(b, rel=1e-14)
    out = np.empty(2)
    cp.prox_norm_into(np.array([3.0, 4.0]), 2.5, cp.PenaltyNorm.l2, out)
    assert np.allclose(out, [1.5, 2.0], rtol=1e-15)
    cp.project_dual_ball_into(np.array([3.0, -0.5]), 1.0, cp.PenaltyNorm.l1, out)
    assert np.array_equal(out, [1.0, -0.5])


def test_trace_and_path_centroids(cp, orc):
    rng = np.random.default_rng(9)
    A = np.concatenate([rng.normal(0, 0.2, (20, 3)), rng.normal(3, 0.2, (20, 3))])
    data = cp.DataMatrix(A)
    g = cp.compute_knn_weights(data, 5, 0.5)
    og = orc.knn_weights(A, 5, 0.5)
    for algo in ("ssnal", "admm", "ama"):
        cfg = cp.SolverConfig(algorithm=cp.algorithm_from_name(algo), collect_trace=True)
        sol = cp.solve(cp.ProblemInstance(data, g, 0.2, 2), cfg)
        tr = sol.trace
        assert tr and tr[0].iter == 0 and tr[-1].gap == sol.termination.gap
        assert all(b.elapsed_s >= a.elapsed_s for a, b in zip(tr, tr[1:]))
    sched = cp.make_schedule(0.01, 5.0, 6)
    res = cp.run_path(data, g, 2, sched, cp.SolverConfig(collect_trace=True))
    ores = orc.run_path(A, og, 2, sched.values, orc.config())
    for t in range(len(sched.values)):
        a = res.assignments[t]
        ol, oK, oc = orc.extract_clusters(ores["X"][t], og)
        assert a.K == oK and a.centroids.shape == (a.K, 3)
        ref = cp.extract_clusters(res.solutions[t].X, g)
        assert np.array_equal(a.centroids, ref.centroids)
        assert np.max(np.abs(a.centroids - oc)) <= 1e-6 * (1 + np.max(np.abs(oc)))
        assert res.solutions[t].trace and res.solutions[t].trace[-1].gap == res.stats[t].gap
