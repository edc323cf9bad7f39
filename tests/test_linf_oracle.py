"""q = infinity in the CPU oracle.

There is no reference implementation (prox.cpp:17-21 rejects q outside
{1, 2}), so this oracle is "parity unpinned": it is checked here against
independent restatements of the math with the same property tests the
reference uses for q in {1, 2} (test_prox.cpp:78-144, test_solvers.cpp:244-414):
prox optimality against a bisection solve, Moreau identity, Jacobian against
finite differences, the dense projected-gradient dual oracle and cross-solver
agreement.  q = infinity is passed as 0 through the C-ABIs.
"""
import numpy as np
import pytest

from test_oracle_kat import FIVE_A, FIVE_E, check_contract_q, dense_incidence

QI = 0


def l1_theta_bisect(v, t):
    """theta with sum max(|v| - theta, 0) = t by bisection (independent of the sort)."""
    a = np.abs(v)
    if a.sum() <= t:
        return -1.0
    lo, hi = 0.0, a.max()
    for _ in range(200):
        mid = 0.5 * (lo + hi)
        if np.maximum(a - mid, 0).sum() > t:
            lo = mid
        else:
            hi = mid
    return 0.5 * (lo + hi)


def test_prox_and_projection_match_bisection(orc):
    rng = np.random.default_rng(7)
    for _ in range(500):
        d = 1 + rng.integers(9)
        v = rng.normal(0, 2.0, d)
        t = rng.uniform(0.0, 4.0)
        th = l1_theta_bisect(v, t)
        p = orc.prox_columns(QI, [v], [t])[0]
        z = orc.project_columns(QI, [v], [t])[0]
        want_p = np.zeros(d) if th < 0 else np.clip(v, -th, th)
        want_z = v if th < 0 else np.sign(v) * np.maximum(np.abs(v) - th, 0)
        assert np.max(np.abs(p - want_p)) <= 1e-12 * (1 + np.abs(v).max())
        assert np.max(np.abs(z - want_z)) <= 1e-12 * (1 + np.abs(v).max())
        # prox optimality: v - p in t * subdifferential of ||.||_inf at p
        r = v - p
        if np.any(p != 0):
            assert abs(np.abs(r).sum() - t) <= 1e-10 * (1 + t)
            big = np.abs(p) >= np.abs(p).max() - 1e-12
            assert np.all((np.abs(r) <= 1e-12) | big)
            assert np.all(r[big] * p[big] >= -1e-12)


def test_norms_and_moreau(orc):
    assert orc.norms(QI, [3.0, -4.0]) == (4.0, 7.0)  # ||.||_inf and its dual ||.||_1
    rng = np.random.default_rng(42)
    for _ in range(1000):
        v = rng.normal(0.0, 2.0, size=1 + rng.integers(6))
        assert orc.moreau_check(QI, v, rng.uniform(0.0, 3.0)) <= 1e-12


def test_prox_edge_cases(orc):
    v = np.array([3.0, -1.0, 0.5])
    assert np.array_equal(orc.prox_columns(QI, [v], [0.0])[0], v)          # t = 0: identity
    assert np.all(orc.prox_columns(QI, [v], [4.5])[0] == 0)                # inside the l1 ball
    assert np.array_equal(orc.prox_columns(QI, [v], [1.0])[0], [2.0, -1.0, 0.5])  # theta = 2
    assert np.array_equal(orc.project_columns(QI, [v], [1.0])[0], [1.0, 0.0, 0.0])
    assert np.all(orc.project_columns(QI, [v], [0.0])[0] == 0)
    J, _, _ = orc.prox_jacobian(QI, v, 0.0)
    assert np.array_equal(J, np.eye(3))
    assert np.all(orc.prox_jacobian(QI, v, 10.0)[0] == 0)
    # theta = 2, S = {0}: M = I - (e0 e0^T - e0 e0^T) = I
    assert np.allclose(orc.prox_jacobian(QI, v, 1.0)[0], np.eye(3))
    # theta = 1.75 with S = {0, 1} for t = 1.25 + 0.75... use a two-element support
    w = np.array([3.0, -2.5, 0.5])
    J, _, _ = orc.prox_jacobian(QI, w, 1.0)  # theta = 2.25, S = {0, 1}, s = (+, -)
    s = np.array([1.0, -1.0, 0.0])
    want = np.eye(3) - (np.diag([1.0, 1.0, 0.0]) - np.outer(s, s) / 2)
    assert np.allclose(J, want, atol=1e-15)
    assert np.allclose(orc.prox_jacobian_diag(QI, w, 1.0), np.diag(want), atol=1e-15)


def test_jacobian_matches_fd(orc):
    rng = np.random.default_rng(5)
    h = 1e-7
    acc = 0
    while acc < 200:
        d = 2 + rng.integers(5)
        v = rng.normal(0, 2.0, d)
        t = rng.uniform(0.1, 3.0)
        th = l1_theta_bisect(v, t)
        if th >= 0 and np.min(np.abs(np.abs(v) - th)) < 1e-2:
            continue  # kink of the support
        if abs(np.abs(v).sum() - t) < 1e-2:
            continue  # boundary of the ball
        acc += 1
        J, _, _ = orc.prox_jacobian(QI, v, t)
        w = rng.normal(0, 1.0, d)
        fd = (orc.prox_columns(QI, [v + h * w], [t])[0] - orc.prox_columns(QI, [v - h * w], [t])[0]) / (2 * h)
        assert np.linalg.norm(J @ w - fd) <= 1e-6 * (1.0 + np.linalg.norm(fd))


def project_l1_cols(Z, r):
    """Column-wise l1-ball projection (sort-based, vectorised over columns)."""
    a = np.abs(Z)
    u = -np.sort(-a, axis=0)
    cs = np.cumsum(u, axis=0)
    j = np.arange(1, Z.shape[0] + 1)[:, None]
    th_all = (cs - r[None, :]) / j
    ok = u - th_all > 0
    rho = Z.shape[0] - 1 - np.argmax(ok[::-1], axis=0)
    th = th_all[rho, np.arange(Z.shape[1])]
    inside = a.sum(axis=0) <= r
    out = np.sign(Z) * np.maximum(a - th[None, :], 0)
    out[:, inside] = Z[:, inside]
    return out


def dense_dual_oracle_inf(A, edges, n, gamma, steps):
    """Projected gradient on the dual with l1-ball projections (the q = inf
    counterpart of test_solvers.cpp:69-96)."""
    Bd = dense_incidence(n, edges)
    r = gamma * np.array([e[2] for e in edges])
    step = 1.0 / np.linalg.eigvalsh(Bd @ Bd.T).max()
    At = A.T
    Z = np.zeros((A.shape[1], len(edges)))
    for _ in range(steps):
        Z += step * ((At - Z @ Bd.T) @ Bd)
        Z = project_l1_cols(Z, r)
    ZBt = Z @ Bd.T
    return -0.5 * np.sum(ZBt * ZBt) + np.sum(ZBt * At)


def test_solvers_match_dense_dual_oracle(orc):
    g = orc.Graph(5, FIVE_E)
    for gamma in (0.05, 0.15):
        oracle = dense_dual_oracle_inf(FIVE_A, FIVE_E, 5, gamma, 20000)
        for algo in ("admm", "ama", "ssnal"):
            sol = orc.solve(FIVE_A, g, gamma, QI, orc.config(algo, epsilon=1e-9))
            assert sol.term["converged"]
            assert abs(orc.primal_objective(FIVE_A, g, gamma, QI, sol.X) - oracle) <= 1e-5
            check_contract_q(orc, FIVE_A, g, gamma, QI, sol, 1e-9)


def test_cross_solver_agreement_mixture(orc):
    A = orc.gaussian_mixture([[-2.0, 0.0, 1.0], [2.0, 0.0, -1.0]], 0.5, 20, 93)
    g = orc.knn_weights(A, 5, 0.5)
    for gamma in (0.1, 0.6):
        sols = [orc.solve(A, g, gamma, QI, orc.config(a, epsilon=1e-8)) for a in ("admm", "ama", "ssnal")]
        for s in sols:
            assert s.term["converged"]
            check_contract_q(orc, A, g, gamma, QI, s, 1e-8)
        f0 = orc.primal_objective(A, g, gamma, QI, sols[0].X)
        for s in sols[1:]:
            assert abs(orc.primal_objective(A, g, gamma, QI, s.X) - f0) <= 1e-6 * (1 + abs(f0))


def test_al_derivatives_fd(orc):
    g = orc.Graph(5, FIVE_E)
    sigma = 1.7
    rng = np.random.default_rng(55)
    Z = 0.1 * rng.standard_normal((10, 2))
    X = FIVE_A + 0.3 * rng.standard_normal((5, 2))
    Dm = rng.standard_normal((5, 2))
    Dm /= np.linalg.norm(Dm)
    h = 1e-6
    fp = orc.phi_value(FIVE_A, g, 0.3, QI, Z, sigma, X + h * Dm)
    fm = orc.phi_value(FIVE_A, g, 0.3, QI, Z, sigma, X - h * Dm)
    G = orc.phi_gradient(FIVE_A, g, 0.3, QI, Z, sigma, X)
    assert (fp - fm) / (2 * h) == pytest.approx(np.sum(G * Dm), rel=1e-5)
    Gp = orc.phi_gradient(FIVE_A, g, 0.3, QI, Z, sigma, X + h * Dm)
    Gm = orc.phi_gradient(FIVE_A, g, 0.3, QI, Z, sigma, X - h * Dm)
    HD = orc.hessian_apply(FIVE_A, g, 0.3, QI, Z, sigma, X, Dm)
    assert np.linalg.norm(HD - (Gp - Gm) / (2 * h)) <= 1e-5 * (1 + np.linalg.norm(HD))
