"""Property tests (hypothesis) of the prox / projection pair the path is built
on (prox.cpp:25-138, and q = infinity from SURVEY.md §8(c)), on the CPU oracle:
Moreau decomposition, dual-ball feasibility, the projection's variational
inequality, and prox optimality against a brute-force line search."""
import numpy as np
import pytest
from hypothesis import given, settings
from hypothesis import strategies as st

vec = st.lists(st.floats(-50, 50, allow_nan=False, allow_infinity=False), min_size=1, max_size=9)
thr = st.floats(0.0, 40.0, allow_nan=False, allow_infinity=False)


def dual_norm(q, z):
    return np.linalg.norm(z) if q == 2 else (np.abs(z).max() if q == 1 else np.abs(z).sum())


def norm(q, x):
    return np.linalg.norm(x) if q == 2 else (np.abs(x).sum() if q == 1 else np.abs(x).max())


@pytest.mark.parametrize("q", [0, 1, 2])
@settings(max_examples=300, deadline=None)
@given(v=vec, t=thr)
def test_moreau_and_feasibility(orc, q, v, t):
    v = np.array(v)
    p = orc.prox_columns(q, [v], [t])[0]
    z = orc.project_columns(q, [v], [t])[0]
    scale = 1.0 + np.abs(v).sum()
    assert np.max(np.abs(p + z - v)) <= 1e-12 * scale           # v = prox + projection
    assert dual_norm(q, z) <= t * (1 + 1e-12) + 1e-12 * scale    # projection is in the dual ball
    # variational inequality of the projection against random points of the ball
    rng = np.random.default_rng(abs(hash((q, len(v)))) % (2 ** 32))
    for _ in range(5):
        y = rng.normal(size=v.shape)
        dn = dual_norm(q, y)
        y = y * (t / dn) if dn > 0 else y
        assert np.dot(v - z, y - z) <= 1e-9 * scale * (1 + t)


@pytest.mark.parametrize("q", [0, 1, 2])
@settings(max_examples=150, deadline=None)
@given(v=vec, t=thr)
def test_prox_minimises_the_model(orc, q, v, t):
    """prox_{t||.||}(v) minimises 1/2||x - v||^2 + t||x||: no random
    perturbation of it does better."""
    v = np.array(v)
    p = orc.prox_columns(q, [v], [t])[0]
    f = lambda x: 0.5 * np.sum((x - v) ** 2) + t * norm(q, x)  # noqa: E731
    fp = f(p)
    rng = np.random.default_rng(len(v) + 17 * q)
    for h in (1e-3, 1e-1, 1.0):
        for _ in range(10):
            assert fp <= f(p + h * rng.normal(size=v.shape)) + 1e-9 * (1 + abs(fp))
