"""run_bench / perf_profile_csv (bench.hpp; bench.cpp:23-116) over GPU solves: the cases of
the reference's test_bench.cpp:34-140 on the same fixture."""
import numpy as np
import pytest

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def task(cp):
    A = cp.generate_gaussian_mixture(np.array([[-2.0, 0.0], [2.0, 0.0]]), 0.4, 10, 11)
    data = cp.DataMatrix(A)
    g = cp.compute_knn_weights(data, 4, 0.5)
    return cp.BenchTask(data, g, cp.PenaltyNorm.l2, cp.make_schedule(0.1, 2.0, 5))


def test_single_method_is_its_own_baseline(cp, task):
    prof = cp.run_bench([task], [cp.Algorithm.SSNAL], cp.BenchOptions(epsilon=1e-6))
    assert prof.problem_count == 5 and prof.baseline_T > 0
    (c,) = prof.curves
    assert c.method == cp.Algorithm.SSNAL and c.solved_total == 5
    assert c.full_time == pytest.approx(prof.baseline_T)
    assert len(c.points) == 10 and c.points[0] == (1.0, 5)
    assert all(s == 5 for _, s in c.points)


def test_curves_nondecreasing_and_bounded(cp, task):
    prof = cp.run_bench([task], [cp.Algorithm.SSNAL, cp.Algorithm.ADMM, cp.Algorithm.FastAMA],
                        cp.BenchOptions(epsilon=1e-6))
    assert prof.problem_count == 5 and len(prof.curves) == 3
    for c in prof.curves:
        solved = [s for _, s in c.points]
        assert len(solved) == 10 and solved == sorted(solved) and max(solved) <= 5
        assert c.solved_total <= 5 and solved[-1] == c.solved_total
    for c in prof.curves:
        if c.solved_total == prof.problem_count:
            assert c.full_time >= prof.baseline_T


def test_zero_cutoff_leaves_curves_at_zero(cp, task):
    prof = cp.run_bench([task], [cp.Algorithm.SSNAL, cp.Algorithm.ADMM],
                        cp.BenchOptions(epsilon=1e-6, cutoff_override=0.0))
    for c in prof.curves:
        assert c.solved_total == 0 and all(s == 0 for _, s in c.points) and c.full_time > 0


def test_throws_when_nothing_converges(cp, task):
    opts = cp.BenchOptions(epsilon=1e-14, base_config=cp.SolverConfig(max_iter=1))
    with pytest.raises(RuntimeError):
        cp.run_bench([task], [cp.Algorithm.ADMM, cp.Algorithm.FastAMA], opts)


def test_validates_inputs(cp, task):
    with pytest.raises(ValueError):
        cp.run_bench([], [cp.Algorithm.SSNAL])
    with pytest.raises(ValueError):
        cp.run_bench([task], [])
    with pytest.raises(ValueError):
        cp.run_bench([cp.BenchTask(None, task.graph, cp.PenaltyNorm.l2, task.schedule)], [cp.Algorithm.SSNAL])
    empty = cp.make_schedule(0.1, 2.0, 5)
    empty.values = []
    with pytest.raises(ValueError):
        cp.run_bench([cp.BenchTask(task.data, task.graph, cp.PenaltyNorm.l2, empty)], [cp.Algorithm.SSNAL])
    with pytest.raises(ValueError):
        cp.run_bench([task], [cp.Algorithm.SSNAL], cp.BenchOptions(tau_max=0))


def test_profile_csv(cp, task):
    prof = cp.run_bench([task], [cp.Algorithm.SSNAL, cp.Algorithm.ADMM], cp.BenchOptions(tau_max=3))
    lines = cp.perf_profile_csv(prof).splitlines()
    assert lines[0] == "method,tau,solved"
    assert len(lines) == 7 and all(x.startswith(("ssnal,", "admm,")) for x in lines[1:])
    assert any(x.startswith("ssnal,1,") for x in lines) and any(x.startswith("admm,3,") for x in lines)
