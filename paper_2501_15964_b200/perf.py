"""Performance profiles over GPU solves (bench.hpp / bench.cpp:23-116 of the
reference): the paper's protocol of an uncapped sweep
per method to fix the baseline T (the method solving most problems, then the
fastest), then a capped sweep with a 10 T wall-clock budget from which the
curve "problems solved within tau T", tau = 1..tau_max, is read.

Problems are timed by each solve's own wall clock (TerminationRecord.wall_time,
bench.cpp:18-20), so host bookkeeping and the warm-start transfers stay out of
the measurement.  Every solve runs on the B200 through cp_solve.
"""
from __future__ import annotations

import copy
from dataclasses import dataclass, field
from typing import List, Optional, Sequence, Tuple

from .cluspath import (Algorithm, DataMatrix, GammaSchedule, PenaltyNorm, ProblemInstance, SolverConfig, WeightedGraph,
                       algorithm_name, solve)
from .io import format_double


@dataclass
class BenchTask:
    """One workload: a dataset, its graph and a gamma schedule; every gamma is one problem."""
    data: Optional[DataMatrix]
    graph: Optional[WeightedGraph]
    norm: object = PenaltyNorm.l2
    schedule: GammaSchedule = None


@dataclass
class MethodCurve:
    method: Algorithm
    points: List[Tuple[float, int]] = field(default_factory=list)  # (tau, solved within tau T)
    solved_total: int = 0
    full_time: float = 0.0  # uncapped full-sweep wall time


@dataclass
class PerfProfile:
    baseline_T: float = 0.0
    problem_count: int = 0
    curves: List[MethodCurve] = field(default_factory=list)


@dataclass
class BenchOptions:
    epsilon: float = 1e-6
    tau_max: int = 10
    cutoff_override: Optional[float] = None  # replaces 10 T (testing hook; 0: no problem may start)
    base_config: SolverConfig = field(default_factory=SolverConfig)  # algorithm overridden per method
    warm_start: bool = True


@dataclass
class _Sweep:
    finish: List[float] = field(default_factory=list)  # cumulative wall time at each solved problem
    total_time: float = 0.0


def _sweep(tasks: Sequence[BenchTask], method, options: BenchOptions, budget: Optional[float]) -> _Sweep:
    """bench.cpp:23-50: every task's schedule with one method; a budget is checked before each
    solve and passed down as the remaining per-solve time limit."""
    out = _Sweep()
    for task in tasks:
        prev = None
        for gamma in task.schedule.values:
            if budget is not None and out.total_time >= budget:
                return out
            cfg = copy.copy(options.base_config)
            cfg.algorithm = method
            cfg.epsilon = options.epsilon
            if budget is not None:
                remaining = budget - out.total_time
                cfg.time_limit = min(cfg.time_limit, remaining) if cfg.time_limit else remaining
            inst = ProblemInstance(task.data, task.graph, gamma, task.norm)
            sol = solve(inst, cfg, prev if options.warm_start else None)
            out.total_time += sol.termination.wall_time
            if sol.termination.converged and (budget is None or out.total_time <= budget):
                out.finish.append(out.total_time)
            prev = sol  # unconverged paths continue from the best iterate
    return out


def run_bench(tasks: Sequence[BenchTask], methods: Sequence, options: Optional[BenchOptions] = None) -> PerfProfile:
    """run_bench (bench.hpp:50-52; bench.cpp:54-116)."""
    options = options or BenchOptions()
    if not methods:
        raise ValueError("run_bench: no methods given")
    if not tasks:
        raise ValueError("run_bench: no tasks given")
    problems = 0
    for t in tasks:
        if t.data is None or t.graph is None:
            raise ValueError("run_bench: task is missing data or graph")
        if t.schedule is None or len(t.schedule.values) == 0:
            raise ValueError("run_bench: task has an empty schedule")
        problems += len(t.schedule.values)
    if options.tau_max < 1:
        raise ValueError("run_bench: tau_max must be >= 1")
    options.base_config.to_c()  # validates (objective.cpp:43-61)
    uncapped = [_sweep(tasks, m, options, None) for m in methods]
    best = 0
    for i in range(1, len(methods)):
        more = len(uncapped[i].finish) > len(uncapped[best].finish)
        tie_faster = (len(uncapped[i].finish) == len(uncapped[best].finish)
                      and uncapped[i].total_time < uncapped[best].total_time)
        if more or tie_faster:
            best = i
    if not uncapped[best].finish:
        raise RuntimeError("run_bench: no baseline (no method solved any problem)")
    T = uncapped[best].total_time
    cutoff = options.cutoff_override if options.cutoff_override is not None else 10.0 * T
    prof = PerfProfile(baseline_T=T, problem_count=problems)
    for i, m in enumerate(methods):
        # a sweep that already fits inside the budget replays identically under the cap
        capped = uncapped[i] if uncapped[i].total_time <= cutoff else _sweep(tasks, m, options, cutoff)
        curve = MethodCurve(method=m, full_time=uncapped[i].total_time, solved_total=len(capped.finish))
        for tau in range(1, options.tau_max + 1):
            horizon = min(float(tau) * T, cutoff)
            curve.points.append((float(tau), sum(1 for t in capped.finish if t <= horizon)))
        prof.curves.append(curve)
    return prof


def perf_profile_csv(profile: PerfProfile) -> str:
    """perf_profile_csv (bench.hpp:55): header "method,tau,solved", one row per curve point."""
    rows = ["method,tau,solved"]
    for c in profile.curves:
        for tau, solved in c.points:
            rows.append(f"{algorithm_name(c.method)},{format_double(tau)},{solved}")
    return "\n".join(rows) + "\n"
