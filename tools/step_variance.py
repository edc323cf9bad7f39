"""Full-path step times back to back, with and without kernel statistics."""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import bench  # noqa: E402
import paper_2501_15964_b200 as cp  # noqa: E402

cfg = bench.CONFIGS[sys.argv[1] if len(sys.argv) > 1 else "c3"]
A = bench.make_input(cp, cfg)
ctx = cp.default_context()
data = cp.DataMatrix(A)
sched = cp.make_schedule(cfg["gamma"][0], cfg["gamma"][1], cfg["T"])
conf = cp.SolverConfig(algorithm=cp.algorithm_from_name(cfg["algorithm"]))
for stats in (False, True, False):
    ctx.stats_enable(stats)
    for s in range(3):
        cp.flush_l2(ctx)
        ctx.synchronize()
        t0 = time.perf_counter()
        cp.timer_start(ctx)
        g = cp.compute_knn_weights(data, cfg["k"], cfg["phi"])
        ctx.synchronize()
        t1 = time.perf_counter()
        res = cp.run_path(data, g, cfg["q"], sched, conf, keep_solutions=False)
        t2 = time.perf_counter()
        print(f"   knn+graph {t1 - t0:.4f} s run_path {t2 - t1:.4f} s sum(wall_time) {sum(t.wall_time for t in res.stats):.4f}")
        dev = cp.timer_stop(ctx) / 1e3
        print(f"stats={stats} step {s}: device {dev:.4f} s wall {time.perf_counter() - t0:.4f} s "
              f"cg {sum(t.cg for t in res.stats)} per-gamma " + " ".join(f"{t.wall_time:.3f}" for t in res.stats),
              flush=True)
