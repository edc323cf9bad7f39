"""Where does the end-to-end C3 path (host in, every X and Z out) spend its time?  Runs the
bench's e2e call twice (the first fills the pinned pool) with CPB_TRACE timestamps."""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import bench  # noqa: E402
import paper_2501_15964_b200 as cp  # noqa: E402

cfg = bench.CONFIGS[sys.argv[1] if len(sys.argv) > 1 else "c3"]
A = bench.make_input(cp, cfg)
ctx = cp.default_context()
sched = cp.make_schedule(cfg["gamma"][0], cfg["gamma"][1], cfg["T"])
scfg = cp.SolverConfig(algorithm=cp.algorithm_from_name(cfg["algorithm"]))
for rep in range(3):
    t0 = time.perf_counter()
    dA = cp.DataMatrix(A, ctx=ctx)
    t1 = time.perf_counter()
    g = cp.compute_knn_weights(dA, cfg["k"], cfg["phi"])
    t2 = time.perf_counter()
    res = cp.run_path(dA, g, cfg["q"], sched, scfg, keep_solutions=True, keep_z=True)
    t3 = time.perf_counter()
    del res
    t4 = time.perf_counter()
    print(f"rep {rep}: data {t1 - t0:.3f} knn {t2 - t1:.3f} run_path {t3 - t2:.3f} del {t4 - t3:.3f} total {t4 - t0:.3f}",
          file=sys.stderr, flush=True)
