"""Where the C3 end-to-end time goes: run_path with every X, Z returned (pinned
host buffers) vs X only vs labels only, same graph, warm context."""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import bench  # noqa: E402
import paper_2501_15964_b200 as cp  # noqa: E402

cfg = bench.CONFIGS[sys.argv[1] if len(sys.argv) > 1 else "c3"]
A = bench.make_input(cp, cfg)
data = cp.DataMatrix(A)
g = cp.compute_knn_weights(data, cfg["k"], cfg["phi"])
sched = cp.make_schedule(cfg["gamma"][0], cfg["gamma"][1], cfg["T"])
scfg = cp.SolverConfig()
modes = (("labels only", False, False), ("X", True, False), ("X+Z", True, True))
if len(sys.argv) > 2 and sys.argv[2] == "xz":
    modes = modes[2:]
for name, ks, kz in modes:
    for rep in range(3):
        t0 = time.perf_counter()
        res = cp.run_path(data, g, cfg["q"], sched, scfg, keep_solutions=ks, keep_z=kz)
        dt = time.perf_counter() - t0
        del res
        print(f"{name:12s} rep {rep}: {dt:.3f} s", flush=True)
