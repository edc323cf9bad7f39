"""Overhead of the partitioned code path at one rank: plain context vs an
in-process group of one vs an NCCL communicator of one (same inputs)."""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import bench  # noqa: E402
import paper_2501_15964_b200 as cp  # noqa: E402

cfg = bench.CONFIGS[sys.argv[1] if len(sys.argv) > 1 else "c3"]
A = bench.make_input(cp, cfg)
sched = cp.make_schedule(cfg["gamma"][0], cfg["gamma"][1], cfg["T"])
grp = cp.LocalGroup(1)
for tag in ("plain", "local1", "nccl1"):
    ctx = cp.Context(0)
    if tag == "local1":
        ctx.set_local_comm(grp, 0)
    elif tag == "nccl1":
        ctx.set_comm(1, 0, cp.nccl_unique_id())
    data = cp.DataMatrix(A, ctx=ctx)
    g = cp.compute_knn_weights(data, cfg["k"], cfg["phi"])
    for rep in range(2):
        ctx.synchronize()
        t0 = time.perf_counter()
        res = cp.run_path(data, g, cfg["q"], sched, cp.SolverConfig(), keep_solutions=False)
        ctx.synchronize()
        dt = time.perf_counter() - t0
    print(tag, "path", round(dt, 4), "solve sum", round(sum(s.wall_time for s in res.stats), 4), flush=True)
