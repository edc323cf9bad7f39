"""Short profiling driver: C2-shaped input, GPU kNN graph, and the first
`ngamma` warm-started solves of the path, with per-kernel CUDA-event stats."""
import json
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import bench  # noqa: E402
import paper_2501_15964_b200 as cp  # noqa: E402

cfg = dict(bench.CONFIGS[sys.argv[1] if len(sys.argv) > 1 else "c2"])
ngamma = int(sys.argv[2]) if len(sys.argv) > 2 else 10
stats = len(sys.argv) > 3 and sys.argv[3] == "stats"
A = bench.make_input(cp, cfg)
data = cp.DataMatrix(A)
g = cp.compute_knn_weights(data, cfg["k"], cfg["phi"])
sched = cp.make_schedule(cfg["gamma"][0], cfg["gamma"][1], cfg["T"])
sched.values = sched.values[:ngamma]
ctx = cp.default_context()
if stats:
    ctx.stats_enable(True)
    ctx.stats_reset()
ctx.synchronize()
t0 = time.perf_counter()
res = cp.run_path(data, g, cfg["q"], sched, cp.SolverConfig(algorithm=cp.algorithm_from_name(cfg["algorithm"])),
                  keep_solutions=False)
wall = time.perf_counter() - t0
print("E", g.edge_count(), "K", [a.K for a in res.assignments], "cg", sum(s.cg for s in res.stats),
      "wall", round(wall, 4), "NFMAX", os.environ.get("CPB_NFMAX"))
if stats:
    st = ctx.stats()
    tot = sum(v["ms"] for v in st.values())
    for k, v in sorted(st.items(), key=lambda kv: -kv[1]["ms"]):
        gbs = v["alg_bytes"] / (v["ms"] / 1e3) / 1e9 if v["ms"] > 0 and v["alg_bytes"] > 0 else 0
        print(f"  {k:18s} n={v['launches']:6d} ms={v['ms']:9.2f} us/launch={1e3 * v['ms'] / max(1, v['launches']):8.1f} GB/s={gbs:7.0f}")
    print("  kernel sum ms", round(tot, 1))
