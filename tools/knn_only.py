"""kNN graph only, on a C5-shaped mixture of n points (default 200000, d=64, k=15)."""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import bench  # noqa: E402
import paper_2501_15964_b200 as cp  # noqa: E402

cfg = dict(bench.CONFIGS["c5"])
cfg["n"] = int(sys.argv[1]) if len(sys.argv) > 1 else 200000
A = bench.make_input(cp, cfg)
ctx = cp.default_context()
data = cp.DataMatrix(A)
for _ in range(2):
    ctx.stats_enable(True)
    ctx.stats_reset()
    t0 = time.perf_counter()
    g = cp.compute_knn_weights(data, cfg["k"], cfg["phi"])
    ctx.synchronize()
    st = ctx.stats()
    print("n", cfg["n"], "E", g.edge_count(), "wall", round(time.perf_counter() - t0, 4),
          {k: round(v["ms"], 2) for k, v in st.items() if k.startswith("knn")}, ctx.knn_info(), flush=True)
