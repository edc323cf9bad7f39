"""Where does the variable host time of compute_knn_weights go?"""
import gc
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import bench  # noqa: E402
import paper_2501_15964_b200 as cp  # noqa: E402

cfg = bench.CONFIGS["c3"]
A = bench.make_input(cp, cfg)
ctx = cp.default_context()
data = cp.DataMatrix(A)
n, k = cfg["n"], cfg["k"]
kd = torch.zeros((n, k), dtype=torch.float64, device="cuda")
kj = torch.zeros((n, k), dtype=torch.int32, device="cuda")
import ctypes as C  # noqa: E402
from paper_2501_15964_b200 import _lib as L  # noqa: E402
for it in range(8):
    ctx.synchronize()
    t0 = time.perf_counter()
    cp.knn_rows_into(data, k, 0, n, kd, kj)
    t1 = time.perf_counter()
    h = C.c_void_p()
    L.check(L.load().cp_graph_from_knn(ctx._h, n, k, 0.5, C.c_void_p(kd.data_ptr()), C.c_void_p(kj.data_ptr()),
                                       C.byref(h)))
    ctx.synchronize()
    t2 = time.perf_counter()
    L.load().cp_graph_destroy(h)
    ctx.synchronize()
    t3 = time.perf_counter()
    g = cp.compute_knn_weights(data, k, 0.5)
    ctx.synchronize()
    t4 = time.perf_counter()
    del g
    gc.collect()
    t5 = time.perf_counter()
    print(f"rows {t1 - t0:.4f} graph {t2 - t1:.4f} destroy {t3 - t2:.4f} full {t4 - t3:.4f} del {t5 - t4:.4f}",
          flush=True)
