"""Standalone SSNAL operators at C2 size (X = A, Z = 0, every edge active):
used to profile the Hessian apply / gradient kernels in isolation."""
import os
import sys
import time

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import bench  # noqa: E402
import paper_2501_15964_b200 as cp  # noqa: E402

cfg = dict(bench.CONFIGS[sys.argv[1] if len(sys.argv) > 1 else "c2"])
reps = int(sys.argv[2]) if len(sys.argv) > 2 else 3
A = bench.make_input(cp, cfg)
data = cp.DataMatrix(A)
g = cp.compute_knn_weights(data, cfg["k"], cfg["phi"])
inst = cp.ProblemInstance(data, g, 0.3)
Z = np.zeros((g.edge_count(), cfg["d"]))
D = np.random.default_rng(0).standard_normal(A.shape)
for r in range(reps):
    t = time.perf_counter()
    H = cp.ssnal_hessian_apply(inst, Z, 1.0, A, D)
    G = cp.ssnal_phi_gradient(inst, Z, 1.0, A)
    print("rep", r, "host s", round(time.perf_counter() - t, 4), float(np.linalg.norm(H)), float(np.linalg.norm(G)))
