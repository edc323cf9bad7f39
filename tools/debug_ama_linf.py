"""Where do the device and oracle fast-AMA iterates first differ (q = inf, d = 40)?"""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "oracle"))
import numpy as np  # noqa: E402

import paper_2501_15964_b200 as cp  # noqa: E402
import pyoracle as orc  # noqa: E402

d, n_per, m = 40, 60, 5
centers = (3.0 / np.sqrt(d)) * orc.normals(1001, m * d).reshape(m, d)
A = orc.gaussian_mixture(centers, 1.0 / np.sqrt(d), n_per, 3)
g = cp.compute_knn_weights(cp.DataMatrix(A), 10, 0.5)
gi, gj, gw, gd2 = g.arrays()
og = orc.Graph.from_arrays(len(A), gi, gj, gw)
print("lambda", cp.IncidenceOperator(g).laplacian_lambda_max() == orc.power_laplacian(og))
sched = cp.make_schedule(0.01, 10.0, 6)
q = int(sys.argv[1]) if len(sys.argv) > 1 else 0
data = cp.DataMatrix(A)
for gamma in sched.values[:4]:
    for it in (1, 2, 3, 10, 11, 20, 100, 1000):
        s = cp.solve(cp.ProblemInstance(data, g, gamma, q), cp.SolverConfig(algorithm=cp.Algorithm.FastAMA, max_iter=it))
        o = orc.solve(A, og, gamma, q, orc.config("ama", max_iter=it))
        dz = np.max(np.abs(s.Z - o.Z))
        dx = np.max(np.abs(s.X - o.X))
        print(f"gamma {gamma:.4g} it {it}: dX {dx:.3e} dZ {dz:.3e} gpu_it {s.termination.iterations} orc_it {o.term['iterations']} "
              f"gap {s.termination.gap:.6e} {o.term['gap']:.6e}", flush=True)
        if dz > 0:
            l = int(np.argmax(np.max(np.abs(s.Z - o.Z), axis=1)))
            print("  worst edge", l, s.Z[l][:8], o.Z[l][:8])
            break
