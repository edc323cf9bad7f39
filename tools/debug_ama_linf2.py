"""Warm-started d = 40, q = inf path: at the gamma where device and oracle stop one gap check
apart, evaluate gap and KKT of both iterates with both implementations."""
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
data = cp.DataMatrix(A)
g = cp.compute_knn_weights(data, 10, 0.5)
gi, gj, gw, gd2 = g.arrays()
og = orc.Graph.from_arrays(len(A), gi, gj, gw)
sched = cp.make_schedule(0.01, 10.0, 6)
q = 0
ws = wo = None
for t, gamma in enumerate(sched.values):
    s = cp.solve(cp.ProblemInstance(data, g, gamma, q), cp.SolverConfig(algorithm=cp.Algorithm.FastAMA), ws)
    o = orc.solve(A, og, gamma, q, orc.config("ama"), warm=wo)
    print(t, gamma, s.termination.iterations, o.term["iterations"], flush=True)
    if s.termination.iterations != o.term["iterations"]:
        k = min(s.termination.iterations, o.term["iterations"])
        s2 = cp.solve(cp.ProblemInstance(data, g, gamma, q), cp.SolverConfig(algorithm=cp.Algorithm.FastAMA, max_iter=k), ws)
        o2 = orc.solve(A, og, gamma, q, orc.config("ama", max_iter=k), warm=wo)
        print(" at", k, "dX", np.max(np.abs(s2.X - o2.X)), "dZ", np.max(np.abs(s2.Z - o2.Z)))
        inst = cp.ProblemInstance(data, g, gamma, q)
        for nm, X, Z in (("gpu-iter", s2.X, s2.Z), ("orc-iter", o2.X, o2.Z)):
            fp_c, fd_c = cp.primal_objective(inst, X), cp.dual_objective(inst, Z)
            fp_o, fd_o = orc.primal_objective(A, og, gamma, q, X), orc.dual_objective(A, og, gamma, q, Z)
            print(f"  {nm}: gpu fp {fp_c!r} fd {fd_c!r} gap {cp.duality_gap(fp_c, fd_c)!r} kkt {cp.kkt_residual(inst, X, Z)!r}")
            print(f"  {nm}: orc fp {fp_o!r} fd {fd_o!r} gap {cp.duality_gap(fp_o, fd_o)!r} kkt {orc.kkt_residual(A, og, gamma, q, X, Z)!r}")
        print("  term gpu", s2.termination)
        print("  term orc", o2.term)
        break
    ws, wo = s, o
