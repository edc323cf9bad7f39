"""Compare SSNAL iteration counts GPU vs oracle on a small C4-shaped instance."""
import os
import sys
import time

sys.path.insert(0, os.getcwd())
sys.path.insert(0, os.path.join(os.getcwd(), "oracle"))
import numpy as np

import bench
import paper_2501_15964_b200 as cp
import pyoracle as orc

n, q = int(sys.argv[1]), int(sys.argv[2])
cfg = dict(bench.CONFIGS["c4"])
cfg["n"] = n
A = bench.make_input(cp, cfg)
g = cp.compute_knn_weights(cp.DataMatrix(A), 10, 0.5)
og = orc.knn_weights(A, 10, 0.5)
sched = cp.make_schedule(0.01, 10.0, 20)
for gi in [int(x) for x in sys.argv[3].split(",")]:
    gam = sched.values[gi]
    t0 = time.perf_counter()
    s = cp.solve(cp.ProblemInstance(cp.DataMatrix(A), g, gam, q), cp.SolverConfig(time_limit=120.0))
    t1 = time.perf_counter()
    o = orc.solve(A, og, gam, q, orc.config("ssnal", time_limit=600.0))
    t2 = time.perf_counter()
    st = s.termination
    print(f"gamma {gam:.4f} gpu it={st.iterations} newton={st.newton} cg={st.cg} conv={st.converged} {t1-t0:.2f}s | "
          f"orc it={o.term['iterations']} newton={o.term.get('newton')} cg={o.term.get('cg')} conv={o.term['converged']} "
          f"{t2-t1:.2f}s | relX {np.linalg.norm(s.X - o.X) / np.linalg.norm(o.X):.2e}", flush=True)
