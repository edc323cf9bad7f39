import sys, time, os
sys.path.insert(0, os.getcwd())
import numpy as np
import bench
import paper_2501_15964_b200 as cp
n = int(sys.argv[1]); q = int(sys.argv[2]); algo = sys.argv[3] if len(sys.argv) > 3 else "ssnal"
cfg = dict(bench.CONFIGS["c4"]); cfg["n"] = n
A = bench.make_input(cp, cfg)
ctx = cp.default_context()
data = cp.DataMatrix(A)
t0 = time.perf_counter()
g = cp.compute_knn_weights(data, 10, 0.5)
ctx.synchronize()
print("knn s", time.perf_counter() - t0, "E", g.edge_count(), flush=True)
sched = cp.make_schedule(0.01, 10.0, 20)
for gi in (0, 5, 10):
    ctx.stats_enable(True); ctx.stats_reset()
    inst = cp.ProblemInstance(data, g, sched.values[gi], q)
    t0 = time.perf_counter()
    sol = cp.solve(inst, cp.SolverConfig(algorithm=cp.algorithm_from_name(algo), time_limit=60.0))
    dt = time.perf_counter() - t0
    st = sol.termination
    print("gamma", sched.values[gi], "s", round(dt, 2), "iters", st.iterations, "newton", st.newton, "cg", st.cg, "conv", st.converged, flush=True)
    for k, v in sorted(ctx.stats().items(), key=lambda kv: -kv[1]["ms"])[:6]:
        print("   ", k, v["launches"], round(v["ms"], 1), flush=True)
