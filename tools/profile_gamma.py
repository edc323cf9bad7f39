"""Per-gamma kernel profile of a path: the warm-started schedule solved one
gamma at a time through cp.solve (the same per-gamma solve run_path does),
with the library's CUDA-event stats reset per gamma.
usage: profile_gamma.py <config> [t0] [t1] [out.json] [time_limit_s]
(gammas t0..t1-1 are profiled; earlier ones run unprofiled)"""
import json
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import bench  # noqa: E402
import paper_2501_15964_b200 as cp  # noqa: E402

name = sys.argv[1] if len(sys.argv) > 1 else "c3"
cfg = dict(bench.CONFIGS[name])
t0 = int(sys.argv[2]) if len(sys.argv) > 2 else 0
t1 = int(sys.argv[3]) if len(sys.argv) > 3 else cfg["T"]
out = sys.argv[4] if len(sys.argv) > 4 and sys.argv[4] != "-" else None
tlim = float(sys.argv[5]) if len(sys.argv) > 5 else None
A = bench.make_input(cp, cfg)
ctx = cp.default_context()
data = cp.DataMatrix(A, ctx=ctx)
g = cp.compute_knn_weights(data, cfg["k"], cfg["phi"])
sched = cp.make_schedule(cfg["gamma"][0], cfg["gamma"][1], cfg["T"])
scfg = cp.SolverConfig(algorithm=cp.algorithm_from_name(cfg["algorithm"]), time_limit=tlim)
warm = None
rep = {"config": name, "env": {k: v for k, v in os.environ.items() if k.startswith("CPB_")}, "per_gamma": []}
for t in range(t1):
    inst = cp.ProblemInstance(data, g, sched.values[t], cfg["q"])
    prof = t >= t0
    if prof:
        ctx.stats_enable(True)
        ctx.stats_reset()
    ctx.synchronize()
    w0 = time.perf_counter()
    sol = cp.solve(inst, scfg, warm)
    wall = time.perf_counter() - w0
    tm = sol.termination
    if prof:
        st = ctx.stats()
        ctx.stats_enable(False)
        rec = {"t": t, "gamma": sched.values[t], "wall_s": round(wall, 4),
               "counts": [tm.iterations, tm.newton, tm.cg, tm.armijo, tm.converged],
               "kernels": {k: {"n": v["launches"], "ms": round(v["ms"], 3),
                               "us": round(1e3 * v["ms"] / max(1, v["launches"]), 1),
                               "GBps": round(v["alg_bytes"] / (v["ms"] / 1e3) / 1e9) if v["ms"] > 0 and v["alg_bytes"] > 0 else None}
                           for k, v in sorted(st.items(), key=lambda kv: -kv[1]["ms"])}}
        rep["per_gamma"].append(rec)
        top = list(rec["kernels"].items())[:5]
        print(t, rec["counts"], rec["wall_s"], [(k, v["ms"], v["us"]) for k, v in top], flush=True)
    warm = sol
if out:
    with open(out, "w") as f:
        json.dump(rep, f, indent=1)
