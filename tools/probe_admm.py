"""SSNAL vs ADMM (and AMA) on the same path (C3's comparison):
per-gamma iterations, convergence and wall time, with a per-solve time limit."""
import json
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import bench  # noqa: E402
import paper_2501_15964_b200 as cp  # noqa: E402

name = sys.argv[1] if len(sys.argv) > 1 else "c3"
algos = (sys.argv[2] if len(sys.argv) > 2 else "ssnal,admm").split(",")
limit = float(sys.argv[3]) if len(sys.argv) > 3 else 60.0
cfg = bench.CONFIGS[name]
A = bench.make_input(cp, cfg)
data = cp.DataMatrix(A)
g = cp.compute_knn_weights(data, cfg["k"], cfg["phi"])
sched = cp.make_schedule(cfg["gamma"][0], cfg["gamma"][1], cfg["T"])
out = {"config": name, "E": g.edge_count(), "time_limit_per_solve_s": limit}
for a in algos:
    conf = cp.SolverConfig(algorithm=cp.algorithm_from_name(a), time_limit=limit)
    t0 = time.perf_counter()
    res = cp.run_path(data, g, cfg["q"], sched, conf, keep_solutions=False)
    wall = time.perf_counter() - t0
    out[a] = {"wall_s": wall, "all_converged": res.all_converged(),
              "per_gamma": [{"gamma": gm, "iterations": s.iterations, "converged": s.converged,
                             "wall_s": round(s.wall_time, 4), "K": asg.K}
                            for gm, s, asg in zip(sched.values, res.stats, res.assignments)]}
    print(a, "wall", round(wall, 3), "converged", res.all_converged(),
          "K", [x.K for x in res.assignments], flush=True)
print(json.dumps(out))
