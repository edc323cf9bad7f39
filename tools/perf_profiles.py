"""Paper-style performance profiles (bench.cpp:23-116 protocol) of SSNAL, ADMM and fast AMA
on one config's 20-gamma path, all solves on the GPU.
usage: perf_profiles.py <config> [per_solve_time_limit_s] [out_prefix]"""
import json
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import bench  # noqa: E402
import paper_2501_15964_b200 as cp  # noqa: E402

name = sys.argv[1] if len(sys.argv) > 1 else "c2"
tlim = float(sys.argv[2]) if len(sys.argv) > 2 else 60.0
prefix = sys.argv[3] if len(sys.argv) > 3 else os.path.join(ROOT, "gpurun_out", f"perf_profile_{name}")
cfg = bench.CONFIGS[name]
A = bench.make_input(cp, cfg)
data = cp.DataMatrix(A)
g = cp.compute_knn_weights(data, cfg["k"], cfg["phi"])
task = cp.BenchTask(data, g, cfg["q"], cp.make_schedule(cfg["gamma"][0], cfg["gamma"][1], cfg["T"]))
opts = cp.BenchOptions(epsilon=1e-6, base_config=cp.SolverConfig(time_limit=tlim))
t0 = time.perf_counter()
prof = cp.run_bench([task], [cp.Algorithm.SSNAL, cp.Algorithm.ADMM, cp.Algorithm.FastAMA], opts)
wall = time.perf_counter() - t0
csv = cp.perf_profile_csv(prof)
with open(prefix + ".csv", "w") as f:
    f.write(csv)
rep = {"config": name, "n": cfg["n"], "d": cfg["d"], "k": cfg["k"], "q": cfg["q"], "gammas": cfg["T"],
       "per_solve_time_limit_s": tlim, "baseline_T_s": prof.baseline_T, "problem_count": prof.problem_count,
       "cutoff_s": 10 * prof.baseline_T, "harness_wall_s": wall,
       "curves": [{"method": cp.algorithm_name(c.method), "full_time_s": c.full_time, "solved_total": c.solved_total,
                   "points": c.points} for c in prof.curves]}
with open(prefix + ".json", "w") as f:
    json.dump(rep, f, indent=1)
print(json.dumps({k: v for k, v in rep.items() if k != "curves"}))
print(csv)
