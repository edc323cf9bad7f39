"""Full-path parity report (north-star correctness bar) on one config: the GPU
path vs the CPU oracle on identical inputs — kNN edge set / order / squared
distances bitwise, weights <= 1 ulp, and for every gamma X within 1e-6
relative Frobenius, labels identical, iteration counts side by side.
Slow (the oracle is single-threaded): C2 takes ~25 min of CPU."""
import json
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "oracle"))
import numpy as np  # noqa: E402

import bench  # noqa: E402
import paper_2501_15964_b200 as cp  # noqa: E402
import pyoracle as orc  # noqa: E402

name = sys.argv[1] if len(sys.argv) > 1 else "c2"
out = sys.argv[2] if len(sys.argv) > 2 else os.path.join(ROOT, "gpurun_out", f"validate_{name}.json")
cfg = bench.CONFIGS[name]
A = bench.make_input(cp, cfg)
rep = {"config": name, "n": cfg["n"], "d": cfg["d"], "k": cfg["k"], "q": cfg["q"], "algorithm": cfg["algorithm"]}
t0 = time.perf_counter()
g = cp.compute_knn_weights(cp.DataMatrix(A), cfg["k"], cfg["phi"])
sched = cp.make_schedule(cfg["gamma"][0], cfg["gamma"][1], cfg["T"])
res = cp.run_path(cp.DataMatrix(A), g, cfg["q"], sched, cp.SolverConfig(algorithm=cp.algorithm_from_name(cfg["algorithm"])),
                  keep_z=False)
rep["gpu_seconds"] = time.perf_counter() - t0
t1 = time.perf_counter()
og = orc.knn_weights(A, cfg["k"], cfg["phi"])
rep["oracle_knn_seconds"] = time.perf_counter() - t1
gi, gj, gw, gd2 = g.arrays()
oi, oj, ow, od2 = og.arrays()
rep["edges"] = int(len(gi))
rep["edges_identical"] = bool(np.array_equal(gi, oi) and np.array_equal(gj, oj))
rep["d2_bitwise"] = bool(np.array_equal(gd2, od2))
rep["w_max_rel_diff"] = float(np.max(np.abs(gw - ow) / ow)) if len(ow) else 0.0
print(json.dumps(rep), flush=True)
t2 = time.perf_counter()
ores = orc.run_path(A, og, cfg["q"], sched.values, orc.config(cfg["algorithm"]), keep_z=False)
rep["oracle_path_seconds"] = time.perf_counter() - t2
per = []
for t in range(len(sched.values)):
    X, OX = res.solutions[t].X, ores["X"][t]
    st, ot = res.stats[t], ores["terms"][t]
    per.append({"gamma": sched.values[t], "rel_X": float(np.linalg.norm(X - OX) / np.linalg.norm(OX)),
                "labels_equal": bool(np.array_equal(res.assignments[t].labels, ores["labels"][t])),
                "K": int(res.assignments[t].K), "K_oracle": int(ores["K"][t]),
                "gpu": [st.iterations, st.newton, st.cg, st.armijo, bool(st.converged)],
                "oracle": [int(ot["iterations"]), int(ot["newton"]), int(ot["cg"]), int(ot["armijo"]),
                           bool(ot["converged"])]})
rep["per_gamma"] = per
rep["max_rel_X"] = max(p["rel_X"] for p in per)
rep["all_labels_equal"] = all(p["labels_equal"] for p in per)
rep["iteration_paths_identical"] = all(p["gpu"] == p["oracle"] for p in per)
os.makedirs(os.path.dirname(out), exist_ok=True)
with open(out, "w") as f:
    json.dump(rep, f, indent=1)
print(json.dumps({k: v for k, v in rep.items() if k != "per_gamma"}), flush=True)
