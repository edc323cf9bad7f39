"""Path parity at large n without the O(n^2 d) CPU kNN: the oracle solves the
path on the GPU-built graph (whose edge set is pinned bitwise elsewhere),
for the first `ngamma` gammas of the config's schedule (warm-started), and
X / labels / iteration counts are compared gamma by gamma.
usage: validate_path_graph.py <config> <ngamma> [oracle_budget_s] [out.json]"""
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

name = sys.argv[1] if len(sys.argv) > 1 else "c3"
ngamma = int(sys.argv[2]) if len(sys.argv) > 2 else 10
budget = float(sys.argv[3]) if len(sys.argv) > 3 else 1e30  # oracle seconds; stops after the gamma that crosses it
out = sys.argv[4] if len(sys.argv) > 4 else os.path.join(ROOT, "gpurun_out", f"validate_{name}_g{ngamma}.json")
cfg = bench.CONFIGS[name]
A = bench.make_input(cp, cfg)
g = cp.compute_knn_weights(cp.DataMatrix(A), cfg["k"], cfg["phi"])
sched = cp.make_schedule(cfg["gamma"][0], cfg["gamma"][1], cfg["T"])
gam = sched.values[:ngamma]
sub = cp.GammaSchedule(gam, gam[0], gam[-1], len(gam), sched.spacing)
t0 = time.perf_counter()
res = cp.run_path(cp.DataMatrix(A), g, cfg["q"], sub, cp.SolverConfig(), keep_z=False)
gpu_s = time.perf_counter() - t0
gi, gj, gw, _ = g.arrays()
og = orc.Graph.from_arrays(cfg["n"], gi, gj, gw)
rep = {"config": name, "gammas": gam, "edges": int(len(gi)), "gpu_seconds": gpu_s, "per_gamma": [],
       "oracle_seconds": 0.0, "budget_s": budget}


def dump():
    done = rep["per_gamma"]
    rep["gammas_checked"] = len(done)
    rep["max_rel_X"] = max((p["rel_X"] for p in done), default=None)
    rep["all_labels_equal"] = all(p["labels_equal"] for p in done)
    rep["iteration_paths_identical"] = all(p["gpu"] == p["oracle"] for p in done)
    with open(out, "w") as f:
        json.dump(rep, f, indent=1)


# the oracle follows run_path (path.cpp:110-142) one gamma at a time, warm-started from the previous
# solution, so a time budget still leaves the gammas it finished on disk
warm = None
for t in range(len(gam)):
    if rep["oracle_seconds"] > budget:
        break
    t1 = time.perf_counter()
    sol = orc.solve(A, og, gam[t], cfg["q"], orc.config("ssnal"), warm=warm)
    lab, K, _ = orc.extract_clusters(sol.X, og)
    rep["oracle_seconds"] += time.perf_counter() - t1
    warm = sol
    X, OX = res.solutions[t].X, sol.X
    st, ot = res.stats[t], sol.term
    rep["per_gamma"].append({
        "gamma": gam[t], "rel_X": float(np.linalg.norm(X - OX) / np.linalg.norm(OX)),
        "labels_equal": bool(np.array_equal(res.assignments[t].labels, lab)),
        "K": int(res.assignments[t].K), "K_oracle": int(K),
        "gpu": [st.iterations, st.newton, st.cg, st.armijo, bool(st.converged)],
        "oracle": [int(ot["iterations"]), int(ot["newton"]), int(ot["cg"]), int(ot["armijo"]), bool(ot["converged"])],
        "oracle_s": round(time.perf_counter() - t1, 1)})
    dump()
dump()
print(json.dumps({k: v for k, v in rep.items() if k != "per_gamma"}), flush=True)
