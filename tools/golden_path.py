"""Generate the committed path goldens of one config with the CPU oracle
(TEST INFRASTRUCTURE; runs in the GPU-less build container, never on the
product path).

  ORC_THREADS=8 python tools/golden_path.py c3 [ngamma]

Inputs are made by the oracle's own restatement of generate_gaussian_mixture
(io.cpp:142-165; libstdc++ <random>, the same toolchain as the product's
host generator).  Stage 1: the oracle kNN graph (graph.cpp:75-114; rows
split across ORC_THREADS, per-row arithmetic unchanged) -> edge count and a
sha256 over (i, j, d2) bytes.  Stage 2: the warm-started path (path.cpp:110-
142) one gamma at a time -> per gamma the iteration counts, objectives, K,
labels and the X / Z sketches of tests/golden/sketch.py.  Outputs:
tests/golden/<cfg>_path.json (scalars) and tests/golden/<cfg>_arrays.npz (labels,
sketches); the full
graph and every X go to scratch/ (git- and gpurun-ignored).
"""
import json
import math
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, os.path.join(ROOT, "oracle"))
sys.path.insert(0, os.path.join(ROOT, "tests", "golden"))
import numpy as np  # noqa: E402

import pyoracle as orc  # noqa: E402
import sketch as sk  # noqa: E402

CONFIGS = {  # bench.py CONFIGS (kept in sync by tests/test_abi_cpu.py)
    "c1": dict(n=1000, d=2, k=10, phi=0.5, q=2, algorithm="ama", centers="circle", gamma=(0.01, 10.0), T=20),
    "c2": dict(n=10000, d=784, k=10, phi=0.5, q=2, algorithm="ssnal", centers="gauss", gamma=(0.01, 10.0), T=20),
    "c3": dict(n=70000, d=784, k=10, phi=0.5, q=2, algorithm="ssnal", centers="gauss", gamma=(0.01, 10.0), T=20),
    # C4-shaped rows (d = 3072) at n = 3000 with capped solves (C4's own gamma_1 needs hundreds of
    # Newton steps): every solve stops after 2 outer iterations of <= 5 Newton steps of <= 60 CG
    # iterations, identically on both sides, so the whole capped path is comparable
    "c4s_q1": dict(n=3000, d=3072, k=10, phi=0.5, q=1, algorithm="ssnal", centers="gauss", gamma=(0.01, 10.0),
                   T=20, max_iter=2, ssnal_newton_max=5, pcg_max_iter=60),
    "c4s_qinf": dict(n=3000, d=3072, k=10, phi=0.5, q=0, algorithm="ssnal", centers="gauss", gamma=(0.01, 10.0),
                     T=20, max_iter=2, ssnal_newton_max=5, pcg_max_iter=60),
}


def oracle_input(cfg):
    n, d, m = cfg["n"], cfg["d"], 10
    if cfg["centers"] == "circle":
        ang = 2 * np.pi * np.arange(m) / m
        centers = np.stack([4 * np.cos(ang), 4 * np.sin(ang)], axis=1)
        spread = 0.5
    else:
        centers = (3.0 / np.sqrt(d)) * orc.normals(1001, m * d).reshape(m, d)
        spread = 1.0 / np.sqrt(d)
    return orc.gaussian_mixture(centers, spread, n // m, 42)


def main():
    name = sys.argv[1]
    ngamma = int(sys.argv[2]) if len(sys.argv) > 2 else None
    cfg = dict(CONFIGS[name])
    if len(sys.argv) > 3:
        cfg.update(json.loads(sys.argv[3]))
    scratch = os.path.join(ROOT, "scratch")
    os.makedirs(scratch, exist_ok=True)
    out_json = os.path.join(ROOT, "tests", "golden", f"{name}_path.json")
    out_lab = os.path.join(ROOT, "tests", "golden", f"{name}_arrays.npz")
    A = oracle_input(cfg)
    gfile = os.path.join(scratch, f"graph_{name}.npz")
    rep = {"config": name, "cfg": cfg, "oracle_threads": orc_threads(), "generator": "tools/golden_path.py"}
    if os.path.exists(gfile):
        z = np.load(gfile)
        i, j, w, d2 = z["i"], z["j"], z["w"], z["d2"]
        rep["knn_seconds"] = float(z["seconds"])
    else:
        t0 = time.perf_counter()
        g = orc.knn_weights(A, cfg["k"], cfg["phi"])
        rep["knn_seconds"] = time.perf_counter() - t0
        i, j, w, d2 = g.arrays()
        np.savez(gfile, i=i, j=j, w=w, d2=d2, seconds=rep["knn_seconds"])
    # weights: glibc exp of the (bitwise) squared distances
    assert all(w[e] == math.exp(-cfg["phi"] * d2[e]) for e in range(0, len(w), max(1, len(w) // 1000)))
    rep["graph"] = {"E": int(len(i)), "edge_hash": sk.edge_hash(i, j, d2),
                    "first": [[int(i[e]), int(j[e]), float(d2[e])] for e in range(min(5, len(i)))]}
    print(json.dumps(rep["graph"]), flush=True)
    og = orc.Graph.from_arrays(cfg["n"], i, j, w)
    gam = orc.make_schedule(cfg["gamma"][0], cfg["gamma"][1], cfg["T"], True)
    T = len(gam) if ngamma is None else ngamma
    rep["gammas"] = [float(x) for x in gam]
    rep["per_gamma"] = []
    labels = {}
    if os.path.exists(out_json):  # resume
        old = json.load(open(out_json))
        if old.get("graph", {}).get("edge_hash") == rep["graph"]["edge_hash"]:
            rep["per_gamma"] = old.get("per_gamma", [])
            if os.path.exists(out_lab):
                labels = dict(np.load(out_lab))
    warm = None
    t_start = len(rep["per_gamma"])
    if t_start > 0:
        wx = np.load(os.path.join(scratch, f"{name}_X_{t_start - 1}.npy"))
        wz = np.load(os.path.join(scratch, f"{name}_Z_last.npy"))
        warm = orc.Solution(wx, wz, {})
    ocfg = orc.config(cfg["algorithm"], max_iter=cfg.get("max_iter", 0),
                      ssnal_newton_max=cfg.get("ssnal_newton_max", 50), pcg_max_iter=cfg.get("pcg_max_iter", 500))
    for t in range(t_start, T):
        t1 = time.perf_counter()
        sol = orc.solve(A, og, gam[t], cfg["q"], ocfg, warm=warm)
        secs = time.perf_counter() - t1
        lab, K, cent = orc.extract_clusters(sol.X, og)
        tm = sol.term
        rec = {"t": t, "gamma": float(gam[t]), "seconds": round(secs, 1),
               "counts": [int(tm["iterations"]), int(tm["newton"]), int(tm["cg"]), int(tm["armijo"]),
                          bool(tm["converged"])],
               "f_primal": tm["f_primal"], "f_dual": tm["f_dual"], "gap": tm["gap"], "K": int(K),
               "X_fro": float(np.linalg.norm(sol.X)), "Z_fro": float(np.linalg.norm(sol.Z))}
        rep["per_gamma"].append(rec)
        labels[f"labels_{t}"] = lab.astype(np.int32)
        labels[f"X_sketch_{t}"] = sk.sketch(sol.X)
        labels[f"Z_sketch_{t}"] = sk.sketch(sol.Z)
        labels[f"centroid_sketch_{t}"] = sk.sketch(cent, m=8)
        np.save(os.path.join(scratch, f"{name}_X_{t}.npy"), sol.X)
        np.save(os.path.join(scratch, f"{name}_Z_last.npy"), sol.Z)
        warm = sol
        with open(out_json, "w") as f:
            json.dump(rep, f, indent=0)
        np.savez_compressed(out_lab, **labels)
        print(json.dumps({k: rec[k] for k in ("t", "gamma", "seconds", "counts", "K")}), flush=True)


def orc_threads():
    return int(os.environ.get("ORC_THREADS", "1"))


if __name__ == "__main__":
    main()
