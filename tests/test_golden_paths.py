"""Full-size parity against committed oracle goldens (SURVEY.md §8(d) gates).

The CPU oracle cannot run at C3/C5 sizes inside a test, so tools/golden_path.py
and tools/golden_knn_rows.py ran it offline (the C3 path took hours on 8 host
threads; per-element arithmetic is the single-threaded restatement's) and
committed, per config:
  * the kNN edge set as a sha256 over (i, j, d2) bytes (bitwise gate) and the
    weights' rule w = exp(-phi d2) in glibc (1 ulp gate, checked here with
    math.exp on the same toolchain);
  * per gamma: outer/Newton/CG/Armijo counts, K, labels, and Psi^T X Omega
    sketches (tests/golden/sketch.py) for the 1e-6 relative-Frobenius gate;
  * C5: the k-nearest lists of a row sample (bitwise).
The GPU side runs the product's own input generator and path, exactly as
bench.py does.
"""
import json
import math
import os
import sys

import numpy as np
import pytest

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, os.path.join(HERE, "golden"))
import sketch as sk  # noqa: E402

GOLD = os.path.join(HERE, "golden")
CFGS = [c for c in ("c1", "c2", "c3", "c4s_q1", "c4s_qinf") if os.path.exists(os.path.join(GOLD, f"{c}_path.json"))]


def load(name):
    rep = json.load(open(os.path.join(GOLD, f"{name}_path.json")))
    arr = dict(np.load(os.path.join(GOLD, f"{name}_arrays.npz")))
    return rep, arr


def product_input(cp, cfg):
    n, d, m = cfg["n"], cfg["d"], 10
    if cfg["centers"] == "circle":
        ang = 2 * np.pi * np.arange(m) / m
        centers = np.stack([4 * np.cos(ang), 4 * np.sin(ang)], axis=1)
        spread = 0.5
    else:
        centers = (3.0 / np.sqrt(d)) * cp.normals(1001, m * d).reshape(m, d)
        spread = 1.0 / np.sqrt(d)
    return cp.generate_gaussian_mixture(centers, spread, n // m, 42)


def test_goldens_are_complete():
    for name in CFGS:
        rep, arr = load(name)
        T = rep["cfg"]["T"]
        assert len(rep["gammas"]) == T
        for t in range(len(rep["per_gamma"])):
            assert f"labels_{t}" in arr and f"X_sketch_{t}" in arr


@pytest.mark.gpu
@pytest.mark.parametrize("name", CFGS)
def test_path_matches_oracle_goldens(cp, name):
    rep, arr = load(name)
    cfg = rep["cfg"]
    A = product_input(cp, cfg)
    data = cp.DataMatrix(A)
    g = cp.compute_knn_weights(data, cfg["k"], cfg["phi"])
    gi, gj, gw, gd2 = g.arrays()
    assert len(gi) == rep["graph"]["E"]
    assert sk.edge_hash(gi, gj, gd2) == rep["graph"]["edge_hash"], "kNN edge set / order / d2 differ from the oracle"
    exact = np.array([math.exp(-cfg["phi"] * x) for x in gd2])
    assert np.max(np.abs(gw - exact) / exact) <= 2.3e-16
    T = len(rep["per_gamma"])
    sched = cp.make_schedule(cfg["gamma"][0], cfg["gamma"][1], cfg["T"])
    assert np.array_equal(np.array(sched.values), np.array(rep["gammas"]))
    sched.values = sched.values[:T]
    keep_z = cfg["n"] * cfg["d"] <= 10 ** 7
    scfg = cp.SolverConfig(algorithm=cp.algorithm_from_name(cfg["algorithm"]), max_iter=cfg.get("max_iter", 0),
                           ssnal_newton_max=cfg.get("ssnal_newton_max", 50), pcg_max_iter=cfg.get("pcg_max_iter", 500))
    res = cp.run_path(data, g, cfg["q"], sched, scfg, keep_z=keep_z)
    worst = 0.0
    for t, rec in enumerate(rep["per_gamma"]):
        st = res.stats[t]
        got = [st.iterations, st.newton, st.cg, st.armijo, bool(st.converged)]
        if cfg["q"] == 0:  # q = inf: the Hessian's dots round differently; capped solves keep the outer counts
            assert got[0] == rec["counts"][0] and got[4] == rec["counts"][4], f"gamma {t}: {got} vs {rec['counts']}"
        else:
            assert got == rec["counts"], f"gamma {t}: counts {got} vs oracle {rec['counts']}"
        assert res.assignments[t].K == rec["K"]
        assert np.array_equal(res.assignments[t].labels, arr[f"labels_{t}"])
        X = res.solutions[t].X
        rel = sk.rel_sketch_error(sk.sketch(X), arr[f"X_sketch_{t}"])
        worst = max(worst, rel)
        assert rel <= 1e-6, f"gamma {t}: X sketch rel {rel}"
        assert abs(np.linalg.norm(X) - rec["X_fro"]) <= 1e-9 * rec["X_fro"]
        if keep_z:
            assert sk.rel_sketch_error(sk.sketch(res.solutions[t].Z), arr[f"Z_sketch_{t}"]) <= 1e-6
        assert abs(st.f_primal - rec["f_primal"]) <= 1e-9 * (1 + abs(rec["f_primal"]))
    print(f"{name}: {T} gammas, worst X sketch rel {worst:.3e}")


@pytest.mark.gpu
def test_c5_knn_row_sample(cp):
    path = os.path.join(GOLD, "c5_knn_rows.npz")
    z = np.load(path)
    cfg = json.loads(str(z["cfg"]))
    A = product_input(cp, cfg)
    data = cp.DataMatrix(A)
    k = cfg["k"]
    rows = z["rows"]
    import torch
    kd = torch.zeros((cfg["n"], k), dtype=torch.float64, device="cuda")
    kj = torch.zeros((cfg["n"], k), dtype=torch.int32, device="cuda")
    for r in rows:  # the sharded-kNN entry point, one query row at a time
        cp.knn_rows_into(data, k, int(r), int(r) + 1, kd, kj)
    kd_h, kj_h = kd.cpu().numpy()[rows], kj.cpu().numpy()[rows]
    for a, r in enumerate(rows):
        assert np.array_equal(kj_h[a], z["kj"][a]) and np.array_equal(kd_h[a], z["kd"][a]), f"row {r}"
    g = cp.compute_knn_weights(data, k, cfg["phi"])
    gi, gj, gw, gd2 = g.arrays()
    key = gi.astype(np.int64) * cfg["n"] + gj
    for a, r in enumerate(rows):
        for m in range(k):
            j = int(z["kj"][a, m])
            lo, hi = min(int(r), j), max(int(r), j)
            pos = np.searchsorted(key, lo * cfg["n"] + hi)
            assert pos < len(key) and key[pos] == lo * cfg["n"] + hi, f"edge ({lo},{hi}) missing"
            assert gd2[pos] == z["kd"][a, m]
