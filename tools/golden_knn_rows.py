"""Golden per-row kNN lists for a row sample of a large config (TEST
INFRASTRUCTURE; CPU oracle, graph.cpp:79-98 per row):

  python tools/golden_knn_rows.py c5 [rows]

-> tests/golden/<cfg>_knn_rows.npz with the sampled row ids, their k smallest
(d2, j) pairs (bitwise) and the config.  The full C5 kNN (10^12 pairs) is out
of reach on the CPU; rows are independent, so a sample pins the edge lists."""
import json
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, os.path.join(ROOT, "oracle"))
sys.path.insert(0, os.path.join(ROOT, "tools"))
import numpy as np  # noqa: E402

import pyoracle as orc  # noqa: E402
from golden_path import CONFIGS, oracle_input  # noqa: E402

CONFIGS = dict(CONFIGS)
CONFIGS["c5"] = dict(n=1000000, d=64, k=15, phi=0.5, q=2, algorithm="ssnal", centers="gauss", gamma=(0.01, 10.0), T=20)


def main():
    name = sys.argv[1] if len(sys.argv) > 1 else "c5"
    nrows = int(sys.argv[2]) if len(sys.argv) > 2 else 96
    cfg = CONFIGS[name]
    A = oracle_input(cfg)
    n = cfg["n"]
    rows = np.unique(np.concatenate([np.arange(8), n - 1 - np.arange(8),
                                     np.linspace(0, n - 1, nrows - 16).astype(np.int64)]))
    t0 = time.perf_counter()
    kd = np.empty((len(rows), cfg["k"]))
    kj = np.empty((len(rows), cfg["k"]), np.int64)
    for a, r in enumerate(rows):
        d_, j_ = orc.knn_rows(A, cfg["k"], int(r), int(r) + 1)
        kd[a], kj[a] = d_[0], j_[0]
    out = os.path.join(ROOT, "tests", "golden", f"{name}_knn_rows.npz")
    np.savez_compressed(out, rows=rows, kd=kd, kj=kj, cfg=json.dumps(cfg), seconds=time.perf_counter() - t0)
    print(out, len(rows), round(time.perf_counter() - t0, 1), "s")


if __name__ == "__main__":
    main()
