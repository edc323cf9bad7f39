"""On-disk formats of the reference's path outputs, so
the CLI and tools can consume GPU results unchanged:

* ``format_double``       io.cpp:14-18 (``std::to_chars`` shortest round-trip)
* ``write_matrix_csv``    io.cpp:120-131 (one matrix row per line)
* ``export_graph_csv``    io.cpp:133-140 (``i,j,w`` header, one edge per line)
* ``path_result_to_json`` path.cpp:144-177 (schedule, solver echo, per-gamma records)

Host-only formatting: the numbers come from the GPU path unchanged.
"""
from __future__ import annotations

import json
import math
from typing import Optional

import numpy as np


def format_double(value: float) -> str:
    """``std::to_chars(first, last, double)`` without a format: the shortest
    digit string that round-trips, printed as fixed or scientific notation,
    whichever is shorter (fixed on a tie; exponent with at least two digits)."""
    v = float(value)
    if math.isnan(v):
        return "-nan" if math.copysign(1.0, v) < 0 else "nan"
    if math.isinf(v):
        return "-inf" if v < 0 else "inf"
    sign = "-" if math.copysign(1.0, v) < 0 else ""
    a = abs(v)
    if a == 0.0:
        return sign + "0"
    # shortest round-trip digits and decimal exponent (repr is shortest round-trip too)
    r = repr(a)
    if "e" in r:
        mant, ex = r.split("e")
        exp10 = int(ex)
    else:
        mant, exp10 = r, 0
    if "." in mant:
        ip, fp = mant.split(".")
    else:
        ip, fp = mant, ""
    digits = (ip + fp).lstrip("0")
    # position of the decimal point relative to the first significant digit
    point = len(ip.lstrip("0")) + exp10 if ip.strip("0") else exp10 - (len(fp) - len(fp.lstrip("0")))
    digits = digits.rstrip("0") or "0"
    nd = len(digits)
    # fixed notation
    if point <= 0:
        fixed = "0." + "0" * (-point) + digits
    elif point >= nd:
        # integral: among equally short spellings the standard picks the one
        # closest to the value, i.e. the exact integer (matters above 2^53)
        fixed = str(int(a))
    else:
        fixed = digits[:point] + "." + digits[point:]
    # scientific notation: d[.ddd]e+XX
    e = point - 1
    sci = digits[0] + ("." + digits[1:] if nd > 1 else "") + "e" + ("-" if e < 0 else "+") + f"{abs(e):02d}"
    return sign + (fixed if len(fixed) <= len(sci) else sci)


def write_matrix_csv(path: str, M) -> None:
    """io.cpp:120-131: one line per matrix row, comma-separated, to_chars values."""
    M = np.asarray(M, dtype=np.float64)
    if M.ndim != 2:
        raise ValueError("write_matrix_csv: a 2-D matrix is required")
    try:
        with open(path, "w", newline="") as f:
            for row in M:
                f.write(",".join(format_double(x) for x in row))
                f.write("\n")
    except OSError as e:
        raise RuntimeError(f"cannot open '{path}' for writing") from e


def export_graph_csv(path: str, graph=None, *, i=None, j=None, w=None) -> None:
    """io.cpp:133-140: ``i,j,w`` header, then one edge per line in the graph's
    lexicographic order.  Pass a WeightedGraph, or the edge arrays."""
    if graph is not None:
        i, j, w, _ = graph.arrays()
    i, j, w = np.asarray(i, dtype=np.int64), np.asarray(j, dtype=np.int64), np.asarray(w, dtype=np.float64)
    try:
        with open(path, "w", newline="") as f:
            f.write("i,j,w\n")
            for a, b, c in zip(i.tolist(), j.tolist(), w.tolist()):
                f.write(f"{a},{b},{format_double(c)}\n")
    except OSError as e:
        raise RuntimeError(f"cannot open '{path}' for writing") from e


def _resolved_max_iter(cfg) -> int:  # objective.cpp:38-41
    if cfg.max_iter > 0:
        return int(cfg.max_iter)
    return 100 if int(cfg.algorithm) == 2 else 20000


def path_result_to_json(result, indent: Optional[int] = 2) -> str:
    """path.cpp:144-177: {schedule, solver, per_gamma[]} with the reference's keys
    (sorted, as nlohmann::json's std::map objects print them)."""
    from .cluspath import algorithm_name
    sch = result.schedule
    cfg = result.solver
    solver = {"algorithm": algorithm_name(cfg.algorithm), "epsilon": cfg.epsilon, "kkt_factor": cfg.kkt_factor,
              "max_iter": _resolved_max_iter(cfg), "admm_rho": cfg.admm_rho, "ssnal_sigma0": cfg.ssnal_sigma0,
              "ama_step_safety": cfg.ama_step_safety}
    if cfg.time_limit is not None:
        solver["time_limit"] = cfg.time_limit
    per = []
    for t, (rec, asg) in enumerate(zip(result.stats, result.assignments)):
        per.append({"gamma": float(sch.values[t]), "converged": bool(rec.converged), "iterations": int(rec.iterations),
                    "gap": float(rec.gap), "f_p": float(rec.f_primal), "f_d": float(rec.f_dual),
                    "wall_time_s": float(rec.wall_time), "labels": [int(x) for x in np.asarray(asg.labels)],
                    "K": int(asg.K)})
    doc = {"schedule": {"start": float(sch.start), "end": float(sch.end), "count": int(sch.count),
                        "spacing": "linear" if int(sch.spacing) == 0 else "geometric",
                        "values": [float(x) for x in sch.values]},
           "solver": solver, "per_gamma": per}
    return json.dumps(doc, indent=indent, sort_keys=True)
