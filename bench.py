#!/usr/bin/env python
"""Benchmark: the warm-started 20-gamma convex-clustering path (BASELINE.json).

One *step* = one full clustering path on one synthetic Gaussian-mixture input:
GPU kNN Gaussian-weight graph + 20 warm-started solves (SSNAL by default) +
per-gamma labels.  Metric: path wall seconds (lower is better), KKT 1e-6.

  python bench.py [--gpus N] [--steps K] [--warmup W] [--config c3] [--impl ours|reference]

Default workload: C3, n=70000 d=784 k=10 (the north-star target; configs[2]
of BASELINE.json).  c2 (n=10000, configs[1]) and c1 are selectable.

* value  — device-timed (CUDA events on the library stream, max over ranks)
           path seconds with the input already resident in HBM; L2 flushed
           between steps.
* e2e    — the same path through the public API with host buffers: host A ->
           DataMatrix (H2D), kNN, run_path returning every X(gamma), Z(gamma)
           and the labels to pinned-free host numpy arrays (D2H), wall clock.
* roofline — the dominant kernel (SSNAL Hessian apply) from the library's
           per-launch CUDA-event statistics during the timed steps:
           algorithmic bytes per launch / event time vs MEASURED_PEAKS hbm_gbs.
* knn    — the tcgen05 3xTF32 distance contraction: TF32 TFLOP/s executed
           (3 x 2 n^2 d / time) against half the measured BF16 peak.
* edge_op_gbps — sum of algorithmic bytes / sum of time over the edge, prox,
           CG, line-search and KKT kernels.
* cpu_baseline — the CPU oracle (oracle/, a restatement of the single-threaded
           reference) on the box's host with every host thread (ORC_THREADS; the
           parallel loops are bitwise the one-thread result), bounded sample: kNN of 400 query rows
           and one call of each SSNAL building block at this config, scaled by
           the GPU path's own iteration counts (which match the oracle's; see
           tests/test_gpu_parity.py::test_ssnal_iteration_path_matches).
* --impl reference — the same CPU extrapolation as the line's value (rank 0).

Multi-GPU (N > 1, one process per GPU under torchrun, NCCL): the kNN is
sharded by query-row blocks with an all-gather of the per-row lists (every
rank then builds the bit-identical graph), and the SSNAL solves are node-
partitioned (each rank owns a node range and the edges it starts: edge passes,
node gathers, Hessian applies and PCG vector updates cover the owned part; sums
are all-reduced, p / D all-gathered, Z assembled after each solve).  Labels and
the graph build stay replicated.  "scaling": "strong" (one path).
"""
from __future__ import annotations

import argparse
import json
import os
import subprocess
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

# Frozen workloads.  Gamma endpoints were
# calibrated once on this engine so that K(gamma_1) ~ n and K(gamma_20) is the
# component floor; see profiles/calibration_*.json.
CONFIGS = {
    "c1": dict(n=1000, d=2, k=10, phi=0.5, q=2, algorithm="ama", centers="circle", gamma=(0.01, 10.0), T=20),
    "c2": dict(n=10000, d=784, k=10, phi=0.5, q=2, algorithm="ssnal", centers="gauss", gamma=(0.01, 10.0), T=20),
    "c3": dict(n=70000, d=784, k=10, phi=0.5, q=2, algorithm="ssnal", centers="gauss", gamma=(0.01, 10.0), T=20),
    "c3admm": dict(n=70000, d=784, k=10, phi=0.5, q=2, algorithm="admm", centers="gauss", gamma=(0.01, 10.0), T=20),
    "c4": dict(n=60000, d=3072, k=10, phi=0.5, q=1, algorithm="ssnal", centers="gauss", gamma=(0.01, 10.0), T=20),
    "c4inf": dict(n=60000, d=3072, k=10, phi=0.5, q=0, algorithm="ssnal", centers="gauss", gamma=(0.01, 10.0),
                  T=20),
    "c5": dict(n=1000000, d=64, k=15, phi=0.5, q=2, algorithm="ssnal", centers="gauss", gamma=(0.01, 10.0), T=20),
}
COUNTS_FILE = os.path.join(ROOT, "profiles", "path_counts_{}.json")


def make_input(cp, cfg):
    """The synthetic mixture through `cp`'s generator: the product package
    for our arm, pyoracle for the reference arm (both restate io.cpp:142-165 on libstdc++
    <random>, so A is bit-identical)."""
    n, d = cfg["n"], cfg["d"]
    m = 10
    if cfg["centers"] == "circle":
        ang = 2 * np.pi * np.arange(m) / m
        centers = np.stack([4 * np.cos(ang), 4 * np.sin(ang)], axis=1)
        spread = 0.5
    else:
        centers = (3.0 / np.sqrt(d)) * cp.normals(1001, m * d).reshape(m, d)
        spread = 1.0 / np.sqrt(d)
    gen = getattr(cp, "generate_gaussian_mixture", None) or cp.gaussian_mixture
    return gen(centers, spread, n // m, 42)


def host_cores():
    try:
        return len(os.sched_getaffinity(0))
    except Exception:
        return os.cpu_count()


def oracle_threads():
    """Host threads for the CPU arms: every core of this box unless ORC_THREADS is set.  The
    oracle's parallel loops (kNN rows, per-edge prox / Jacobian, node-partitioned scatters) give
    results bitwise equal to one thread; its reductions stay sequential in Eigen's order.
    Must run before the oracle's first call (the thread count is read once)."""
    os.environ.setdefault("ORC_THREADS", str(host_cores()))
    return int(os.environ["ORC_THREADS"])


def oracle_counts(name):
    """The oracle's own per-gamma counts of this config (tests/golden/<cfg>_path.json, made by
    tools/golden_path.py), when the golden covers the whole schedule."""
    f = os.path.join(ROOT, "tests", "golden", f"{name}_path.json")
    if not os.path.exists(f):
        return None
    g = json.load(open(f))
    if len(g.get("per_gamma", [])) != g["cfg"]["T"]:
        return None
    return [{"gamma": r["gamma"], "iterations": r["counts"][0], "newton": r["counts"][1], "cg": r["counts"][2],
             "armijo": r["counts"][3], "converged": r["counts"][4], "K": r["K"]} for r in g["per_gamma"]]


def _peaks_file():
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as f:
            return json.load(f)
    except Exception:
        return {}


PEAKS = _peaks_file()


def load_peaks():
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as f:
            p = json.load(f)
        return float(p["hbm_gbs"]), "measured"
    except Exception:
        return 6650.0, "fallback"


class ClockSampler:
    """nvidia-smi clocks / throttle reasons sampled during the timed region."""

    Q = ("clocks.sm,clocks.max.sm,clocks_event_reasons.active,clocks_event_reasons.hw_slowdown,"
         "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
         "clocks_event_reasons.sw_power_cap")

    def __init__(self, index):
        self.index = index
        self.rows = []
        self.proc = None
        self.th = None

    def start(self):
        try:
            self.proc = subprocess.Popen(["nvidia-smi", "-i", str(self.index), f"--query-gpu={self.Q}",
                                          "--format=csv,noheader,nounits", "-lms", "200"],
                                         stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
        except Exception:
            self.proc = None
            return
        self.th = threading.Thread(target=self._read, daemon=True)
        self.th.start()

    def _read(self):
        for line in self.proc.stdout:
            parts = [x.strip() for x in line.split(",")]
            if len(parts) >= 7:
                self.rows.append(parts)

    def stop(self):
        if self.proc is not None:
            self.proc.terminate()
            try:
                self.proc.wait(timeout=5)
            except Exception:
                self.proc.kill()
        if self.th is not None:
            self.th.join(timeout=2)
        sm = []
        mx = 0.0
        reasons = set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for r in self.rows:
            try:
                sm.append(float(r[0]))
                mx = max(mx, float(r[1]))
            except ValueError:
                continue
            for k, nm in enumerate(names):
                if r[3 + k].lower().startswith("active"):
                    reasons.add(nm)
        return {"sm_mhz": float(np.median(sm)) if sm else None, "sm_max_mhz": mx or None,
                "reasons": sorted(reasons), "samples": len(sm)}


def dist_setup():
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    if world > 1:
        import torch
        import torch.distributed as dist
        torch.cuda.set_device(local)
        dist.init_process_group("nccl")
        return world, rank, local, dist
    return 1, 0, 0, None


def allmax(dist, x):
    if dist is None:
        return x
    import torch
    t = torch.tensor([float(x)], device="cuda")
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    return float(t.item())


def barrier(dist):
    if dist is not None:
        dist.barrier()


# ---- CPU side (oracle; cpu_baseline leg and --impl reference only) -------------------
def cpu_estimate(cfg, A, counts, knn_rows=400, reps=2):
    """Extrapolated single-core reference path seconds from a bounded sample."""
    sys.path.insert(0, os.path.join(ROOT, "oracle"))
    import pyoracle as orc

    t0 = time.perf_counter()
    n, k = cfg["n"], cfg["k"]
    rows = min(knn_rows, n)
    t_knn = orc.time_knn_rows(A, k, rows) * (n / rows)
    if counts.get("algorithm") != "ssnal":
        # small configs: time the whole oracle path directly
        g = orc.knn_weights(A, k, cfg["phi"])
        gam = orc.make_schedule(cfg["gamma"][0], cfg["gamma"][1], cfg["T"], True)
        ts = time.perf_counter()
        orc.run_path(A, g, cfg["q"], gam, orc.config(cfg["algorithm"]), keep_z=False)
        est = t_knn + (time.perf_counter() - ts)
        sample = f"full oracle path (kNN {rows} rows scaled x{n / rows:.0f})"
        return est, sample, time.perf_counter() - t0
    # Graph from the GPU-identical edge set is not needed for unit costs; build a
    # cheap same-size graph: the exact kNN graph costs O(n^2 d) on one core, so
    # use the edge list recorded with the counts.
    ef = os.path.join(ROOT, counts.get("edges_file", "")) if counts.get("edges_file") else None
    ed = np.load(ef) if ef and os.path.exists(ef) else None
    if ed is not None:
        g = orc.Graph.from_arrays(n, ed["i"], ed["j"], ed["w"])
    else:  # same degree structure: chain each sample to its k successors inside its cluster
        per = n // 10
        ii, jj = [], []
        for c in range(10):
            base = c * per
            for a in range(per):
                for s in range(1, k // 2 + 1):
                    ii.append(base + a)
                    jj.append(base + (a + s) % per)
        ii, jj = np.array(ii), np.array(jj)
        lo, hi = np.minimum(ii, jj), np.maximum(ii, jj)
        key = np.unique(lo * n + hi)
        g = orc.Graph.from_arrays(n, key // n, key % n, np.full(len(key), 0.4))
    units = orc.time_ssnal_units(A, g, counts["gamma_mid"], cfg["q"], 1.0, reps)
    E_scale = counts["E"] / max(1, g.E)
    for key in ("eval_phi", "gradient", "jacobian_diag", "hess_apply", "multiplier"):
        units[key] *= E_scale  # edge-dominated units scale with |E|
    est = t_knn
    for c in counts["per_gamma"]:
        outer, N, C, R = c["iterations"], c["newton"], c["cg"], c["armijo"]
        est += units["gap"] * (1 + outer)
        est += outer * (units["eval_phi"] + units["multiplier"])
        est += (N + outer) * units["gradient"]
        est += N * (units["jacobian_diag"] + 2 * units["hess_apply"])  # + PCG's exit residual apply (linalg.cpp:188)
        est += C * (units["hess_apply"] + units["pcg_vec"])
        est += R * units["eval_phi"]
    sample = (f"oracle kNN of {rows} query rows (x{n / rows:.0f}) + one call of each SSNAL block at n={n}, "
              f"d={cfg['d']}, scaled by the path's counts (newton {sum(c['newton'] for c in counts['per_gamma'])}, "
              f"cg {sum(c['cg'] for c in counts['per_gamma'])}, armijo {sum(c['armijo'] for c in counts['per_gamma'])})")
    return est, sample, time.perf_counter() - t0


def run_reference(args, cfg):
    """The reference arm: the CPU restatement of the reference's single-threaded path (oracle/;
    the reference itself needs Eigen 3.4, absent from this image) on this box's host, rank 0
    only.  Inputs come from the oracle's own generator and the iteration counts from the
    oracle's own run of this config (tests/golden); nothing of the product is loaded."""
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return
    threads = oracle_threads()
    sys.path.insert(0, os.path.join(ROOT, "oracle"))
    import pyoracle as orc
    A = make_input(orc, cfg)
    cf = COUNTS_FILE.format(args.config)
    counts = json.load(open(cf)) if os.path.exists(cf) else {"algorithm": cfg["algorithm"]}
    oc = oracle_counts(args.config)
    if oc is not None:
        counts["per_gamma"] = oc
        counts["counts_source"] = f"tests/golden/{args.config}_path.json (the oracle's own path)"
    vals = []
    sample = ""
    for s in range(args.warmup + args.steps):
        timed = s >= args.warmup
        # warm-up steps use a smaller sample (untimed); timed steps the bounded one
        est, sample, spent = cpu_estimate(cfg, A, counts, knn_rows=200 if timed else 40, reps=1)
        if timed:
            vals.append(est)
    v = float(np.median(vals))
    line = {"metric": "clustering-path wall s (20 gamma, KKT 1e-6)", "value": v, "unit": "s", "impl": "reference",
            "n_gpus": world, "steps": args.steps, "warmup": args.warmup, "higher_is_better": False,
            "dtype": "f64", "data": "synthetic", "config": workload_config(args, cfg, world),
            "cpu_baseline": {"value": v, "unit": "s", "cores": threads, "host_cores": host_cores(), "kind": "port",
                             "extrapolated": counts.get("algorithm") == "ssnal",
                             "counts_source": counts.get("counts_source", "profiles/path_counts (GPU path)"),
                             "sample": sample},
            "e2e": {"value": v, "unit": "s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(line), flush=True)


def workload_config(args, cfg, world):
    return {"workload": f"{args.config}: Gaussian mixture n={cfg['n']} d={cfg['d']}, kNN k={cfg['k']} phi={cfg['phi']}, "
                        f"q={'inf' if cfg['q'] == 0 else cfg['q']}, {cfg['algorithm'].upper()} {cfg['T']}-gamma warm-started path "
                        f"[{cfg['gamma'][0]}, {cfg['gamma'][1]}] geometric, eps=1e-6",
            "n": cfg["n"], "d": cfg["d"], "k": cfg["k"], "T": cfg["T"], "solver": cfg["algorithm"],
            "l2": "flushed between steps (512 MB write); edge arrays > L2",
            "parallelism": ("kNN query rows sharded over the ranks (NCCL all-gather of the n x k lists); "
                            "SSNAL node-partitioned: owned nodes / owned+ghost edges per rank, NCCL all-reduce "
                            "of sums, all-gather of p and D, Z assembled per gamma") if world > 1 else "single"}


# Kernels whose timer bytes are algorithmic HBM bytes; the kNN entries carry
# flops (knn_gemm, knn_band) or nothing and are reported under "knn".
def per_kernel_entry(name, v, peak):
    e = {"launches": v["launches"], "ms": round(v["ms"], 3)}
    if v["ms"] > 0 and v["alg_bytes"] > 0 and not name.startswith("knn"):
        gbps = v["alg_bytes"] / (v["ms"] / 1e3) / 1e9
        e.update({"GBps": round(gbps, 1), "frac": round(gbps / peak, 3) if peak else None})
    return e


def run_ours(args, cfg):
    world, rank, local, dist = dist_setup()
    if world != args.gpus:
        raise SystemExit(f"bench.py: --gpus {args.gpus} but WORLD_SIZE={world}: refusing to report a "
                         f"{args.gpus}-GPU number from {world} process(es)")
    import paper_2501_15964_b200 as cp
    ctx = cp.default_context(local)
    if world > 1:
        cp.init_comm_from_torch(ctx)  # NCCL communicator: node-partitioned Newton PCG
    A = make_input(cp, cfg)
    cpcfg = cp.SolverConfig(algorithm=cp.algorithm_from_name(cfg["algorithm"]), time_limit=args.time_limit)
    sched = cp.make_schedule(cfg["gamma"][0], cfg["gamma"][1], cfg["T"])
    data = cp.DataMatrix(A, ctx=ctx)

    knn = cp.compute_knn_weights  # row-sharded over the communicator's ranks when world > 1

    def step():
        g = knn(data, cfg["k"], cfg["phi"])
        res = cp.run_path(data, g, cfg["q"], sched, cpcfg, keep_solutions=False, centroids=False)
        return g, res

    for _ in range(args.warmup):
        cp.flush_l2(ctx)
        g, res = step()
    ctx.stats_enable(True)
    ctx.stats_reset()
    clocks = ClockSampler(local)
    clocks.start()
    times = []
    l0 = cp.launch_count()
    for _ in range(args.steps):
        cp.flush_l2(ctx)
        barrier(dist)
        ctx.synchronize()
        cp.timer_start(ctx)
        g, res = step()
        times.append(cp.timer_stop(ctx) / 1e3)
    launches = cp.launch_count() - l0
    clk = clocks.stop()
    stats = ctx.stats()
    ctx.stats_enable(False)
    per_step = allmax(dist, float(np.mean(times)))
    E = g.edge_count()
    # ---- e2e through the public API with host buffers ------------------------------
    e2e_times = []
    T = cfg["T"]
    # every X(gamma) and labels always come back; the 20 E x d multipliers too
    # unless they exceed 96 GB of host memory (C4, C5)
    keep_z = T * E * cfg["d"] * 8 <= (96 << 30)
    e2e_cold = None
    for s in range(0 if args.no_e2e else 1 + max(1, min(args.steps, 2))):  # the first call also allocates the pinned output pool
        barrier(dist)
        t0 = time.perf_counter()
        dA = cp.DataMatrix(A, ctx=ctx)
        g2 = knn(dA, cfg["k"], cfg["phi"])
        # one copy of the path's outputs comes back to the host: rank 0's (every rank holds the same)
        res2 = cp.run_path(dA, g2, cfg["q"], sched, cpcfg, keep_solutions=(rank == 0), keep_z=keep_z)
        if s > 0:
            e2e_times.append(time.perf_counter() - t0)
        else:
            e2e_cold = time.perf_counter() - t0
        del res2
    e2e = allmax(dist, float(np.mean(e2e_times))) if e2e_times else None
    e2e_cold = allmax(dist, e2e_cold) if e2e_cold is not None else None
    h2d = cfg["n"] * cfg["d"] * 8
    d2h = T * (cfg["n"] * cfg["d"] + (E * cfg["d"] if keep_z else 0)) * 8 + T * cfg["n"] * 8
    # ---- roofline of the dominant kernel --------------------------------------------
    peak, peak_kind = load_peaks()
    top = max(stats.items(), key=lambda kv: kv[1]["ms"]) if stats else ("none", {"ms": 0, "alg_bytes": 0, "launches": 0})
    roof_kernel = "hess_apply" if "hess_apply" in stats else top[0]  # AMA/ADMM paths have no Hessian
    hs = stats[roof_kernel] if roof_kernel in stats else top[1]
    achieved = hs["alg_bytes"] / (hs["ms"] / 1e3) / 1e9 if hs["ms"] > 0 else 0.0
    total_ms = sum(v["ms"] for v in stats.values())
    traffic = None
    try:  # one ncu --set full capture of this config's Hessian (profiles/ncu_traffic_r02.json)
        with open(os.path.join(ROOT, "profiles", "ncu_traffic_r02.json")) as f:
            traffic = json.load(f).get(args.config)
    except Exception:
        traffic = None
    if roof_kernel != "hess_apply":
        traffic = None  # the committed captures are of the Hessian
    roof = {"bound": "hbm", "kernel": roof_kernel, "achieved": achieved, "peak": peak, "peak_kind": peak_kind,
            "unit": "GB/s", "frac": achieved / peak if peak else None,
            "traffic": traffic["dram_bytes"] if traffic else None,
            "traffic_launch": ({k: traffic[k] for k in ("kernel", "launch", "alg_bytes", "duration_ms", "source")}
                               if traffic else None),
            "launches": hs["launches"], "avg_launch_us": 1e3 * hs["ms"] / max(1, hs["launches"]),
            "share_of_timed_kernels": hs["ms"] / total_ms if total_ms else None,
            "per_kernel": {k: per_kernel_entry(k, v, peak) for k, v in sorted(stats.items(), key=lambda kv: -kv[1]["ms"])}}
    # ---- the dense contraction on the tensor cores (north-star subsystem 1) ----------
    ki = ctx.knn_info()
    kg = stats.get("knn_gemm")
    knn = {"tensor_cores": bool(ki["tensor_cores"]), "segments": ki["segments"], "band_rows": ki["band_rows"],
           "exact_rows": ki["exact_rows"], "worst_bound_ratio": ki["worst_ratio"],
           "total_ms": round(stats.get("knn_topk", {"ms": 0.0})["ms"] / max(1, args.steps), 3)}
    if kg and kg["ms"] > 0:
        alg = kg["alg_bytes"] / (kg["ms"] / 1e3) / 1e12  # alg_bytes holds 2 n^2 d flops for this kernel
        tf32_peak = PEAKS.get("bf16_tflops", 2250.0) / 2.0
        knn.update({"gemm_ms": round(kg["ms"] / kg["launches"], 3), "alg_tflops": round(alg, 1),
                    "tf32_exec_tflops": round(3 * alg, 1), "bound": "tensor", "peak_tf32_tflops": tf32_peak,
                    "peak_kind": "MEASURED_PEAKS bf16 burst / 2 (dense TF32 = half of BF16)",
                    "frac": round(3 * alg / tf32_peak, 3)})
    edge_ops = {k: v for k, v in stats.items() if v["alg_bytes"] > 0 and not k.startswith("knn")}
    eb, et = sum(v["alg_bytes"] for v in edge_ops.values()), sum(v["ms"] for v in edge_ops.values())
    edge_op_gbps = eb / (et / 1e3) / 1e9 if et > 0 else None
    counts = {"algorithm": cfg["algorithm"], "E": E, "gamma_mid": sched.values[len(sched.values) // 2],
              "per_gamma": [{"gamma": gm, "iterations": s.iterations, "newton": s.newton, "cg": s.cg,
                             "armijo": s.armijo, "converged": s.converged, "K": a.K}
                            for gm, s, a in zip(sched.values, res.stats, res.assignments)]}
    if rank == 0 and args.write_counts:
        os.makedirs(os.path.dirname(COUNTS_FILE), exist_ok=True)
        gi, gj, gw, _ = g.arrays()
        rel = os.path.join("profiles", f"graph_{args.config}.npz")
        np.savez_compressed(os.path.join(ROOT, rel), i=gi.astype(np.int32), j=gj.astype(np.int32),
                            w=gw.astype(np.float32))
        counts["edges_file"] = rel
        with open(COUNTS_FILE.format(args.config), "w") as f:
            json.dump(counts, f, indent=1)
    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu:
        ccounts = dict(counts)
        oc = oracle_counts(args.config)
        if oc is not None:  # the oracle's own iteration counts of this path
            ccounts["per_gamma"] = oc
        threads = oracle_threads()
        sys.path.insert(0, os.path.join(ROOT, "oracle"))
        import pyoracle as orc
        est, sample, spent = cpu_estimate(cfg, make_input(orc, cfg), ccounts)
        cpu = {"value": est, "unit": "s", "cores": threads, "host_cores": host_cores(), "kind": "port",
               "extrapolated": cfg["algorithm"] == "ssnal",
               "counts_source": "oracle goldens" if oc is not None else "this GPU path (identical to the oracle's at C2)",
               "sample": sample, "sample_cpu_seconds": round(spent, 1)}
    if rank == 0:
        line = {"metric": "clustering-path wall s (20 gamma, KKT 1e-6)", "value": per_step, "unit": "s",
                "n_gpus": world, "steps": args.steps, "warmup": args.warmup, "ms_per_step": 1e3 * per_step,
                "higher_is_better": False, "scaling": "strong" if world > 1 else "weak", "vs_baseline": None,
                "dtype": "f64",
                "data": "synthetic", "config": workload_config(args, cfg, world),
                "e2e": {"value": e2e, "unit": "s", "h2d_bytes_per_step": h2d, "d2h_bytes_per_step": d2h,
                        "cold_value": e2e_cold,
                        "cold_note": "first call of the process: includes allocating/pinning the host output pool",
                        "returns": "X, labels, records per gamma" + (", Z per gamma" if keep_z else ""),
                        "d2h_note": "bytes of results delivered to host buffers; a gamma accepted as is with an "
                                    "unchanged dual projection gets its X/Z as a host copy of the previous "
                                    "gamma's (bitwise equal), not a second transfer over the link"},
                "roofline": roof, "cpu_baseline": cpu, "clocks": clk, "gpu_launches": int(launches),
                "knn": knn, "edge_op_gbps": edge_op_gbps,
                "path": {"E": E, "K": [a.K for a in res.assignments], "converged": all(s.converged for s in res.stats),
                         "outer": [s.iterations for s in res.stats], "newton": sum(s.newton for s in res.stats),
                         "cg": sum(s.cg for s in res.stats), "armijo": sum(s.armijo for s in res.stats),
                         "per_gamma": [[s.iterations, s.newton, s.cg, s.armijo, bool(s.converged),
                                        round(s.wall_time, 3)] for s in res.stats],
                         "time_limit_per_gamma_s": args.time_limit,
                         "step_seconds": [round(t, 4) for t in times]}}
        print(json.dumps(line), flush=True)
    if dist is not None:
        dist.destroy_process_group()


def spawn_ranks(args):
    """`bench.py --gpus N` started without a launcher: re-exec under torch.distributed.run with N
    ranks (one per GPU), or fail loudly when the box has fewer GPUs than asked for."""
    import torch
    have = torch.cuda.device_count()
    if have < args.gpus:
        raise SystemExit(f"bench.py: --gpus {args.gpus} requested but this box has {have} GPU(s); "
                         f"not reporting a {args.gpus}-GPU number")
    import socket
    with socket.socket() as so:
        so.bind(("127.0.0.1", 0))
        port = so.getsockname()[1]
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={args.gpus}",
           "--master-addr=127.0.0.1", f"--master-port={port}", os.path.abspath(__file__)] + sys.argv[1:]
    os.execv(sys.executable, cmd)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=3)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--config", default="c3", choices=sorted(CONFIGS))
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--no-cpu", action="store_true", help="skip the CPU-baseline sample")
    ap.add_argument("--write-counts", action="store_true", help="record the path counts for the reference arm")
    ap.add_argument("--time-limit", type=float, default=None,
                    help="SolverConfig.time_limit per gamma (seconds); a capped gamma reports converged=false")
    ap.add_argument("--no-e2e", action="store_true", help="skip the end-to-end API timing (long configs)")
    args = ap.parse_args()
    cfg = CONFIGS[args.config]
    if args.impl == "ours" and args.gpus > 1 and "WORLD_SIZE" not in os.environ:
        spawn_ranks(args)
    if args.impl == "reference":
        run_reference(args, cfg)
    else:
        run_ours(args, cfg)


if __name__ == "__main__":
    main()
