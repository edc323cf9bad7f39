"""paper_2501_15964_b200 — B200-native convex-clustering path engine.

A drop-in for the hot path of the reference ``cluspath`` solver (arXiv
2501.15964): kNN Gaussian-weight graph, edge operators B / Bᵀ, per-edge
prox/projection, the SSNAL semismooth-Newton/PCG inner loop (plus fast AMA and
ADMM), and GPU connected-component labels, swept over a warm-started gamma
path.  All numerics run in hand-written sm_100a CUDA (libcluspath_b200.so)
behind the C-ABI of include/cluspath_b200.h; this package is the host-side
mirror of the reference API.
"""
from .cluspath import (Algorithm, ClusterAssignment, Context, DataMatrix, GammaSchedule, IncidenceOperator, LocalGroup,
                       PathOptions, PathResult, PenaltyNorm, ProblemInstance, Solution, SolverConfig, Spacing,
                       TerminationRecord, WeightedGraph, algorithm_from_name, algorithm_name, component_count,
                       compute_knn_weights, compute_knn_weights_sharded, connected_components, default_context, dual_objective, duality_gap,
                       extract_clusters, flush_l2, gather_row_lists, init_comm_from_torch, knn_rows_into, nccl_unique_id, generate_gaussian_mixture, kkt_residual, launch_count,
                       make_data_matrix, make_schedule, normals, penalty_norm_from_q, timer_start, timer_stop,
                       primal_objective, project_columns, prox_jacobian, prox_jacobian_apply, ProxJacobian, shard_rows, prox_columns, prox_jacobian_diag, recover_primal, run_path,
                       solve, ssnal_hessian_apply, ssnal_phi_gradient, ssnal_phi_value, two_point_closed_form,
                       CholeskyFactor, LinearOperator, PcgResult, TraceRow, dual_norm_value, moreau_check, norm_value,
                       pcg, pinned_empty, power_iteration, project_dual_ball, project_dual_ball_into, prox_norm,
                       prox_norm_into)

from .io import export_graph_csv, format_double, path_result_to_json, write_matrix_csv
from .perf import BenchOptions, BenchTask, MethodCurve, PerfProfile, perf_profile_csv, run_bench

__all__ = [n for n in dir() if not n.startswith("_")]
