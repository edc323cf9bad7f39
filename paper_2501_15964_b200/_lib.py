"""ctypes binding of libcluspath_b200.so (the C-ABI in include/cluspath_b200.h).

The shared library is built in-tree (``python __graft_entry__.py build`` or
``make -C paper_2501_15964_b200/csrc``) for sm_100a only.  There is no CPU
fallback: if the library is missing or no CUDA device is visible, every call
raises.
"""
from __future__ import annotations

import ctypes as C
import os

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(_HERE, "libcluspath_b200.so")

D = C.POINTER(C.c_double)
I64 = C.POINTER(C.c_int64)
VP = C.c_void_p


class SolverConfigC(C.Structure):
    """cp_solver_config (SolverConfig, solvers.hpp:72-93)."""
    _fields_ = [("algorithm", C.c_int32), ("collect_trace", C.c_int32), ("epsilon", C.c_double),
                ("kkt_factor", C.c_double), ("max_iter", C.c_int64), ("time_limit", C.c_double),
                ("admm_rho", C.c_double), ("ama_step_safety", C.c_double), ("ssnal_sigma0", C.c_double),
                ("armijo_mu", C.c_double), ("backtrack_beta", C.c_double), ("ssnal_newton_max", C.c_int64),
                ("pcg_max_iter", C.c_int64)]


class TerminationC(C.Structure):
    """cp_termination (TerminationRecord, solvers.hpp:45-52, plus work counters)."""
    _fields_ = [("f_primal", C.c_double), ("f_dual", C.c_double), ("gap", C.c_double),
                ("iterations", C.c_int64), ("converged", C.c_int32), ("pad", C.c_int32),
                ("wall_time", C.c_double), ("newton", C.c_int64), ("cg", C.c_int64),
                ("armijo", C.c_int64), ("hess_apply", C.c_int64)]


class PathOptionsC(C.Structure):
    _fields_ = [("warm_start", C.c_int32), ("require_connected", C.c_int32), ("fuse_tol", C.c_double)]


class TraceRowC(C.Structure):
    """cp_trace_row (TraceRow, solvers.hpp:54-60)."""
    _fields_ = [("iter", C.c_int64), ("f_p", C.c_double), ("f_d", C.c_double), ("gap", C.c_double),
                ("elapsed_s", C.c_double)]


APPLY_FN = C.CFUNCTYPE(C.c_int, VP, D, D, C.c_int64, C.c_int64)
CENT_FN = C.CFUNCTYPE(None, VP, C.c_int64, C.c_int64, C.c_int64, D)
TRACE_FN = C.CFUNCTYPE(None, VP, C.c_int64, C.POINTER(TraceRowC), C.c_int64)


class PathSinkC(C.Structure):
    _fields_ = [("user", VP), ("centroids", CENT_FN), ("trace", TRACE_FN), ("skip_identity", C.c_int32)]


class KernelStatC(C.Structure):
    _fields_ = [("name", C.c_char * 40), ("launches", C.c_int64), ("ms", C.c_double), ("alg_bytes", C.c_double)]


# (name, restype, argtypes)
_SIGS = [
    ("cp_ctx_create", C.c_int, [C.c_int, C.POINTER(VP)]),
    ("cp_ctx_destroy", None, [VP]),
    ("cp_last_error", C.c_char_p, []),
    ("cp_ctx_synchronize", C.c_int, [VP]),
    ("cp_solver_config_default", None, [C.POINTER(SolverConfigC)]),
    ("cp_path_options_default", None, [C.POINTER(PathOptionsC)]),
    ("cp_stats_enable", C.c_int, [VP, C.c_int]),
    ("cp_stats_reset", C.c_int, [VP]),
    ("cp_stats_get", C.c_int, [VP, C.POINTER(KernelStatC), C.c_int, C.POINTER(C.c_int)]),
    ("cp_device_info", C.c_int, [VP, C.POINTER(C.c_int), C.POINTER(C.c_int), C.POINTER(C.c_int),
                                 C.POINTER(C.c_int)]),
    ("cp_knn_info", C.c_int, [VP, C.POINTER(C.c_int), C.POINTER(C.c_int), C.POINTER(C.c_int64),
                              C.POINTER(C.c_int64), D]),
    ("cp_launch_count", C.c_ulonglong, []),
    ("cp_timer_start", C.c_int, [VP]),
    ("cp_timer_stop", C.c_int, [VP, D]),
    ("cp_flush_l2", C.c_int, [VP]),
    ("cp_host_alloc", C.c_int, [C.c_uint64, C.POINTER(VP)]),
    ("cp_host_free", None, [VP]),
    ("cp_gaussian_mixture", C.c_int, [D, C.c_int64, C.c_int64, C.c_double, C.c_int64, C.c_uint64, D]),
    ("cp_normals", C.c_int, [C.c_uint64, C.c_int64, D]),
    ("cp_data_create", C.c_int, [VP, D, C.c_int64, C.c_int64, C.POINTER(VP)]),
    ("cp_data_destroy", None, [VP]),
    ("cp_knn_graph", C.c_int, [VP, VP, C.c_int64, C.c_double, C.POINTER(VP)]),
    ("cp_knn_rows", C.c_int, [VP, VP, C.c_int64, C.c_int64, C.c_int64, VP, VP]),
    ("cp_graph_laplacian", C.c_int, [VP, VP, C.POINTER(C.c_int64), C.POINTER(C.c_int64), D,
                                     C.POINTER(C.c_int64)]),
    ("cp_graph_from_knn", C.c_int, [VP, C.c_int64, C.c_int64, C.c_double, VP, VP, C.POINTER(VP)]),
    ("cp_shard_rows", C.c_int, [C.c_int64, C.c_int, C.c_int, C.POINTER(C.c_int64), C.POINTER(C.c_int64)]),
    ("cp_nccl_unique_id", C.c_int, [C.c_char_p]),
    ("cp_ctx_set_comm", C.c_int, [VP, C.c_int, C.c_int, C.c_char_p]),
    ("cp_local_group_create", C.c_int, [C.c_int, C.POINTER(VP)]),
    ("cp_local_group_destroy", None, [VP]),
    ("cp_ctx_set_local_comm", C.c_int, [VP, VP, C.c_int]),
    ("cp_graph_from_edges", C.c_int, [VP, C.c_int64, I64, I64, D, C.c_int64, C.POINTER(VP)]),
    ("cp_graph_destroy", None, [VP]),
    ("cp_graph_nodes", C.c_int64, [VP]),
    ("cp_graph_edge_count", C.c_int64, [VP]),
    ("cp_graph_export", C.c_int, [VP, VP, I64, I64, D, D]),
    ("cp_graph_degrees", C.c_int, [VP, VP, I64]),
    ("cp_incidence_apply", C.c_int, [VP, VP, D, C.c_int64, C.c_int64, D]),
    ("cp_incidence_apply_t", C.c_int, [VP, VP, D, C.c_int64, C.c_int64, D]),
    ("cp_connected_components", C.c_int, [VP, VP, I64, I64]),
    ("cp_laplacian_lambda_max", C.c_int, [VP, VP, C.c_double, C.c_int64, D]),
    ("cp_prox_columns", C.c_int, [VP, C.c_int, D, D, C.c_int64, C.c_int64, D]),
    ("cp_project_columns", C.c_int, [VP, C.c_int, D, D, C.c_int64, C.c_int64, D]),
    ("cp_prox_jacobian_apply", C.c_int, [VP, C.c_int, D, D, D, C.c_int64, C.c_int64, D]),
    ("cp_prox_jacobian_diag", C.c_int, [VP, C.c_int, D, D, C.c_int64, C.c_int64, D]),
    ("cp_primal_objective", C.c_int, [VP, VP, VP, C.c_double, C.c_int, D, D]),
    ("cp_dual_objective", C.c_int, [VP, VP, VP, C.c_double, C.c_int, D, D]),
    ("cp_kkt_residual", C.c_int, [VP, VP, VP, C.c_double, C.c_int, D, D, D]),
    ("cp_ssnal_phi_value", C.c_int, [VP, VP, VP, C.c_double, C.c_int, D, C.c_double, D, D]),
    ("cp_ssnal_phi_gradient", C.c_int, [VP, VP, VP, C.c_double, C.c_int, D, C.c_double, D, D]),
    ("cp_ssnal_hessian_apply", C.c_int, [VP, VP, VP, C.c_double, C.c_int, D, C.c_double, D, D, D]),
    ("cp_solve", C.c_int, [VP, VP, VP, C.c_double, C.c_int, C.POINTER(SolverConfigC), D, C.c_int64, C.c_int64, D,
                           C.c_int64, D, D, C.POINTER(TerminationC)]),
    ("cp_make_schedule", C.c_int, [C.c_double, C.c_double, C.c_int64, C.c_int, D]),
    ("cp_extract_clusters", C.c_int, [VP, VP, D, C.c_int64, C.c_int64, C.c_double, I64, I64, D]),
    ("cp_run_path", C.c_int, [VP, VP, VP, C.c_int, D, C.c_int64, C.POINTER(SolverConfigC),
                              C.POINTER(PathOptionsC), D, D, I64, I64, C.POINTER(TerminationC)]),
    ("cp_run_path_ex", C.c_int, [VP, VP, VP, C.c_int, D, C.c_int64, C.POINTER(SolverConfigC),
                                 C.POINTER(PathOptionsC), D, D, I64, I64, C.POINTER(TerminationC),
                                 C.POINTER(PathSinkC)]),
    ("cp_last_trace", C.c_int, [VP, C.POINTER(TraceRowC), C.c_int64, I64]),
    ("cp_linop_identity", C.c_int, [VP, C.c_int64, C.POINTER(VP)]),
    ("cp_linop_dense", C.c_int, [VP, D, C.c_int64, C.c_int, C.POINTER(VP)]),
    ("cp_linop_sparse", C.c_int, [VP, C.c_int64, I64, I64, D, C.c_int, C.POINTER(VP)]),
    ("cp_linop_jacobi", C.c_int, [VP, D, C.c_int64, C.c_int64, C.POINTER(VP)]),
    ("cp_linop_callback", C.c_int, [VP, C.c_int64, APPLY_FN, VP, C.c_int, C.c_int, C.POINTER(VP)]),
    ("cp_linop_info", C.c_int, [VP, I64, C.POINTER(C.c_int), C.POINTER(C.c_int)]),
    ("cp_linop_destroy", None, [VP]),
    ("cp_linop_apply", C.c_int, [VP, VP, D, C.c_int64, D]),
    ("cp_pcg", C.c_int, [VP, VP, D, C.c_int64, VP, C.c_double, C.c_int64, D, I64, D, C.POINTER(C.c_int32)]),
    ("cp_power_iteration", C.c_int, [VP, VP, C.c_double, C.c_int64, D]),
    ("cp_factor_create", C.c_int, [VP, C.c_int64, I64, I64, D, C.c_double, C.POINTER(VP)]),
    ("cp_factor_solve", C.c_int, [VP, VP, D, C.c_int64, D]),
    ("cp_factor_destroy", None, [VP]),
    ("cp_norm_values", C.c_int, [VP, C.c_int, D, C.c_int64, C.c_int64, D, D]),
]

EXPORTED = [s[0] for s in _SIGS]

_lib = None


def _point_at_torch_nccl():
    """The library dlopens NCCL on first use.  A process that also imports torch must end up with
    torch's NCCL (the pip nvidia-nccl wheel), not the system one: if the older system library
    is loaded first, torch's import later fails on missing symbols.  CPB_NCCL_LIB names the
    wheel's library when it is installed (comm.cu tries an already-loaded NCCL first)."""
    if os.environ.get("CPB_NCCL_LIB"):
        return
    try:
        import importlib.util
        spec = importlib.util.find_spec("nvidia.nccl")
    except (ImportError, ValueError):
        spec = None
    for base in (list(spec.submodule_search_locations) if spec and spec.submodule_search_locations else []):
        cand = os.path.join(base, "lib", "libnccl.so.2")
        if os.path.exists(cand):
            os.environ["CPB_NCCL_LIB"] = cand
            return


def load():
    """Load the in-tree shared library (raises when it has not been built)."""
    global _lib
    if _lib is not None:
        return _lib
    if not os.path.exists(LIB_PATH):
        raise ImportError(f"{LIB_PATH} is missing: build it with `python __graft_entry__.py` (build()) — "
                          "paper_2501_15964_b200 has no CPU fallback")
    _point_at_torch_nccl()
    lib = C.CDLL(LIB_PATH)
    for name, res, args in _SIGS:
        f = getattr(lib, name)
        f.restype = res
        f.argtypes = args
    _lib = lib
    return lib


def check(rc):
    if rc == 0:
        return
    msg = (load().cp_last_error() or b"").decode()
    if rc == 1:
        raise ValueError(msg)
    raise RuntimeError(msg)
