"""Host-side mirror of the reference's ``cluspath`` API over the C-ABI.

Names, argument meaning and error behaviour follow the reference headers
(include/cluspath/*.hpp): ``compute_knn_weights``, ``WeightedGraph``,
``IncidenceOperator``, ``connected_components``, the prox helpers,
``SolverConfig``/``ProblemInstance``/``solve``, ``run_path``,
``extract_clusters`` and ``make_schedule``.  std::invalid_argument surfaces as
ValueError and std::runtime_error as RuntimeError.

Layout: a reference d x n column-major matrix is a C-contiguous float64 numpy
array of shape (n, d) here — identical bytes, one sample (or edge) per row.
Every computation runs on the B200 through libcluspath_b200.so.
"""
from __future__ import annotations

import bisect
import ctypes as C
import enum
import math
from dataclasses import dataclass, field
from typing import List, Optional, Sequence

import numpy as np

from . import _lib as L

_ctx_cache = {}


class Context:
    """One CUDA device with its stream and workspace (cp_ctx)."""

    def __init__(self, device: int = 0):
        lib = L.load()
        h = C.c_void_p()
        L.check(lib.cp_ctx_create(int(device), C.byref(h)))
        self._h = h
        self.device = device

    def close(self):
        if getattr(self, "_h", None) is not None and L._lib is not None:
            L._lib.cp_ctx_destroy(self._h)
            self._h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    def synchronize(self):
        L.check(L.load().cp_ctx_synchronize(self._h))

    def device_info(self):
        a, b, c, d = C.c_int(), C.c_int(), C.c_int(), C.c_int()
        L.check(L.load().cp_device_info(self._h, C.byref(a), C.byref(b), C.byref(c), C.byref(d)))
        return {"sm": f"{a.value}{b.value}", "sm_count": c.value, "built_arch": d.value}

    def set_comm(self, nranks: int, rank: int, unique_id: bytes):
        """Attach an NCCL communicator (cp_ctx_set_comm): the SSNAL Newton
        systems' PCG is then node-partitioned over the ranks."""
        if len(unique_id) != 128:
            raise ValueError("NCCL unique id must be 128 bytes")
        L.check(L.load().cp_ctx_set_comm(self._h, int(nranks), int(rank), C.c_char_p(bytes(unique_id))))

    def set_local_comm(self, group: "LocalGroup", rank: int):
        """Join an in-process group (cp_ctx_set_local_comm): the partitioned
        path with several ranks in one process (one host thread per rank)."""
        L.check(L.load().cp_ctx_set_local_comm(self._h, group._h, int(rank)))

    def knn_info(self):
        """How the last compute_knn_weights on this context ran (tensor-core
        candidate pass, segments, rows re-done exactly, worst |d2~-d2|/bound)."""
        tc, seg, band, ex, wr = C.c_int(), C.c_int(), C.c_int64(), C.c_int64(), C.c_double()
        L.check(L.load().cp_knn_info(self._h, C.byref(tc), C.byref(seg), C.byref(band), C.byref(ex), C.byref(wr)))
        return {"tensor_cores": tc.value, "segments": seg.value, "band_rows": band.value, "exact_rows": ex.value,
                "worst_ratio": wr.value}

    # kernel statistics for roofline accounting
    def stats_enable(self, on=True):
        L.check(L.load().cp_stats_enable(self._h, 1 if on else 0))

    def stats_reset(self):
        L.check(L.load().cp_stats_reset(self._h))

    def stats(self):
        arr = (L.KernelStatC * 64)()
        cnt = C.c_int()
        L.check(L.load().cp_stats_get(self._h, arr, 64, C.byref(cnt)))
        return {arr[k].name.decode(): {"launches": arr[k].launches, "ms": arr[k].ms, "alg_bytes": arr[k].alg_bytes}
                for k in range(min(cnt.value, 64))}


def launch_count() -> int:
    """Library kernel launches so far in this process."""
    return int(L.load().cp_launch_count())


def timer_start(ctx: Context):
    L.check(L.load().cp_timer_start(ctx._h))


def timer_stop(ctx: Context) -> float:
    ms = C.c_double()
    L.check(L.load().cp_timer_stop(ctx._h, C.byref(ms)))
    return ms.value


def flush_l2(ctx: Context):
    L.check(L.load().cp_flush_l2(ctx._h))


def normals(seed: int, count: int):
    """libstdc++ N(0,1) draws over mt19937_64(seed) (the generator io.cpp uses)."""
    out = np.empty(int(count))
    L.check(L.load().cp_normals(C.c_uint64(seed), int(count), _dp(out)))
    return out


def generate_gaussian_mixture(centers, spread, per_center, seed):
    """generate_gaussian_mixture (io.cpp:142-165); centers (m, d) -> samples (m*per_center, d)."""
    c = np.ascontiguousarray(centers, dtype=np.float64)
    m, d = c.shape
    out = np.empty((m * int(per_center), d))
    L.check(L.load().cp_gaussian_mixture(_dp(c), d, m, float(spread), int(per_center), C.c_uint64(seed), _dp(out)))
    return out


def default_context(device: int = 0) -> Context:
    ctx = _ctx_cache.get(device)
    if ctx is None:
        ctx = Context(device)
        _ctx_cache[device] = ctx
    return ctx


def _f64(a):
    return np.ascontiguousarray(a, dtype=np.float64)


class _PinnedBlock:
    """A page-locked host block (cp_host_alloc) exposed to numpy; returned to
    the pool when the last array viewing it is released."""

    _pool = {}

    def __init__(self, shape, dtype=np.float64):
        dtype = np.dtype(dtype)
        self.nbytes = int(np.prod(shape)) * dtype.itemsize
        free = _PinnedBlock._pool.get(self.nbytes)
        if free:
            self.ptr = free.pop()
        else:
            h = C.c_void_p()
            L.check(L.load().cp_host_alloc(self.nbytes, C.byref(h)))
            self.ptr = h.value
        self.__array_interface__ = {"shape": tuple(int(s) for s in shape), "typestr": dtype.str,
                                    "data": (self.ptr, False), "version": 3}

    def __del__(self):
        try:
            _PinnedBlock._pool.setdefault(self.nbytes, []).append(self.ptr)
        except Exception:
            pass


def pinned_empty(shape, dtype=np.float64):
    """numpy array in page-locked host memory (fast, asynchronous D2H target)."""
    return np.asarray(_PinnedBlock(shape, dtype))


def _dp(a):
    return a.ctypes.data_as(L.D) if a is not None else None


def _ip(a):
    return a.ctypes.data_as(L.I64) if a is not None else None


# ---- types.hpp ---------------------------------------------------------------

class DataMatrix:
    """DataMatrix (types.hpp:16-22) held in HBM.  ``values``: (n, d) samples."""

    def __init__(self, values, feature_names: Optional[Sequence[str]] = None, ctx: Optional[Context] = None):
        v = np.asarray(values, dtype=np.float64)
        if v.ndim != 2 or v.shape[0] < 1 or v.shape[1] < 1:
            raise ValueError("data matrix must have at least one feature and one sample")
        self.values = np.ascontiguousarray(v)
        names = list(feature_names or [])
        if names:
            if len(names) != v.shape[1]:
                raise ValueError("feature_names size does not match feature count")
            if any(not s for s in names):
                raise ValueError("feature_names entries must be non-empty")
        self.feature_names = names
        self.ctx = ctx or default_context()
        h = C.c_void_p()
        L.check(L.load().cp_data_create(self.ctx._h, _dp(self.values), v.shape[1], v.shape[0], C.byref(h)))
        self._h = h

    def __del__(self):
        if getattr(self, "_h", None) is not None and L._lib is not None:
            L._lib.cp_data_destroy(self._h)
            self._h = None

    @property
    def d(self):
        return self.values.shape[1]

    @property
    def n(self):
        return self.values.shape[0]


def make_data_matrix(values, feature_names=None, ctx=None) -> DataMatrix:
    """make_data_matrix (graph.cpp:10-23)."""
    return DataMatrix(values, feature_names, ctx)


# ---- graph.hpp ---------------------------------------------------------------

class WeightedGraph:
    """WeightedGraph (graph.hpp:23-51): sorted, validated, device-resident."""

    def __init__(self, n: int = 0, edges: Optional[Sequence] = None, ctx: Optional[Context] = None, _handle=None):
        self.ctx = ctx or default_context()
        if _handle is not None:
            self._h = _handle
        else:
            edges = list(edges or [])
            i = np.array([e[0] for e in edges], dtype=np.int64)
            j = np.array([e[1] for e in edges], dtype=np.int64)
            w = np.array([e[2] for e in edges], dtype=np.float64)
            h = C.c_void_p()
            L.check(L.load().cp_graph_from_edges(self.ctx._h, int(n), _ip(i), _ip(j), _dp(w), len(edges), C.byref(h)))
            self._h = h
        self._arrays = None

    @classmethod
    def from_arrays(cls, n, i, j, w, ctx=None):
        ctx = ctx or default_context()
        i = np.ascontiguousarray(i, dtype=np.int64)
        j = np.ascontiguousarray(j, dtype=np.int64)
        w = _f64(w)
        h = C.c_void_p()
        L.check(L.load().cp_graph_from_edges(ctx._h, int(n), _ip(i), _ip(j), _dp(w), len(i), C.byref(h)))
        return cls(ctx=ctx, _handle=h)

    def __del__(self):
        if getattr(self, "_h", None) is not None and L._lib is not None:
            L._lib.cp_graph_destroy(self._h)
            self._h = None

    def nodes(self) -> int:
        return L.load().cp_graph_nodes(self._h)

    def edge_count(self) -> int:
        return L.load().cp_graph_edge_count(self._h)

    def arrays(self):
        """(i, j, w, d2) in list order; d2 = kNN squared distances (NaN otherwise)."""
        if self._arrays is None:
            E = self.edge_count()
            i = np.empty(E, np.int64)
            j = np.empty(E, np.int64)
            w = np.empty(E, np.float64)
            d2 = np.empty(E, np.float64)
            L.check(L.load().cp_graph_export(self.ctx._h, self._h, _ip(i), _ip(j), _dp(w), _dp(d2)))
            self._arrays = (i, j, w, d2)
        return self._arrays

    def edges(self):
        i, j, w, _ = self.arrays()
        return [(int(a), int(b), float(c)) for a, b, c in zip(i, j, w)]

    def edge(self, l):
        i, j, w, _ = self.arrays()
        return (int(i[l]), int(j[l]), float(w[l]))

    def weights(self):
        return self.arrays()[2].copy()

    def degrees(self):
        deg = np.empty(self.nodes(), np.int64)
        L.check(L.load().cp_graph_degrees(self.ctx._h, self._h, _ip(deg)))
        return deg

    def degree(self, v):
        if v < 0 or v >= self.nodes():
            raise ValueError("node index out of range")
        return int(self.degrees()[v])

    def max_degree(self):
        deg = self.degrees()
        return int(deg.max()) if len(deg) else 0

    def find_edge(self, i, j):
        """graph.cpp:47-56: position of (i, j) in the sorted list, or None."""
        if i > j:
            i, j = j, i
        a, b, _, _ = self.arrays()
        keys = list(zip(a.tolist(), b.tolist()))
        p = bisect.bisect_left(keys, (i, j))
        return p if p < len(keys) and keys[p] == (i, j) else None


def compute_knn_weights(data: DataMatrix, k: int, phi: float) -> WeightedGraph:
    """compute_knn_weights (graph.hpp:58; graph.cpp:75-114), on the GPU."""
    h = C.c_void_p()
    L.check(L.load().cp_knn_graph(data.ctx._h, data._h, int(k), float(phi), C.byref(h)))
    return WeightedGraph(ctx=data.ctx, _handle=h)


class LocalGroup:
    """In-process rank group (cp_local_group): collectives meet at host
    barriers, so several ranks can share one GPU without any kernel waiting
    on another rank."""

    def __init__(self, nranks: int):
        h = C.c_void_p()
        L.check(L.load().cp_local_group_create(int(nranks), C.byref(h)))
        self._h = h
        self.nranks = int(nranks)

    def __del__(self):
        if getattr(self, "_h", None) is not None and L._lib is not None:
            L._lib.cp_local_group_destroy(self._h)
            self._h = None


def nccl_unique_id() -> bytes:
    """A fresh 128-byte NCCL unique id (cp_nccl_unique_id)."""
    buf = C.create_string_buffer(128)
    L.check(L.load().cp_nccl_unique_id(buf))
    return buf.raw


def init_comm_from_torch(ctx: "Context", group=None) -> None:
    """One process per GPU: rank 0 creates the NCCL id, torch.distributed
    broadcasts it, every rank attaches the communicator to its context."""
    import torch.distributed as dist
    world = dist.get_world_size(group)
    rank = dist.get_rank(group)
    obj = [nccl_unique_id() if rank == 0 else None]
    dist.broadcast_object_list(obj, src=0, group=group)
    ctx.set_comm(world, rank, obj[0])


def shard_rows(n: int, nranks: int, rank: int):
    """Query rows [r0, r1) of `rank` in the row-sharded kNN (cp_shard_rows)."""
    r0, r1 = C.c_int64(), C.c_int64()
    L.check(L.load().cp_shard_rows(int(n), int(nranks), int(rank), C.byref(r0), C.byref(r1)))
    return r0.value, r1.value


def knn_rows_into(data: DataMatrix, k: int, r0: int, r1: int, kd, kj) -> None:
    """cp_knn_rows: rows [r0, r1) of the per-row kNN lists into the CUDA
    tensors kd (n x k float64) and kj (n x k int32) at their global rows."""
    n = data.n
    if kd.shape[0] < n or kj.shape[0] < n or kd.shape[1] != k or kj.shape[1] != k or not kd.is_cuda or not kj.is_cuda:
        raise ValueError("knn_rows_into: kd / kj must be CUDA tensors of at least n x k")
    if str(kd.dtype) != "torch.float64" or str(kj.dtype) != "torch.int32" or not kd.is_contiguous() \
            or not kj.is_contiguous():
        raise ValueError("knn_rows_into: kd must be contiguous float64 and kj contiguous int32")
    L.check(L.load().cp_knn_rows(data.ctx._h, data._h, int(k), int(r0), int(r1), C.c_void_p(kd.data_ptr()),
                                 C.c_void_p(kj.data_ptr())))


def gather_row_lists(n: int, k: int, rows_fn, device, group=None):
    """Row-sharded kNN lists: this rank fills its rows with
    ``rows_fn(r0, r1, kd, kj)`` (kd, kj: (n_pad, k) float64 / int32 tensors on
    `device`), then every rank receives every rank's equal-size row chunk
    through torch.distributed (NCCL over NVLink on GPUs, gloo on CPU).
    Returns the complete (n, k) lists, identical on every rank."""
    import torch
    import torch.distributed as dist
    P = dist.get_world_size(group) if dist.is_initialized() else 1
    rank = dist.get_rank(group) if dist.is_initialized() else 0
    chunk = -(-n // P)
    kd = torch.zeros((chunk * P, k), dtype=torch.float64, device=device)
    kj = torch.zeros((chunk * P, k), dtype=torch.int32, device=device)
    r0, r1 = shard_rows(n, P, rank)
    if r1 > r0:
        rows_fn(r0, r1, kd, kj)
    if P > 1:
        mine_d = kd[rank * chunk:(rank + 1) * chunk].contiguous()
        mine_j = kj[rank * chunk:(rank + 1) * chunk].contiguous()
        outs_d = [torch.empty_like(mine_d) for _ in range(P)]
        outs_j = [torch.empty_like(mine_j) for _ in range(P)]
        dist.all_gather(outs_d, mine_d, group=group)
        dist.all_gather(outs_j, mine_j, group=group)
        kd = torch.cat(outs_d)
        kj = torch.cat(outs_j)
    return kd[:n], kj[:n]


def compute_knn_weights_sharded(data: DataMatrix, k: int, phi: float, group=None) -> WeightedGraph:
    """compute_knn_weights with the n^2 d distance work split by query-row
    blocks over the ranks of `group` (one process per GPU, NCCL all-gather of
    the n x k lists); every rank returns the same graph, bit-identical to
    compute_knn_weights on one GPU."""
    import torch
    n = data.n
    dev = torch.device("cuda", torch.cuda.current_device())

    def rows_fn(r0, r1, kd, kj):
        torch.cuda.synchronize(dev)
        knn_rows_into(data, k, r0, r1, kd, kj)

    kd, kj = gather_row_lists(n, int(k), rows_fn, dev, group)
    kd, kj = kd.contiguous(), kj.contiguous()
    torch.cuda.synchronize(dev)
    h = C.c_void_p()
    L.check(L.load().cp_graph_from_knn(data.ctx._h, n, int(k), float(phi), C.c_void_p(kd.data_ptr()),
                                       C.c_void_p(kj.data_ptr()), C.byref(h)))
    return WeightedGraph(ctx=data.ctx, _handle=h)


class IncidenceOperator:
    """IncidenceOperator (graph.hpp:62-86): X B and Z B^T on the GPU."""

    def __init__(self, graph: WeightedGraph):
        self.graph = graph

    def nodes(self):
        return self.graph.nodes()

    def edge_count(self):
        return self.graph.edge_count()

    def apply(self, X):
        X = _f64(X)
        if X.ndim != 2:
            raise ValueError("incidence apply: operand must be a matrix")
        out = np.empty((self.graph.edge_count(), X.shape[1]))
        L.check(L.load().cp_incidence_apply(self.graph.ctx._h, self.graph._h, _dp(X), X.shape[1], X.shape[0],
                                            _dp(out)))
        return out

    def apply_transpose(self, Z):
        Z = _f64(Z)
        if Z.ndim != 2:
            raise ValueError("incidence adjoint: operand must be a matrix")
        out = np.empty((self.graph.nodes(), Z.shape[1]))
        L.check(L.load().cp_incidence_apply_t(self.graph.ctx._h, self.graph._h, _dp(Z), Z.shape[1], Z.shape[0],
                                              _dp(out)))
        return out

    def laplacian(self):
        """IncidenceOperator::laplacian (graph.cpp:154-167): B B^T as a
        scipy.sparse.csc_matrix, built on the GPU."""
        import scipy.sparse as sp
        n = self.graph.nodes()
        nnz = C.c_int64()
        h = self.graph.ctx._h
        L.check(L.load().cp_graph_laplacian(h, self.graph._h, None, None, None, C.byref(nnz)))
        colptr = np.empty(n + 1, np.int64)
        rows = np.empty(max(1, nnz.value), np.int64)
        vals = np.empty(max(1, nnz.value))
        L.check(L.load().cp_graph_laplacian(h, self.graph._h, _ip(colptr), _ip(rows), _dp(vals), C.byref(nnz)))
        return sp.csc_matrix((vals[:nnz.value], rows[:nnz.value], colptr), shape=(n, n))

    def laplacian_lambda_max(self, tol=1e-9, max_iter=10000):
        """power_iteration(LinearOperator::sparse(laplacian())) (linalg.cpp:194-242)."""
        out = C.c_double()
        L.check(L.load().cp_laplacian_lambda_max(self.graph.ctx._h, self.graph._h, tol, int(max_iter), C.byref(out)))
        return out.value


def connected_components(graph: WeightedGraph):
    """connected_components (graph.cpp:169-196): first-appearance labels."""
    lab = np.empty(graph.nodes(), np.int64)
    K = C.c_int64()
    L.check(L.load().cp_connected_components(graph.ctx._h, graph._h, _ip(lab), C.byref(K)))
    return lab


def component_count(labels) -> int:
    labels = np.asarray(labels)
    return int(labels.max()) + 1 if len(labels) else 0


# ---- prox.hpp ----------------------------------------------------------------

class PenaltyNorm(enum.IntEnum):
    """prox.hpp:8 PenaltyNorm{l1, l2}, extended with linf (q = infinity, code 0;
    no reference counterpart)."""
    linf = 0
    l1 = 1
    l2 = 2


def penalty_norm_from_q(q) -> PenaltyNorm:
    """q in {1, 2} as the reference (prox.cpp:17-21), plus q = inf / "inf"."""
    if q == 1:
        return PenaltyNorm.l1
    if q == 2:
        return PenaltyNorm.l2
    if (isinstance(q, float) and math.isinf(q) and q > 0) or (isinstance(q, str) and q.lower() in ("inf", "linf")):
        return PenaltyNorm.linf
    raise ValueError(f"penalty norm exponent must be 1, 2 or inf, got {q}")


def _qcode(norm) -> int:
    """C-ABI code of a penalty norm: PenaltyNorm / 0, 1, 2 / inf / "inf"."""
    if isinstance(norm, PenaltyNorm):
        return int(norm)
    if isinstance(norm, (int, np.integer)) and int(norm) in (0, 1, 2):
        return int(norm)
    return int(penalty_norm_from_q(norm))


def _cols_call(fn, q, V, t, ctx):
    V = _f64(V)
    if V.ndim != 2:
        raise ValueError("columns must be given as a matrix")
    t = _f64(t).reshape(-1)
    if len(t) != V.shape[0]:
        raise ValueError("one threshold per column required")
    out = np.empty_like(V)
    ctx = ctx or default_context()
    L.check(fn(ctx._h, int(q), _dp(V), _dp(t), V.shape[1], V.shape[0], _dp(out)))
    return out


def prox_columns(V, thresholds, norm=PenaltyNorm.l2, ctx=None):
    """prox_columns_into (prox.cpp:73-80): per-column prox of t_l ||.||_q."""
    return _cols_call(L.load().cp_prox_columns, _qcode(norm), V, thresholds, ctx)


def project_columns(Z, radii, norm=PenaltyNorm.l2, ctx=None):
    """project_columns (prox.cpp:82-93): per-column dual-ball projection."""
    return _cols_call(L.load().cp_project_columns, _qcode(norm), Z, radii, ctx)


def prox_jacobian_apply(V, thresholds, W, norm=PenaltyNorm.l2, ctx=None):
    """Columnwise M_l W_l with M_l = Jacobian of prox at V_l (prox.cpp:95-132), on the GPU."""
    ctx = ctx or default_context()
    V, W = _f64(V), _f64(W)
    if V.shape != W.shape or V.ndim != 2:
        raise ValueError("prox_jacobian_apply: V and W must have the same (E, d) shape")
    t = _f64(thresholds)
    out = np.empty_like(V)
    L.check(L.load().cp_prox_jacobian_apply(ctx._h, _qcode(norm), _dp(V), _dp(t), _dp(W), V.shape[1], V.shape[0],
                                            _dp(out)))
    return out


class ProxJacobian:
    """prox_jacobian(v, t, norm) (prox.hpp:38-47): apply(w) and diag(r) of the
    structured Jacobian of prox_{t||.||} at v, evaluated on the GPU."""

    def __init__(self, v, t, norm=PenaltyNorm.l2, ctx=None):
        self.v = _f64(v).reshape(-1)
        self.t = float(t)
        self.norm = norm
        self.ctx = ctx

    def apply(self, w):
        w = _f64(w).reshape(-1)
        if w.shape != self.v.shape:
            raise ValueError("ProxJacobian::apply: size mismatch")
        return prox_jacobian_apply(self.v[None, :], [self.t], w[None, :], self.norm, self.ctx)[0]

    def diag(self, r=None):
        dg = prox_jacobian_diag(self.v[None, :], [self.t], self.norm, self.ctx)[0]
        return dg if r is None else dg[r]


def prox_jacobian(v, t, norm=PenaltyNorm.l2, ctx=None) -> ProxJacobian:
    if not (t >= 0) or not math.isfinite(t):
        raise ValueError("prox_jacobian: threshold must be finite and >= 0")
    return ProxJacobian(v, t, norm, ctx)


def prox_jacobian_diag(V, thresholds, norm=PenaltyNorm.l2, ctx=None):
    """ProxJacobian::diag per column (prox.cpp:106-132)."""
    return _cols_call(L.load().cp_prox_jacobian_diag, _qcode(norm), V, thresholds, ctx)


def norm_value(v, norm=PenaltyNorm.l2, ctx=None) -> float:
    """norm_value (prox.hpp:14; prox.cpp:25-31): ||v||_q on the GPU."""
    return _norms(v, norm, ctx)[0]


def dual_norm_value(v, norm=PenaltyNorm.l2, ctx=None) -> float:
    """dual_norm_value (prox.hpp:15; prox.cpp:25-31): ||v||_q' on the GPU."""
    return _norms(v, norm, ctx)[1]


def _norms(v, norm, ctx):
    v = _f64(v).reshape(-1)
    ctx = ctx or default_context()
    a, b = C.c_double(), C.c_double()
    L.check(L.load().cp_norm_values(ctx._h, _qcode(norm), _dp(v), len(v), 1, C.byref(a), C.byref(b)))
    return a.value, b.value


def prox_norm(v, t, norm=PenaltyNorm.l2, ctx=None):
    """prox_norm (prox.hpp:19-21): prox_{t ||.||_q}(v)."""
    if not (t >= 0) or not math.isfinite(t):
        raise ValueError("prox_norm: threshold must be finite and >= 0")
    return prox_columns(_f64(v).reshape(1, -1), [t], norm, ctx)[0]


def prox_norm_into(v, t, norm, out, ctx=None):
    """prox_norm_into (prox.hpp:20-21): writes prox_{t ||.||_q}(v) into `out`."""
    out[...] = prox_norm(v, t, norm, ctx).reshape(np.shape(out))


def project_dual_ball(z, r, norm=PenaltyNorm.l2, ctx=None):
    """project_dual_ball (prox.hpp:24-26): projection onto {||.||_q' <= r}."""
    if not (r >= 0) or not math.isfinite(r):
        raise ValueError("project_dual_ball: threshold must be finite and >= 0")
    return project_columns(_f64(z).reshape(1, -1), [r], norm, ctx)[0]


def project_dual_ball_into(z, r, norm, out, ctx=None):
    """project_dual_ball_into (prox.hpp:25-26)."""
    out[...] = project_dual_ball(z, r, norm, ctx).reshape(np.shape(out))


def moreau_check(v, t, norm=PenaltyNorm.l2, ctx=None) -> float:
    """moreau_check (prox.hpp:51-54): ||prox(v) + Pi(v) - v||_inf."""
    v = _f64(v).reshape(-1)
    return float(np.max(np.abs(prox_norm(v, t, norm, ctx) + project_dual_ball(v, t, norm, ctx) - v), initial=0.0))


# ---- linalg.hpp (linalg.hpp:17-87) ----------------------------------------------
# Operands are (rows,) vectors or (rows, cols) blocks in the reference's own
# orientation (Eigen d x k), passed column-major to the device.

def _fblock(x, rows=None):
    x = np.asarray(x, dtype=np.float64)
    vec = x.ndim == 1
    x2 = x.reshape(-1, 1) if vec else x
    if x2.ndim != 2:
        raise ValueError("operand must be a vector or a matrix")
    return np.asfortranarray(x2), vec


class LinearOperator:
    """LinearOperator (linalg.hpp:38-65).  LinearOperator(rows, fn) wraps a
    Python callable (host round trip per apply); the static factories build
    device-resident operators."""

    def __init__(self, rows, fn=None, symmetric=True, positive_definite=False, ctx=None, _handle=None):
        self.ctx = ctx or default_context()
        self._h = None
        self._keep = None
        if _handle is not None:
            self._h = _handle
            return
        if fn is None:
            raise ValueError("LinearOperator: empty apply function")
        self._err = None

        def tramp(user, xin, xout, r, c):
            try:
                X = np.ctypeslib.as_array(xin, shape=(int(c) * int(r),)).reshape((int(r), int(c)), order="F")
                Y = np.asarray(fn(X.copy(order="F") if c > 1 else X[:, 0].copy()), dtype=np.float64)
                Y = Y.reshape((int(r), int(c)), order="F") if Y.ndim == 1 else Y
                if Y.shape != (int(r), int(c)):
                    raise RuntimeError("LinearOperator::apply: image shape mismatch")
                np.ctypeslib.as_array(xout, shape=(int(c) * int(r),))[:] = Y.reshape(-1, order="F")
                return 0
            except Exception as e:  # noqa: BLE001 — re-raised by the caller after the C call returns
                self._err = e
                return 1

        self._keep = L.APPLY_FN(tramp)
        h = C.c_void_p()
        L.check(L.load().cp_linop_callback(self.ctx._h, int(rows), self._keep, None, int(bool(symmetric)),
                                           int(bool(positive_definite)), C.byref(h)))
        self._h = h

    def __del__(self):
        if getattr(self, "_h", None) is not None and L._lib is not None:
            L._lib.cp_linop_destroy(self._h)
            self._h = None

    def _info(self):
        r, s, p = C.c_int64(), C.c_int(), C.c_int()
        L.check(L.load().cp_linop_info(self._h, C.byref(r), C.byref(s), C.byref(p)))
        return r.value, bool(s.value), bool(p.value)

    def rows(self):
        return self._info()[0]

    def symmetric(self):
        return self._info()[1]

    def positive_definite(self):
        return self._info()[2]

    def _raise_callback(self, rc):
        err = getattr(self, "_err", None)
        if rc != 0 and err is not None:
            self._err = None
            raise err
        L.check(rc)

    def apply(self, x):
        X, vec = _fblock(x)
        if X.shape[0] != self.rows():
            raise ValueError("LinearOperator::apply: operand has wrong row count")
        out = np.empty(X.shape, order="F")
        self._raise_callback(L.load().cp_linop_apply(self.ctx._h, self._h, _dp(X), X.shape[1], _dp(out)))
        return out[:, 0].copy() if vec else out

    @staticmethod
    def _make(fn, ctx, *args):
        ctx = ctx or default_context()
        h = C.c_void_p()
        L.check(fn(ctx._h, *args, C.byref(h)))
        return LinearOperator(0, ctx=ctx, _handle=h)

    @staticmethod
    def identity(n, ctx=None):
        return LinearOperator._make(L.load().cp_linop_identity, ctx, int(n))

    @staticmethod
    def dense(M, positive_definite=False, ctx=None):
        M = np.asarray(M, dtype=np.float64)
        if M.ndim != 2 or M.shape[0] != M.shape[1]:
            raise ValueError("LinearOperator::dense: matrix must be square")
        M = np.asfortranarray(M)
        return LinearOperator._make(L.load().cp_linop_dense, ctx, _dp(M), M.shape[0], int(bool(positive_definite)))

    @staticmethod
    def sparse(M, positive_definite=False, ctx=None):
        import scipy.sparse as sp
        M = sp.csc_matrix(M)
        if M.shape[0] != M.shape[1]:
            raise ValueError("LinearOperator::sparse: matrix must be square")
        cp_ = np.ascontiguousarray(M.indptr, dtype=np.int64)
        ri = np.ascontiguousarray(M.indices, dtype=np.int64)
        va = np.ascontiguousarray(M.data, dtype=np.float64)
        return LinearOperator._make(L.load().cp_linop_sparse, ctx, M.shape[0], _ip(cp_), _ip(ri), _dp(va),
                                    int(bool(positive_definite)))

    @staticmethod
    def jacobi(diag, ctx=None):
        """jacobi(Vector) for a 1-D diagonal, jacobi(Matrix) for a 2-D block."""
        D, vec = _fblock(diag)
        return LinearOperator._make(L.load().cp_linop_jacobi, ctx, _dp(D), D.shape[0], D.shape[1])


@dataclass
class PcgResult:
    """PcgResult (linalg.hpp:67-72)."""
    x: np.ndarray
    iterations: int = 0
    residual: float = 0.0
    converged: bool = False


def pcg(op: LinearOperator, rhs, preconditioner: Optional[LinearOperator] = None, tol: float = 1e-10,
        max_iter: int = 1000) -> PcgResult:
    """pcg (linalg.hpp:76-77; linalg.cpp:143-192) on the GPU."""
    B, vec = _fblock(rhs)
    if B.shape[0] != op.rows():
        raise ValueError("pcg: rhs row count does not match the operator")
    x = np.empty(B.shape, order="F")
    it, res, conv = C.c_int64(), C.c_double(), C.c_int32()
    rc = L.load().cp_pcg(op.ctx._h, op._h, _dp(B), B.shape[1], preconditioner._h if preconditioner else None,
                         float(tol), int(max_iter), _dp(x), C.byref(it), C.byref(res), C.byref(conv))
    for o in (op, preconditioner):
        if o is not None and getattr(o, "_err", None) is not None:
            o._raise_callback(rc)
    L.check(rc)
    return PcgResult(x[:, 0].copy() if vec else x, it.value, res.value, bool(conv.value))


def power_iteration(op: LinearOperator, tol: float = 1e-9, max_iter: int = 10000) -> float:
    """power_iteration (linalg.hpp:82-83; linalg.cpp:194-242) on the GPU."""
    out = C.c_double()
    op._raise_callback(L.load().cp_power_iteration(op.ctx._h, op._h, float(tol), int(max_iter), C.byref(out)))
    return out.value


class CholeskyFactor:
    """CholeskyFactor(L, rho) (linalg.hpp:17-33): solve() returns (I + rho L)^{-1} rhs,
    computed on the GPU by Jacobi-preconditioned CG to 1e-14 relative residual per column."""

    def __init__(self, Lap, rho, ctx=None):
        import scipy.sparse as sp
        self.ctx = ctx or default_context()
        Lc = sp.csc_matrix(Lap)
        if Lc.shape[0] != Lc.shape[1]:
            raise ValueError("cholesky: matrix must be square")
        self._n, self._rho = Lc.shape[0], float(rho)
        cp_ = np.ascontiguousarray(Lc.indptr, dtype=np.int64)
        ri = np.ascontiguousarray(Lc.indices, dtype=np.int64)
        va = np.ascontiguousarray(Lc.data, dtype=np.float64)
        h = C.c_void_p()
        self._h = None
        L.check(L.load().cp_factor_create(self.ctx._h, self._n, _ip(cp_), _ip(ri), _dp(va), float(rho), C.byref(h)))
        self._h = h

    def __del__(self):
        if getattr(self, "_h", None) is not None and L._lib is not None:
            L._lib.cp_factor_destroy(self._h)
            self._h = None

    def size(self):
        return self._n

    def rho(self):
        return self._rho

    def solve(self, rhs):
        B, vec = _fblock(rhs)
        if B.shape[0] != self._n:
            raise ValueError("cholesky solve: rhs has wrong row count")
        out = np.empty(B.shape, order="F")
        L.check(L.load().cp_factor_solve(self.ctx._h, self._h, _dp(B), B.shape[1], _dp(out)))
        return out[:, 0].copy() if vec else out


# ---- solvers.hpp ---------------------------------------------------------------

class Algorithm(enum.IntEnum):
    ADMM = 0
    FastAMA = 1
    SSNAL = 2


def algorithm_from_name(name: str) -> Algorithm:
    if name == "admm":
        return Algorithm.ADMM
    if name in ("ama", "fast-ama", "fastama"):
        return Algorithm.FastAMA
    if name == "ssnal":
        return Algorithm.SSNAL
    raise ValueError(f"unknown solver '{name}' (expected ssnal, admm or ama)")


def algorithm_name(a) -> str:
    return {0: "admm", 1: "ama", 2: "ssnal"}[int(a)]


@dataclass
class SolverConfig:
    """SolverConfig (solvers.hpp:72-93) with the reference defaults."""
    algorithm: Algorithm = Algorithm.SSNAL
    epsilon: float = 1e-6
    kkt_factor: float = 10.0
    max_iter: int = 0
    time_limit: Optional[float] = None
    admm_rho: float = 1.0
    ama_step_safety: float = 0.99
    ssnal_sigma0: float = 1.0
    armijo_mu: float = 1e-4
    backtrack_beta: float = 0.5
    ssnal_newton_max: int = 50
    pcg_max_iter: int = 500
    collect_trace: bool = False

    def to_c(self):
        if self.time_limit is not None and not (self.time_limit > 0):
            raise ValueError("config: time_limit must be positive when set")
        alg = self.algorithm if not isinstance(self.algorithm, str) else algorithm_from_name(self.algorithm)
        return L.SolverConfigC(int(alg), int(self.collect_trace), self.epsilon, self.kkt_factor, int(self.max_iter),
                               float(self.time_limit or 0.0), self.admm_rho, self.ama_step_safety, self.ssnal_sigma0,
                               self.armijo_mu, self.backtrack_beta, int(self.ssnal_newton_max),
                               int(self.pcg_max_iter))

    def resolved_max_iter(self):
        if self.max_iter > 0:
            return self.max_iter
        return 100 if int(self.algorithm) == 2 else 20000


@dataclass
class TerminationRecord:
    f_primal: float = 0.0
    f_dual: float = 0.0
    gap: float = 0.0
    iterations: int = 0
    converged: bool = False
    wall_time: float = 0.0
    newton: int = 0
    cg: int = 0
    armijo: int = 0
    hess_apply: int = 0

    @classmethod
    def from_c(cls, t):
        return cls(t.f_primal, t.f_dual, t.gap, t.iterations, bool(t.converged), t.wall_time, t.newton, t.cg,
                   t.armijo, t.hess_apply)


@dataclass
class TraceRow:
    """TraceRow (solvers.hpp:54-60)."""
    iter: int = 0
    f_p: float = 0.0
    f_d: float = 0.0
    gap: float = 0.0
    elapsed_s: float = 0.0


def _trace_rows(rows, count):
    return [TraceRow(rows[k].iter, rows[k].f_p, rows[k].f_d, rows[k].gap, rows[k].elapsed_s) for k in range(count)]


@dataclass
class Solution:
    X: np.ndarray
    Z: np.ndarray
    termination: TerminationRecord = field(default_factory=TerminationRecord)
    trace: List[TraceRow] = field(default_factory=list)  # filled when SolverConfig.collect_trace


class ProblemInstance:
    """ProblemInstance (solvers.hpp:26-43)."""

    def __init__(self, data: DataMatrix, graph: WeightedGraph, gamma: float, norm=PenaltyNorm.l2):
        if data.n != graph.nodes():
            raise ValueError(f"instance: graph has {graph.nodes()} nodes for {data.n} samples")
        if not (gamma >= 0.0) or not np.isfinite(gamma):
            raise ValueError("instance: gamma must be finite and >= 0")
        self.data, self.graph, self.gamma, self.norm = data, graph, float(gamma), _qcode(norm)
        self.B = IncidenceOperator(graph)

    def penalty_radii(self):
        return self.gamma * self.graph.weights()

    def d(self):
        return self.data.d

    def n(self):
        return self.data.n

    def edge_count(self):
        return self.graph.edge_count()

    def _args(self):
        return self.data.ctx._h, self.data._h, self.graph._h, self.gamma, self.norm


def primal_objective(inst: ProblemInstance, X) -> float:
    X = _f64(X)
    if X.shape != (inst.n(), inst.d()):
        raise ValueError("primal_objective: X has the wrong shape")
    out = C.c_double()
    L.check(L.load().cp_primal_objective(*inst._args(), _dp(X), C.byref(out)))
    return out.value


def dual_objective(inst: ProblemInstance, Z) -> float:
    Z = _f64(Z)
    if Z.shape != (inst.edge_count(), inst.d()):
        raise ValueError("dual_objective: Z has the wrong shape")
    out = C.c_double()
    L.check(L.load().cp_dual_objective(*inst._args(), _dp(Z), C.byref(out)))
    return out.value


def duality_gap(f_p, f_d) -> float:
    return abs(f_p - f_d) / (1.0 + abs(f_p) + abs(f_d))


def recover_primal(inst: ProblemInstance, Z):
    return inst.data.values - inst.B.apply_transpose(Z)


def kkt_residual(inst: ProblemInstance, X, Z) -> float:
    X, Z = _f64(X), _f64(Z)
    if X.shape != (inst.n(), inst.d()):
        raise ValueError("kkt_residual: X has the wrong shape")
    if Z.shape != (inst.edge_count(), inst.d()):
        raise ValueError("kkt_residual: Z has the wrong shape")
    out = C.c_double()
    L.check(L.load().cp_kkt_residual(*inst._args(), _dp(X), _dp(Z), C.byref(out)))
    return out.value


def ssnal_phi_value(inst, Z, sigma, X) -> float:
    out = C.c_double()
    L.check(L.load().cp_ssnal_phi_value(*inst._args(), _dp(_f64(Z)), float(sigma), _dp(_f64(X)), C.byref(out)))
    return out.value


def ssnal_phi_gradient(inst, Z, sigma, X):
    out = np.empty((inst.n(), inst.d()))
    L.check(L.load().cp_ssnal_phi_gradient(*inst._args(), _dp(_f64(Z)), float(sigma), _dp(_f64(X)), _dp(out)))
    return out


def ssnal_hessian_apply(inst, Z, sigma, X, D):
    out = np.empty((inst.n(), inst.d()))
    L.check(L.load().cp_ssnal_hessian_apply(*inst._args(), _dp(_f64(Z)), float(sigma), _dp(_f64(X)), _dp(_f64(D)),
                                            _dp(out)))
    return out


def solve(inst: ProblemInstance, config: Optional[SolverConfig] = None, warm: Optional[Solution] = None) -> Solution:
    """solve (objective.cpp:115-123) -> solve_ssnal / solve_admm / solve_fast_ama on the GPU."""
    config = config or SolverConfig()
    cfg = config.to_c()
    n, d, E = inst.n(), inst.d(), inst.edge_count()
    X = np.empty((n, d))
    Z = np.empty((E, d))
    t = L.TerminationC()
    wx = wz = None
    wshape = (0, 0, 0)
    if warm is not None:
        wx, wz = _f64(warm.X), _f64(warm.Z)
        if wx.ndim != 2 or wz.ndim != 2 or wx.shape[1] != wz.shape[1]:
            raise ValueError("warm start does not match the instance shapes")
        wshape = (wx.shape[1], wx.shape[0], wz.shape[0])
    L.check(L.load().cp_solve(*inst._args(), C.byref(cfg), _dp(wx), wshape[0], wshape[1], _dp(wz), wshape[2], _dp(X),
                              _dp(Z), C.byref(t)))
    trace = []
    if config.collect_trace:
        cnt = C.c_int64()
        L.check(L.load().cp_last_trace(inst.data.ctx._h, None, 0, C.byref(cnt)))
        rows = (L.TraceRowC * max(1, cnt.value))()
        L.check(L.load().cp_last_trace(inst.data.ctx._h, rows, cnt.value, C.byref(cnt)))
        trace = _trace_rows(rows, cnt.value)
    return Solution(X, Z, TerminationRecord.from_c(t), trace)


# ---- path.hpp --------------------------------------------------------------------

class Spacing(enum.IntEnum):
    linear = 0
    geometric = 1


@dataclass
class GammaSchedule:
    values: List[float]
    start: float = 0.0
    end: float = 0.0
    count: int = 0
    spacing: Spacing = Spacing.geometric


def make_schedule(start, end, count, spacing=Spacing.geometric) -> GammaSchedule:
    """make_schedule (path.cpp:21-58)."""
    out = np.empty(max(int(count), 1))
    L.check(L.load().cp_make_schedule(float(start), float(end), int(count), int(spacing), _dp(out)))
    return GammaSchedule(out[:int(count)].tolist(), float(start), float(end), int(count), Spacing(int(spacing)))


@dataclass
class ClusterAssignment:
    labels: np.ndarray
    K: int
    centroids: np.ndarray


def extract_clusters(X, graph: WeightedGraph, fuse_tol: float = 1e-3) -> ClusterAssignment:
    """extract_clusters (path.cpp:60-89) on the GPU."""
    X = _f64(X)
    n, d = X.shape
    lab = np.empty(n, np.int64)
    K = C.c_int64()
    cent = np.empty((n, d))
    L.check(L.load().cp_extract_clusters(graph.ctx._h, graph._h, _dp(X), d, n, float(fuse_tol), _ip(lab), C.byref(K),
                                         _dp(cent)))
    return ClusterAssignment(lab, K.value, cent[:K.value].copy())


@dataclass
class PathOptions:
    warm_start: bool = True
    require_connected: bool = False
    fuse_tol: float = 1e-3


@dataclass
class PathResult:
    schedule: GammaSchedule
    solutions: List[Solution]
    assignments: List[ClusterAssignment]
    stats: List[TerminationRecord]
    solver: SolverConfig

    def all_converged(self):
        return all(s.converged for s in self.stats)


def run_path(data: DataMatrix, graph: WeightedGraph, norm, schedule: GammaSchedule, config: Optional[SolverConfig] = None,
             options: Optional[PathOptions] = None, keep_solutions: bool = True, keep_z: bool = True,
             centroids: bool = True) -> PathResult:
    """run_path (path.cpp:110-142): warm-started gamma sweep, all on the GPU.
    keep_solutions=False returns labels and records only; keep_z=False keeps
    every X(gamma) but not the E x d multipliers (their host copy is the
    dominant cost of a large path: 20 x E x d doubles).  centroids=False skips
    ClusterAssignment.centroids (path.cpp:135; one d x K D2H per gamma)."""
    config = config or SolverConfig()
    options = options or PathOptions()
    gam = _f64(schedule.values)
    T = len(gam)
    if T == 0:
        raise ValueError("run_path: empty schedule")
    n, d, E = data.n, data.d, graph.edge_count()
    X = pinned_empty((T, n, d)) if keep_solutions else None
    Z = pinned_empty((T, E, d)) if keep_solutions and keep_z else None
    lab = np.empty((T, n), np.int64)
    K = np.empty(T, np.int64)
    terms = (L.TerminationC * T)()
    cfg = config.to_c()
    opt = L.PathOptionsC(int(options.warm_start), int(options.require_connected), float(options.fuse_tol))
    cents = [None] * T
    traces = [[] for _ in range(T)]

    def on_cent(user, t, k, dd, ptr):  # ClusterAssignment::centroids, d x K -> (K, d) rows
        cents[t] = np.ctypeslib.as_array(ptr, shape=(int(k) * int(dd),)).reshape(int(k), int(dd)).copy() \
            if k > 0 else np.empty((0, int(dd)))

    def on_trace(user, t, rows, cnt):
        traces[t] = _trace_rows(rows, int(cnt))

    sink = L.PathSinkC(None, L.CENT_FN(on_cent) if centroids else L.CENT_FN(),
                       L.TRACE_FN(on_trace) if config.collect_trace else L.TRACE_FN(), int(X is not None))
    L.check(L.load().cp_run_path_ex(data.ctx._h, data._h, graph._h, _qcode(norm), _dp(gam), T, C.byref(cfg),
                                    C.byref(opt), _dp(X), _dp(Z), _ip(lab), _ip(K), terms, C.byref(sink)))
    stats = [TerminationRecord.from_c(t) for t in terms]
    sols = [Solution(X[t] if X is not None else None, Z[t] if Z is not None else None, stats[t], traces[t])
            for t in range(T)]
    if centroids and X is not None:  # K = n: every node its own cluster, centroids = X (skip_identity)
        for t in range(T):
            if cents[t] is None and int(K[t]) == n:
                cents[t] = X[t]
    asg = [ClusterAssignment(lab[t], int(K[t]), cents[t]) for t in range(T)]
    return PathResult(schedule, sols, asg, stats, config)


def two_point_closed_form(a1, a2, w, gamma):
    """path.cpp:91-103 (host arithmetic, used by tests)."""
    a1, a2 = np.asarray(a1, float), np.asarray(a2, float)
    if a1.shape != a2.shape:
        raise ValueError("two_point_closed_form: dimension mismatch")
    if not w > 0:
        raise ValueError("two_point_closed_form: weight must be positive")
    if not gamma >= 0:
        raise ValueError("two_point_closed_form: gamma must be >= 0")
    c = a1 - a2
    nc = float(np.linalg.norm(c))
    if nc == 0.0:
        return a1.copy(), a2.copy()
    s = min(2.0 * gamma * w / nc, 1.0)
    return a1 - 0.5 * s * c, a2 + 0.5 * s * c
