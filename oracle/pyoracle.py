"""TEST INFRASTRUCTURE ONLY — ctypes driver for the CPU oracle (oracle/*.cpp).

Only tests/, ``__graft_entry__.smoke()`` and bench.py's CPU-baseline legs may
import this module, and only as the checker (or the timed CPU reference).  The
product package ``paper_2501_15964_b200`` never imports it.

Every function mirrors one reference entry point (cited) and takes/returns
numpy arrays in the reference layout: a d x n FP64 column-major matrix is a
C-contiguous numpy array of shape (n, d) — one sample per row, the same bytes.
Errors raise ValueError (std::invalid_argument) or RuntimeError
(std::runtime_error), as the reference's tests expect.
"""
from __future__ import annotations

import ctypes as C
import os
import subprocess
from dataclasses import dataclass

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_LIB_PATH = os.path.join(_HERE, "_build", "liborc.so")
_lib = None

D = C.POINTER(C.c_double)
I64 = C.POINTER(C.c_int64)


class OrcConfig(C.Structure):
    _fields_ = [("algorithm", C.c_int32), ("collect_trace", C.c_int32), ("epsilon", C.c_double),
                ("kkt_factor", C.c_double), ("max_iter", C.c_int64), ("time_limit", C.c_double),
                ("admm_rho", C.c_double), ("ama_step_safety", C.c_double), ("ssnal_sigma0", C.c_double),
                ("armijo_mu", C.c_double), ("backtrack_beta", C.c_double), ("ssnal_newton_max", C.c_int64),
                ("pcg_max_iter", C.c_int64)]


class OrcTerm(C.Structure):
    _fields_ = [("f_primal", C.c_double), ("f_dual", C.c_double), ("gap", C.c_double),
                ("iterations", C.c_int64), ("converged", C.c_int32), ("pad", C.c_int32),
                ("wall_time", C.c_double), ("newton", C.c_int64), ("cg", C.c_int64),
                ("armijo", C.c_int64), ("hess_apply", C.c_int64)]

    def as_dict(self):
        return {k: getattr(self, k) for k, _ in self._fields_ if k != "pad"}


ALGOS = {"admm": 0, "ama": 1, "ssnal": 2}


def config(algorithm="ssnal", epsilon=1e-6, kkt_factor=10.0, max_iter=0, time_limit=0.0, admm_rho=1.0,
           ama_step_safety=0.99, ssnal_sigma0=1.0, armijo_mu=1e-4, backtrack_beta=0.5, ssnal_newton_max=50,
           pcg_max_iter=500):
    """SolverConfig defaults (solvers.hpp:72-93)."""
    return OrcConfig(ALGOS[algorithm] if isinstance(algorithm, str) else algorithm, 0, epsilon, kkt_factor, max_iter,
                     time_limit, admm_rho, ama_step_safety, ssnal_sigma0, armijo_mu, backtrack_beta,
                     ssnal_newton_max, pcg_max_iter)


def build():
    subprocess.run(["make", "-s", "-C", _HERE], check=True)


def lib():
    global _lib
    if _lib is None:
        if not os.path.exists(_LIB_PATH):
            build()
        _lib = C.CDLL(_LIB_PATH)
        _lib.orc_error.restype = C.c_char_p
        for name in ("orc_graph_E", "orc_graph_n", "orc_graph_find"):
            getattr(_lib, name).restype = C.c_int64
        _lib.orc_graph_find.argtypes = [C.c_void_p, C.c_int64, C.c_int64]
        _lib.orc_graph_E.argtypes = [C.c_void_p]
        _lib.orc_graph_n.argtypes = [C.c_void_p]
        _lib.orc_graph_free.argtypes = [C.c_void_p]
    return _lib


def _dp(a):
    return a.ctypes.data_as(D) if a is not None else None


def _ip(a):
    return a.ctypes.data_as(I64) if a is not None else None


def _f64(a):
    return np.ascontiguousarray(a, dtype=np.float64)


def _check(rc):
    if rc == 0:
        return
    msg = lib().orc_error().decode()
    if rc == 1:
        raise ValueError(msg)
    raise RuntimeError(msg)


def _cd(x):
    return C.c_double(float(x))


def _ci(x):
    return C.c_int64(int(x))


class Graph:
    """WeightedGraph (graph.hpp:23-51): sorted, validated edge list."""

    def __init__(self, n, edges=None, _handle=None):
        self._h = None
        if _handle is not None:
            self._h = _handle
            return
        edges = list(edges or [])
        i = np.array([e[0] for e in edges], dtype=np.int64)
        j = np.array([e[1] for e in edges], dtype=np.int64)
        w = np.array([e[2] for e in edges], dtype=np.float64)
        h = C.c_void_p()
        _check(lib().orc_graph_new(_ci(n), _ip(i), _ip(j), _dp(w), _ci(len(edges)), C.byref(h)))
        self._h = h

    @classmethod
    def from_arrays(cls, n, i, j, w):
        i = np.ascontiguousarray(i, dtype=np.int64)
        j = np.ascontiguousarray(j, dtype=np.int64)
        w = _f64(w)
        h = C.c_void_p()
        _check(lib().orc_graph_new(_ci(n), _ip(i), _ip(j), _dp(w), _ci(len(i)), C.byref(h)))
        return cls(n, _handle=h)

    def __del__(self):
        if self._h is not None and _lib is not None:
            _lib.orc_graph_free(self._h)
            self._h = None

    @property
    def n(self):
        return lib().orc_graph_n(self._h)

    @property
    def E(self):
        return lib().orc_graph_E(self._h)

    def arrays(self):
        E = self.E
        i = np.empty(E, np.int64)
        j = np.empty(E, np.int64)
        w = np.empty(E, np.float64)
        d2 = np.full(E, np.nan)
        lib().orc_graph_export(self._h, _ip(i), _ip(j), _dp(w), _dp(d2))
        return i, j, w, d2

    def degree(self):
        deg = np.empty(self.n, np.int64)
        lib().orc_graph_degree(self._h, _ip(deg))
        return deg

    def find_edge(self, i, j):
        r = lib().orc_graph_find(self._h, i, j)
        return None if r < 0 else r


def knn_weights(A, k, phi):
    """compute_knn_weights (graph.cpp:75-114).  A: (n, d) samples."""
    A = _f64(A)
    n, d = A.shape
    h = C.c_void_p()
    _check(lib().orc_knn(_dp(A), _ci(d), _ci(n), _ci(k), _cd(phi), C.byref(h)))
    return Graph(n, _handle=h)


def validate_data(A):
    A = _f64(A)
    n, d = A.shape if A.ndim == 2 else (0, 0)
    _check(lib().orc_validate_data(_dp(A), _ci(d), _ci(n)))


def B(g, X):
    X = _f64(X)
    out = np.empty((g.E, X.shape[1]))
    _check(lib().orc_B(g._h, _dp(X), _ci(X.shape[1]), _ci(X.shape[0]), _dp(out)))
    return out


def Bt(g, Z):
    Z = _f64(Z)
    out = np.empty((g.n, Z.shape[1]))
    _check(lib().orc_Bt(g._h, _dp(Z), _ci(Z.shape[1]), _ci(Z.shape[0]), _dp(out)))
    return out


def laplacian_dense(g):
    out = np.empty((g.n, g.n))
    _check(lib().orc_laplacian_dense(g._h, _dp(out)))
    return out


def connected_components(g):
    lab = np.empty(g.n, np.int64)
    K = C.c_int64()
    _check(lib().orc_cc(g._h, _ip(lab), C.byref(K)))
    return lab, K.value


def prox_columns(q, V, t):
    V = _f64(V)
    t = _f64(t)
    out = np.empty_like(V)
    _check(lib().orc_prox_columns(q, _dp(V), _dp(t), _ci(V.shape[1]), _ci(V.shape[0]), _dp(out)))
    return out


def project_columns(q, Z, r):
    Z = _f64(Z)
    r = _f64(r)
    out = np.empty_like(Z)
    _check(lib().orc_project_columns(q, _dp(Z), _dp(r), _ci(Z.shape[1]), _ci(Z.shape[0]), _dp(out)))
    return out


def prox_jacobian(q, v, t):
    v = _f64(v)
    d = v.shape[0]
    J = np.empty((d, d))
    a, b = C.c_double(), C.c_double()
    _check(lib().orc_prox_jacobian(q, _dp(v), _ci(d), _cd(t), _dp(J), C.byref(a), C.byref(b)))
    return J.T.copy(), a.value, b.value   # J[r, c] = (J e_c)_r


def prox_jacobian_diag(q, v, t):
    v = _f64(v)
    out = np.empty_like(v)
    _check(lib().orc_prox_jacobian_diag(q, _dp(v), _ci(v.shape[0]), _cd(t), _dp(out)))
    return out


def moreau_check(q, v, t):
    v = _f64(v)
    r = C.c_double()
    _check(lib().orc_moreau(q, _dp(v), _ci(v.shape[0]), _cd(t), C.byref(r)))
    return r.value


def norms(q, v):
    v = _f64(v)
    a, b = C.c_double(), C.c_double()
    _check(lib().orc_norms(q, _dp(v), _ci(v.shape[0]), C.byref(a), C.byref(b)))
    return a.value, b.value


def pcg_dense(M, rhs, tol, maxit, pdiag=None):
    """pcg (linalg.cpp:143-192) on a dense operator; rhs is (n,) or (n, m)."""
    M = _f64(M)
    rhs = _f64(rhs)
    vec = rhs.ndim == 1
    R = rhs.reshape(rhs.shape[0], -1)
    n, m = R.shape
    Rc = np.asfortranarray(R)  # Eigen column-major n x m
    x = np.empty((m, n))
    it, res, conv = C.c_int64(), C.c_double(), C.c_int()
    Mc = np.asfortranarray(M)
    pd = _f64(pdiag) if pdiag is not None else None
    _check(lib().orc_pcg_dense(Mc.ctypes.data_as(D), _ci(n), Rc.ctypes.data_as(D), _ci(m), _dp(pd), _cd(tol),
                               _ci(maxit), _dp(x), C.byref(it), C.byref(res), C.byref(conv)))
    X = x.T
    return (X[:, 0] if vec else X), it.value, res.value, bool(conv.value)


def power_dense(M, tol=1e-9, maxit=10000):
    M = np.asfortranarray(_f64(M))
    out = C.c_double()
    _check(lib().orc_power_dense(M.ctypes.data_as(D), _ci(M.shape[0]), _cd(tol), _ci(maxit), C.byref(out)))
    return out.value


def power_laplacian(g, tol=1e-9, maxit=10000):
    out = C.c_double()
    _check(lib().orc_power_laplacian(g._h, _cd(tol), _ci(maxit), C.byref(out)))
    return out.value


def cholesky_solve(g, rho, rhs):
    rhs = _f64(rhs)
    R = np.asfortranarray(rhs.reshape(rhs.shape[0], -1))
    out = np.empty((R.shape[1], R.shape[0]))
    _check(lib().orc_cholesky_solve(g._h, _cd(rho), R.ctypes.data_as(D), _ci(R.shape[1]), _dp(out)))
    return out.T.reshape(rhs.shape)


def _inst(A):
    A = _f64(A)
    return A, A.shape[1], A.shape[0]


def primal_objective(A, g, gamma, q, X):
    A, d, n = _inst(A)
    out = C.c_double()
    _check(lib().orc_primal(_dp(A), _ci(d), _ci(n), g._h, _cd(gamma), q, _dp(_f64(X)), C.byref(out)))
    return out.value


def dual_objective(A, g, gamma, q, Z):
    A, d, n = _inst(A)
    out = C.c_double()
    _check(lib().orc_dual(_dp(A), _ci(d), _ci(n), g._h, _cd(gamma), q, _dp(_f64(Z)), C.byref(out)))
    return out.value


def kkt_residual(A, g, gamma, q, X, Z):
    A, d, n = _inst(A)
    out = C.c_double()
    _check(lib().orc_kkt(_dp(A), _ci(d), _ci(n), g._h, _cd(gamma), q, _dp(_f64(X)), _dp(_f64(Z)), C.byref(out)))
    return out.value


def phi_value(A, g, gamma, q, Z, sigma, X):
    A, d, n = _inst(A)
    out = C.c_double()
    _check(lib().orc_phi(_dp(A), _ci(d), _ci(n), g._h, _cd(gamma), q, _dp(_f64(Z)), _cd(sigma), _dp(_f64(X)),
                         C.byref(out)))
    return out.value


def phi_gradient(A, g, gamma, q, Z, sigma, X):
    A, d, n = _inst(A)
    out = np.empty((n, d))
    _check(lib().orc_phi_grad(_dp(A), _ci(d), _ci(n), g._h, _cd(gamma), q, _dp(_f64(Z)), _cd(sigma),
                              _dp(_f64(X)), _dp(out)))
    return out


def hessian_apply(A, g, gamma, q, Z, sigma, X, Dm):
    A, d, n = _inst(A)
    out = np.empty((n, d))
    _check(lib().orc_hess_apply(_dp(A), _ci(d), _ci(n), g._h, _cd(gamma), q, _dp(_f64(Z)), _cd(sigma),
                                _dp(_f64(X)), _dp(_f64(Dm)), _dp(out)))
    return out


@dataclass
class Solution:
    X: np.ndarray
    Z: np.ndarray
    term: dict


def solve(A, g, gamma, q, cfg=None, warm=None):
    A, d, n = _inst(A)
    cfg = cfg or config()
    X = np.empty((n, d))
    Z = np.empty((g.E, d))
    t = OrcTerm()
    wx = _f64(warm.X) if warm is not None else None
    wz = _f64(warm.Z) if warm is not None else None
    wxs = wx.shape if wx is not None else (0, 0)
    wzs = wz.shape if wz is not None else (0, 0)
    _check(lib().orc_solve(_dp(A), _ci(d), _ci(n), g._h, _cd(gamma), q, C.byref(cfg), _dp(wx), _ci(wxs[1]),
                           _ci(wxs[0]), _dp(wz), _ci(wzs[1]), _ci(wzs[0]), _dp(X), _dp(Z), C.byref(t)))
    return Solution(X, Z, t.as_dict())


def run_path(A, g, q, gammas, cfg=None, warm_start=True, require_connected=False, fuse_tol=1e-3, keep_z=True):
    A, d, n = _inst(A)
    cfg = cfg or config()
    gam = _f64(gammas)
    T = len(gam)
    X = np.empty((T, n, d))
    Z = np.empty((T, g.E, d)) if keep_z else None
    lab = np.empty((T, n), np.int64)
    K = np.empty(T, np.int64)
    terms = (OrcTerm * T)()
    _check(lib().orc_run_path(_dp(A), _ci(d), _ci(n), g._h, q, _dp(gam), _ci(T), C.byref(cfg), int(warm_start),
                              int(require_connected), _cd(fuse_tol), _dp(X), _dp(Z), _ip(lab), _ip(K), terms))
    return {"X": X, "Z": Z, "labels": lab, "K": K, "terms": [t.as_dict() for t in terms]}


def extract_clusters(X, g, fuse_tol=1e-3):
    X = _f64(X)
    n, d = X.shape
    lab = np.empty(n, np.int64)
    K = C.c_int64()
    cent = np.empty((n, d))
    _check(lib().orc_extract_clusters(_dp(X), _ci(d), _ci(n), g._h, _cd(fuse_tol), _ip(lab), C.byref(K), _dp(cent)))
    return lab, K.value, cent[:K.value].copy()


def make_schedule(start, end, count, geometric=True):
    out = np.empty(max(int(count), 0))
    _check(lib().orc_make_schedule(_cd(start), _cd(end), _ci(count), int(geometric), _dp(out)))
    return out


def gaussian_mixture(centers, spread, per_center, seed):
    """generate_gaussian_mixture (io.cpp:142-165); centers: (m, d)."""
    c = _f64(centers)
    m, d = c.shape
    out = np.empty((m * per_center, d))
    _check(lib().orc_mixture(_dp(c), _ci(d), _ci(m), _cd(spread), _ci(per_center), C.c_uint64(seed), _dp(out)))
    return out


def knn_rows(A, k, r0, r1):
    """Per-row k nearest (d2, j) of rows [r0, r1) (graph.cpp:79-88)."""
    A = _f64(A)
    n, d = A.shape
    kd = np.zeros((r1 - r0, k))
    kj = np.zeros((r1 - r0, k), dtype=np.int64)
    _check(lib().orc_knn_rows(_dp(A), _ci(d), _ci(n), _ci(k), _ci(r0), _ci(r1), _dp(kd), _ip(kj)))
    return kd, kj


def time_knn_rows(A, k, rows):
    """Seconds for the reference kNN of the first `rows` samples (graph.cpp:90-103)."""
    A = _f64(A)
    n, d = A.shape
    s = C.c_double()
    _check(lib().orc_time_knn_rows(_dp(A), _ci(d), _ci(n), _ci(k), _ci(rows), C.byref(s)))
    return s.value


SSNAL_UNITS = ("eval_phi", "gradient", "jacobian_diag", "hess_apply", "pcg_vec", "gap", "multiplier")


def time_ssnal_units(A, g, gamma, q=2, sigma=1.0, reps=1):
    """Seconds per call of each SSNAL building block (ssnal.cpp), dict keyed by SSNAL_UNITS."""
    A, d, n = _inst(A)
    out = np.empty(7)
    _check(lib().orc_time_ssnal_units(_dp(A), _ci(d), _ci(n), g._h, _cd(gamma), q, _cd(sigma), int(reps),
                                      _dp(out)))
    return dict(zip(SSNAL_UNITS, out.tolist()))


def normals(seed, count):
    out = np.empty(int(count))
    lib().orc_normals(C.c_uint64(seed), _ci(count), _dp(out))
    return out
