"""Size-independent fingerprints of a path's solutions, shared by the golden
generator (tools/golden_path.py, CPU oracle) and the GPU parity tests.

X is (n, d) in the reference layout (one sample per row = Eigen d x n column
major).  sketch(X) = Psi^T X Omega with Rademacher Psi (n x m) and Omega
(d x m), entries +-1/sqrt(m): E ||Psi^T D Omega||_F^2 = ||D||_F^2, so
||sketch(X1) - sketch(X2)||_F / ||sketch(X2)||_F estimates the relative
Frobenius error ||X1 - X2|| / ||X2|| (the 1e-6 bar of SURVEY.md §8(d)) from
m*m numbers instead of n*d.  The signs come from numpy's PCG64 with fixed
seeds, so both sides build the same Psi / Omega.
"""
import hashlib

import numpy as np

M = 32


def _signs(rows, m, seed):
    rng = np.random.Generator(np.random.PCG64(seed))
    return (rng.integers(0, 2, size=(rows, m), dtype=np.int8).astype(np.float64) * 2.0 - 1.0) / np.sqrt(m)


def sketch(X, m=M, seed=(20250127, 1)):
    X = np.asarray(X, dtype=np.float64)
    psi = _signs(X.shape[0], m, seed[0])
    om = _signs(X.shape[1], m, seed[1])
    return (psi.T @ X) @ om


def rel_sketch_error(S, S_ref):
    S, S_ref = np.asarray(S), np.asarray(S_ref)
    return float(np.linalg.norm(S - S_ref) / max(np.linalg.norm(S_ref), 1e-300))


def edge_hash(i, j, d2):
    """sha256 over the lexicographic edge list and its squared distances (int64, int64, float64 bytes)."""
    h = hashlib.sha256()
    h.update(np.ascontiguousarray(i, dtype=np.int64).tobytes())
    h.update(np.ascontiguousarray(j, dtype=np.int64).tobytes())
    h.update(np.ascontiguousarray(d2, dtype=np.float64).tobytes())
    return h.hexdigest()
