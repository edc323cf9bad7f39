// linalg.hpp:17-87 of the reference on the device: LinearOperator (identity,
// dense, sparse, Jacobi and host-callback operators), pcg (linalg.cpp:143-192,
// with the reference's exit residual), power_iteration (linalg.cpp:194-242)
// and CholeskyFactor (linalg.cpp:32-54).
//
// These are the general-purpose entry points of the boundary (the solvers run
// their own fused PCG, pcg.cu, and Laplacian power iteration, graph.cu).  The
// loop control is on the host with one scalar read per iteration; operands
// stay in HBM.  The factor of I + rho L is replaced by a Jacobi-preconditioned
// CG to 1e-14 relative residual per right-hand-side column: the same M^{-1} b
// up to rounding, without the fill of a sparse factor.
#include <algorithm>
#include <cmath>
#include <random>
#include <vector>

#include "linalg.cuh"

namespace cpb {

namespace {

// Y(r, c) = sum_k M(r, k) X(k, c), k ascending (column-major n x n M, n x cols X).
__global__ void k_dense_mv(const double* __restrict__ M, const double* __restrict__ X, int64_t n, int64_t cols,
                           double* __restrict__ Y) {
  const int64_t total = n * cols;
  for (int64_t p = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; p < total;
       p += static_cast<int64_t>(gridDim.x) * blockDim.x) {
    const int64_t r = p % n, c = p / n;
    const double* x = X + c * n;
    double s = 0.0;
    for (int64_t k = 0; k < n; ++k) s = s + M[k * n + r] * x[k];
    Y[p] = s;
  }
}
// Eigen's column-major sparse * dense accumulates res(row) += val * x(col) over
// columns in increasing order; per row that is the row's entries by ascending
// column, which CSR rows hold.
__global__ void k_csr_mv(const int* __restrict__ rowptr, const int* __restrict__ col, const double* __restrict__ val,
                         const double* __restrict__ X, int64_t n, int64_t cols, double* __restrict__ Y) {
  const int64_t total = n * cols;
  for (int64_t p = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; p < total;
       p += static_cast<int64_t>(gridDim.x) * blockDim.x) {
    const int64_t r = p % n, c = p / n;
    const double* x = X + c * n;
    double s = 0.0;
    for (int q = rowptr[r]; q < rowptr[r + 1]; ++q) s = s + val[q] * x[col[q]];
    Y[p] = s;
  }
}
// jacobi: Y = X ./ D, D a column (broadcast over columns) or a full block
__global__ void k_div(const double* __restrict__ X, const double* __restrict__ D, int64_t n, int64_t cols,
                      int full, double* __restrict__ Y) {
  const int64_t total = n * cols;
  for (int64_t p = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; p < total;
       p += static_cast<int64_t>(gridDim.x) * blockDim.x)
    Y[p] = X[p] / D[full ? p : p % n];
}
__global__ void k_scale(const double* __restrict__ X, double s, int64_t m, double* __restrict__ Y) {
  for (int64_t p = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; p < m;
       p += static_cast<int64_t>(gridDim.x) * blockDim.x)
    Y[p] = X[p] / s;
}
// p = z + beta p
__global__ void k_xpby(const double* __restrict__ z, double beta, int64_t m, double* __restrict__ p) {
  for (int64_t i = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; i < m;
       i += static_cast<int64_t>(gridDim.x) * blockDim.x)
    p[i] = z[i] + beta * p[i];
}
// Per-row (mode 0) or per-column (mode 1) Euclidean norms of an n x cols block.
__global__ void k_line_norms(const double* __restrict__ X, int64_t n, int64_t cols, int mode, double* __restrict__ out) {
  const int64_t lines = mode == 0 ? n : cols, len = mode == 0 ? cols : n;
  for (int64_t i = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; i < lines;
       i += static_cast<int64_t>(gridDim.x) * blockDim.x) {
    double s = 0.0;
    for (int64_t k = 0; k < len; ++k) {
      const double v = mode == 0 ? X[k * n + i] : X[i * n + k];
      s = s + v * v;
    }
    out[i] = sqrt(s);
  }
}
// worst line ratio ||r_line|| / (||b_line|| or 1): block maxima
__global__ void k_line_ratio(const double* __restrict__ R, const double* __restrict__ bn, int64_t n, int64_t cols,
                             int mode, double* part) {
  __shared__ double sh[32];
  const int64_t lines = mode == 0 ? n : cols, len = mode == 0 ? cols : n;
  double worst = 0.0;
  for (int64_t i = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; i < lines;
       i += static_cast<int64_t>(gridDim.x) * blockDim.x) {
    double s = 0.0;
    for (int64_t k = 0; k < len; ++k) {
      const double v = mode == 0 ? R[k * n + i] : R[i * n + k];
      s = s + v * v;
    }
    const double b = bn[i];
    worst = fmax(worst, sqrt(s) / (b > 0.0 ? b : 1.0));
  }
  worst = block_max(worst, sh);
  if (threadIdx.x == 0) part[blockIdx.x] = worst;
}
// ||v||_q and the dual norm per column (prox.cpp:25-31; q = 0: infinity)
__global__ void k_norms(int q, const double* __restrict__ V, int64_t d, int64_t cols, double* nrm, double* dual) {
  __shared__ double sh[32];
  for (int64_t c = blockIdx.x; c < cols; c += gridDim.x) {
    const double* v = V + c * d;
    double s2 = 0.0, s1 = 0.0, mx = 0.0;
    for (int64_t k = threadIdx.x; k < d; k += blockDim.x) {
      const double a = fabs(v[k]);
      s2 += v[k] * v[k];
      s1 += a;
      mx = fmax(mx, a);
    }
    s2 = block_sum(s2, sh);
    s1 = block_sum(s1, sh);
    mx = block_max(mx, sh);
    if (threadIdx.x == 0) {
      const double l2 = sqrt(s2);
      nrm[c] = q == 2 ? l2 : (q == 1 ? s1 : mx);
      dual[c] = q == 2 ? l2 : (q == 1 ? mx : s1);
    }
  }
}

int grid_for(Ctx& c, int64_t m) { return std::max(1, std::min(cdiv(m, 256), c.sm_count * 8)); }

}  // namespace

// ---- LinearOperator (linalg.cpp:56-122) -----------------------------------------------
void linop_apply(Ctx& c, const LinOp& op, const double* X, int64_t cols, double* Y) {
  const int64_t n = op.n, m = n * cols;
  if (cols < 0) invalid("LinearOperator::apply: negative column count");
  if (m == 0) return;
  switch (op.kind) {
    case LinOp::Identity:
      copy_dev(c, Y, X, m);
      break;
    case LinOp::Dense:
      k_dense_mv<<<grid_for(c, m), 256, 0, c.s>>>(op.vals.p, X, n, cols, Y);
      CPB_LAUNCH_CHECK();
      break;
    case LinOp::Sparse:
      k_csr_mv<<<grid_for(c, m), 256, 0, c.s>>>(op.rowptr.p, op.col.p, op.vals.p, X, n, cols, Y);
      CPB_LAUNCH_CHECK();
      break;
    case LinOp::Jacobi:
      if (op.jcols > 1 && cols != op.jcols) invalid("jacobi: operand shape mismatch");
      k_div<<<grid_for(c, m), 256, 0, c.s>>>(X, op.vals.p, n, cols, op.jcols > 1, Y);
      CPB_LAUNCH_CHECK();
      break;
    case LinOp::Callback: {
      // host functor (LinearOperator(rows, fn, ...)): one round trip per apply
      std::vector<double> hx(static_cast<size_t>(m)), hy(static_cast<size_t>(m));
      d2h(c, hx.data(), X, m * sizeof(double));
      if (op.fn(op.user, hx.data(), hy.data(), n, cols) != 0) runtime("LinearOperator::apply: callback failed");
      h2d(c, Y, hy.data(), m * sizeof(double));
      break;
    }
  }
}

namespace {
// linalg.cpp:128-139 (mode 0: rows, or the plain 2-norm for one column) / per column (mode 1)
struct Relres {
  Ctx& c;
  int64_t n, cols;
  int mode;  // 0 rows, 1 columns, 2 single vector
  double* bn;
  double* part;
  double nb = 1.0;
  Relres(Ctx& c_, const double* b, int64_t n_, int64_t cols_, int per_column) : c(c_), n(n_), cols(cols_) {
    mode = cols == 1 ? 2 : (per_column ? 1 : 0);
    const int64_t lines = mode == 0 ? n : cols;
    bn = c.buf<double>("la.bn", lines + 1);
    part = c.buf<double>("la.part", static_cast<size_t>(c.sm_count) * 8 + 2);
    if (mode == 2) {
      nb = std::sqrt(dot_dev(c, b, b, n));
    } else {
      k_line_norms<<<grid_for(c, lines), 256, 0, c.s>>>(b, n, cols, mode, bn);
      CPB_LAUNCH_CHECK();
    }
  }
  double operator()(const double* r) {
    if (mode == 2) return std::sqrt(dot_dev(c, r, r, n)) / (nb > 0.0 ? nb : 1.0);
    const int64_t lines = mode == 0 ? n : cols;
    const int g = grid_for(c, lines);
    k_line_ratio<<<g, 256, 0, c.s>>>(r, bn, n, cols, mode, part);
    CPB_LAUNCH_CHECK();
    reduce_max(c, part, g, c.dscal);
    double h;
    c.fetch(0, 1, &h);
    return h;
  }
};
}  // namespace

// pcg (linalg.cpp:143-192): x0 = 0, Frobenius inner products, the reference's
// stopping rule, the exit residual recomputed from op.
PcgResultDev pcg_generic(Ctx& c, const LinOp& op, const double* rhs, int64_t cols, const LinOp* pre, double tol,
                         int64_t max_iter, double* x, int per_column) {
  if (!(tol > 0.0)) invalid("pcg: tol must be positive");
  if (max_iter < 1) invalid("pcg: max_iter must be >= 1");
  const int64_t n = op.n, m = n * cols;
  if (pre && pre->n != n) invalid("LinearOperator::apply: operand has wrong row count");
  PcgResultDev res;
  if (m > 0) CPB_CUDA(cudaMemsetAsync(x, 0, m * sizeof(double), c.s));
  if (m == 0) {
    res.converged = true;
    return res;
  }
  double* r = c.buf<double>("la.r", m);
  double* z = c.buf<double>("la.z", m);
  double* p = c.buf<double>("la.p", m);
  double* Ap = c.buf<double>("la.Ap", m);
  copy_dev(c, r, rhs, m);
  Relres relres(c, rhs, n, cols, per_column);
  {
    const double r0 = relres(r);
    if (r0 <= tol) {
      res.residual = r0;
      res.converged = true;
      return res;
    }
  }
  auto precond = [&](const double* v, double* out) {
    if (pre)
      linop_apply(c, *pre, v, cols, out);
    else
      copy_dev(c, out, v, m);
  };
  precond(r, z);
  copy_dev(c, p, z, m);
  double rz = dot_dev(c, r, z, m);
  int64_t it = 0;
  while (it < max_iter) {
    ++it;
    linop_apply(c, op, p, cols, Ap);
    const double pAp = dot_dev(c, p, Ap, m);
    if (pAp <= 0.0) {
      if (dot_dev(c, p, p, m) == 0.0) break;
      runtime("pcg: operator is not positive definite (p'Ap <= 0)");
    }
    const double alpha = rz / pAp;
    axpy_dev(c, x, x, alpha, p, m);
    axpy_dev(c, r, r, -alpha, Ap, m);
    if (relres(r) <= tol) break;
    precond(r, z);
    const double rz_next = dot_dev(c, r, z, m);
    k_xpby<<<grid_for(c, m), 256, 0, c.s>>>(z, rz_next / rz, m, p);
    CPB_LAUNCH_CHECK();
    rz = rz_next;
  }
  res.iterations = it;
  linop_apply(c, op, x, cols, Ap);      // true residual (linalg.cpp:188)
  axpy_dev(c, r, rhs, -1.0, Ap, m);
  res.residual = relres(r);
  res.converged = res.residual <= tol;
  return res;
}

// power_iteration (linalg.cpp:194-242): two fixed-seed libstdc++ Gaussian
// probes and e_0, best estimate over the probes that were not annihilated.
double power_generic(Ctx& c, const LinOp& op, double tol, int64_t max_iter) {
  if (!(tol > 0.0)) invalid("power_iteration: tol must be positive");
  if (max_iter < 1) invalid("power_iteration: max_iter must be >= 1");
  const int64_t n = op.n;
  if (n == 0) return 0.0;
  std::vector<std::vector<double>> starts;
  for (uint64_t seed : {0x5851f42d4c957f2dULL, 0x14057b7ef767814fULL}) {
    std::mt19937_64 rng(seed);
    std::normal_distribution<double> gauss;
    std::vector<double> s(static_cast<size_t>(n));
    for (auto& x : s) x = gauss(rng);
    starts.push_back(std::move(s));
  }
  starts.emplace_back(static_cast<size_t>(n), 0.0);
  starts.back()[0] = 1.0;
  double* v = c.buf<double>("la.pv", n);
  double* w = c.buf<double>("la.pw", n);
  double best = 0.0;
  bool any = false;
  for (const auto& s : starts) {
    h2d(c, w, s.data(), n * sizeof(double));
    const double ns = std::sqrt(dot_dev(c, w, w, n));
    k_scale<<<grid_for(c, n), 256, 0, c.s>>>(w, ns, n, v);
    CPB_LAUNCH_CHECK();
    double prev = 0.0, est = 0.0;
    bool dead = false;
    for (int64_t it = 1; it <= max_iter; ++it) {
      linop_apply(c, op, v, 1, w);
      const double nw = std::sqrt(dot_dev(c, w, w, n));
      if (nw <= 1e-300) {
        dead = true;
        break;
      }
      const double lambda = dot_dev(c, v, w, n);
      est = lambda;
      k_scale<<<grid_for(c, n), 256, 0, c.s>>>(w, nw, n, v);
      CPB_LAUNCH_CHECK();
      if (it > 1 && std::abs(lambda - prev) <= tol * std::max(std::abs(lambda), 1e-300)) break;
      prev = lambda;
    }
    if (!dead) {
      any = true;
      best = std::max(best, est);
    }
  }
  return any ? best : 0.0;
}

// CSC (Eigen compressed columns, int64) -> device CSR rows by ascending column.
void linop_set_sparse(Ctx& c, LinOp& op, int64_t n, const int64_t* colptr, const int64_t* rowidx, const double* values,
                      double scale, double shift) {
  if (n < 0) invalid("LinearOperator::sparse: negative dimension");
  const int64_t nnz = n > 0 ? colptr[n] : 0;
  if (n > 0 && colptr[0] != 0) invalid("sparse: colptr[0] must be 0");
  std::vector<std::vector<std::pair<int, double>>> rows(static_cast<size_t>(n));
  for (int64_t j = 0; j < n; ++j) {
    if (colptr[j + 1] < colptr[j]) invalid("sparse: colptr must be nondecreasing");
    for (int64_t q = colptr[j]; q < colptr[j + 1]; ++q) {
      const int64_t r = rowidx[q];
      if (r < 0 || r >= n) invalid("sparse: row index out of range");
      rows[static_cast<size_t>(r)].emplace_back(static_cast<int>(j), scale * values[q]);
    }
  }
  std::vector<int> rp(static_cast<size_t>(n) + 1, 0), cl;
  std::vector<double> vl;
  cl.reserve(static_cast<size_t>(nnz) + static_cast<size_t>(n));
  vl.reserve(cl.capacity());
  for (int64_t r = 0; r < n; ++r) {
    auto& row = rows[static_cast<size_t>(r)];
    std::stable_sort(row.begin(), row.end(), [](auto& a, auto& b) { return a.first < b.first; });
    bool diag = false;
    for (auto& [j, v] : row) {  // duplicates summed like Eigen's compressed storage would hold them
      if (shift != 0.0 && !diag && j >= r) {
        if (j == r) {
          cl.push_back(j), vl.push_back(shift + v), diag = true;
          continue;
        }
        cl.push_back(static_cast<int>(r)), vl.push_back(shift), diag = true;
      }
      cl.push_back(j), vl.push_back(v);
    }
    if (shift != 0.0 && !diag) cl.push_back(static_cast<int>(r)), vl.push_back(shift);
    rp[static_cast<size_t>(r) + 1] = static_cast<int>(cl.size());
  }
  op.kind = LinOp::Sparse;
  op.n = n;
  op.rowptr.resize(rp.size());
  op.col.resize(cl.size() + 1);
  op.vals.resize(vl.size() + 1);
  h2d(c, op.rowptr.p, rp.data(), rp.size() * sizeof(int));
  if (!cl.empty()) {
    h2d(c, op.col.p, cl.data(), cl.size() * sizeof(int));
    h2d(c, op.vals.p, vl.data(), vl.size() * sizeof(double));
  }
  c.sync();
}

void norm_values_dev(Ctx& c, int q, const double* V, int64_t d, int64_t cols, double* nrm, double* dual) {
  if (cols == 0) return;
  k_norms<<<std::max(1, std::min(static_cast<int>(cols), c.sm_count * 8)), 256, 0, c.s>>>(q, V, d, cols, nrm, dual);
  CPB_LAUNCH_CHECK();
}

}  // namespace cpb
