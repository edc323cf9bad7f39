// TEST INFRASTRUCTURE ONLY (see oracle.hpp).  Restates prox.cpp (prox,
// projection, structural Jacobian, Moreau check) and linalg.cpp (operators,
// block PCG, power iteration, the ADMM factor) of the reference.
#include "oracle.hpp"

#include <algorithm>
#include <deque>
#include <functional>

namespace oracle {

namespace {
void check_t(double t, const char* what) {
  if (!(t >= 0.0) || !std::isfinite(t)) throw std::invalid_argument(std::string(what) + ": threshold must be finite and >= 0");
}
double sgn(double x) { return static_cast<double>((x > 0.0) - (x < 0.0)); }  // Eigen's sign()
}  // namespace

// prox.cpp:25-31 (+ q = inf: ||.||_inf with dual ||.||_1)
double norm_value(const double* v, Index n, Norm q) {
  if (q == Norm::linf) return max_abs(v, n);
  return q == Norm::l1 ? esum(n, [&](Index k) { return std::abs(v[k]); }) : norm2(v, n);
}
double dual_norm_value(const double* v, Index n, Norm q) {
  if (q == Norm::linf) return esum(n, [&](Index k) { return std::abs(v[k]); });
  return q == Norm::l1 ? max_abs(v, n) : norm2(v, n);
}

// The l1-ball threshold by Michelot's fixed point, with every sum in the
// "32-lane" order the device uses (linf.cuh, group_sum over lane-strided
// partials): element k goes to partial k mod 32 in increasing k, then the
// partials meet in an xor butterfly (16, 8, 4, 2, 1).  Same algorithm and same
// rounding on both sides, so theta, S and everything derived from them are
// bitwise equal to the device's (no reference exists for q = inf; the
// bisection / sort-based checks in tests/test_linf_oracle.py pin the math).
namespace {
template <class F>
double lane32_sum(Index n, F f) {  // f(k, &x) -> include?
  double p[32] = {0.0};
  for (Index k = 0; k < n; ++k) {
    double x;
    if (f(k, &x)) p[k & 31] += x;
  }
  for (int o = 16; o >= 1; o >>= 1) {
    double q[32];
    for (int v = 0; v < 32; ++v) q[v] = p[v] + p[v ^ o];
    for (int v = 0; v < 32; ++v) p[v] = q[v];
  }
  return p[0];
}
}  // namespace

double l1_theta(const double* v, Index n, double t, Index* count) {
  const double s1 = lane32_sum(n, [&](Index k, double* x) {
    *x = std::abs(v[k]);
    return true;
  });
  if (!(s1 > t)) {
    if (count) *count = 0;
    return -1.0;
  }
  double theta = (s1 - t) / static_cast<double>(n);
  Index support = n;
  // the support shrinks strictly on every pass that continues, so this ends
  // within n passes; a pass whose support does not shrink (the fixed point,
  // or a rounding-induced regrowth) keeps the previous theta
  for (;;) {
    Index c = 0;
    const double th = theta;
    const double s = lane32_sum(n, [&](Index k, double* x) {
      *x = std::abs(v[k]);
      if (*x > th) {
        ++c;
        return true;
      }
      return false;
    });
    if (c == 0) {
      support = 0;
      break;
    }
    if (c >= support) break;
    theta = (s - t) / static_cast<double>(c);
    support = c;
  }
  if (count) *count = support;
  return theta;
}

// prox.cpp:33-45
void prox_norm_into(const double* v, Index n, double t, Norm q, double* out) {
  check_t(t, "prox_norm");
  if (q == Norm::l2) {
    const double nv = norm2(v, n);
    if (nv <= t) {
      for (Index k = 0; k < n; ++k) out[k] = 0.0;
    } else {
      const double s = 1.0 - t / nv;
      for (Index k = 0; k < n; ++k) out[k] = s * v[k];
    }
  } else if (q == Norm::linf) {
    const double th = l1_theta(v, n, t, nullptr);
    for (Index k = 0; k < n; ++k) out[k] = th < 0.0 ? 0.0 : std::max(std::min(v[k], th), -th);
  } else {
    for (Index k = 0; k < n; ++k) out[k] = sgn(v[k]) * std::max(std::abs(v[k]) - t, 0.0);
  }
}

// prox.cpp:53-65
void project_dual_ball_into(const double* z, Index n, double r, Norm q, double* out) {
  check_t(r, "project_dual_ball");
  if (q == Norm::l2) {
    const double nz = norm2(z, n);
    if (nz <= r) {
      for (Index k = 0; k < n; ++k) out[k] = z[k];
    } else {
      const double s = r / nz;
      for (Index k = 0; k < n; ++k) out[k] = s * z[k];
    }
  } else if (q == Norm::linf) {
    const double th = l1_theta(z, n, r, nullptr);
    for (Index k = 0; k < n; ++k) out[k] = th < 0.0 ? z[k] : sgn(z[k]) * std::max(std::abs(z[k]) - th, 0.0);
  } else {
    for (Index k = 0; k < n; ++k) out[k] = std::max(std::min(z[k], r), -r);
  }
}

// prox.cpp:73-93
void prox_columns_into(const Mat& V, const std::vector<double>& t, Norm q, Mat& out) {
  if (static_cast<Index>(t.size()) != V.cols) throw std::invalid_argument("prox_columns: one threshold per column required");
  out = Mat(V.rows, V.cols);
  par_for(V.cols, [&](Index l) { prox_norm_into(V.col(l), V.rows, t[static_cast<size_t>(l)], q, out.col(l)); });
}
void project_columns_inplace(Mat& Z, const std::vector<double>& r, Norm q) {
  if (static_cast<Index>(r.size()) != Z.cols) throw std::invalid_argument("project_columns: one radius per column required");
  par_ranges(Z.cols, [&](Index lo, Index hi) {
    std::vector<double> tmp(static_cast<size_t>(Z.rows));
    for (Index l = lo; l < hi; ++l) {
      project_dual_ball_into(Z.col(l), Z.rows, r[static_cast<size_t>(l)], q, tmp.data());
      std::copy(tmp.begin(), tmp.end(), Z.col(l));
    }
  });
}

// prox.cpp:95-110
void ProxJac::apply(const double* w, Index n, double* out) const {
  if (q == Norm::l2) {
    for (Index k = 0; k < n; ++k) out[k] = alpha * w[k];
    if (beta != 0.0) {
      const double c = beta * dotp(dir.data(), w, n);
      for (Index k = 0; k < n; ++k) out[k] += c * dir[static_cast<size_t>(k)];
    }
    return;
  }
  if (static_cast<Index>(active.size()) != n) throw std::invalid_argument("ProxJacobian::apply: size mismatch");
  if (q == Norm::linf) {  // M = I - (diag(1_S) - s s^T / |S|), or 0 inside the ball
    if (theta < 0.0) {
      for (Index k = 0; k < n; ++k) out[k] = 0.0;
      return;
    }
    double c = 0.0;
    for (Index k = 0; k < n; ++k) c += dir[static_cast<size_t>(k)] * w[k];
    const double b = support > 0 ? c / static_cast<double>(support) : 0.0;
    for (Index k = 0; k < n; ++k)
      out[k] = active[static_cast<size_t>(k)] ? b * dir[static_cast<size_t>(k)] : w[k];
    return;
  }
  for (Index k = 0; k < n; ++k) out[k] = active[static_cast<size_t>(k)] ? w[k] : 0.0;
}
double ProxJac::diag(Index r) const {
  if (q == Norm::l2) return alpha + (beta != 0.0 ? beta * dir[static_cast<size_t>(r)] * dir[static_cast<size_t>(r)] : 0.0);
  if (q == Norm::linf) {
    if (theta < 0.0) return 0.0;
    return active[static_cast<size_t>(r)] ? 1.0 / static_cast<double>(support) : 1.0;
  }
  return active[static_cast<size_t>(r)] ? 1.0 : 0.0;
}

// prox.cpp:112-132: q=2 smooth region alpha I + beta v v^T, zero map at and
// inside the kink, identity at t = 0; q=1 strict |v_r| > t mask.
ProxJac prox_jacobian(const double* v, Index n, double t, Norm q) {
  check_t(t, "prox_jacobian");
  ProxJac J;
  J.q = q;
  if (q == Norm::l2) {
    if (t == 0.0) {
      J.alpha = 1.0;
      return J;
    }
    const double nv = norm2(v, n);
    if (nv > t) {
      J.alpha = 1.0 - t / nv;
      J.beta = t / (nv * nv * nv);
      J.dir.assign(v, v + n);
    }
  } else if (q == Norm::linf) {
    J.theta = l1_theta(v, n, t, &J.support);
    J.active.assign(static_cast<size_t>(n), 0);
    J.dir.assign(static_cast<size_t>(n), 0.0);
    if (J.theta >= 0.0)
      for (Index k = 0; k < n; ++k)
        if (std::abs(v[k]) > J.theta) {
          J.active[static_cast<size_t>(k)] = 1;
          J.dir[static_cast<size_t>(k)] = sgn(v[k]);
        }
  } else {
    J.active.resize(static_cast<size_t>(n));
    for (Index k = 0; k < n; ++k) J.active[static_cast<size_t>(k)] = std::abs(v[k]) > t;
  }
  return J;
}

// prox.cpp:134-138
double moreau_check(const double* v, Index n, double t, Norm q) {
  std::vector<double> p(static_cast<size_t>(n)), z(static_cast<size_t>(n)), s(static_cast<size_t>(n));
  prox_norm_into(v, n, t, q, p.data());
  project_dual_ball_into(v, n, t, q, z.data());
  for (Index k = 0; k < n; ++k) s[static_cast<size_t>(k)] = p[static_cast<size_t>(k)] + z[static_cast<size_t>(k)] - v[k];
  return max_abs(s.data(), n);
}

// ---- linalg ----------------------------------------------------------------
Mat LinOp::apply(const Mat& x) const {
  if (x.rows != rows) throw std::invalid_argument("LinearOperator::apply: operand has wrong row count");
  Mat out = fn(x);
  if (out.rows != x.rows || out.cols != x.cols) throw std::runtime_error("LinearOperator::apply: image shape mismatch");
  return out;
}

// Dense M * X; Eigen's GEMV/GEMM kernels reorder sums, so tests on dense
// operators compare at tolerance.
LinOp op_dense(const Mat& M) {
  if (M.rows != M.cols) throw std::invalid_argument("LinearOperator::dense: matrix must be square");
  LinOp op;
  op.rows = M.rows;
  op.fn = [M](const Mat& x) {
    Mat y(M.rows, x.cols, 0.0);
    for (Index c = 0; c < x.cols; ++c)
      for (Index k = 0; k < M.cols; ++k) {
        const double xk = x(k, c);
        for (Index r = 0; r < M.rows; ++r) y(r, c) += M(r, k) * xk;
      }
    return y;
  };
  return op;
}

// Eigen column-major sparse * dense: res(row) += val * x(col) for columns in
// increasing order (SparseDenseProduct.h, ColMajor branch).
LinOp op_csc(const Csc& L) {
  LinOp op;
  op.rows = L.n;
  op.fn = [L](const Mat& x) {
    Mat y(L.n, x.cols, 0.0);
    for (Index c = 0; c < x.cols; ++c)
      for (Index j = 0; j < L.n; ++j) {
        const double xj = x(j, c);
        for (Index p = L.colptr[static_cast<size_t>(j)]; p < L.colptr[static_cast<size_t>(j + 1)]; ++p)
          y(L.row[static_cast<size_t>(p)], c) += L.val[static_cast<size_t>(p)] * xj;
      }
    return y;
  };
  return op;
}

// linalg.cpp:110-122
LinOp op_jacobi(const Mat& diag) {
  for (double x : diag.v)
    if (x <= 0.0) throw std::invalid_argument("jacobi: diagonal must be positive");
  LinOp op;
  op.rows = diag.rows;
  op.fn = [diag](const Mat& x) {
    if (x.cols != diag.cols) throw std::invalid_argument("jacobi: operand shape mismatch");
    Mat y(x.rows, x.cols);
    par_for(x.size(), [&](Index k) { y.v[static_cast<size_t>(k)] = x.v[static_cast<size_t>(k)] / diag.v[static_cast<size_t>(k)]; });
    return y;
  };
  return op;
}
LinOp op_jacobi_vec(const std::vector<double>& diag) {
  for (double x : diag)
    if (x <= 0.0) throw std::invalid_argument("jacobi: diagonal must be positive");
  LinOp op;
  op.rows = static_cast<Index>(diag.size());
  op.fn = [diag](const Mat& x) {
    Mat y(x.rows, x.cols);
    for (Index c = 0; c < x.cols; ++c)
      for (Index r = 0; r < x.rows; ++r) y(r, c) = x(r, c) / diag[static_cast<size_t>(r)];
    return y;
  };
  return op;
}

namespace {
// linalg.cpp:128-139: single column -> plain relative 2-norm; block -> the
// worst relative row norm (rows are strided: sequential order).
double relres(const Mat& r, const Mat& b) {
  if (b.cols == 1) {
    const double nb = norm2(b.v.data(), b.size());
    return norm2(r.v.data(), r.size()) / (nb > 0.0 ? nb : 1.0);
  }
  std::vector<double> rel(static_cast<size_t>(b.rows));
  par_for(b.rows, [&](Index i) {
    const double nb = std::sqrt(ssum(b.cols, [&](Index c) { return b(i, c) * b(i, c); }));
    const double nr = std::sqrt(ssum(r.cols, [&](Index c) { return r(i, c) * r(i, c); }));
    rel[static_cast<size_t>(i)] = nr / (nb > 0.0 ? nb : 1.0);
  });
  double worst = 0.0;
  for (double x : rel) worst = std::max(worst, x);
  return worst;
}
double fdot(const Mat& a, const Mat& b) { return dotp(a.v.data(), b.v.data(), a.size()); }
}  // namespace

// linalg.cpp:143-192
PcgOut pcg(const LinOp& op, const Mat& rhs, const LinOp* pre, double tol, Index max_iter) {
  if (!(tol > 0.0)) throw std::invalid_argument("pcg: tol must be positive");
  if (max_iter < 1) throw std::invalid_argument("pcg: max_iter must be >= 1");
  if (rhs.rows != op.rows) throw std::invalid_argument("pcg: rhs row count does not match the operator");
  PcgOut res;
  res.x = Mat(rhs.rows, rhs.cols, 0.0);
  Mat r = rhs;
  auto precond = [&](const Mat& v) { return pre ? pre->apply(v) : v; };
  if (relres(r, rhs) <= tol) {
    res.residual = relres(r, rhs);
    res.converged = true;
    return res;
  }
  Mat z = precond(r);
  Mat p = z;
  double rz = fdot(r, z);
  Index it = 0;
  while (it < max_iter) {
    ++it;
    Mat Ap = op.apply(p);
    const double pAp = fdot(p, Ap);
    if (pAp <= 0.0) {
      if (sq_norm(p.v.data(), p.size()) == 0.0) break;
      throw std::runtime_error("pcg: operator is not positive definite (p'Ap <= 0)");
    }
    const double alpha = rz / pAp;
    par_for(p.size(), [&](Index k) {
      res.x.v[static_cast<size_t>(k)] += alpha * p.v[static_cast<size_t>(k)];
      r.v[static_cast<size_t>(k)] -= alpha * Ap.v[static_cast<size_t>(k)];
    });
    if (relres(r, rhs) <= tol) break;
    z = precond(r);
    const double rz_next = fdot(r, z);
    const double beta = rz_next / rz;
    par_for(p.size(), [&](Index k) { p.v[static_cast<size_t>(k)] = z.v[static_cast<size_t>(k)] + beta * p.v[static_cast<size_t>(k)]; });
    rz = rz_next;
  }
  res.iterations = it;
  Mat Ax = op.apply(res.x);
  Mat tr(rhs.rows, rhs.cols);
  for (Index k = 0; k < tr.size(); ++k) tr.v[static_cast<size_t>(k)] = rhs.v[static_cast<size_t>(k)] - Ax.v[static_cast<size_t>(k)];
  res.residual = relres(tr, rhs);
  res.converged = res.residual <= tol;
  return res;
}

// linalg.cpp:194-242: two fixed-seed Gaussian probes plus e_0; best estimate
// over the probes that were not annihilated.
double power_iteration(const LinOp& op, double tol, Index max_iter) {
  if (!(tol > 0.0)) throw std::invalid_argument("power_iteration: tol must be positive");
  if (max_iter < 1) throw std::invalid_argument("power_iteration: max_iter must be >= 1");
  const Index n = op.rows;
  if (n == 0) return 0.0;
  std::vector<std::vector<double>> starts;
  for (std::uint64_t seed : {0x5851f42d4c957f2dULL, 0x14057b7ef767814fULL}) {
    std::mt19937_64 rng(seed);
    std::normal_distribution<double> gauss;
    std::vector<double> s(static_cast<size_t>(n));
    for (Index i = 0; i < n; ++i) s[static_cast<size_t>(i)] = gauss(rng);
    starts.push_back(std::move(s));
  }
  starts.emplace_back(static_cast<size_t>(n), 0.0);
  starts.back()[0] = 1.0;

  double best = 0.0;
  bool any = false;
  for (const auto& s : starts) {
    Mat v(n, 1);
    const double ns = norm2(s.data(), n);
    for (Index i = 0; i < n; ++i) v.v[static_cast<size_t>(i)] = s[static_cast<size_t>(i)] / ns;
    double prev = 0.0, est = 0.0;
    bool dead = false;
    for (Index it = 1; it <= max_iter; ++it) {
      Mat w = op.apply(v);
      const double nw = norm2(w.v.data(), n);
      if (nw <= 1e-300) {
        dead = true;
        break;
      }
      const double lambda = dotp(v.v.data(), w.v.data(), n);
      est = lambda;
      for (Index i = 0; i < n; ++i) v.v[static_cast<size_t>(i)] = w.v[static_cast<size_t>(i)] / nw;
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

// ---- ADMM factor (linalg.cpp:32-54 semantics; envelope Cholesky + RCM) ------
Cholesky::Cholesky(const Csc& Lap, double rho_) : n(Lap.n), rho(rho_) {
  if (!(rho > 0.0) || !std::isfinite(rho)) throw std::invalid_argument("cholesky: rho must be positive and finite");
  // symmetry check (linalg.cpp:16-31)
  double scale = 0.0, asym = 0.0;
  for (double x : Lap.val) scale = std::max(scale, std::abs(x));
  auto at = [&](Index r, Index c) {
    for (Index p = Lap.colptr[static_cast<size_t>(c)]; p < Lap.colptr[static_cast<size_t>(c + 1)]; ++p)
      if (Lap.row[static_cast<size_t>(p)] == r) return Lap.val[static_cast<size_t>(p)];
    return 0.0;
  };
  for (Index c = 0; c < n; ++c)
    for (Index p = Lap.colptr[static_cast<size_t>(c)]; p < Lap.colptr[static_cast<size_t>(c + 1)]; ++p)
      asym = std::max(asym, std::abs(Lap.val[static_cast<size_t>(p)] - at(c, Lap.row[static_cast<size_t>(p)])));
  if (asym > 1e-12 * (1.0 + scale)) throw std::invalid_argument("cholesky: matrix is not symmetric");

  // reverse Cuthill-McKee ordering
  std::vector<Index> deg(static_cast<size_t>(n));
  for (Index c = 0; c < n; ++c) deg[static_cast<size_t>(c)] = Lap.colptr[static_cast<size_t>(c + 1)] - Lap.colptr[static_cast<size_t>(c)];
  std::vector<char> seen(static_cast<size_t>(n), 0);
  std::vector<Index> order;
  order.reserve(static_cast<size_t>(n));
  for (Index s0 = 0; s0 < n; ++s0) {
    if (seen[static_cast<size_t>(s0)]) continue;
    std::deque<Index> q{s0};
    seen[static_cast<size_t>(s0)] = 1;
    while (!q.empty()) {
      Index v = q.front();
      q.pop_front();
      order.push_back(v);
      std::vector<Index> nb;
      for (Index p = Lap.colptr[static_cast<size_t>(v)]; p < Lap.colptr[static_cast<size_t>(v + 1)]; ++p) {
        Index u = Lap.row[static_cast<size_t>(p)];
        if (!seen[static_cast<size_t>(u)]) {
          seen[static_cast<size_t>(u)] = 1;
          nb.push_back(u);
        }
      }
      std::sort(nb.begin(), nb.end(), [&](Index a, Index b) { return deg[static_cast<size_t>(a)] < deg[static_cast<size_t>(b)] || (deg[static_cast<size_t>(a)] == deg[static_cast<size_t>(b)] && a < b); });
      for (Index u : nb) q.push_back(u);
    }
  }
  std::reverse(order.begin(), order.end());
  perm = order;
  std::vector<Index> inv(static_cast<size_t>(n));
  for (Index k = 0; k < n; ++k) inv[static_cast<size_t>(perm[static_cast<size_t>(k)])] = k;

  // M = I + rho L in the new ordering, row-envelope storage
  first.assign(static_cast<size_t>(n), 0);
  for (Index i = 0; i < n; ++i) {
    Index f = i, old = perm[static_cast<size_t>(i)];
    for (Index p = Lap.colptr[static_cast<size_t>(old)]; p < Lap.colptr[static_cast<size_t>(old + 1)]; ++p)
      f = std::min(f, inv[static_cast<size_t>(Lap.row[static_cast<size_t>(p)])]);
    first[static_cast<size_t>(i)] = f;
  }
  rowptr.assign(static_cast<size_t>(n + 1), 0);
  for (Index i = 0; i < n; ++i) rowptr[static_cast<size_t>(i + 1)] = rowptr[static_cast<size_t>(i)] + static_cast<size_t>(i - first[static_cast<size_t>(i)] + 1);
  L.assign(rowptr[static_cast<size_t>(n)], 0.0);
  auto Lref = [&](Index i, Index j) -> double& { return L[rowptr[static_cast<size_t>(i)] + static_cast<size_t>(j - first[static_cast<size_t>(i)])]; };
  for (Index i = 0; i < n; ++i) {
    Index old = perm[static_cast<size_t>(i)];
    Lref(i, i) = 1.0;
    for (Index p = Lap.colptr[static_cast<size_t>(old)]; p < Lap.colptr[static_cast<size_t>(old + 1)]; ++p) {
      Index j = inv[static_cast<size_t>(Lap.row[static_cast<size_t>(p)])];
      if (j <= i) Lref(i, j) += rho * Lap.val[static_cast<size_t>(p)];
    }
  }
  for (Index i = 0; i < n; ++i) {
    const Index fi = first[static_cast<size_t>(i)];
    for (Index j = fi; j < i; ++j) {
      const Index lo = std::max(fi, first[static_cast<size_t>(j)]);
      double s = Lref(i, j);
      for (Index k = lo; k < j; ++k) s -= Lref(i, k) * Lref(j, k);
      Lref(i, j) = s / Lref(j, j);
    }
    double s = Lref(i, i);
    for (Index k = fi; k < i; ++k) s -= Lref(i, k) * Lref(i, k);
    if (!(s > 0.0)) throw std::runtime_error("cholesky: factorization of I + rho*L failed");
    Lref(i, i) = std::sqrt(s);
  }
}

Mat Cholesky::solve(const Mat& rhs) const {
  if (rhs.rows != n) throw std::invalid_argument("cholesky solve: rhs has wrong row count");
  Mat out(n, rhs.cols);
  std::vector<double> y(static_cast<size_t>(n));
  auto Lv = [&](Index i, Index j) { return L[rowptr[static_cast<size_t>(i)] + static_cast<size_t>(j - first[static_cast<size_t>(i)])]; };
  for (Index c = 0; c < rhs.cols; ++c) {
    for (Index i = 0; i < n; ++i) {
      double s = rhs(perm[static_cast<size_t>(i)], c);
      for (Index k = first[static_cast<size_t>(i)]; k < i; ++k) s -= Lv(i, k) * y[static_cast<size_t>(k)];
      y[static_cast<size_t>(i)] = s / Lv(i, i);
    }
    // back substitution with L^T (column access through row envelopes)
    for (Index i = n - 1; i >= 0; --i) {
      y[static_cast<size_t>(i)] /= Lv(i, i);
      const double yi = y[static_cast<size_t>(i)];
      for (Index k = first[static_cast<size_t>(i)]; k < i; ++k) y[static_cast<size_t>(k)] -= Lv(i, k) * yi;
    }
    for (Index i = 0; i < n; ++i) out(perm[static_cast<size_t>(i)], c) = y[static_cast<size_t>(i)];
  }
  return out;
}

}  // namespace oracle
