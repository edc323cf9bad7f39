// Fused solver kernels (see ops.cuh).  Geometry conventions:
//  * "group" kernels: one row (edge or node) per group of gx = min(32, 2^ceil(log2 d))
//    lanes of a warp, 256/gx rows per block, lanes striding over the d features;
//    per-row reductions are group shuffles (no shared memory, no atomics);
//  * node-gather kernels walk the node CSR (incident edges in ascending edge
//    id) in descending-degree order so hubs start first;
//  * "feature-major" kernels (PCG) give every thread a fixed set of features
//    so per-feature row norms reduce without atomics;
//  * every reduction is a block partial over a static row partition, then a
//    fixed-order column reduce: bitwise run-to-run reproducible.
// All arithmetic is compiled with -fmad=false (elementwise rounding matches the
// reference's SSE2 build); the cited reference line is given per kernel.
#include <cmath>

#include "gather.cuh"
#include "ops.cuh"
#include "ptx.cuh"
#include "comm.cuh"
#include "linf.cuh"
#include <cooperative_groups.h>
namespace cg = cooperative_groups;

namespace cpb {

namespace {

// ---------------------------------------------------------------------------------
struct GroupGeom {
  int gx, gy, grid;
};
// short = true (q = 1 / 2 edge passes): rows of 17..128 features take 8 lanes each, four rows
// per warp, so the per-row reductions cost 3 shuffle levels shared by four rows instead of 5
// for one (C5, d = 64).  q = inf keeps 32-lane rows: its threshold sums follow the oracle's
// 32-lane order.
GroupGeom group_geom(Ctx& c, int64_t rows, int64_t d, int per_sm = 8, bool short_rows = false) {
  int gx = 1;
  while (gx < d && gx < 32) gx <<= 1;
  if (short_rows && d > 16 && d <= 128) gx = 8;
  const int gy = 256 / gx;
  const int grid = std::max(1, std::min(cdiv(rows, gy), c.sm_count * per_sm));
  return {gx, gy, grid};
}
inline int flat_grid(Ctx& c, int64_t m) { return std::max(1, std::min(cdiv(m, 256), c.sm_count * 4)); }

__device__ __forceinline__ double sgnd(double x) { return static_cast<double>((x > 0.0) - (x < 0.0)); }
// q=1 prox: sign(v) max(|v| - t, 0) (prox.cpp:42)
__device__ __forceinline__ double soft(double v, double t) { return sgnd(v) * fmax(fabs(v) - t, 0.0); }

#define ROWS_BEGIN(rows)                                                                               \
  for (int64_t row_ = blockIdx.x * static_cast<int64_t>(blockDim.y) + threadIdx.y; row_ < (rows); \
       row_ += static_cast<int64_t>(gridDim.x) * blockDim.y)

// A node-partitioned SSNAL solve is running on this context (solve.cu sets the
// owned node range for the whole solve when a communicator is attached).
inline bool partitioned(const Ctx& c) { return c.comm && c.own_v1 >= 0; }

// Edge rows of an EdgeSel, one group (blockDim.x lanes) per edge.
#define EDGES_BEGIN(sel)                                                                                    \
  for (int64_t i_ = blockIdx.x * static_cast<int64_t>(blockDim.y) + threadIdx.y; i_ < (sel).count;       \
       i_ += static_cast<int64_t>(gridDim.x) * blockDim.y)                                                 \
    if (const int64_t row_ = (sel).at(i_); true)

// ---- flat vector kernels ----------------------------------------------------------
__global__ void k_scale(const double* __restrict__ x, double s, int64_t m, double* __restrict__ out) {
  for (int64_t p = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; p < m;
       p += static_cast<int64_t>(gridDim.x) * blockDim.x)
    out[p] = s * x[p];
}
__global__ void k_div(const double* __restrict__ x, double s, int64_t m, double* __restrict__ out) {
  for (int64_t p = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; p < m;
       p += static_cast<int64_t>(gridDim.x) * blockDim.x)
    out[p] = x[p] / s;
}
__global__ void k_dot(const double* __restrict__ a, const double* __restrict__ b, int64_t m, double* part) {
  __shared__ double sh[32];
  double s = 0.0;
  const int64_t step = static_cast<int64_t>(gridDim.x) * blockDim.x;
  int64_t p = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x;
  for (; p + 7 * step < m; p += 8 * step) {  // 8 elements' loads ahead of the ordered sum
    double x[8], y[8];
#pragma unroll
    for (int u = 0; u < 8; ++u) x[u] = a[p + u * step], y[u] = b[p + u * step];
#pragma unroll
    for (int u = 0; u < 8; ++u) s += x[u] * y[u];
  }
  for (; p < m; p += step) s += a[p] * b[p];
  s = block_sum(s, sh);
  if (threadIdx.x == 0) part[blockIdx.x] = s;
}
__global__ void k_maxabs(const double* __restrict__ a, int64_t m, double* part) {
  __shared__ double sh[32];
  double s = 0.0;
  for (int64_t p = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; p < m;
       p += static_cast<int64_t>(gridDim.x) * blockDim.x)
    s = fmax(s, fabs(a[p]));
  s = block_max(s, sh);
  if (threadIdx.x == 0) part[blockIdx.x] = s;
}
__global__ void k_axpy(double* __restrict__ out, const double* __restrict__ x, double a, const double* __restrict__ y,
                       int64_t m) {
  for (int64_t p = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; p < m;
       p += static_cast<int64_t>(gridDim.x) * blockDim.x)
    out[p] = x[p] + a * y[p];
}
__global__ void k_neg(double* __restrict__ out, const double* __restrict__ x, int64_t m) {
  for (int64_t p = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; p < m;
       p += static_cast<int64_t>(gridDim.x) * blockDim.x)
    out[p] = -x[p];
}
// Xt = X + alpha D (when D) and the partial of ||Xt - A||^2 (ssnal.cpp:37, :174)
__global__ void k_trial_x(const double* __restrict__ X, const double* __restrict__ D, double alpha,
                          double* __restrict__ Xt, const double* __restrict__ A, int64_t m, double* part) {
  __shared__ double sh[32];
  double s = 0.0;
  const int64_t step = static_cast<int64_t>(gridDim.x) * blockDim.x;
  int64_t p = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x;
  // batches of 4 grid-stride elements: all loads first (the sum keeps the element order)
  for (; p + 3 * step < m; p += 4 * step) {
    double x[4], dd[4], a[4];
#pragma unroll
    for (int u = 0; u < 4; ++u) {
      x[u] = X[p + u * step];
      dd[u] = D ? D[p + u * step] : 0.0;
      a[u] = A[p + u * step];
    }
#pragma unroll
    for (int u = 0; u < 4; ++u) {
      double xv = x[u];
      if (D) {
        xv = xv + alpha * dd[u];
        Xt[p + u * step] = xv;
      }
      const double t = xv - a[u];
      s += t * t;
    }
  }
  for (; p < m; p += step) {
    double x = X[p];
    if (D) {
      x = x + alpha * D[p];
      Xt[p] = x;
    }
    const double t = x - A[p];
    s += t * t;
  }
  s = block_sum(s, sh);
  if (threadIdx.x == 0) part[blockIdx.x] = s;
}

// ---- prox / projection columns (prox.cpp:33-93, :112-132) -----------------------------
__global__ void k_prox_cols(int q, const double* __restrict__ V, const double* __restrict__ t, int64_t E, int d,
                            double* __restrict__ out) {
  const unsigned gm = group_mask();
  ROWS_BEGIN(E) {
    const double* v = V + row_ * d;
    double* o = out + row_ * d;
    const double tl = t[row_];
    if (q == Q_L2) {
      double ss = 0.0;
      for (int f = threadIdx.x; f < d; f += blockDim.x) ss += v[f] * v[f];
      const double nv = sqrt(group_sum(ss, gm));
      const double s = 1.0 - tl / nv;
      for (int f = threadIdx.x; f < d; f += blockDim.x) o[f] = (nv <= tl) ? 0.0 : s * v[f];
    } else if (q == Q_LINF) {
      int cnt;
      const double th = linf_theta([&](int f) { return v[f]; }, d, tl, gm, &cnt);
      for (int f = threadIdx.x; f < d; f += blockDim.x) o[f] = th < 0.0 ? 0.0 : clampd(v[f], th);
    } else {
      for (int f = threadIdx.x; f < d; f += blockDim.x) o[f] = soft(v[f], tl);
    }
  }
}
// In place (out == Z), rows inside the ball are not rewritten (the values would be the same
// bits); `changed` (nullable) is set when any row moves.
__global__ void k_project_cols(int q, const double* __restrict__ Z, const double* __restrict__ r, int64_t E, int d,
                               double* __restrict__ out, int* changed) {
  const unsigned gm = group_mask();
  const bool inplace = out == Z;
  ROWS_BEGIN(E) {
    const double* z = Z + row_ * d;
    double* o = out + row_ * d;
    const double rl = r[row_];
    if (q == Q_L2) {
      double ss = 0.0;
      for (int f = threadIdx.x; f < d; f += blockDim.x) ss += z[f] * z[f];
      const double nz = sqrt(group_sum(ss, gm));
      const double s = rl / nz;
      const bool inside = nz <= rl;
      if (!inside && changed) *changed = 1;
      if (!(inplace && inside))
        for (int f = threadIdx.x; f < d; f += blockDim.x) o[f] = inside ? z[f] : s * z[f];
    } else if (q == Q_LINF) {
      int cnt;
      const double th = linf_theta([&](int f) { return z[f]; }, d, rl, gm, &cnt);
      if (th >= 0.0 && changed) *changed = 1;
      if (!(inplace && th < 0.0))
        for (int f = threadIdx.x; f < d; f += blockDim.x) o[f] = th < 0.0 ? z[f] : soft(z[f], th);
    } else {
      for (int f = threadIdx.x; f < d; f += blockDim.x) {
        const double v = fmax(fmin(z[f], rl), -rl);
        if (v != z[f] && changed) *changed = 1;
        if (!inplace || v != z[f]) o[f] = v;
      }
    }
  }
}
__global__ void k_jac_diag_cols(int q, const double* __restrict__ V, const double* __restrict__ t, int64_t E, int d,
                                double* __restrict__ out) {
  const unsigned gm = group_mask();
  ROWS_BEGIN(E) {
    const double* v = V + row_ * d;
    double* o = out + row_ * d;
    const double tl = t[row_];
    if (q == Q_L2) {
      double ss = 0.0;
      for (int f = threadIdx.x; f < d; f += blockDim.x) ss += v[f] * v[f];
      const double nv = sqrt(group_sum(ss, gm));
      double al = 0.0, be = 0.0;
      if (tl == 0.0) {
        al = 1.0;
      } else if (nv > tl) {
        al = 1.0 - tl / nv;
        be = tl / (nv * nv * nv);
      }
      for (int f = threadIdx.x; f < d; f += blockDim.x) o[f] = al + (be != 0.0 ? be * v[f] * v[f] : 0.0);
    } else if (q == Q_LINF) {  // diag of M = I - (diag(1_S) - s s^T / |S|); 0 inside the ball
      int cnt;
      const double th = linf_theta([&](int f) { return v[f]; }, d, tl, gm, &cnt);
      const double b = cnt > 0 ? 1.0 / cnt : 0.0;
      for (int f = threadIdx.x; f < d; f += blockDim.x) o[f] = th < 0.0 ? 0.0 : (fabs(v[f]) > th ? b : 1.0);
    } else {
      for (int f = threadIdx.x; f < d; f += blockDim.x) o[f] = fabs(v[f]) > tl ? 1.0 : 0.0;
    }
  }
}

// ProxJacobian::apply (prox.cpp:95-104, :112-132) column-wise: out_l = M_l w_l
// with M_l the structured Jacobian of prox_{t_l ||.||} at v_l.
__global__ void k_jac_apply_cols(int q, const double* __restrict__ V, const double* __restrict__ t,
                                 const double* __restrict__ W, int64_t E, int d, double* __restrict__ out) {
  const unsigned gm = group_mask();
  ROWS_BEGIN(E) {
    const double* v = V + row_ * d;
    const double* w = W + row_ * d;
    double* o = out + row_ * d;
    const double tl = t[row_];
    if (q == Q_L2) {  // alpha w + beta <v, w> v outside the ball, 0 at/inside the kink, w at t = 0
      double ss = 0.0, vw = 0.0;
      for (int f = threadIdx.x; f < d; f += blockDim.x) ss += v[f] * v[f], vw += v[f] * w[f];
      const double nv = sqrt(group_sum(ss, gm));
      vw = group_sum(vw, gm);
      double al = 0.0, be = 0.0;
      if (tl == 0.0) {
        al = 1.0;
      } else if (nv > tl) {
        al = 1.0 - tl / nv;
        be = tl / (nv * nv * nv);
      }
      for (int f = threadIdx.x; f < d; f += blockDim.x) o[f] = al * w[f] + (be != 0.0 ? be * vw * v[f] : 0.0);
    } else if (q == Q_LINF) {  // w - (1_S w - s <s, w> / |S|); 0 inside the l1 ball
      int cnt;
      const double th = linf_theta([&](int f) { return v[f]; }, d, tl, gm, &cnt);
      double sw = 0.0;
      for (int f = threadIdx.x; f < d; f += blockDim.x)
        if (th >= 0.0 && fabs(v[f]) > th) sw += (v[f] > 0.0 ? w[f] : -w[f]);
      sw = group_sum(sw, gm);
      const double b = cnt > 0 ? sw / cnt : 0.0;
      for (int f = threadIdx.x; f < d; f += blockDim.x)
        o[f] = th < 0.0 ? 0.0 : (fabs(v[f]) > th ? (v[f] > 0.0 ? b : -b) : w[f]);
    } else {  // strict |v_r| > t mask
      for (int f = threadIdx.x; f < d; f += blockDim.x) o[f] = fabs(v[f]) > tl ? w[f] : 0.0;
    }
  }
}

// ---- SSNAL: phi edge pass (ssnal.cpp:24-39) -------------------------------------------
// V = X B + Z / sigma (write), nv = ||V_l||, envelope partial
//   sum_l gamma w_l ||P_l||_q + sigma/2 ||P_l - V_l||^2.
__global__ void k_phi_edge(const double* __restrict__ X, const double* __restrict__ Z, const int* __restrict__ ei,
                           const int* __restrict__ ej, const double* __restrict__ thr, const double* __restrict__ rad,
                           EdgeSel sel, int d, double sigma, int q, double* __restrict__ V, double* __restrict__ nv,
                           double* __restrict__ nvc, double* part) {
  __shared__ double sh[32];
  const unsigned gm = group_mask();
  double acc = 0.0;
  EDGES_BEGIN(sel) {
    const double* xa = X + static_cast<int64_t>(ei[row_]) * d;
    const double* xb = X + static_cast<int64_t>(ej[row_]) * d;
    const double* z = Z + row_ * d;
    double* v = V + row_ * d;
    const double t = thr[row_];
    double env;
    if (q == Q_L2) {
      double ss = 0.0;
#pragma unroll 4
      for (int f = threadIdx.x; f < d; f += blockDim.x) {
        const double x = (xa[f] - xb[f]) + __ldcs(z + f) / sigma;
        __stcs(v + f, x);
        ss += x * x;
      }
      ss = group_sum(ss, gm);
      const double nvl = sqrt(ss);
      double pn = 0.0, sq = ss;
      if (!(nvl <= t)) {
        // P = s V with s = 1 - t/||V||: ||P|| = s ||V||, ||P - V||^2 = (s - 1)^2 ||V||^2
        // (closed forms of the reference's two vector norms, one pass over V).
        const double s = 1.0 - t / nvl;
        pn = s * nvl;
        sq = (s - 1.0) * (s - 1.0) * ss;
      }
      env = rad[row_] * pn + (0.5 * sigma) * sq;
      if (threadIdx.x == 0) nv[row_] = nvl;
    } else if (q == Q_LINF) {
      // P = clamp(V, theta): ||P||_inf = theta, ||P - V||^2 = sum soft(V, theta)^2
      for (int f = threadIdx.x; f < d; f += blockDim.x) v[f] = (xa[f] - xb[f]) + z[f] / sigma;
      int cnt;
      const double th = linf_theta([&](int f) { return v[f]; }, d, t, gm, &cnt);
      double sq = 0.0;
      for (int f = threadIdx.x; f < d; f += blockDim.x) {
        const double r = th < 0.0 ? v[f] : soft(v[f], th);
        sq += r * r;
      }
      env = rad[row_] * (th < 0.0 ? 0.0 : th) + (0.5 * sigma) * group_sum(sq, gm);
      if (threadIdx.x == 0) {
        nv[row_] = th;
        nvc[row_] = cnt;
      }
    } else {
      double a = 0.0, b = 0.0;
#pragma unroll 4
      for (int f = threadIdx.x; f < d; f += blockDim.x) {
        const double x = (xa[f] - xb[f]) + __ldcs(z + f) / sigma;
        __stcs(v + f, x);
        const double p = soft(x, t);
        a += fabs(p);
        b += (p - x) * (p - x);
      }
      env = rad[row_] * group_sum(a, gm) + (0.5 * sigma) * group_sum(b, gm);
      if (threadIdx.x == 0) nv[row_] = 0.0;
    }
    if (threadIdx.x == 0) acc += env;
  }
  acc = block_sum(acc, sh);
  if (threadIdx.x == 0 && threadIdx.y == 0) part[blockIdx.x] = acc;
}

// Per-edge prox scale and structural Jacobian (prox.cpp:39-44, :112-132).
__global__ void k_jac(const double* __restrict__ nv, const double* __restrict__ thr, int64_t E, int q,
                      double* __restrict__ ps, double* __restrict__ jal, double* __restrict__ jbe, double* part) {
  __shared__ double sh[32];
  double cnt = 0.0;
  for (int64_t l = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; l < E;
       l += static_cast<int64_t>(gridDim.x) * blockDim.x) {
    if (q == Q_L2) {
      const double n = nv[l], t = thr[l];
      const double s = (n <= t) ? 0.0 : 1.0 - t / n;
      const double be = (t > 0.0 && n > t) ? t / (n * n * n) : 0.0;
      ps[l] = s;
      jal[l] = (t == 0.0) ? 1.0 : s;
      jbe[l] = be;
      cnt += (be != 0.0) ? 1.0 : 0.0;
    } else if (q == Q_LINF) {  // nv = (theta, |S|) from the phi edge pass
      const double th = nv[l], sc = nv[E + l];
      ps[l] = th;
      jal[l] = th;
      jbe[l] = (th >= 0.0 && sc > 0.0) ? 1.0 / sc : 0.0;
      cnt += 1.0;
    } else {
      cnt += 1.0;
    }
  }
  cnt = block_sum(cnt, sh);
  if (threadIdx.x == 0) part[blockIdx.x] = cnt;
}

// ---- objectives / gap (objective.cpp:63-113) ------------------------------------------
// Edge terms at (X, Z): [0] sum w_l ||XB_l||_q, [1] ||XB - prox_r(XB + Z)||^2,
// [2] ||XB||^2, [3] ||Z||^2; max dual-ball excess into partmax.
__device__ __forceinline__ void gap_edge_terms(const double* xa, const double* xb, const double* z, double rl,
                                               double wl, int d, int q, unsigned gm, double* t4, double& excess) {
  if (q == Q_LINF) {  // ||XB_l||_inf, prox_{r||.||inf}(XB + Z) = clamp at theta_r, dual norm l1
    double xb2 = 0.0, zz = 0.0, xm = 0.0, z1 = 0.0;
    for (int f = threadIdx.x; f < d; f += blockDim.x) {
      const double x = xa[f] - xb[f];
      xb2 += x * x;
      zz += z[f] * z[f];
      xm = fmax(xm, fabs(x));
      z1 += fabs(z[f]);
    }
    int cnt;
    const double th = linf_theta([&](int f) { return (xa[f] - xb[f]) + z[f]; }, d, rl, gm, &cnt);
    double al = 0.0;
    for (int f = threadIdx.x; f < d; f += blockDim.x) {
      const double x = xa[f] - xb[f];
      const double e = x - (th < 0.0 ? 0.0 : clampd(x + z[f], th));
      al += e * e;
    }
    t4[0] = wl * group_max(xm, gm);
    t4[1] = group_sum(al, gm);
    t4[2] = group_sum(xb2, gm);
    t4[3] = group_sum(zz, gm);
    excess = fmax(excess, group_sum(z1, gm) - (rl + 1e-9));
    return;
  }
  double xb2 = 0.0, zz = 0.0, uu = 0.0, l1 = 0.0, zmax = 0.0;
  for (int f = threadIdx.x; f < d; f += blockDim.x) {
    const double x = xa[f] - xb[f];
    const double u = x + z[f];
    xb2 += x * x;
    zz += z[f] * z[f];
    uu += u * u;
    l1 += fabs(x);
    zmax = fmax(zmax, fabs(z[f]));
  }
  xb2 = group_sum(xb2, gm);
  zz = group_sum(zz, gm);
  double al = 0.0;
  if (q == Q_L2) {
    const double nu = sqrt(group_sum(uu, gm));
    if (nu <= rl) {
      al = xb2;
    } else {
      const double s = 1.0 - rl / nu;
      for (int f = threadIdx.x; f < d; f += blockDim.x) {
        const double x = xa[f] - xb[f];
        const double e = x - s * (x + z[f]);
        al += e * e;
      }
      al = group_sum(al, gm);
    }
    t4[0] = wl * sqrt(xb2);
    excess = fmax(excess, sqrt(zz) - (rl + 1e-9));
  } else {
    for (int f = threadIdx.x; f < d; f += blockDim.x) {
      const double x = xa[f] - xb[f];
      const double e = x - soft(x + z[f], rl);
      al += e * e;
    }
    al = group_sum(al, gm);
    t4[0] = wl * group_sum(l1, gm);
    excess = fmax(excess, group_max(zmax, gm) - (rl + 1e-9));
  }
  t4[1] = al;
  t4[2] = xb2;
  t4[3] = zz;
}

__global__ void k_gap_edge(const double* __restrict__ X, const double* __restrict__ Z, const int* __restrict__ ei,
                           const int* __restrict__ ej, const double* __restrict__ rad, const double* __restrict__ w,
                           EdgeSel sel, int d, int q, double* part) {
  __shared__ double sh[32];
  const unsigned gm = group_mask();
  double s[4] = {0, 0, 0, 0}, excess = -1.0;
  EDGES_BEGIN(sel) {
    double t4[4];
    gap_edge_terms(X + static_cast<int64_t>(ei[row_]) * d, X + static_cast<int64_t>(ej[row_]) * d, Z + row_ * d,
                   rad[row_], w[row_], d, q, gm, t4, excess);
    if (threadIdx.x == 0)
      for (int k = 0; k < 4; ++k) s[k] += t4[k];
  }
  for (int k = 0; k < 4; ++k) {
    const double r = block_sum(s[k], sh);
    if (threadIdx.x == 0 && threadIdx.y == 0) part[5 * blockIdx.x + k] = r;
  }
  const double m = block_max(excess, sh);
  if (threadIdx.x == 0 && threadIdx.y == 0) part[5 * blockIdx.x + 4] = m;
}

// ---- SSNAL multiplier (ssnal.cpp:183-195, :205) fused with the edge gap terms -----------
// part per block: [0..3] gap edge terms at the new Z, [4] ||XB - PV||^2, [5] ||XB||^2 (same as [2]),
// [6] max |Z + sigma XB| (pre-projection), [7] max |Zenv - Zsum|, [8] dual excess
__global__ void k_mult(const double* __restrict__ X, double* __restrict__ Z, const double* __restrict__ V,
                       const double* __restrict__ ps, const double* __restrict__ thr, const double* __restrict__ rad,
                       const double* __restrict__ w, const int* __restrict__ ei, const int* __restrict__ ej, EdgeSel sel,
                       int d, double sigma, int q, double* part) {
  __shared__ double sh[32];
  const unsigned gm = group_mask();
  double s[5] = {0, 0, 0, 0, 0}, mx = 0.0, err = 0.0, excess = -1.0;
  EDGES_BEGIN(sel) {
    const double* xa = X + static_cast<int64_t>(ei[row_]) * d;
    const double* xb = X + static_cast<int64_t>(ej[row_]) * d;
    double* z = Z + row_ * d;
    const double* v = V + row_ * d;
    const double rl = rad[row_], tl = thr[row_], sl = ps[row_];
    double nn = 0.0, m = 0.0;
#pragma unroll 4
    for (int f = threadIdx.x; f < d; f += blockDim.x) {
      const double zs = z[f] + sigma * (xa[f] - xb[f]);
      nn += zs * zs;
      m = fmax(m, fabs(zs));
    }
    mx = fmax(mx, m);
    const double nz = sqrt(group_sum(nn, gm));
    const double sc = rl / nz;
    // pass 2: project, self-check, write Z, and the gap's edge sums at the new Z
    double fr = 0.0, e = 0.0, xb2 = 0.0, zz = 0.0, uu = 0.0, l1 = 0.0, zmax = 0.0, al = 0.0;
#pragma unroll 4
    for (int f = threadIdx.x; f < d; f += blockDim.x) {
      const double x = xa[f] - xb[f];
      const double zs = z[f] + sigma * x;
      const double zp = (q == Q_L2) ? ((nz <= rl) ? zs : sc * zs) : fmax(fmin(zs, rl), -rl);
      const double vf = __ldcs(v + f);
      const double pv = (q == Q_L2) ? sl * vf : soft(vf, tl);
      const double zenv = sigma * (vf - pv);
      e = fmax(e, fabs(zenv - zp));
      z[f] = zp;
      fr += (x - pv) * (x - pv);
      const double u = x + zp;
      xb2 += x * x;
      zz += zp * zp;
      uu += u * u;
      l1 += fabs(x);
      zmax = fmax(zmax, fabs(zp));
      if (q != Q_L2) {
        const double ee = x - soft(u, rl);
        al += ee * ee;
      }
    }
    err = fmax(err, e);
    fr = group_sum(fr, gm);
    xb2 = group_sum(xb2, gm);
    zz = group_sum(zz, gm);
    double t4[4];
    if (q == Q_L2) {
      const double nu = sqrt(group_sum(uu, gm));
      if (nu <= rl) {
        al = xb2;
      } else {  // pass 3 (objective.cpp:110-111): XB - prox(XB + Z) needs ||XB + Z|| first
        const double s2 = 1.0 - rl / nu;
#pragma unroll 4
        for (int f = threadIdx.x; f < d; f += blockDim.x) {
          const double x = xa[f] - xb[f];
          const double ee = x - s2 * (x + z[f]);
          al += ee * ee;
        }
        al = group_sum(al, gm);
      }
      t4[0] = w[row_] * sqrt(xb2);
      excess = fmax(excess, sqrt(zz) - (rl + 1e-9));
    } else {
      al = group_sum(al, gm);
      t4[0] = w[row_] * group_sum(l1, gm);
      excess = fmax(excess, group_max(zmax, gm) - (rl + 1e-9));
    }
    t4[1] = al;
    t4[2] = xb2;
    t4[3] = zz;
    if (threadIdx.x == 0) {
      for (int k = 0; k < 4; ++k) s[k] += t4[k];
      s[4] += fr;
    }
  }
  for (int k = 0; k < 5; ++k) {
    const double r = block_sum(s[k], sh);
    if (threadIdx.x == 0 && threadIdx.y == 0) part[9 * blockIdx.x + k] = r;
  }
  const double a = block_max(mx, sh);
  const double b = block_max(err, sh);
  const double c = block_max(excess, sh);
  if (threadIdx.x == 0 && threadIdx.y == 0) {
    part[9 * blockIdx.x + 5] = 0.0;
    part[9 * blockIdx.x + 6] = a;
    part[9 * blockIdx.x + 7] = b;
    part[9 * blockIdx.x + 8] = c;
  }
}

// q = infinity multiplier (ssnal.cpp:183-206 with the l1 dual ball): Zsum =
// Pi_{B1(r)}(Z + sigma XB) at its own threshold, the self-check against
// Zenv = sigma (V - clamp(V, theta_v)) (theta_v = ps from the phi pass), and
// the gap's edge terms at the new Z (prox_{r||.||inf}(XB + Z) needs a third
// threshold).  Same part layout as k_mult.
__global__ void k_mult_inf(const double* __restrict__ X, double* __restrict__ Z, const double* __restrict__ V,
                           const double* __restrict__ ps, const double* __restrict__ rad,
                           const double* __restrict__ w, const int* __restrict__ ei, const int* __restrict__ ej,
                           EdgeSel sel, int d, double sigma, double* part) {
  __shared__ double sh[32];
  const unsigned gm = group_mask();
  double s[5] = {0, 0, 0, 0, 0}, mx = 0.0, err = 0.0, excess = -1.0;
  EDGES_BEGIN(sel) {
    const double* xa = X + static_cast<int64_t>(ei[row_]) * d;
    const double* xb = X + static_cast<int64_t>(ej[row_]) * d;
    double* z = Z + row_ * d;
    const double* v = V + row_ * d;
    const double rl = rad[row_], thv = ps[row_];
    double m = 0.0;
    for (int f = threadIdx.x; f < d; f += blockDim.x) m = fmax(m, fabs(z[f] + sigma * (xa[f] - xb[f])));
    mx = fmax(mx, m);
    int cnt;
    const double thz = linf_theta([&](int f) { return z[f] + sigma * (xa[f] - xb[f]); }, d, rl, gm, &cnt);
    double fr = 0.0, e = 0.0, xb2 = 0.0, zz = 0.0, xm = 0.0, z1 = 0.0;
    for (int f = threadIdx.x; f < d; f += blockDim.x) {
      const double x = xa[f] - xb[f];
      const double zs = z[f] + sigma * x;
      const double zp = thz < 0.0 ? zs : soft(zs, thz);
      const double vf = v[f];
      const double pv = thv < 0.0 ? 0.0 : clampd(vf, thv);
      e = fmax(e, fabs(sigma * (vf - pv) - zp));
      z[f] = zp;
      fr += (x - pv) * (x - pv);
      xb2 += x * x;
      zz += zp * zp;
      xm = fmax(xm, fabs(x));
      z1 += fabs(zp);
    }
    err = fmax(err, e);
    const double thu = linf_theta([&](int f) { return (xa[f] - xb[f]) + z[f]; }, d, rl, gm, &cnt);
    double al = 0.0;
    for (int f = threadIdx.x; f < d; f += blockDim.x) {
      const double x = xa[f] - xb[f];
      const double ee = x - (thu < 0.0 ? 0.0 : clampd(x + z[f], thu));
      al += ee * ee;
    }
    al = group_sum(al, gm);
    fr = group_sum(fr, gm);
    xb2 = group_sum(xb2, gm);
    zz = group_sum(zz, gm);
    const double pen = w[row_] * group_max(xm, gm);
    excess = fmax(excess, group_sum(z1, gm) - (rl + 1e-9));
    if (threadIdx.x == 0) {
      s[0] += pen;
      s[1] += al;
      s[2] += xb2;
      s[3] += zz;
      s[4] += fr;
    }
  }
  for (int k = 0; k < 5; ++k) {
    const double r = block_sum(s[k], sh);
    if (threadIdx.x == 0 && threadIdx.y == 0) part[9 * blockIdx.x + k] = r;
  }
  const double a = block_max(mx, sh);
  const double b = block_max(err, sh);
  const double c = block_max(excess, sh);
  if (threadIdx.x == 0 && threadIdx.y == 0) {
    part[9 * blockIdx.x + 5] = 0.0;
    part[9 * blockIdx.x + 6] = a;
    part[9 * blockIdx.x + 7] = b;
    part[9 * blockIdx.x + 8] = c;
  }
}

// Shared-memory variant of k_mult for d <= kMultSmemMaxD with 32-lane rows:
// pass 1 stages x = x_i - x_j and Zsum in the warp's shared-memory rows, so
// passes 2 and 3 never touch HBM/L2 again (k_mult re-reads the three rows
// per pass, and at C3 its 60 % L2 hit rate left it latency-bound at ~1.2 TB/s).
// Each lane reads back only the elements it wrote (f = lane + 32 k), so no
// synchronisation is needed.  Per-edge arithmetic and per-lane accumulation
// order are those of k_mult (only the rows-to-block partition of the
// deterministic block partials differs).
constexpr int kMultSmemMaxD = 1024, kMultWarps = 4;
// Ring depth of the TMA edge kernels (edges in flight per warp).  One stage
// for long rows: at d = 784 eight warps per SM already keep ~150 KB in
// flight, and two stages halve the warps per SM (C3 phi 230 -> 511 ms,
// multiplier 187 -> 294 ms per 10 gammas).  Two stages for short rows (C5,
// d = 64: phi 242 -> 230 ms, multiplier 201 -> 197 ms); eight were much
// slower (phi 14.3 vs 6.4 ms per launch).
constexpr int kEdgeMaxStages = 8;
inline int edge_stages(int64_t d, int rows) {
  (void)rows;
  return d <= 128 ? 2 : 1;
}
template <int Q>
__global__ void __launch_bounds__(32 * kMultWarps) k_mult_s(
    const double* __restrict__ X, double* __restrict__ Z, const double* __restrict__ V, const double* __restrict__ ps,
    const double* __restrict__ thr, const double* __restrict__ rad, const double* __restrict__ w,
    const int* __restrict__ ei, const int* __restrict__ ej, EdgeSel sel, int d, double sigma, double* part) {
  extern __shared__ double srow[];
  __shared__ double sh[32];
  double* sx = srow + static_cast<size_t>(threadIdx.y) * 2 * d;
  double* sz = sx + d;
  double s[5] = {0, 0, 0, 0, 0}, mx = 0.0, err = 0.0, excess = -1.0;
  EDGES_BEGIN(sel) {
    const double* xa = X + static_cast<int64_t>(ei[row_]) * d;
    const double* xb = X + static_cast<int64_t>(ej[row_]) * d;
    double* z = Z + row_ * d;
    const double* v = V + row_ * d;
    const double rl = rad[row_], tl = thr[row_], sl = ps[row_];
    double nn = 0.0, m = 0.0;
#pragma unroll 4
    for (int f = threadIdx.x; f < d; f += 32) {
      const double x = xa[f] - xb[f];
      const double zs = z[f] + sigma * x;
      sx[f] = x;
      sz[f] = zs;
      nn += zs * zs;
      m = fmax(m, fabs(zs));
    }
    mx = fmax(mx, m);
    const double nz = sqrt(warp_sum(nn));
    const double sc = rl / nz;
    double fr = 0.0, e = 0.0, xb2 = 0.0, zz = 0.0, uu = 0.0, l1 = 0.0, zmax = 0.0, al = 0.0;
#pragma unroll 4
    for (int f = threadIdx.x; f < d; f += 32) {
      const double x = sx[f];
      const double zs = sz[f];
      const double zp = (Q == Q_L2) ? ((nz <= rl) ? zs : sc * zs) : fmax(fmin(zs, rl), -rl);
      const double vf = __ldcs(v + f);
      const double pv = (Q == Q_L2) ? sl * vf : soft(vf, tl);
      const double zenv = sigma * (vf - pv);
      e = fmax(e, fabs(zenv - zp));
      z[f] = zp;
      sz[f] = zp;
      fr += (x - pv) * (x - pv);
      const double u = x + zp;
      xb2 += x * x;
      zz += zp * zp;
      if (Q == Q_L2) {
        uu += u * u;
      } else {
        l1 += fabs(x);
        zmax = fmax(zmax, fabs(zp));
        const double ee = x - soft(u, rl);
        al += ee * ee;
      }
    }
    err = fmax(err, e);
    fr = warp_sum(fr);
    xb2 = warp_sum(xb2);
    zz = warp_sum(zz);
    double t0;
    if (Q == Q_L2) {
      const double nu = sqrt(warp_sum(uu));
      if (nu <= rl) {
        al = xb2;
      } else {  // pass 3 (objective.cpp:110-111) from shared memory
        const double s2 = 1.0 - rl / nu;
#pragma unroll 4
        for (int f = threadIdx.x; f < d; f += 32) {
          const double x = sx[f];
          const double ee = x - s2 * (x + sz[f]);
          al += ee * ee;
        }
        al = warp_sum(al);
      }
      t0 = w[row_] * sqrt(xb2);
      excess = fmax(excess, sqrt(zz) - (rl + 1e-9));
    } else {
      al = warp_sum(al);
      t0 = w[row_] * warp_sum(l1);
      excess = fmax(excess, warp_max(zmax) - (rl + 1e-9));
    }
    if (threadIdx.x == 0) {
      s[0] += t0;
      s[1] += al;
      s[2] += xb2;
      s[3] += zz;
      s[4] += fr;
    }
  }
  for (int k = 0; k < 5; ++k) {
    const double r = block_sum(s[k], sh);
    if (threadIdx.x == 0 && threadIdx.y == 0) part[9 * blockIdx.x + k] = r;
  }
  const double a = block_max(mx, sh);
  const double b = block_max(err, sh);
  const double c = block_max(excess, sh);
  if (threadIdx.x == 0 && threadIdx.y == 0) {
    part[9 * blockIdx.x + 5] = 0.0;
    part[9 * blockIdx.x + 6] = a;
    part[9 * blockIdx.x + 7] = b;
    part[9 * blockIdx.x + 8] = c;
  }
}

// TMA variant (even d): one lane streams the edge's four rows (x_i, x_j, Z_l,
// V_l) into the warp's shared-memory slot with cp.async.bulk, so each warp
// keeps 4 d doubles in flight without spending registers on them; the three
// passes then run from shared memory (x_i's slot is reused for x, Z_l's for
// Zsum / the projected Z).  Per-element arithmetic is that of k_mult_s.
// VM = 1: V_l staged by TMA with the other rows.  VM = 2: V_l recomputed from the staged
// rows, v = (x_i - x_j) + z_l / sigma — the exact expression (and rounding) of the phi edge
// pass that wrote V at the same X and Z, so it is bitwise the stored row; one HBM row fewer
// per edge.  The host picks VM = 2 unless the last Armijo search failed (then X moved past
// the last trial point, ssnal.cpp:172-179, and the stored V is read).
template <int Q, int VM>
__global__ void __launch_bounds__(32 * kMultWarps) k_mult_t(
    const double* __restrict__ X, double* __restrict__ Z, const double* __restrict__ V, const double* __restrict__ ps,
    const double* __restrict__ thr, const double* __restrict__ rad, const double* __restrict__ w,
    const int* __restrict__ ei, const int* __restrict__ ej, EdgeSel sel, int d, double sigma, double* part, int S) {
  extern __shared__ __align__(16) double trow[];
  __shared__ double sh[32];
  __shared__ uint64_t bars[kMultWarps][kEdgeMaxStages];
  const int lane = threadIdx.x;
  uint64_t* bar = bars[threadIdx.y];
  if (lane == 0)
    for (int q = 0; q < S; ++q) mbar_init(&bar[q], 1);
  fence_mbar_init();
  __syncwarp();
  const unsigned rb = static_cast<unsigned>(d) * 8u;
  const int64_t wid = static_cast<int64_t>(blockIdx.x) * blockDim.y + threadIdx.y;
  const int64_t nw = static_cast<int64_t>(gridDim.x) * blockDim.y;
  const int64_t cnt = wid < sel.count ? (sel.count - wid + nw - 1) / nw : 0;  // this warp's edges: wid + e nw
  constexpr int NR = VM == 1 ? 4 : 3;  // staged rows per edge
  double* const base = trow + static_cast<size_t>(threadIdx.y) * S * NR * d;
  auto issue = [&](int64_t e, int q) {  // lane 0: x_i, x_j, Z_l, V_l of edge wid + e nw into slot q
    const int64_t l = sel.at(wid + e * nw);
    double* sx = base + static_cast<size_t>(q) * NR * d;
    uint64_t* b = &bar[q];
    fence_proxy_async();
    mbar_expect_tx(b, NR * rb);
    bulk_g2s(sx, X + static_cast<int64_t>(ei[l]) * d, rb, b);
    bulk_g2s(sx + d, X + static_cast<int64_t>(ej[l]) * d, rb, b);
    const uint64_t ef = policy_evict_first();
    bulk_g2s_hint(sx + 2 * d, Z + l * d, rb, b, ef);
    if (VM == 1) bulk_g2s_hint(sx + 3 * d, V + l * d, rb, b, ef);
  };
  if (lane == 0)
    for (int q = 0; q < S && q < cnt; ++q) issue(q, q);
  double s[5] = {0, 0, 0, 0, 0}, mx = 0.0, err = 0.0, excess = -1.0;
  int q = 0;
  unsigned ph = 0;
  for (int64_t it = 0; it < cnt; ++it) {
    const int64_t row_ = sel.at(wid + it * nw);
    double* sx = base + static_cast<size_t>(q) * NR * d;  // x_i, then x = x_i - x_j
    double* sb = sx + d;   // x_j, then (VM = 2) V_l
    double* sz = sb + d;   // Z_l, then Zsum, then Z_l new
    const double* sv = VM == 1 ? sz + d : sb;  // V_l
    double* z = Z + row_ * d;
    const double rl = rad[row_], tl = thr[row_], sl = ps[row_];
    mbar_wait(&bar[q], ph);
    double nn = 0.0, m = 0.0;
#pragma unroll 4
    for (int f = lane; f < d; f += 32) {
      const double x = sx[f] - sb[f];
      const double zo = sz[f];
      const double zs = zo + sigma * x;
      sx[f] = x;
      if (VM == 2) sb[f] = x + zo / sigma;
      sz[f] = zs;
      nn += zs * zs;
      m = fmax(m, fabs(zs));
    }
    mx = fmax(mx, m);
    const double nz = sqrt(warp_sum(nn));
    const double sc = rl / nz;
    double fr = 0.0, e = 0.0, xb2 = 0.0, zz = 0.0, uu = 0.0, l1 = 0.0, zmax = 0.0, al = 0.0;
#pragma unroll 4
    for (int f = lane; f < d; f += 32) {
      const double x = sx[f];
      const double zs = sz[f];
      const double zp = (Q == Q_L2) ? ((nz <= rl) ? zs : sc * zs) : fmax(fmin(zs, rl), -rl);
      const double vf = sv[f];
      const double pv = (Q == Q_L2) ? sl * vf : soft(vf, tl);
      const double zenv = sigma * (vf - pv);
      e = fmax(e, fabs(zenv - zp));
      z[f] = zp;
      sz[f] = zp;
      fr += (x - pv) * (x - pv);
      const double u = x + zp;
      xb2 += x * x;
      zz += zp * zp;
      if (Q == Q_L2) {
        uu += u * u;
      } else {
        l1 += fabs(x);
        zmax = fmax(zmax, fabs(zp));
        const double ee = x - soft(u, rl);
        al += ee * ee;
      }
    }
    err = fmax(err, e);
    fr = warp_sum(fr);
    xb2 = warp_sum(xb2);
    zz = warp_sum(zz);
    double t0;
    if (Q == Q_L2) {
      const double nu = sqrt(warp_sum(uu));
      if (nu <= rl) {
        al = xb2;
      } else {  // pass 3 (objective.cpp:110-111) from shared memory
        const double s2 = 1.0 - rl / nu;
#pragma unroll 4
        for (int f = lane; f < d; f += 32) {
          const double x = sx[f];
          const double ee = x - s2 * (x + sz[f]);
          al += ee * ee;
        }
        al = warp_sum(al);
      }
      t0 = w[row_] * sqrt(xb2);
      excess = fmax(excess, sqrt(zz) - (rl + 1e-9));
    } else {
      al = warp_sum(al);
      t0 = w[row_] * warp_sum(l1);
      excess = fmax(excess, warp_max(zmax) - (rl + 1e-9));
    }
    if (lane == 0) {
      s[0] += t0;
      s[1] += al;
      s[2] += xb2;
      s[3] += zz;
      s[4] += fr;
    }
    __syncwarp();  // every lane is done with the slot before lane 0 refills it
    if (lane == 0 && it + S < cnt) issue(it + S, q);
    if (++q == S) q = 0, ph ^= 1u;
  }
  for (int k = 0; k < 5; ++k) {
    const double r = block_sum(s[k], sh);
    if (threadIdx.x == 0 && threadIdx.y == 0) part[9 * blockIdx.x + k] = r;
  }
  const double a = block_max(mx, sh);
  const double b = block_max(err, sh);
  const double c = block_max(excess, sh);
  if (threadIdx.x == 0 && threadIdx.y == 0) {
    part[9 * blockIdx.x + 5] = 0.0;
    part[9 * blockIdx.x + 6] = a;
    part[9 * blockIdx.x + 7] = b;
    part[9 * blockIdx.x + 8] = c;
  }
}

// ---- q = inf edge passes with the rows staged in shared memory ----------------------------
// Michelot's threshold (linf.cuh) walks a row several times; the generic kernels re-read it
// from L1/L2 on every pass, which at C4 (d = 3072, 24 KB per row, 8 rows per block) thrashes
// L1 (phi 57 ms, multiplier 175 ms per launch).  Here one warp per edge stages the rows its
// passes revisit, 4 warps per block, and every pass after the first reads shared memory.
// Each lane touches only the elements it wrote (f = lane + 32 k): no block barriers.
// The threshold passes visit only each lane's surviving candidates (linf_theta_bits).
// Per-element arithmetic and per-lane order are those of the generic kernels.
constexpr int kLinfWarps = 4;
inline bool linf_staged(int64_t d, int rows) {
  return d > 32 && d <= 32 * 32 * kLinfWords && static_cast<size_t>(kLinfWarps) * rows * d * sizeof(double) <= 200 * 1024;
}
__global__ void __launch_bounds__(32 * kLinfWarps) k_phi_edge_linf_s(
    const double* __restrict__ X, const double* __restrict__ Z, const int* __restrict__ ei,
    const int* __restrict__ ej, const double* __restrict__ thr, const double* __restrict__ rad, EdgeSel sel, int d,
    double sigma, double* __restrict__ V, double* __restrict__ nv, double* __restrict__ nvc, double* part) {
  extern __shared__ double srow[];
  __shared__ double sh[32];
  const unsigned gm = group_mask();
  double* sv = srow + static_cast<size_t>(threadIdx.y) * d;
  double acc = 0.0;
  EDGES_BEGIN(sel) {
    const double* xa = X + static_cast<int64_t>(ei[row_]) * d;
    const double* xb = X + static_cast<int64_t>(ej[row_]) * d;
    const double* z = Z + row_ * d;
    double* v = V + row_ * d;
    const double t = thr[row_];
    // 8 elements per lane per batch: 24 independent loads in flight (the pass is latency-bound otherwise)
    for (int f0 = threadIdx.x; f0 < d; f0 += 8 * 32) {
      double a[8], b[8], c[8];
#pragma unroll
      for (int u = 0; u < 8; ++u) {
        const int f = f0 + 32 * u;
        a[u] = f < d ? xa[f] : 0.0;
        b[u] = f < d ? xb[f] : 0.0;
        c[u] = f < d ? __ldcs(z + f) : 0.0;
      }
#pragma unroll
      for (int u = 0; u < 8; ++u) {
        const int f = f0 + 32 * u;
        if (f < d) {
          const double x = (a[u] - b[u]) + c[u] / sigma;
          sv[f] = x;
          __stcs(v + f, x);
        }
      }
    }
    int cnt;
    const double th = linf_theta_bits([&](int f) { return sv[f]; }, d, t, &cnt);
    double sq = 0.0;
    for (int f = threadIdx.x; f < d; f += blockDim.x) {
      const double r = th < 0.0 ? sv[f] : soft(sv[f], th);
      sq += r * r;
    }
    const double env = rad[row_] * (th < 0.0 ? 0.0 : th) + (0.5 * sigma) * group_sum(sq, gm);
    if (threadIdx.x == 0) {
      nv[row_] = th;
      nvc[row_] = cnt;
      acc += env;
    }
    __syncwarp();
  }
  acc = block_sum(acc, sh);
  if (threadIdx.x == 0 && threadIdx.y == 0) part[blockIdx.x] = acc;
}
// k_mult_inf with x = x_i - x_j and Z + sigma x (then the new Z) staged
__global__ void __launch_bounds__(32 * kLinfWarps) k_mult_inf_s(
    const double* __restrict__ X, double* __restrict__ Z, const double* __restrict__ V, const double* __restrict__ ps,
    const double* __restrict__ rad, const double* __restrict__ w, const int* __restrict__ ei,
    const int* __restrict__ ej, EdgeSel sel, int d, double sigma, double* part) {
  extern __shared__ double srow[];
  __shared__ double sh[32];
  const unsigned gm = group_mask();
  double* sx = srow + static_cast<size_t>(threadIdx.y) * 2 * d;
  double* sz = sx + d;
  double s[5] = {0, 0, 0, 0, 0}, mx = 0.0, err = 0.0, excess = -1.0;
  EDGES_BEGIN(sel) {
    const double* xa = X + static_cast<int64_t>(ei[row_]) * d;
    const double* xb = X + static_cast<int64_t>(ej[row_]) * d;
    double* z = Z + row_ * d;
    const double* v = V + row_ * d;
    const double rl = rad[row_], thv = ps[row_];
    double m = 0.0;
    for (int f0 = threadIdx.x; f0 < d; f0 += 8 * 32) {  // batched loads (see k_phi_edge_linf_s)
      double a[8], b[8], c[8];
#pragma unroll
      for (int u = 0; u < 8; ++u) {
        const int f = f0 + 32 * u;
        a[u] = f < d ? xa[f] : 0.0;
        b[u] = f < d ? xb[f] : 0.0;
        c[u] = f < d ? z[f] : 0.0;
      }
#pragma unroll
      for (int u = 0; u < 8; ++u) {
        const int f = f0 + 32 * u;
        if (f < d) {
          const double x = a[u] - b[u];
          const double zs = c[u] + sigma * x;
          sx[f] = x;
          sz[f] = zs;
          m = fmax(m, fabs(zs));
        }
      }
    }
    mx = fmax(mx, m);
    int cnt;
    const double thz = linf_theta_bits([&](int f) { return sz[f]; }, d, rl, &cnt);
    double fr = 0.0, e = 0.0, xb2 = 0.0, zz = 0.0, xm = 0.0, z1 = 0.0;
#pragma unroll 8
    for (int f = threadIdx.x; f < d; f += blockDim.x) {
      const double x = sx[f];
      const double zs = sz[f];
      const double zp = thz < 0.0 ? zs : soft(zs, thz);
      const double vf = __ldcs(v + f);
      const double pv = thv < 0.0 ? 0.0 : clampd(vf, thv);
      e = fmax(e, fabs(sigma * (vf - pv) - zp));
      z[f] = zp;
      sz[f] = zp;
      fr += (x - pv) * (x - pv);
      xb2 += x * x;
      zz += zp * zp;
      xm = fmax(xm, fabs(x));
      z1 += fabs(zp);
    }
    err = fmax(err, e);
    const double thu = linf_theta_bits([&](int f) { return sx[f] + sz[f]; }, d, rl, &cnt);
    double al = 0.0;
    for (int f = threadIdx.x; f < d; f += blockDim.x) {
      const double x = sx[f];
      const double ee = x - (thu < 0.0 ? 0.0 : clampd(x + sz[f], thu));
      al += ee * ee;
    }
    al = group_sum(al, gm);
    fr = group_sum(fr, gm);
    xb2 = group_sum(xb2, gm);
    zz = group_sum(zz, gm);
    const double pen = w[row_] * group_max(xm, gm);
    excess = fmax(excess, group_sum(z1, gm) - (rl + 1e-9));
    if (threadIdx.x == 0) {
      s[0] += pen;
      s[1] += al;
      s[2] += xb2;
      s[3] += zz;
      s[4] += fr;
    }
    __syncwarp();
  }
  for (int k = 0; k < 5; ++k) {
    const double r = block_sum(s[k], sh);
    if (threadIdx.x == 0 && threadIdx.y == 0) part[9 * blockIdx.x + k] = r;
  }
  const double a = block_max(mx, sh);
  const double b = block_max(err, sh);
  const double c = block_max(excess, sh);
  if (threadIdx.x == 0 && threadIdx.y == 0) {
    part[9 * blockIdx.x + 5] = 0.0;
    part[9 * blockIdx.x + 6] = a;
    part[9 * blockIdx.x + 7] = b;
    part[9 * blockIdx.x + 8] = c;
  }
}
// gap edge terms (gap_edge_terms) with x = x_i - x_j and z staged: one streaming pass with
// batched loads, later passes from shared memory (the generic kernel re-reads the rows)
template <int Q>
__global__ void __launch_bounds__(32 * kLinfWarps) k_gap_edge_s(
    const double* __restrict__ X, const double* __restrict__ Z, const int* __restrict__ ei,
    const int* __restrict__ ej, const double* __restrict__ rad, const double* __restrict__ w, EdgeSel sel, int d,
    double* part) {
  extern __shared__ double srow[];
  __shared__ double sh[32];
  const unsigned gm = group_mask();
  double* sx = srow + static_cast<size_t>(threadIdx.y) * 2 * d;
  double* sz = sx + d;
  double s[4] = {0, 0, 0, 0}, excess = -1.0;
  EDGES_BEGIN(sel) {
    const double* xa = X + static_cast<int64_t>(ei[row_]) * d;
    const double* xb = X + static_cast<int64_t>(ej[row_]) * d;
    const double* z = Z + row_ * d;
    const double rl = rad[row_];
    double xb2 = 0.0, zz = 0.0, xm = 0.0, z1 = 0.0, uu = 0.0, l1 = 0.0, zmax = 0.0;
    for (int f0 = threadIdx.x; f0 < d; f0 += 8 * 32) {
      double a[8], b[8], c[8];
#pragma unroll
      for (int u = 0; u < 8; ++u) {
        const int f = f0 + 32 * u;
        a[u] = f < d ? xa[f] : 0.0;
        b[u] = f < d ? xb[f] : 0.0;
        c[u] = f < d ? __ldcs(z + f) : 0.0;
      }
#pragma unroll
      for (int u = 0; u < 8; ++u) {
        const int f = f0 + 32 * u;
        if (f < d) {
          const double x = a[u] - b[u];
          const double zf = c[u];
          sx[f] = x;
          sz[f] = zf;
          xb2 += x * x;
          zz += zf * zf;
          if (Q == Q_LINF) {
            xm = fmax(xm, fabs(x));
            z1 += fabs(zf);
          } else {
            const double uv = x + zf;
            uu += uv * uv;
            l1 += fabs(x);
            zmax = fmax(zmax, fabs(zf));
          }
        }
      }
    }
    double t0, al = 0.0;
    xb2 = group_sum(xb2, gm);
    zz = group_sum(zz, gm);
    if (Q == Q_LINF) {
      int cnt;
      const double th = linf_theta_bits([&](int f) { return sx[f] + sz[f]; }, d, rl, &cnt);
      for (int f = threadIdx.x; f < d; f += blockDim.x) {
        const double x = sx[f];
        const double e = x - (th < 0.0 ? 0.0 : clampd(x + sz[f], th));
        al += e * e;
      }
      al = group_sum(al, gm);
      t0 = w[row_] * group_max(xm, gm);
      excess = fmax(excess, group_sum(z1, gm) - (rl + 1e-9));
    } else if (Q == Q_L2) {
      const double nu = sqrt(group_sum(uu, gm));
      if (nu <= rl) {
        al = xb2;
      } else {
        const double sc = 1.0 - rl / nu;
        for (int f = threadIdx.x; f < d; f += blockDim.x) {
          const double x = sx[f];
          const double e = x - sc * (x + sz[f]);
          al += e * e;
        }
        al = group_sum(al, gm);
      }
      t0 = w[row_] * sqrt(xb2);
      excess = fmax(excess, sqrt(zz) - (rl + 1e-9));
    } else {
      for (int f = threadIdx.x; f < d; f += blockDim.x) {
        const double x = sx[f];
        const double e = x - soft(x + sz[f], rl);
        al += e * e;
      }
      al = group_sum(al, gm);
      t0 = w[row_] * group_sum(l1, gm);
      excess = fmax(excess, group_max(zmax, gm) - (rl + 1e-9));
    }
    if (threadIdx.x == 0) s[0] += t0, s[1] += al, s[2] += xb2, s[3] += zz;
    __syncwarp();
  }
  for (int k = 0; k < 4; ++k) {
    const double r = block_sum(s[k], sh);
    if (threadIdx.x == 0 && threadIdx.y == 0) part[5 * blockIdx.x + k] = r;
  }
  const double m = block_max(excess, sh);
  if (threadIdx.x == 0 && threadIdx.y == 0) part[5 * blockIdx.x + 4] = m;
}
// project_columns (prox.cpp:82-93) with the row staged: q = 2 needs ||z|| before scaling and
// q = inf its threshold passes; one streaming read with batched loads, then shared memory
template <int Q>
__global__ void __launch_bounds__(32 * kLinfWarps) k_project_cols_s(const double* __restrict__ Z,
                                                                     const double* __restrict__ r, int64_t E, int d,
                                                                     double* __restrict__ out, int* changed) {
  const bool inplace = out == Z;
  extern __shared__ double srow[];
  const unsigned gm = group_mask();
  double* sz = srow + static_cast<size_t>(threadIdx.y) * d;
  ROWS_BEGIN(E) {
    const double* z = Z + row_ * d;
    double* o = out + row_ * d;
    const double rl = r[row_];
    double ss = 0.0;
    for (int f0 = threadIdx.x; f0 < d; f0 += 8 * 32) {
      double a[8];
#pragma unroll
      for (int u = 0; u < 8; ++u) {
        const int f = f0 + 32 * u;
        a[u] = f < d ? __ldcs(z + f) : 0.0;
      }
#pragma unroll
      for (int u = 0; u < 8; ++u) {
        const int f = f0 + 32 * u;
        if (f < d) {
          sz[f] = a[u];
          if (Q == Q_L2) ss += a[u] * a[u];
        }
      }
    }
    if (Q == Q_L2) {
      const double nz = sqrt(group_sum(ss, gm));
      const double sc = rl / nz;
      const bool inside = nz <= rl;
      if (!inside && changed) *changed = 1;
      if (!(inplace && inside))
        for (int f = threadIdx.x; f < d; f += blockDim.x) o[f] = inside ? sz[f] : sc * sz[f];
    } else {
      int cnt;
      const double th = linf_theta_bits([&](int f) { return sz[f]; }, d, rl, &cnt);
      if (th >= 0.0 && changed) *changed = 1;
      if (!(inplace && th < 0.0))
        for (int f = threadIdx.x; f < d; f += blockDim.x) o[f] = th < 0.0 ? sz[f] : soft(sz[f], th);
    }
    __syncwarp();
  }
}
// Launch one of the staged q = inf kernels on `grid` blocks (the generic kernel's grid, so the
// partial tables keep their shape).
template <class K, class... Args>
void launch_linf_s(K kernel, int rows, int64_t d, int grid, cudaStream_t s, Args... args) {
  const size_t smem = static_cast<size_t>(kLinfWarps) * rows * d * sizeof(double);
  CPB_CUDA(cudaFuncSetAttribute(kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(smem)));
  kernel<<<grid, dim3(32, kLinfWarps), smem, s>>>(args...);
  CPB_LAUNCH_CHECK();
}
static_assert(kMultWarps == kLinfWarps, "k_gap_edge_t must assign edges to warps like k_gap_edge_s");
// TMA variant of k_gap_edge_s for q = 2 / 1 (even d <= 1024): x_i, x_j and Z_l stream into
// the warp's shared-memory slot by cp.async.bulk instead of batched loads.  Same edges per
// warp, per-lane element order and group sums as k_gap_edge_s, so the partial table is
// bitwise the same.
template <int Q>
__global__ void __launch_bounds__(32 * kMultWarps) k_gap_edge_t(
    const double* __restrict__ X, const double* __restrict__ Z, const int* __restrict__ ei,
    const int* __restrict__ ej, const double* __restrict__ rad, const double* __restrict__ w, EdgeSel sel, int d,
    double* part, int S) {
  extern __shared__ __align__(16) double prow[];
  __shared__ double sh[32];
  __shared__ uint64_t bars[kMultWarps][kEdgeMaxStages];
  const int lane = threadIdx.x;
  const unsigned gm = 0xffffffffu;
  uint64_t* bar = bars[threadIdx.y];
  if (lane == 0)
    for (int q = 0; q < S; ++q) mbar_init(&bar[q], 1);
  fence_mbar_init();
  __syncwarp();
  const unsigned rb = static_cast<unsigned>(d) * 8u;
  const int64_t wid = static_cast<int64_t>(blockIdx.x) * blockDim.y + threadIdx.y;
  const int64_t nw = static_cast<int64_t>(gridDim.x) * blockDim.y;
  const int64_t cnt = wid < sel.count ? (sel.count - wid + nw - 1) / nw : 0;
  double* const base = prow + static_cast<size_t>(threadIdx.y) * S * 3 * d;
  auto issue = [&](int64_t e, int q) {
    const int64_t l = sel.at(wid + e * nw);
    double* sa = base + static_cast<size_t>(q) * 3 * d;
    uint64_t* b = &bar[q];
    fence_proxy_async();
    mbar_expect_tx(b, 3 * rb);
    bulk_g2s(sa, X + static_cast<int64_t>(ei[l]) * d, rb, b);
    bulk_g2s(sa + d, X + static_cast<int64_t>(ej[l]) * d, rb, b);
    bulk_g2s_hint(sa + 2 * d, Z + l * d, rb, b, policy_evict_first());
  };
  if (lane == 0)
    for (int q = 0; q < S && q < cnt; ++q) issue(q, q);
  double s[4] = {0, 0, 0, 0}, excess = -1.0;
  int q = 0;
  unsigned ph = 0;
  for (int64_t e = 0; e < cnt; ++e) {
    const int64_t row_ = sel.at(wid + e * nw);
    const double* sa = base + static_cast<size_t>(q) * 3 * d;
    const double* sb = sa + d;
    const double* sz = sb + d;
    const double rl = rad[row_];
    mbar_wait(&bar[q], ph);
    double xb2 = 0.0, zz = 0.0, uu = 0.0, l1 = 0.0, zmax = 0.0;
    for (int f = lane; f < d; f += 32) {
      const double x = sa[f] - sb[f];
      const double zf = sz[f];
      xb2 += x * x;
      zz += zf * zf;
      const double uv = x + zf;
      uu += uv * uv;
      l1 += fabs(x);
      zmax = fmax(zmax, fabs(zf));
    }
    double t0, al = 0.0;
    xb2 = group_sum(xb2, gm);
    zz = group_sum(zz, gm);
    if (Q == Q_L2) {
      const double nu = sqrt(group_sum(uu, gm));
      if (nu <= rl) {
        al = xb2;
      } else {
        const double sc = 1.0 - rl / nu;
        for (int f = lane; f < d; f += 32) {
          const double x = sa[f] - sb[f];
          const double ev = x - sc * (x + sz[f]);
          al += ev * ev;
        }
        al = group_sum(al, gm);
      }
      t0 = w[row_] * sqrt(xb2);
      excess = fmax(excess, sqrt(zz) - (rl + 1e-9));
    } else {
      for (int f = lane; f < d; f += 32) {
        const double x = sa[f] - sb[f];
        const double ev = x - soft(x + sz[f], rl);
        al += ev * ev;
      }
      al = group_sum(al, gm);
      t0 = w[row_] * group_sum(l1, gm);
      excess = fmax(excess, group_max(zmax, gm) - (rl + 1e-9));
    }
    if (lane == 0) s[0] += t0, s[1] += al, s[2] += xb2, s[3] += zz;
    __syncwarp();
    if (lane == 0 && e + S < cnt) issue(e + S, q);
    if (++q == S) q = 0, ph ^= 1u;
  }
  for (int k = 0; k < 4; ++k) {
    const double r = block_sum(s[k], sh);
    if (threadIdx.x == 0 && threadIdx.y == 0) part[5 * blockIdx.x + k] = r;
  }
  const double m = block_max(excess, sh);
  if (threadIdx.x == 0 && threadIdx.y == 0) part[5 * blockIdx.x + 4] = m;
}

// gap edge terms over `sel` on `grid` blocks (5 partials per block)
void gap_edge_launch(Ctx& c, int grid, const GroupGeom& ge, const double* X, const double* Z, const Prob& P,
                     EdgeSel sel, int64_t d, double* pe) {
  if (ge.gx == 32 && P.q != Q_LINF && d > 32 && d % 2 == 0 && d <= kMultSmemMaxD && linf_staged(d, 2)) {
    const int S = edge_stages(d, 3);
    const size_t smem = static_cast<size_t>(kMultWarps) * S * 3 * d * sizeof(double);
    if (first_on_device("k_gap_edge_t.smem")) {
      CPB_CUDA(cudaFuncSetAttribute(k_gap_edge_t<Q_L2>, cudaFuncAttributeMaxDynamicSharedMemorySize, 220 * 1024));
      CPB_CUDA(cudaFuncSetAttribute(k_gap_edge_t<Q_L1>, cudaFuncAttributeMaxDynamicSharedMemorySize, 220 * 1024));
    }
    const dim3 blk(32, kMultWarps);
    if (P.q == Q_L2)
      k_gap_edge_t<Q_L2><<<grid, blk, smem, c.s>>>(X, Z, P.g->ei.p, P.g->ej.p, P.rad, P.g->w.p, sel,
                                                   static_cast<int>(d), pe, S);
    else
      k_gap_edge_t<Q_L1><<<grid, blk, smem, c.s>>>(X, Z, P.g->ei.p, P.g->ej.p, P.rad, P.g->w.p, sel,
                                                   static_cast<int>(d), pe, S);
    CPB_LAUNCH_CHECK();
    return;
  }
  if (ge.gx == 32 && linf_staged(d, 2)) {  // 32-lane rows that fit two staged rows per warp
    auto args = [&](auto kernel) {
      launch_linf_s(kernel, 2, d, grid, c.s, X, Z, (const int*)P.g->ei.p, (const int*)P.g->ej.p,
                    (const double*)P.rad, (const double*)P.g->w.p, sel, static_cast<int>(d), pe);
    };
    if (P.q == Q_LINF)
      args(k_gap_edge_s<Q_LINF>);
    else if (P.q == Q_L2)
      args(k_gap_edge_s<Q_L2>);
    else
      args(k_gap_edge_s<Q_L1>);
    return;
  }
  k_gap_edge<<<grid, dim3(ge.gx, ge.gy), 0, c.s>>>(X, Z, P.g->ei.p, P.g->ej.p, P.rad, P.g->w.p, sel,
                                                   static_cast<int>(d), P.q, pe);
  CPB_LAUNCH_CHECK();
}

// TMA variant of k_phi_edge (even d, 32-lane rows): x_i, x_j and Z_l are
// streamed into the warp's shared-memory slot by cp.async.bulk (three rows in
// flight per warp regardless of registers); V_l is written with streaming
// stores.  Per-element arithmetic and per-lane order are those of k_phi_edge.
template <int Q>
__global__ void __launch_bounds__(32 * kMultWarps) k_phi_edge_t(
    const double* __restrict__ X, const double* __restrict__ Z, const int* __restrict__ ei,
    const int* __restrict__ ej, const double* __restrict__ thr, const double* __restrict__ rad, EdgeSel sel, int d,
    double sigma, double* __restrict__ V, double* __restrict__ nv, double* part, int S) {
  extern __shared__ __align__(16) double prow[];
  __shared__ double sh[32];
  __shared__ uint64_t bars[kMultWarps][kEdgeMaxStages];
  const int lane = threadIdx.x;
  uint64_t* bar = bars[threadIdx.y];
  if (lane == 0)
    for (int q = 0; q < S; ++q) mbar_init(&bar[q], 1);
  fence_mbar_init();
  __syncwarp();
  const unsigned rb = static_cast<unsigned>(d) * 8u;
  const int64_t wid = static_cast<int64_t>(blockIdx.x) * blockDim.y + threadIdx.y;
  const int64_t nw = static_cast<int64_t>(gridDim.x) * blockDim.y;
  const int64_t cnt = wid < sel.count ? (sel.count - wid + nw - 1) / nw : 0;
  double* const base = prow + static_cast<size_t>(threadIdx.y) * S * 3 * d;
  auto issue = [&](int64_t e, int q) {
    const int64_t l = sel.at(wid + e * nw);
    double* sa = base + static_cast<size_t>(q) * 3 * d;
    uint64_t* b = &bar[q];
    fence_proxy_async();
    mbar_expect_tx(b, 3 * rb);
    bulk_g2s(sa, X + static_cast<int64_t>(ei[l]) * d, rb, b);
    bulk_g2s(sa + d, X + static_cast<int64_t>(ej[l]) * d, rb, b);
    bulk_g2s_hint(sa + 2 * d, Z + l * d, rb, b, policy_evict_first());
  };
  if (lane == 0)
    for (int q = 0; q < S && q < cnt; ++q) issue(q, q);
  double acc = 0.0;
  int q = 0;
  unsigned ph = 0;
  for (int64_t e = 0; e < cnt; ++e) {
    const int64_t row_ = sel.at(wid + e * nw);
    double* sa = base + static_cast<size_t>(q) * 3 * d;
    double* sb = sa + d;
    double* sz = sb + d;
    double* v = V + row_ * d;
    const double t = thr[row_];
    mbar_wait(&bar[q], ph);
    double env;
    if (Q == Q_L2) {
      double ss = 0.0;
#pragma unroll 4
      for (int f = lane; f < d; f += 32) {
        const double x = (sa[f] - sb[f]) + sz[f] / sigma;
        __stcs(v + f, x);
        ss += x * x;
      }
      ss = warp_sum(ss);
      const double nvl = sqrt(ss);
      double pn = 0.0, sq = ss;
      if (!(nvl <= t)) {
        const double sc = 1.0 - t / nvl;
        pn = sc * nvl;
        sq = (sc - 1.0) * (sc - 1.0) * ss;
      }
      env = rad[row_] * pn + (0.5 * sigma) * sq;
      if (lane == 0) nv[row_] = nvl;
    } else {
      double a = 0.0, b = 0.0;
#pragma unroll 4
      for (int f = lane; f < d; f += 32) {
        const double x = (sa[f] - sb[f]) + sz[f] / sigma;
        __stcs(v + f, x);
        const double p = soft(x, t);
        a += fabs(p);
        b += (p - x) * (p - x);
      }
      env = rad[row_] * warp_sum(a) + (0.5 * sigma) * warp_sum(b);
      if (lane == 0) nv[row_] = 0.0;
    }
    if (lane == 0) acc += env;
    __syncwarp();
    if (lane == 0 && e + S < cnt) issue(e + S, q);
    if (++q == S) q = 0, ph ^= 1u;
  }
  acc = block_sum(acc, sh);
  if (threadIdx.x == 0 && threadIdx.y == 0) part[blockIdx.x] = acc;
}

// ---- fast AMA (ama.cpp:57-72) -----------------------------------------------------------
// One edge row of the dual step: z~ = Zh_l + step (x_i - x_j), Z+ = proj_{dual ball}(z~),
// Zh_l = Z+ + mom (Z+ - Zp_l), Zp_l = Z+.  Loads bypass L1 (__ldcg): the fused block kernel
// below reads rows other SMs wrote before its grid barrier.
__device__ __forceinline__ void ama_edge_row(int64_t row, const double* __restrict__ Xh, double* __restrict__ Zh,
                                             double* __restrict__ Zp, int ia, int ib, double rl, int d, double step,
                                             double mom, int q, unsigned gm) {
  const double* xa = Xh + static_cast<int64_t>(ia) * d;
  const double* xb = Xh + static_cast<int64_t>(ib) * d;
  double* zh = Zh + row * d;
  double* zp = Zp + row * d;
  if (q == Q_LINF) {
    int cnt;
    const double th =
        linf_theta([&](int f) { return __ldcg(zh + f) + step * (__ldcg(xa + f) - __ldcg(xb + f)); }, d, rl, gm, &cnt);
    for (int f = threadIdx.x; f < d; f += blockDim.x) {
      const double zn = __ldcg(zh + f) + step * (__ldcg(xa + f) - __ldcg(xb + f));
      const double zpr = th < 0.0 ? zn : soft(zn, th);
      const double old = __ldcg(zp + f);
      zh[f] = zpr + mom * (zpr - old);
      zp[f] = zpr;
    }
    return;
  }
  double nn = 0.0;
  if (q == Q_L2) {
    for (int f = threadIdx.x; f < d; f += blockDim.x) {
      const double zn = __ldcg(zh + f) + step * (__ldcg(xa + f) - __ldcg(xb + f));
      nn += zn * zn;
    }
  }
  const double nz = sqrt(group_sum(nn, gm));
  const double sc = rl / nz;
  for (int f = threadIdx.x; f < d; f += blockDim.x) {
    const double zn = __ldcg(zh + f) + step * (__ldcg(xa + f) - __ldcg(xb + f));
    const double zpr = (q == Q_L2) ? ((nz <= rl) ? zn : sc * zn) : fmax(fmin(zn, rl), -rl);
    const double old = __ldcg(zp + f);
    zh[f] = zpr + mom * (zpr - old);
    zp[f] = zpr;
  }
}

__global__ void k_ama_edge(const double* __restrict__ Xh, double* __restrict__ Zh, double* __restrict__ Zp,
                           const double* __restrict__ rad, const int* __restrict__ ei, const int* __restrict__ ej,
                           int64_t E, int d, double step, double mom, int q, const double* __restrict__ momp) {
  if (momp) mom = *momp;  // graph-launched blocks read the momentum the block's k_ama_mom wrote
  const unsigned gm = group_mask();
  ROWS_BEGIN(E) { ama_edge_row(row_, Xh, Zh, Zp, ei[row_], ej[row_], rad[row_], d, step, mom, q, gm); }
}

// k_g_gap's per-(node, feature) terms: ||X - A||^2, ||B^T Z||^2, <B^T Z, A>, ||X - A + B^T Z||^2
__device__ __forceinline__ void gap_node_acc(double* s, double xv, double a, double acc) {
  const double xa = xv - a;
  const double st = xa + acc;
  s[0] += xa * xa;
  s[1] += acc * acc;
  s[2] += acc * a;
  s[3] += st * st;
}

// Fused block of `cnt` AMA iterations for small problems (d <= 32), one cooperative launch:
// per iteration X^ = A - Z^ B^T (node-CSR gather, incident edges in ascending id: k_g_bt mode
// 1's exact order), grid barrier, the edge step with the iteration's Nesterov momentum
// (computed per thread from t0 exactly like the host loop), grid barrier; finally
// X = A - Z B^T of the new iterate (recover_primal).  Bitwise the same as the per-kernel loop;
// replaces 2 cnt + 1 launches by one (C1: n = 1000, d = 2, launch-bound).
__global__ void __launch_bounds__(256) k_ama_block(const double* __restrict__ A, double* Xh, double* Zh, double* Zp,
                                                   double* Xout, const double* __restrict__ rad,
                                                   const int* __restrict__ ei, const int* __restrict__ ej,
                                                   const int* __restrict__ off, const int* __restrict__ adj_e,
                                                   const int* __restrict__ adj_o, const int* __restrict__ order,
                                                   int64_t n, int64_t E, int d, double step, int q, double t0,
                                                   int cnt, const double* __restrict__ wt, double* part) {
  cg::grid_group grid = cg::this_grid();
  const unsigned gm = group_mask();
  const int tid = threadIdx.y * blockDim.x + threadIdx.x;
  const int lane = tid & 31;
  const int64_t w0 = (static_cast<int64_t>(blockIdx.x) * 256 + tid) >> 5, nw = static_cast<int64_t>(gridDim.x) * 8;
  double t = t0;
  double sn[4] = {0, 0, 0, 0};
  // When every warp owns at most one node and every group at most one edge for the whole
  // kernel (C1), the node's incident edge ids / sides and the edge's endpoints stay in
  // registers, so an iteration's loads are all independent (one L2 latency per phase).
  const bool one_node = nw >= n;
  const int64_t row0 = blockIdx.x * static_cast<int64_t>(blockDim.y) + threadIdx.y;
  const bool one_row = static_cast<int64_t>(gridDim.x) * blockDim.y >= E;
  int my_v = -1, my_deg = 0, my_e = 0, my_o = 0;
  if (one_node && w0 < n) {
    my_v = order[w0];
    const int p0 = off[my_v];
    my_deg = off[my_v + 1] - p0;
    if (my_deg <= 32 && lane < my_deg) {
      my_e = adj_e[p0 + lane];
      my_o = adj_o[p0 + lane];
    }
  }
  int r_a = 0, r_b = 0;
  double r_l = 0.0;
  if (one_row && row0 < E) {
    r_a = ei[row0];
    r_b = ej[row0];
    r_l = rad[row0];
  }
  for (int j = 0;; ++j) {
    const bool last = j == cnt;
    const double* Zs = last ? Zp : Zh;
    double* Xd = last ? Xout : Xh;
    if (one_node && my_deg <= 32) {
      if (my_v >= 0) {  // warp-uniform
        double acc = 0.0;
        for (int u0 = 0; u0 < my_deg; u0 += 8) {
          double x[8];
          bool pl[8];
#pragma unroll
          for (int u = 0; u < 8; ++u) {
            const int e = __shfl_sync(0xffffffffu, my_e, (u0 + u) & 31);
            pl[u] = __shfl_sync(0xffffffffu, my_o, (u0 + u) & 31) > my_v;
            x[u] = (u0 + u < my_deg && lane < d) ? __ldcg(Zs + static_cast<int64_t>(e) * d + lane) : 0.0;
          }
#pragma unroll
          for (int u = 0; u < 8; ++u)
            if (u0 + u < my_deg) acc = pl[u] ? acc + x[u] : acc - x[u];
        }
        if (lane < d) {
          const int64_t i = static_cast<int64_t>(my_v) * d + lane;
          const double xv = A[i] - acc;
          Xd[i] = xv;
          if (last) gap_node_acc(sn, xv, A[i], acc);
        }
      }
    } else
    for (int64_t it = w0; it < n; it += nw) {
      const int v = order[it];
      if (lane < d) {
        const int p0 = off[v], p1 = off[v + 1];
        double acc = 0.0;
        for (int p = p0; p < p1; ++p) {
          const double x = __ldcg(Zs + static_cast<int64_t>(adj_e[p]) * d + lane);
          acc = adj_o[p] > v ? acc + x : acc - x;
        }
        const int64_t i = static_cast<int64_t>(v) * d + lane;
        const double xv = A[i] - acc;
        Xd[i] = xv;
        if (last) gap_node_acc(sn, xv, A[i], acc);
      }
    }
    if (last) break;
    grid.sync();
    const double tn = 0.5 * (1.0 + sqrt(1.0 + 4.0 * t * t));
    const double mom = (t - 1.0) / tn;
    t = tn;
    if (one_row) {
      if (row0 < E) ama_edge_row(row0, Xh, Zh, Zp, r_a, r_b, r_l, d, step, mom, q, gm);
    } else {
      for (int64_t row = row0; row < E; row += static_cast<int64_t>(gridDim.x) * blockDim.y)
        ama_edge_row(row, Xh, Zh, Zp, ei[row], ej[row], rad[row], d, step, mom, q, gm);
    }
    grid.sync();
  }
  // The gap check's partials at (Xout, Zp) (k_g_gap / k_gap_edge terms): the node terms came
  // with the last gather (acc = the B^T Zp row k_g_gap forms, same order); the edge terms need
  // every Xout row, hence one more barrier.  X, Z rows are first touched here by this SM (earlier
  // phases load with __ldcg), so plain loads see the other SMs' writes.
  __shared__ double sh[32];
  for (int k = 0; k < 4; ++k) {
    const double r = block_sum(sn[k], sh);
    if (tid == 0) part[4 * blockIdx.x + k] = r;
  }
  grid.sync();
  double se[4] = {0, 0, 0, 0}, excess = -1.0;
  for (int64_t row = row0; row < E; row += static_cast<int64_t>(gridDim.x) * blockDim.y) {
    double t4[4];
    gap_edge_terms(Xout + static_cast<int64_t>(ei[row]) * d, Xout + static_cast<int64_t>(ej[row]) * d, Zp + row * d,
                   rad[row], wt[row], d, q, gm, t4, excess);
    if (threadIdx.x == 0)
      for (int k = 0; k < 4; ++k) se[k] += t4[k];
  }
  double* pe = part + 4 * static_cast<int64_t>(gridDim.x);
  for (int k = 0; k < 4; ++k) {
    const double r = block_sum(se[k], sh);
    if (tid == 0) pe[5 * blockIdx.x + k] = r;
  }
  const double m = block_max(excess, sh);
  if (tid == 0) pe[5 * blockIdx.x + 4] = m;
}

// ---- host helpers ----------------------------------------------------------------------------
double* part_buf(Ctx& c, const char* name, size_t count) { return c.buf<double>(name, count + 8); }

double fetch1(Ctx& c) {
  double v;
  c.fetch(0, 1, &v);
  return v;
}

}  // namespace

// ====================================================================================
void make_radii(Ctx& c, const Graph& g, double gamma, double* rad) {
  if (g.E == 0) return;
  k_scale<<<flat_grid(c, g.E), 256, 0, c.s>>>(g.w.p, gamma, g.E, rad);
  CPB_LAUNCH_CHECK();
}
void make_thr(Ctx& c, int64_t E, const double* rad, double sigma, double* thr) {
  if (E == 0) return;
  k_div<<<flat_grid(c, E), 256, 0, c.s>>>(rad, sigma, E, thr);
  CPB_LAUNCH_CHECK();
}

double dot_dev(Ctx& c, const double* a, const double* b, int64_t count) {
  const int grid = flat_grid(c, count);
  double* part = part_buf(c, "dot.part", grid);
  k_dot<<<grid, 256, 0, c.s>>>(a, b, count, part);
  CPB_LAUNCH_CHECK();
  reduce_sum(c, part, grid, c.dscal);
  return fetch1(c);
}
double max_abs_dev(Ctx& c, const double* x, int64_t count) {
  const int grid = flat_grid(c, count);
  double* part = part_buf(c, "max.part", grid);
  k_maxabs<<<grid, 256, 0, c.s>>>(x, count, part);
  CPB_LAUNCH_CHECK();
  reduce_max(c, part, grid, c.dscal);
  return fetch1(c);
}
void axpy_dev(Ctx& c, double* out, const double* x, double a, const double* y, int64_t count) {
  if (count == 0) return;
  k_axpy<<<flat_grid(c, count), 256, 0, c.s>>>(out, x, a, y, count);
  CPB_LAUNCH_CHECK();
}
void neg_dev(Ctx& c, double* out, const double* x, int64_t count) {
  if (count == 0) return;
  k_neg<<<flat_grid(c, count), 256, 0, c.s>>>(out, x, count);
  CPB_LAUNCH_CHECK();
}
void copy_dev(Ctx& c, double* dst, const double* src, int64_t count) {
  if (count == 0 || dst == src) return;
  CPB_CUDA(cudaMemcpyAsync(dst, src, count * sizeof(double), cudaMemcpyDeviceToDevice, c.s));
}

void prox_columns_dev(Ctx& c, int q, const double* V, const double* t, int64_t d, int64_t E, double* out) {
  if (E == 0) return;
  GroupGeom gg = group_geom(c, E, d);
  k_prox_cols<<<gg.grid, dim3(gg.gx, gg.gy), 0, c.s>>>(q, V, t, E, static_cast<int>(d), out);
  CPB_LAUNCH_CHECK();
}
void project_columns_dev(Ctx& c, int q, const double* Z, const double* r, int64_t d, int64_t E, double* out) {
  int* changed = c.buf<int>("proj.changed", 1);
  CPB_CUDA(cudaMemsetAsync(changed, 0, sizeof(int), c.s));
  if (E == 0) return;
  GroupGeom gg = group_geom(c, E, d, 8, q != Q_LINF);
  if ((q == Q_L2 || q == Q_LINF) && gg.gx == 32 && linf_staged(d, 1)) {  // one HBM read of Z instead of two
    if (q == Q_L2)
      launch_linf_s(k_project_cols_s<Q_L2>, 1, d, gg.grid, c.s, Z, r, E, static_cast<int>(d), out, changed);
    else
      launch_linf_s(k_project_cols_s<Q_LINF>, 1, d, gg.grid, c.s, Z, r, E, static_cast<int>(d), out, changed);
    return;
  }
  k_project_cols<<<gg.grid, dim3(gg.gx, gg.gy), 0, c.s>>>(q, Z, r, E, static_cast<int>(d), out, changed);
  CPB_LAUNCH_CHECK();
}

bool last_projection_changed(Ctx& c) {
  int h = 1;
  CPB_CUDA(cudaMemcpyAsync(&h, c.buf<int>("proj.changed", 1), sizeof(int), cudaMemcpyDeviceToHost, c.s));
  c.sync();
  return h != 0;
}
void prox_jacobian_apply_dev(Ctx& c, int q, const double* V, const double* t, const double* W, int64_t d, int64_t E,
                             double* out) {
  if (E == 0) return;
  GroupGeom gg = group_geom(c, E, d);
  k_jac_apply_cols<<<gg.grid, dim3(gg.gx, gg.gy), 0, c.s>>>(q, V, t, W, E, static_cast<int>(d), out);
  CPB_LAUNCH_CHECK();
}

void prox_jacobian_diag_dev(Ctx& c, int q, const double* V, const double* t, int64_t d, int64_t E, double* out) {
  if (E == 0) return;
  GroupGeom gg = group_geom(c, E, d);
  k_jac_diag_cols<<<gg.grid, dim3(gg.gx, gg.gy), 0, c.s>>>(q, V, t, E, static_cast<int>(d), out);
  CPB_LAUNCH_CHECK();
}

double eval_phi(const Prob& P, const double* X, const double* D, double alpha, double* Xt, const double* Z,
                double sigma, const double* thr, double zz, double* V, double* nv) {
  Ctx& c = *P.c;
  const int64_t d = P.d(), n = P.n(), E = P.E(), m = d * n;
  const int fg = flat_grid(c, m);
  double* pn = part_buf(c, "phi.pn", fg);
  const double* Xe = D ? Xt : X;
  {
    Ctx::Timer tm(&c, D ? "trial_x" : "phi_node", (D ? 4.0 : 2.0) * m * 8.0);
    k_trial_x<<<fg, 256, 0, c.s>>>(X, D, alpha, Xt, P.A->A.p, m, pn);
    CPB_LAUNCH_CHECK();
  }
  reduce_sum(c, pn, fg, c.dscal);
  if (E > 0) {
    // one launch over an edge selection; returns the number of block partials in pe_
    auto run = [&](EdgeSel sel, double* pe_) -> int {
      GroupGeom gg = group_geom(c, sel.count, d, 8, P.q != Q_LINF);
      int nb = gg.grid;
      if (gg.gx == 32 && d <= kMultSmemMaxD && d % 2 == 0 && (P.q == Q_L2 || P.q == Q_L1)) {
        const int S = edge_stages(d, 3);
        const size_t smem = static_cast<size_t>(kMultWarps) * S * 3 * d * sizeof(double);
        if (first_on_device("k_phi_edge_t.smem")) {
          CPB_CUDA(cudaFuncSetAttribute(k_phi_edge_t<Q_L2>, cudaFuncAttributeMaxDynamicSharedMemorySize, 220 * 1024));
          CPB_CUDA(cudaFuncSetAttribute(k_phi_edge_t<Q_L1>, cudaFuncAttributeMaxDynamicSharedMemorySize, 220 * 1024));
        }
        int per_sm = 0;
        CPB_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, k_phi_edge_t<Q_L2>, 32 * kMultWarps, smem));
        nb = std::max(1, std::min(cdiv(sel.count, kMultWarps), c.sm_count * std::max(1, per_sm)));
        if (P.q == Q_L2)
          k_phi_edge_t<Q_L2><<<nb, dim3(32, kMultWarps), smem, c.s>>>(Xe, Z, P.g->ei.p, P.g->ej.p, thr, P.rad, sel,
                                                                      static_cast<int>(d), sigma, V, nv, pe_, S);
        else
          k_phi_edge_t<Q_L1><<<nb, dim3(32, kMultWarps), smem, c.s>>>(Xe, Z, P.g->ei.p, P.g->ej.p, thr, P.rad, sel,
                                                                      static_cast<int>(d), sigma, V, nv, pe_, S);
        CPB_LAUNCH_CHECK();
      } else if (P.q == Q_LINF && linf_staged(d, 1)) {
        launch_linf_s(k_phi_edge_linf_s, 1, d, gg.grid, c.s, Xe, Z, (const int*)P.g->ei.p, (const int*)P.g->ej.p,
                      thr, (const double*)P.rad, sel, static_cast<int>(d), sigma, V, nv, nv + E, pe_);
      } else {
        k_phi_edge<<<gg.grid, dim3(gg.gx, gg.gy), 0, c.s>>>(Xe, Z, P.g->ei.p, P.g->ej.p, thr, P.rad, sel,
                                                            static_cast<int>(d), sigma, P.q, V, nv, nv + E, pe_);
        CPB_LAUNCH_CHECK();
      }
      return nb;
    };
    const size_t pe_n = std::max(group_geom(c, E, d, 8, P.q != Q_LINF).grid, c.sm_count * 64);
    double* pe = part_buf(c, "phi.pe", pe_n);
    Ctx::Timer tm(&c, "phi_edge", (2.0 * E * d + n * d + 4.0 * E) * 8.0);
    if (!partitioned(c)) {
      reduce_sum(c, pe, run(EdgeSel{nullptr, 0, E}, pe), c.dscal + 1);
    } else {  // owned edges (summed) + ghost edges (their V feeds this rank's gathers)
      const EdgePart& ep = edge_part(c, *P.g);
      reduce_sum(c, pe, run(EdgeSel{nullptr, ep.e0, ep.e1 - ep.e0}, pe), c.dscal + 1);
      if (ep.nghost) run(EdgeSel{ep.ghost.p, 0, ep.nghost}, part_buf(c, "phi.pg", pe_n));
      comm_allreduce_sum(c, c.dscal + 1, 1);
    }
  } else {
    fill(c, c.dscal + 1, 1, 0.0);
  }
  double h[2];
  c.fetch(0, 2, h);
  return 0.5 * h[0] + h[1] - zz / (2.0 * sigma);
}

int64_t jac_params(const Prob& P, const double* nv, const double* thr, double* ps, double* jal, double* jbe) {
  Ctx& c = *P.c;
  const int64_t E = P.E();
  if (E == 0) return 0;
  const int grid = flat_grid(c, E);
  double* part = part_buf(c, "jac.part", grid);
  k_jac<<<grid, 256, 0, c.s>>>(nv, thr, E, P.q, ps, jal, jbe, part);
  CPB_LAUNCH_CHECK();
  reduce_sum(c, part, grid, c.dscal);
  return static_cast<int64_t>(fetch1(c));
}

double grad_diag(const Prob& P, const double* X, const double* V, const double* ps, const double* jal,
                 const double* jbe, const double* thr, double sigma, double* G, double* diag, bool want_diag) {
  Ctx& c = *P.c;
  const int64_t d = P.d(), n = P.n(), E = P.E();
  double* part = part_buf(c, "grad.part", static_cast<size_t>(c.sm_count) * 16);
  int nb;
  {
    // SURVEY.md §8(d) K8/K9 compulsory bytes: V once, the per-edge scalar, X and A read, G (and the
    // Jacobi diagonal) written, the CSR
    Ctx::Timer tm(&c, "grad_diag", (static_cast<double>(E) * d + E + (want_diag ? 4.0 : 3.0) * n * d) * 8.0 +
                                       (2.0 * E + n + 1) * 4.0);
    nb = gather_grad_diag(c, *P.g, X, P.A->A.p, V, ps, jal, jbe, thr, d, sigma, P.q, want_diag, G, diag, part);
  }
  reduce_sum(c, part, nb, c.dscal);
  if (partitioned(c)) comm_allreduce_sum(c, c.dscal, 1);  // ||G||^2 over every rank's rows
  return fetch1(c);
}

int hess_apply(const Prob& P, const double* p, const double* V, const double* jal, const double* jbe,
               const double* thr, double sigma, double* Ap, double* part, const void* st, const unsigned* mask,
               const unsigned* sgn) {
  Ctx& c = *P.c;
  double* bc = c.buf<double>("hess.bc", P.E() + 1);
  return hess_two_pass(c, *P.g, p, V, jal, jbe, thr, P.d(), sigma, P.q, bc, Ap, part,
                       cg_active_ptr(st), mask, sgn);
}

PcgOut pcg_newton(const Prob& P, const double* V, const double* jal, const double* jbe, const double* thr,
                  double sigma, const double* G, PcgWork w, double tol, int64_t max_iter, int64_t n_active) {
  const int64_t d = P.d(), n = P.n(), E = P.E(), m = d * n;
  // Algorithmic bytes per H-apply: p read + Ap write
  // (2 n d) + the active edge rows (E_a d) + two per-edge scalars + the CSR.
  const double hess_bytes = (2.0 * m + static_cast<double>(n_active) * d + 2.0 * E) * 8.0 + (2.0 * E + n + 1) * 4.0;
  // q = 1 / inf: the Jacobian's feature sets as bits, built once for this Newton system, so
  // the per-iteration gathers stop re-reading V (2 bits instead of 8 bytes per feature)
  unsigned *mask = nullptr, *sgn = nullptr;
  if (P.q != Q_L2 && E > 0) {
    const size_t words = static_cast<size_t>(E) * ((d + 31) / 32);
    mask = P.c->buf<unsigned>("hess.mask", words + 1);
    sgn = P.c->buf<unsigned>("hess.sgn", words + 1);
    edge_masks(*P.c, *P.g, V, P.q == Q_L1 ? thr : jal, d, P.q, mask, sgn);
  }
  PcgOp op = [&](const double* p, double* Ap, double* part, const void* st) {
    return hess_apply(P, p, V, jal, jbe, thr, sigma, Ap, part, st, mask, sgn);
  };
  // with a communicator the Newton system is node-partitioned over the ranks
  // (everything outside the PCG stays replicated: identical on every rank)
  const bool dist = P.c->comm != nullptr;
  const double op_b = dist ? hess_bytes / P.c->comm->nranks : hess_bytes;
  return pcg_dev(*P.c, n, d, op, op_b, "hess_apply", G, w, tol, max_iter, false, dist, P.g, true);
}

// Sum (and max) the columns of a (rows x cols) block-partial table on the host,
// in block order: deterministic and cheap (rows <= 8 x SM count).
// Column sums (or maxima for max_cols) of a host copy of a rows x cols block-partial table.
std::vector<double> reduce_cols(const double* all, int rows, int cols, const std::vector<int>& max_cols = {}) {
  std::vector<double> out(cols, 0.0);
  for (int k : max_cols) out[k] = -1e300;
  for (int b = 0; b < rows; ++b)
    for (int k = 0; k < cols; ++k) {
      const double x = all[static_cast<size_t>(b) * cols + k];
      bool is_max = false;
      for (int mk : max_cols) is_max |= (mk == k);
      out[k] = is_max ? std::max(out[k], x) : out[k] + x;
    }
  return out;
}
std::vector<double> host_cols(Ctx& c, const double* part, int rows, int cols, const std::vector<int>& max_cols = {}) {
  std::vector<double> all(static_cast<size_t>(rows) * cols), out(cols, 0.0);
  d2h(c, all.data(), part, all.size() * sizeof(double));
  for (int k : max_cols) out[k] = -1e300;
  for (int b = 0; b < rows; ++b)
    for (int k = 0; k < cols; ++k) {
      const double x = all[static_cast<size_t>(b) * cols + k];
      bool is_max = false;
      for (int mk : max_cols) is_max |= (mk == k);
      out[k] = is_max ? std::max(out[k], x) : out[k] + x;
    }
  return out;
}

GapOut eval_gap(const Prob& P, const double* X, const double* Z) {
  Ctx& c = *P.c;
  const int64_t d = P.d(), n = P.n(), E = P.E();
  // node partials [nbn x 4] and edge partials [grid x 5] share one buffer: both kernels are
  // enqueued first and one D2H brings both tables back (one host round trip per gap check)
  EdgeSel sel{nullptr, 0, E};
  if (E > 0 && partitioned(c)) {
    const EdgePart& ep = edge_part(c, *P.g);
    sel = EdgeSel{nullptr, ep.e0, ep.e1 - ep.e0};
  }
  GroupGeom ge = group_geom(c, sel.count, d, 8, P.q != Q_LINF);
  const size_t node_cap = 4 * static_cast<size_t>(c.sm_count) * 16;  // gather_gap: <= 8 * SMs blocks x 4
  double* pn = part_buf(c, "gap.pp", node_cap + 5 * static_cast<size_t>(ge.grid));
  int nbn;
  {
    Ctx::Timer tm(&c, "gap_node", (static_cast<double>(E) * d + 2.0 * n * d) * 8.0 + (2.0 * E + n + 1) * 4.0);  // Z once, X, A, CSR
    nbn = gather_gap(c, *P.g, X, P.A->A.p, Z, d, pn);
  }
  double* pe = pn + 4 * static_cast<size_t>(nbn);
  if (E > 0) {
    Ctx::Timer tm(&c, "gap_edge", (E * d + n * d) * 8.0);
    gap_edge_launch(c, ge.grid, ge, X, Z, P, sel, d, pe);
  }
  return gap_from_partials(P, pn, nbn, E > 0 ? ge.grid : 0);
}

// The gap / KKT numbers from the device's node partial table [nbn x 4] followed by the edge
// partial table [nbe x 5] (one D2H for both).
GapOut gap_from_partials(const Prob& P, const double* dev_parts, int nbn, int nbe) {
  Ctx& c = *P.c;
  const int64_t E = P.E();
  std::vector<double> all(4 * static_cast<size_t>(nbn) + 5 * static_cast<size_t>(nbe));
  d2h(c, all.data(), dev_parts, all.size() * sizeof(double));
  std::vector<double> h = reduce_cols(all.data(), nbn, 4);
  if (partitioned(c)) comm_allreduce_host(c, h);
  std::vector<double> e(5, 0.0);
  e[4] = -1.0;
  if (E > 0) {
    e = reduce_cols(all.data() + 4 * static_cast<size_t>(nbn), nbe, 5, {4});
    if (partitioned(c)) comm_allreduce_host(c, e, {4});
  }
  if (e[4] > 0.0) invalid("dual_objective: Z violates the dual-ball constraint");
  const double normA = data_fro_norm(c, *P.A);
  GapOut g;
  g.fp = 0.5 * h[0];
  if (E > 0 && P.gamma != 0.0) g.fp = g.fp + P.gamma * e[0];
  g.fd = -0.5 * h[1] + h[2];
  g.gap = std::abs(g.fp - g.fd) / (1.0 + std::abs(g.fp) + std::abs(g.fd));
  const double stat = std::sqrt(h[3]) / (1.0 + normA);
  if (E == 0 || P.gamma == 0.0) {
    g.kkt = stat;
  } else {
    const double align = std::sqrt(e[1]) / (1.0 + std::sqrt(e[2]) + std::sqrt(e[3]));
    g.kkt = std::max(stat, align);
  }
  return g;
}

double primal_objective_dev(const Prob& P, const double* X) {
  Ctx& c = *P.c;
  const int64_t d = P.d(), n = P.n(), E = P.E(), m = d * n;
  const int fg = flat_grid(c, m);
  double* pn = part_buf(c, "po.pn", fg);
  k_trial_x<<<fg, 256, 0, c.s>>>(X, nullptr, 0.0, nullptr, P.A->A.p, m, pn);
  CPB_LAUNCH_CHECK();
  reduce_sum(c, pn, fg, c.dscal);
  double value = 0.5 * fetch1(c);
  if (E == 0 || P.gamma == 0.0) return value;
  // penalty: gap edge term [0] with a zero dual (Z only enters the other terms)
  double* Z0 = c.buf<double>("po.z0", static_cast<size_t>(E) * d);
  CPB_CUDA(cudaMemsetAsync(Z0, 0, static_cast<size_t>(E) * d * sizeof(double), c.s));
  GroupGeom ge = group_geom(c, E, d);
  double* pe = part_buf(c, "po.pe", 5 * static_cast<size_t>(ge.grid));
  gap_edge_launch(c, ge.grid, ge, X, Z0, P, EdgeSel{nullptr, 0, E}, d, pe);
  std::vector<double> e = host_cols(c, pe, ge.grid, 5, {4});
  return value + P.gamma * e[0];
}

double dual_objective_dev(const Prob& P, const double* Z) {
  // fd does not depend on X; evaluate with X = A
  GapOut g = eval_gap(P, P.A->A.p, Z);
  return g.fd;
}
double kkt_residual_dev(const Prob& P, const double* X, const double* Z) {
  Ctx& c = *P.c;
  const int64_t d = P.d(), n = P.n(), E = P.E();
  (void)n;
  double* pn = part_buf(c, "kkt.pn", 4 * static_cast<size_t>(c.sm_count) * 16);
  const int nbn = gather_gap(c, *P.g, X, P.A->A.p, Z, d, pn);
  std::vector<double> h = host_cols(c, pn, nbn, 4);
  const double stat = std::sqrt(h[3]) / (1.0 + data_fro_norm(c, *P.A));
  if (E == 0 || P.gamma == 0.0) return stat;
  GroupGeom ge = group_geom(c, E, d);
  double* pe = part_buf(c, "kkt.pe", 5 * static_cast<size_t>(ge.grid));
  gap_edge_launch(c, ge.grid, ge, X, Z, P, EdgeSel{nullptr, 0, E}, d, pe);
  std::vector<double> e = host_cols(c, pe, ge.grid, 5, {4});
  return std::max(stat, std::sqrt(e[1]) / (1.0 + std::sqrt(e[2]) + std::sqrt(e[3])));
}

MultOut ssnal_multiplier(const Prob& P, const double* X, double* Z, const double* V, const double* ps,
                         const double* thr, double sigma, bool v_at_x) {
  Ctx& c = *P.c;
  const int64_t d = P.d(), n = P.n(), E = P.E();
  const size_t pe_n = 9 * static_cast<size_t>(std::max(group_geom(c, E, d, 8, P.q != Q_LINF).grid, c.sm_count * 64));
  double* pe = part_buf(c, "mult.pe", pe_n);
  // one launch over an edge selection; returns the number of 9-wide block partials
  auto run = [&](EdgeSel sel, double* pe) -> int {
    GroupGeom ge = group_geom(c, sel.count, d, 8, P.q != Q_LINF);
    int nb = ge.grid;
    if (P.q == Q_LINF && linf_staged(d, 2)) {
      launch_linf_s(k_mult_inf_s, 2, d, ge.grid, c.s, X, Z, V, ps, (const double*)P.rad, (const double*)P.g->w.p,
                    (const int*)P.g->ei.p, (const int*)P.g->ej.p, sel, static_cast<int>(d), sigma, pe);
    } else if (P.q == Q_LINF) {
      k_mult_inf<<<ge.grid, dim3(ge.gx, ge.gy), 0, c.s>>>(X, Z, V, ps, P.rad, P.g->w.p, P.g->ei.p, P.g->ej.p, sel,
                                                          static_cast<int>(d), sigma, pe);
      CPB_LAUNCH_CHECK();
    } else if (ge.gx == 32 && d <= kMultSmemMaxD && d % 2 == 0 && (P.q == Q_L2 || P.q == Q_L1)) {
      // V_l staged with the other rows (streaming it from HBM in pass 2 with 3
      // staged rows and more warps per SM measured slower: 4.42 vs 3.46 ms at C3)
      const int VM = v_at_x ? 2 : 1;
      const int NR = VM == 1 ? 4 : 3;
      const int S = edge_stages(d, NR);
      const size_t smem = static_cast<size_t>(kMultWarps) * S * NR * d * sizeof(double);
      if (first_on_device("k_mult_t.smem")) {
        CPB_CUDA(cudaFuncSetAttribute(k_mult_t<Q_L2, 1>, cudaFuncAttributeMaxDynamicSharedMemorySize, 220 * 1024));
        CPB_CUDA(cudaFuncSetAttribute(k_mult_t<Q_L1, 1>, cudaFuncAttributeMaxDynamicSharedMemorySize, 220 * 1024));
        CPB_CUDA(cudaFuncSetAttribute(k_mult_t<Q_L2, 2>, cudaFuncAttributeMaxDynamicSharedMemorySize, 220 * 1024));
        CPB_CUDA(cudaFuncSetAttribute(k_mult_t<Q_L1, 2>, cudaFuncAttributeMaxDynamicSharedMemorySize, 220 * 1024));
      }
      int per_sm = 0;
      CPB_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, k_mult_t<Q_L2, 2>, 32 * kMultWarps, smem));
      nb = std::max(1, std::min(cdiv(sel.count, kMultWarps), c.sm_count * std::max(1, per_sm)));
      const dim3 blk(32, kMultWarps);
      const int di = static_cast<int>(d);
      const int* ei = P.g->ei.p;
      const int* ej = P.g->ej.p;
      const double* wl = P.g->w.p;
      if (P.q == Q_L2 && VM == 1)
        k_mult_t<Q_L2, 1><<<nb, blk, smem, c.s>>>(X, Z, V, ps, thr, P.rad, wl, ei, ej, sel, di, sigma, pe, S);
      else if (P.q == Q_L2)
        k_mult_t<Q_L2, 2><<<nb, blk, smem, c.s>>>(X, Z, V, ps, thr, P.rad, wl, ei, ej, sel, di, sigma, pe, S);
      else if (VM == 1)
        k_mult_t<Q_L1, 1><<<nb, blk, smem, c.s>>>(X, Z, V, ps, thr, P.rad, wl, ei, ej, sel, di, sigma, pe, S);
      else
        k_mult_t<Q_L1, 2><<<nb, blk, smem, c.s>>>(X, Z, V, ps, thr, P.rad, wl, ei, ej, sel, di, sigma, pe, S);
      CPB_LAUNCH_CHECK();
    } else if (ge.gx == 32 && d <= kMultSmemMaxD && (P.q == Q_L2 || P.q == Q_L1)) {
      const size_t smem = static_cast<size_t>(kMultWarps) * 2 * d * sizeof(double);
      if (first_on_device("k_mult_s.smem")) {
        CPB_CUDA(cudaFuncSetAttribute(k_mult_s<Q_L2>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                      kMultWarps * 2 * kMultSmemMaxD * 8));
        CPB_CUDA(cudaFuncSetAttribute(k_mult_s<Q_L1>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                      kMultWarps * 2 * kMultSmemMaxD * 8));
      }
      int per_sm = 0;
      CPB_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, k_mult_s<Q_L2>, 32 * kMultWarps, smem));
      nb = std::max(1, std::min(cdiv(sel.count, kMultWarps), c.sm_count * std::max(1, per_sm)));
      if (P.q == Q_L2)
        k_mult_s<Q_L2><<<nb, dim3(32, kMultWarps), smem, c.s>>>(X, Z, V, ps, thr, P.rad, P.g->w.p, P.g->ei.p,
                                                                P.g->ej.p, sel, static_cast<int>(d), sigma, pe);
      else
        k_mult_s<Q_L1><<<nb, dim3(32, kMultWarps), smem, c.s>>>(X, Z, V, ps, thr, P.rad, P.g->w.p, P.g->ei.p,
                                                                P.g->ej.p, sel, static_cast<int>(d), sigma, pe);
      CPB_LAUNCH_CHECK();
    } else {
      k_mult<<<ge.grid, dim3(ge.gx, ge.gy), 0, c.s>>>(X, Z, V, ps, thr, P.rad, P.g->w.p, P.g->ei.p, P.g->ej.p, sel,
                                                      static_cast<int>(d), sigma, P.q, pe);
      CPB_LAUNCH_CHECK();
    }
    return nb;
  };
  int nb;
  {
    Ctx::Timer tm(&c, "multiplier", (3.0 * E * d + n * d) * 8.0);
    if (!partitioned(c)) {
      nb = run(EdgeSel{nullptr, 0, E}, pe);
    } else {  // ghost edges first (updated, never summed), then the owned range
      const EdgePart& ep = edge_part(c, *P.g);
      if (ep.nghost) run(EdgeSel{ep.ghost.p, 0, ep.nghost}, part_buf(c, "mult.pg", pe_n));
      nb = run(EdgeSel{nullptr, ep.e0, ep.e1 - ep.e0}, pe);
    }
  }
  std::vector<double> s = host_cols(c, pe, nb, 9, {6, 7, 8});
  if (partitioned(c)) comm_allreduce_host(c, s, {6, 7, 8});
  const double mx = s[6], err = s[7], excess = s[8];
  const double scale = 1.0 + mx;
  if (err > 1e-10 * scale) runtime("ssnal: multiplier self-check failed");
  if (excess > 0.0) invalid("dual_objective: Z violates the dual-ball constraint");
  // node terms at (X, new Z)
  double* pn = part_buf(c, "mult.pn", 4 * static_cast<size_t>(c.sm_count) * 16);
  int nbn;
  {
    Ctx::Timer tm(&c, "gap_node", (static_cast<double>(E) * d + 2.0 * n * d) * 8.0 + (2.0 * E + n + 1) * 4.0);  // Z once, X, A, CSR
    nbn = gather_gap(c, *P.g, X, P.A->A.p, Z, d, pn);
  }
  std::vector<double> h = host_cols(c, pn, nbn, 4);
  if (partitioned(c)) comm_allreduce_host(c, h);
  const double normA = data_fro_norm(c, *P.A);
  MultOut o;
  GapOut& g = o.gap;
  g.fp = 0.5 * h[0];
  if (P.gamma != 0.0) g.fp = g.fp + P.gamma * s[0];
  g.fd = -0.5 * h[1] + h[2];
  g.gap = std::abs(g.fp - g.fd) / (1.0 + std::abs(g.fp) + std::abs(g.fd));
  const double stat = std::sqrt(h[3]) / (1.0 + normA);
  const double align = std::sqrt(s[1]) / (1.0 + std::sqrt(s[2]) + std::sqrt(s[3]));
  g.kkt = (P.gamma == 0.0) ? stat : std::max(stat, align);
  o.feas = std::sqrt(s[4]) / (1.0 + std::sqrt(s[2]));
  o.zz = s[3];
  return o;
}

void ama_primal(const Prob& P, const double* Zh, double* Xh) {
  gather_a_minus_bt(*P.c, *P.g, P.A->A.p, Zh, P.d(), Xh);
}
void ama_dual_step(const Prob& P, const double* Xh, double* Zh, double* Zprev, double step, double mom,
                   const double* momp) {
  Ctx& c = *P.c;
  const int64_t d = P.d(), E = P.E();
  GroupGeom ge = group_geom(c, E, d);
  k_ama_edge<<<ge.grid, dim3(ge.gx, ge.gy), 0, c.s>>>(Xh, Zh, Zprev, P.rad, P.g->ei.p, P.g->ej.p, E,
                                                      static_cast<int>(d), step, mom, P.q, momp);
  CPB_LAUNCH_CHECK();
}

// Nesterov momenta of `cnt` consecutive AMA iterations (ama.cpp:66-70): t' = (1 + sqrt(1 + 4t^2)) / 2,
// mom = (t - 1) / t'.  tm[cnt] carries t across blocks.  Same operation order as the host loop and
// -fmad=false, so the values are bitwise the host's.
__global__ void k_ama_mom(double* tm, int cnt) {
  double t = tm[cnt];
  for (int j = 0; j < cnt; ++j) {
    const double tn = 0.5 * (1.0 + sqrt(1.0 + 4.0 * t * t));
    tm[j] = (t - 1.0) / tn;
    t = tn;
  }
  tm[cnt] = t;
}
__global__ void k_set1(double* p, double v) { *p = v; }
void ama_momenta(const Prob& P, double* tm, int cnt) {
  k_ama_mom<<<1, 1, 0, P.c->s>>>(tm, cnt);
  CPB_LAUNCH_CHECK();
}
int ama_block_fused(const Prob& P, double* Xh, double* Zh, double* Zp, double* Xout, double step, double t0,
                    int cnt, double** parts) {
  Ctx& c = *P.c;
  const int64_t d = P.d(), n = P.n(), E = P.E();
  if (d > 32 || E < 1 || E > (1 << 18) || n > (1 << 17) || partitioned(c)) return 0;
  GroupGeom ge = group_geom(c, E, d);
  int occ = 0;
  CPB_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, k_ama_block, 256, 0));
  if (occ < 1) return 0;
  const int64_t want = std::max<int64_t>(cdiv(n, 8), cdiv(E, ge.gy));
  const int grid = static_cast<int>(std::max<int64_t>(1, std::min<int64_t>(want, static_cast<int64_t>(c.sm_count))));
  const double* A = P.A->A.p;
  const int *ei = P.g->ei.p, *ej = P.g->ej.p, *off = P.g->off.p, *ae = P.g->adj_e.p, *ao = P.g->adj_o.p,
            *ord = P.g->order.p;
  const double* rad = P.rad;
  int dd = static_cast<int>(d), qq = P.q;
  const double* wt = P.g->w.p;
  double* part = part_buf(c, "ama.parts", 9 * static_cast<size_t>(grid));
  void* args[] = {(void*)&A,   (void*)&Xh,  (void*)&Zh, (void*)&Zp, (void*)&Xout, (void*)&rad, (void*)&ei,
                  (void*)&ej,  (void*)&off, (void*)&ae, (void*)&ao, (void*)&ord,  (void*)&n,   (void*)&E,
                  (void*)&dd,  (void*)&step, (void*)&qq, (void*)&t0, (void*)&cnt, (void*)&wt, (void*)&part};
  {
    Ctx::Timer tm(&c, "ama_block", static_cast<double>(cnt) * (5.0 * E * d + 3.0 * n * d) * 8.0);
    CPB_CUDA(cudaLaunchCooperativeKernel((const void*)k_ama_block, dim3(grid), dim3(ge.gx, ge.gy), args, 0, c.s));
    CPB_LAUNCH_CHECK();
  }
  *parts = part;
  return grid;
}
void ama_set_t(const Prob& P, double* tm, int cnt, double t) {
  k_set1<<<1, 1, 0, P.c->s>>>(tm + cnt, t);
  CPB_LAUNCH_CHECK();
}

}  // namespace cpb
