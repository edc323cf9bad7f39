// Node-CSR gather kernels (see gather.cuh).
//
// Work item = (node, feature chunk): one warp owns up to 32*NF consecutive
// features (lane l holds f = chunk0 + l + 32 k, k < NF) of one node and walks
// the node's incident edges in ascending id.  Edge metadata (id, other
// endpoint, per-edge scalars) is fetched 32 edges at a time with one
// coalesced load per lane and handed out by warp shuffles; feature rows are
// then loaded 4 edges x NF features at a time (all issued before use).  No
// block-wide barriers: warps never wait on each other, so a hub node only
// delays its own warps.  Items are enumerated hubs-first (descending degree).
// Per-(node, feature) accumulation order = ascending edge id = the reference's
// scatter order (graph.cpp:140-152), bitwise.
#include <cstdlib>

#include <algorithm>
#include <memory>
#include <string>
#include <vector>

#include "comm.cuh"
#include "gather.cuh"
#include "graph.cuh"

namespace cpb {

namespace {

constexpr int kEB = 4;  // edges per load batch
constexpr unsigned kFull = 0xffffffffu;

struct ChunkGeom {
  int nch;  // chunks per node
  int nf;   // features per lane
};
// Up to 32 * 6 features per warp.
inline ChunkGeom chunk_geom(int64_t d) {
  constexpr int nf_max = 6;
  const int nch = static_cast<int>((d + 32 * nf_max - 1) / (32 * nf_max));
  const int nf = static_cast<int>((d + 32 * nch - 1) / (32 * nch));
  return {nch, nf};
}

// Item loop: warp w of the grid takes items w, w + W, ... (static: the
// per-block partial sums are deterministic).
#define ITEMS_BEGIN(n, nch)                                                                               \
  const int lane = threadIdx.x & 31;                                                                      \
  const int64_t nitems_ = (n) * (nch);                                                                    \
  for (int64_t it_ = (blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x) >> 5; it_ < nitems_; \
       it_ += (static_cast<int64_t>(gridDim.x) * blockDim.x) >> 5) {                                      \
    const int v = order[it_ / (nch)];                                                                     \
    const int f0 = static_cast<int>(it_ % (nch)) * 32 * NF + lane;                                        \
    const int p0 = off[v], p1 = off[v + 1];                                                               \
    const int64_t base = static_cast<int64_t>(v) * d;

#define ITEMS_END }

// ---- Bᵀ-type gathers ------------------------------------------------------------------
// mode 0: out = sum z;  1: out = A - sum z;  2: out = A + sum (rho U - L)
template <int NF>
__global__ void __launch_bounds__(256) k_g_bt(const double* __restrict__ Z, const double* __restrict__ Z2,
                                              const double* __restrict__ A, double rho, const int* __restrict__ off,
                                              const int* __restrict__ adj_e, const int* __restrict__ adj_o,
                                              const int* __restrict__ order, int64_t n, int d, int nch, int mode,
                                              double* __restrict__ out) {
  ITEMS_BEGIN(n, nch)
  double acc[NF];
#pragma unroll
  for (int k = 0; k < NF; ++k) acc[k] = 0.0;
  for (int p = p0; p < p1; p += 32) {
    const int cnt = min(32, p1 - p);
    const int my_e = lane < cnt ? adj_e[p + lane] : 0;
    const int my_o = lane < cnt ? adj_o[p + lane] : 0;
    for (int u0 = 0; u0 < cnt; u0 += kEB) {
      int le[kEB];
      bool pl[kEB];
#pragma unroll
      for (int u = 0; u < kEB; ++u) {
        le[u] = __shfl_sync(kFull, my_e, (u0 + u) & 31);
        pl[u] = __shfl_sync(kFull, my_o, (u0 + u) & 31) > v;
      }
      double x[kEB][NF];
#pragma unroll
      for (int u = 0; u < kEB; ++u)
#pragma unroll
        for (int k = 0; k < NF; ++k) {
          const int f = f0 + 32 * k;
          x[u][k] = 0.0;
          if (u0 + u < cnt && f < d) {
            const int64_t i = static_cast<int64_t>(le[u]) * d + f;
            x[u][k] = (mode == 2) ? rho * __ldcs(Z + i) - __ldcs(Z2 + i) : __ldcs(Z + i);
          }
        }
#pragma unroll
      for (int u = 0; u < kEB; ++u)
        if (u0 + u < cnt)
#pragma unroll
          for (int k = 0; k < NF; ++k) acc[k] = pl[u] ? acc[k] + x[u][k] : acc[k] - x[u][k];
    }
  }
#pragma unroll
  for (int k = 0; k < NF; ++k) {
    const int f = f0 + 32 * k;
    if (f < d) out[base + f] = (mode == 0) ? acc[k] : (mode == 1 ? A[base + f] - acc[k] : A[base + f] + acc[k]);
  }
  ITEMS_END
}

// ---- (I + rho L) y and its (pAp, pp) block partials ----------------------------------------
template <int NF>
__global__ void __launch_bounds__(256) k_g_lap(const double* __restrict__ y, double rho, const int* __restrict__ off,
                                               const int* __restrict__ adj_o, const int* __restrict__ order, int64_t n,
                                               int d, int nch, double* __restrict__ out, double* part,
                                               const int* active) {
  if (active && !*active) return;
  __shared__ double sh[32];
  double s_a = 0.0, s_b = 0.0;
  ITEMS_BEGIN(n, nch)
  const double deg = static_cast<double>(p1 - p0);
  double nb[NF];
#pragma unroll
  for (int k = 0; k < NF; ++k) nb[k] = 0.0;
  for (int p = p0; p < p1; p += 32) {
    const int cnt = min(32, p1 - p);
    const int my_o = lane < cnt ? adj_o[p + lane] : 0;
    for (int u0 = 0; u0 < cnt; u0 += kEB) {
      int lo[kEB];
#pragma unroll
      for (int u = 0; u < kEB; ++u) lo[u] = __shfl_sync(kFull, my_o, (u0 + u) & 31);
      double x[kEB][NF];
#pragma unroll
      for (int u = 0; u < kEB; ++u)
#pragma unroll
        for (int k = 0; k < NF; ++k) {
          const int f = f0 + 32 * k;
          x[u][k] = (u0 + u < cnt && f < d) ? y[static_cast<int64_t>(lo[u]) * d + f] : 0.0;
        }
#pragma unroll
      for (int u = 0; u < kEB; ++u)
#pragma unroll
        for (int k = 0; k < NF; ++k) nb[k] += x[u][k];
    }
  }
  double a = 0.0, b = 0.0;
#pragma unroll
  for (int k = 0; k < NF; ++k) {
    const int f = f0 + 32 * k;
    if (f >= d) continue;
    const double yv = y[base + f];
    const double o = yv + rho * (deg * yv - nb[k]);
    out[base + f] = o;
    a += yv * o;
    b += yv * yv;
  }
  s_a += a;
  s_b += b;
  ITEMS_END
  s_a = block_sum(s_a, sh);
  s_b = block_sum(s_b, sh);
  if (threadIdx.x == 0) {
    part[2 * blockIdx.x] = s_a;
    part[2 * blockIdx.x + 1] = s_b;
  }
}

// ---- gap node terms (objective.cpp:76-88, :100-106) ---------------------------------------
// part[4b + k]: ||X - A||^2, ||Z Bᵀ||^2, <Z Bᵀ, A>, ||X - A + Z Bᵀ||^2
template <int NF>
__global__ void __launch_bounds__(256) k_g_gap(const double* __restrict__ X, const double* __restrict__ A,
                                               const double* __restrict__ Z, const int* __restrict__ off,
                                               const int* __restrict__ adj_e, const int* __restrict__ adj_o,
                                               const int* __restrict__ order, int64_t n, int d, int nch,
                                               double* part) {
  __shared__ double sh[32];
  double s[4] = {0, 0, 0, 0};
  ITEMS_BEGIN(n, nch)
  double acc[NF];
#pragma unroll
  for (int k = 0; k < NF; ++k) acc[k] = 0.0;
  for (int p = p0; p < p1; p += 32) {
    const int cnt = min(32, p1 - p);
    const int my_e = lane < cnt ? adj_e[p + lane] : 0;
    const int my_o = lane < cnt ? adj_o[p + lane] : 0;
    for (int u0 = 0; u0 < cnt; u0 += kEB) {
      int le[kEB];
      bool pl[kEB];
#pragma unroll
      for (int u = 0; u < kEB; ++u) {
        le[u] = __shfl_sync(kFull, my_e, (u0 + u) & 31);
        pl[u] = __shfl_sync(kFull, my_o, (u0 + u) & 31) > v;
      }
      double x[kEB][NF];
#pragma unroll
      for (int u = 0; u < kEB; ++u)
#pragma unroll
        for (int k = 0; k < NF; ++k) {
          const int f = f0 + 32 * k;
          x[u][k] = (u0 + u < cnt && f < d) ? __ldcs(Z + static_cast<int64_t>(le[u]) * d + f) : 0.0;
        }
#pragma unroll
      for (int u = 0; u < kEB; ++u)
        if (u0 + u < cnt)
#pragma unroll
          for (int k = 0; k < NF; ++k) acc[k] = pl[u] ? acc[k] + x[u][k] : acc[k] - x[u][k];
    }
  }
#pragma unroll
  for (int k = 0; k < NF; ++k) {
    const int f = f0 + 32 * k;
    if (f >= d) continue;
    const double a = A[base + f];
    const double xa = X[base + f] - a;
    const double st = xa + acc[k];
    s[0] += xa * xa;
    s[1] += acc[k] * acc[k];
    s[2] += acc[k] * a;
    s[3] += st * st;
  }
  ITEMS_END
#pragma unroll
  for (int k = 0; k < 4; ++k) {
    const double r = block_sum(s[k], sh);
    if (threadIdx.x == 0) part[4 * blockIdx.x + k] = r;
  }
}

__device__ __forceinline__ double softd(double v, double t) {
  return static_cast<double>((v > 0.0) - (v < 0.0)) * fmax(fabs(v) - t, 0.0);
}

// ---- SSNAL gradient + Jacobi diagonal (ssnal.cpp:41-44, :68-82) ---------------------------
template <int NF>
__global__ void __launch_bounds__(256) k_g_grad(const double* __restrict__ X, const double* __restrict__ A,
                                                const double* __restrict__ V, const double* __restrict__ ps,
                                                const double* __restrict__ jal, const double* __restrict__ jbe,
                                                const double* __restrict__ thr, const int* __restrict__ off,
                                                const int* __restrict__ adj_e, const int* __restrict__ adj_o,
                                                const int* __restrict__ order, int64_t n, int d, int nch,
                                                double sigma, int q, int want_diag, double* __restrict__ G,
                                                double* __restrict__ diag, double* part) {
  __shared__ double sh[32];
  double s_g = 0.0;
  ITEMS_BEGIN(n, nch)
  double ag[NF], ad[NF];
#pragma unroll
  for (int k = 0; k < NF; ++k) {
    ag[k] = 0.0;
    ad[k] = 1.0;
  }
  for (int p = p0; p < p1; p += 32) {
    const int cnt = min(32, p1 - p);
    const int my_e = lane < cnt ? adj_e[p + lane] : 0;
    const int my_o = lane < cnt ? adj_o[p + lane] : 0;
    // q = 0 (infinity): ps = theta, jbe = 1/|S| (k_jac)
    const double my_s = lane < cnt ? ((q == 2 || q == 0) ? ps[my_e] : thr[my_e]) : 0.0;
    const double my_a = (lane < cnt && q == 2) ? jal[my_e] : 0.0;
    const double my_b = (lane < cnt && (q == 2 || q == 0)) ? jbe[my_e] : 0.0;
    for (int u0 = 0; u0 < cnt; u0 += kEB) {
      int le[kEB];
      bool pl[kEB];
      double es[kEB], ea[kEB], eb[kEB];
#pragma unroll
      for (int u = 0; u < kEB; ++u) {
        const int src = (u0 + u) & 31;
        le[u] = __shfl_sync(kFull, my_e, src);
        pl[u] = __shfl_sync(kFull, my_o, src) > v;
        es[u] = __shfl_sync(kFull, my_s, src);
        ea[u] = __shfl_sync(kFull, my_a, src);
        eb[u] = __shfl_sync(kFull, my_b, src);
      }
      double x[kEB][NF];
#pragma unroll
      for (int u = 0; u < kEB; ++u)
#pragma unroll
        for (int k = 0; k < NF; ++k) {
          const int f = f0 + 32 * k;
          x[u][k] = (u0 + u < cnt && f < d) ? __ldcs(V + static_cast<int64_t>(le[u]) * d + f) : 0.0;
        }
#pragma unroll
      for (int u = 0; u < kEB; ++u) {
        if (u0 + u >= cnt) continue;
#pragma unroll
        for (int k = 0; k < NF; ++k) {
          const double val = x[u][k];
          double uu, jd;
          if (q == 2) {
            uu = val - es[u] * val;
            jd = ea[u] + (eb[u] != 0.0 ? eb[u] * val * val : 0.0);
          } else if (q == 0) {  // V - clamp(V, theta); diag M = 1/|S| on S, 1 off S, 0 inside
            const double th = es[u];
            uu = th < 0.0 ? val : softd(val, th);
            jd = th < 0.0 ? 0.0 : (fabs(val) > th ? eb[u] : 1.0);
          } else {
            uu = val - softd(val, es[u]);
            jd = fabs(val) > es[u] ? 1.0 : 0.0;
          }
          ag[k] = pl[u] ? ag[k] + uu : ag[k] - uu;
          ad[k] += sigma * (1.0 - jd);
        }
      }
    }
  }
#pragma unroll
  for (int k = 0; k < NF; ++k) {
    const int f = f0 + 32 * k;
    if (f >= d) continue;
    const double gv = (X[base + f] - A[base + f]) + sigma * ag[k];
    G[base + f] = gv;
    if (want_diag) diag[base + f] = ad[k];
    s_g += gv * gv;
  }
  ITEMS_END
  s_g = block_sum(s_g, sh);
  if (threadIdx.x == 0) part[blockIdx.x] = s_g;
}

// ---- SSNAL Hessian, pass 1: bc_l = beta_l <v_l, p_i - p_j> (warp per active edge) -----------
__global__ void __launch_bounds__(256) k_edge_dot(const double* __restrict__ P, const double* __restrict__ V,
                                                  const double* __restrict__ jbe, const int* __restrict__ ei,
                                                  const int* __restrict__ ej, const int* __restrict__ elist, int64_t e0, int64_t E, int d,
                                                  double* __restrict__ bc, const int* active) {
  if (active && !*active) return;
  const int lane = threadIdx.x & 31;
  for (int64_t i = (blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x) >> 5; i < E;
       i += (static_cast<int64_t>(gridDim.x) * blockDim.x) >> 5) {
    const int64_t l = elist ? static_cast<int64_t>(elist[i]) : e0 + i;  // an edge selection (see EdgeSel)
    const double be = jbe[l];
    if (be == 0.0) {
      if (lane == 0) bc[l] = 0.0;
      continue;
    }
    const double* pa = P + static_cast<int64_t>(ei[l]) * d;
    const double* pb = P + static_cast<int64_t>(ej[l]) * d;
    const double* vl = V + l * d;
    double c0 = 0.0, c1 = 0.0, c2 = 0.0, c3 = 0.0;
    if ((d & 1) == 0) {  // even d: 16-byte loads of feature pairs, two pairs per lane in flight
      const int h = d >> 1;
      const double2* v2 = reinterpret_cast<const double2*>(vl);
      const double2* a2 = reinterpret_cast<const double2*>(pa);
      const double2* b2 = reinterpret_cast<const double2*>(pb);
      int k = lane;
      for (; k + 32 < h; k += 64) {
        const double2 v0 = __ldcs(v2 + k), v1 = __ldcs(v2 + k + 32);
        const double2 x0 = a2[k], x1 = a2[k + 32], y0 = b2[k], y1 = b2[k + 32];
        c0 = __fma_rn(v0.x, x0.x - y0.x, c0);
        c1 = __fma_rn(v0.y, x0.y - y0.y, c1);
        c2 = __fma_rn(v1.x, x1.x - y1.x, c2);
        c3 = __fma_rn(v1.y, x1.y - y1.y, c3);
      }
      if (k < h) {
        const double2 v0 = __ldcs(v2 + k), x0 = a2[k], y0 = b2[k];
        c0 = __fma_rn(v0.x, x0.x - y0.x, c0);
        c1 = __fma_rn(v0.y, x0.y - y0.y, c1);
      }
      const double c = warp_sum((c0 + c1) + (c2 + c3));
      if (lane == 0) bc[l] = be * c;
      continue;
    }
    int f = lane;
    for (; f + 96 < d; f += 128) {
      const double v0 = __ldcs(vl + f), v1 = __ldcs(vl + f + 32), v2 = __ldcs(vl + f + 64), v3 = __ldcs(vl + f + 96);
      const double a0 = pa[f], a1 = pa[f + 32], a2 = pa[f + 64], a3 = pa[f + 96];
      const double b0 = pb[f], b1 = pb[f + 32], b2 = pb[f + 64], b3 = pb[f + 96];
      c0 = __fma_rn(v0, a0 - b0, c0);
      c1 = __fma_rn(v1, a1 - b1, c1);
      c2 = __fma_rn(v2, a2 - b2, c2);
      c3 = __fma_rn(v3, a3 - b3, c3);
    }
    for (; f < d; f += 32) c0 = __fma_rn(__ldcs(vl + f), pa[f] - pb[f], c0);
    const double c = warp_sum((c0 + c1) + (c2 + c3));
    if (lane == 0) bc[l] = be * c;
  }
}

// q = infinity: bc_l = <s_S, p_i - p_j> / |S| over S = {|v_f| > theta_l}
// (zero inside the ball, where (I - M) = I).
__global__ void __launch_bounds__(256) k_edge_dot_inf(const double* __restrict__ P, const double* __restrict__ V,
                                                      const double* __restrict__ jal, const double* __restrict__ jbe,
                                                      const int* __restrict__ ei, const int* __restrict__ ej,
                                                      const int* __restrict__ elist, int64_t e0, int64_t E, int d, double* __restrict__ bc, const int* active,
                                                      const unsigned* __restrict__ mask, const unsigned* __restrict__ sgn) {
  const int W = (d + 31) >> 5;
  if (active && !*active) return;
  const int lane = threadIdx.x & 31;
  for (int64_t i = (blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x) >> 5; i < E;
       i += (static_cast<int64_t>(gridDim.x) * blockDim.x) >> 5) {
    const int64_t l = elist ? static_cast<int64_t>(elist[i]) : e0 + i;  // an edge selection (see EdgeSel)
    const double th = jal[l], be = jbe[l];
    if (th < 0.0 || be == 0.0) {
      if (lane == 0) bc[l] = 0.0;
      continue;
    }
    const double* pa = P + static_cast<int64_t>(ei[l]) * d;
    const double* pb = P + static_cast<int64_t>(ej[l]) * d;
    const double* vl = V + l * d;
    double c = 0.0;
    if (mask) {  // S and sign(v) as bits (edge_masks): no V row read
      const unsigned* mw = mask + l * W;
      const unsigned* sw = sgn + l * W;
      for (int f = lane, k = 0; f < d; f += 32, ++k) {
        const unsigned bit = 1u << lane;
        if (mw[k] & bit) c += (sw[k] & bit) ? pa[f] - pb[f] : pb[f] - pa[f];
      }
    } else {
      for (int f = lane; f < d; f += 32) {
        const double vf = vl[f];
        if (fabs(vf) > th) c += vf > 0.0 ? pa[f] - pb[f] : pb[f] - pa[f];
      }
    }
    c = warp_sum(c);
    if (lane == 0) bc[l] = be * c;
  }
}

// ---- SSNAL Hessian, pass 2: node gather (ssnal.cpp:56-64) -----------------------------------
// Ap_v = p_v + sigma sum_l +-(w - (alpha w + bc v)),  w = p_i(l) - p_j(l).
// QT = the penalty q as a compile-time constant: 2 reads V_l for active edges; 1 and 0
// (q = inf) read the edge_masks bits instead and carry no V registers (C4: 245 -> fewer
// registers per thread, more warps in flight for the p gathers).
template <int NF, int QT>
__global__ void __launch_bounds__(256, QT == 2 ? 1 : 2) k_g_hess(const double* __restrict__ P, const double* __restrict__ V,
                                                const double* __restrict__ jal, const double* __restrict__ bc,
                                                const double* __restrict__ thr, const int* __restrict__ off,
                                                const int* __restrict__ adj_e, const int* __restrict__ adj_o,
                                                const int* __restrict__ order, int64_t n, int d, int nch,
                                                double sigma, int q_unused, double* __restrict__ Ap, double* part,
                                                const int* active, const unsigned* __restrict__ mask,
                                                const unsigned* __restrict__ sgn) {
  constexpr int q = QT;
  constexpr int EB = QT == 2 ? kEB : 2;  // edges per load batch (mask variants: 2, for 2 blocks per SM)
  (void)q_unused;
  if (active && !*active) return;
  __shared__ double sh[32];
  double s_a = 0.0, s_b = 0.0;
  const int W = (d + 31) >> 5;
  ITEMS_BEGIN(n, nch)
  const int w0 = static_cast<int>(it_ % nch) * NF;  // word of feature f0 + 32 k is w0 + k (bit = lane)
  const unsigned lbit = 1u << lane;
  double pv[NF], acc[NF];
  double diag_coef = 0.0;  // sum over incident edges of (1 - alpha_l), q = 2
#pragma unroll
  for (int k = 0; k < NF; ++k) {
    const int f = f0 + 32 * k;
    pv[k] = f < d ? P[base + f] : 0.0;
    acc[k] = 0.0;
  }
  for (int p = p0; p < p1; p += 32) {
    const int cnt = min(32, p1 - p);
    const int my_e = lane < cnt ? adj_e[p + lane] : 0;
    const int my_o = lane < cnt ? adj_o[p + lane] : v;
    const double my_a = lane < cnt ? ((q == 2 || q == 0) ? jal[my_e] : thr[my_e]) : 0.0;
    const double my_b = (lane < cnt && (q == 2 || q == 0)) ? bc[my_e] : 0.0;
    for (int u0 = 0; u0 < cnt; u0 += EB) {
      int le[EB], lo[EB];
      double ea[EB], eb[EB];
#pragma unroll
      for (int u = 0; u < EB; ++u) {
        const int src = (u0 + u) & 31;
        le[u] = __shfl_sync(kFull, my_e, src);
        lo[u] = __shfl_sync(kFull, my_o, src);
        ea[u] = __shfl_sync(kFull, my_a, src);
        eb[u] = __shfl_sync(kFull, my_b, src);
      }
      constexpr int VE = QT == 2 ? EB : 1, ME = QT == 2 ? 1 : EB, SE = QT == 0 ? EB : 1;
      double po[EB][NF], vv[VE][NF];
      unsigned mb[ME][NF], sb[SE][NF];  // q = 1 / inf: S membership and sign bits (edge_masks)
#pragma unroll
      for (int u = 0; u < EB; ++u) {
        const bool ok = u0 + u < cnt;
#pragma unroll
        for (int k = 0; k < NF; ++k) {
          const int f = f0 + 32 * k;
          po[u][k] = (ok && f < d) ? __ldg(P + static_cast<int64_t>(lo[u]) * d + f) : 0.0;
          if constexpr (QT == 2)
            vv[u][k] = (ok && eb[u] != 0.0 && f < d) ? __ldcs(V + static_cast<int64_t>(le[u]) * d + f) : 0.0;
          else
            mb[u][k] = (ok && f < d) ? mask[static_cast<int64_t>(le[u]) * W + w0 + k] : 0u;
          if constexpr (QT == 0) sb[u][k] = (ok && f < d) ? sgn[static_cast<int64_t>(le[u]) * W + w0 + k] : 0u;
        }
      }
      if (q == 2) {
        // Sign-free form: the edge adds (1 - alpha)(p_v - p_o) - s bc v_l to node v
        // (s = +1 when v is the smaller endpoint); the p_v part is summed as a
        // scalar, the rest is two FMAs per feature.
#pragma unroll
        for (int u = 0; u < EB; ++u) {
          if (u0 + u >= cnt) continue;
          const double ca = 1.0 - ea[u];
          const double cb = (lo[u] > v) ? eb[u] : -eb[u];
          diag_coef += ca;
#pragma unroll
          for (int k = 0; k < NF; ++k) {
            acc[k] = __fma_rn(-ca, po[u][k], acc[k]);
            if constexpr (QT == 2)
              if (cb != 0.0) acc[k] = __fma_rn(-cb, vv[u][k], acc[k]);
          }
        }
      } else if (q == 0) {  // (I - M) w = 1_S (w - s bc), identity inside the ball
#pragma unroll
        for (int u = 0; u < EB; ++u) {
          if (u0 + u >= cnt) continue;
          const bool plus = lo[u] > v;
          const double th = ea[u];
#pragma unroll
          for (int k = 0; k < NF; ++k) {
            const double w = plus ? pv[k] - po[u][k] : po[u][k] - pv[k];
            bool in_s = false, pos = false;
            if constexpr (QT == 0) {
              in_s = (mb[u][k] & lbit) != 0u;
              pos = (sb[u][k] & lbit) != 0u;
            }
            const double y = th < 0.0 ? w : (in_s ? w - (pos ? eb[u] : -eb[u]) : 0.0);
            acc[k] = plus ? acc[k] + y : acc[k] - y;
          }
        }
      } else {
#pragma unroll
        for (int u = 0; u < EB; ++u) {
          if (u0 + u >= cnt) continue;
          const bool plus = lo[u] > v;
#pragma unroll
          for (int k = 0; k < NF; ++k) {
            const double w = plus ? pv[k] - po[u][k] : po[u][k] - pv[k];
            bool act = false;
            if constexpr (QT == 1) act = (mb[u][k] & lbit) != 0u;
            const double y = w - (act ? w : 0.0);
            acc[k] = plus ? acc[k] + y : acc[k] - y;
          }
        }
      }
    }
  }
#pragma unroll
  for (int k = 0; k < NF; ++k) {
    const int f = f0 + 32 * k;
    if (f >= d) continue;
    if (q == 2) acc[k] = __fma_rn(diag_coef, pv[k], acc[k]);
    const double o = pv[k] + sigma * acc[k];
    Ap[base + f] = o;
    s_a += pv[k] * o;
    s_b += pv[k] * pv[k];
  }
  ITEMS_END
  s_a = block_sum(s_a, sh);
  s_b = block_sum(s_b, sh);
  if (threadIdx.x == 0) {
    part[2 * blockIdx.x] = s_a;
    part[2 * blockIdx.x + 1] = s_b;
  }
}


template <int NF>
constexpr auto k_g_hess2 = k_g_hess<NF, 2>;
template <int NF>
constexpr auto k_g_hess1 = k_g_hess<NF, 1>;
template <int NF>
constexpr auto k_g_hess0 = k_g_hess<NF, 0>;

// ---- single-pass Hessian for short rows (q = 2, even d <= 256) --------------------------
// One warp per node; lane l holds the feature pairs 2(l + 32k), k < NP, as
// double2.  Per batch of kEB incident edges it loads p_other and v_l (16-byte
// loads, all in flight together), forms the kEB dots <v_l, p_v - p_o> with
// interleaved butterfly reductions and adds (1 - alpha) w - beta c v_l.  This
// replaces the two-pass path (k_edge_dot + k_g_hess), which read V three times
// and gathered every p row four times, by one pass that reads V once per
// endpoint.
template <int NP>
__global__ void __launch_bounds__(256, NP == 1 ? 3 : 1) k_hess_warp(const double* __restrict__ P, const double* __restrict__ V,
                                                   const double* __restrict__ jal, const double* __restrict__ jbe,
                                                   const int* __restrict__ off, const int* __restrict__ adj_e,
                                                   const int* __restrict__ adj_o, const int* __restrict__ order,
                                                   int64_t n, int d, double sigma, double* __restrict__ Ap,
                                                   double* part, const int* active, const int* __restrict__ wl) {
  if (active && !*active) return;
  __shared__ double sh[32];
  const int lane = threadIdx.x & 31;
  const int h = d >> 1;  // double2 per row
  // node lists per warp (wl: offsets, then node ids) or a grid-stride walk of `order`
  const int64_t wid = (blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x) >> 5;
  const int64_t nwarps = (static_cast<int64_t>(gridDim.x) * blockDim.x) >> 5;
  const int64_t j0 = wl ? wl[wid] : wid, j1 = wl ? wl[wid + 1] : n, jstep = wl ? 1 : nwarps;
  const double2* P2 = reinterpret_cast<const double2*>(P);
  const double2* V2 = reinterpret_cast<const double2*>(V);
  double s_a = 0.0, s_b = 0.0;
  for (int64_t jt = j0; jt < j1; jt += jstep) {
    const int v = wl ? wl[jt] : order[jt];
    const int p0 = off[v], p1 = off[v + 1];
    const int64_t base = static_cast<int64_t>(v) * h;
    double2 pv[NP], acc[NP];
#pragma unroll
    for (int k = 0; k < NP; ++k) {
      const int j = lane + 32 * k;
      pv[k] = j < h ? P2[base + j] : make_double2(0.0, 0.0);
      acc[k] = make_double2(0.0, 0.0);
    }
    double dsum = 0.0;  // sum of (1 - alpha) over edges with beta = 0 (their p_v part)
    for (int p = p0; p < p1; p += 32) {
      const int cnt = min(32, p1 - p);
      const int my_e = lane < cnt ? adj_e[p + lane] : 0;
      const int my_o = lane < cnt ? adj_o[p + lane] : v;
      const double my_a = lane < cnt ? 1.0 - jal[my_e] : 0.0;
      const double my_b = lane < cnt ? jbe[my_e] : 0.0;
      for (int u0 = 0; u0 < cnt; u0 += kEB) {
        int le[kEB], lo[kEB];
        double ca[kEB], be[kEB];
#pragma unroll
        for (int u = 0; u < kEB; ++u) {
          const int src = (u0 + u) & 31;
          le[u] = __shfl_sync(kFull, my_e, src);
          lo[u] = __shfl_sync(kFull, my_o, src);
          ca[u] = __shfl_sync(kFull, my_a, src);
          be[u] = __shfl_sync(kFull, my_b, src);
        }
        double2 po[kEB][NP], vv[kEB][NP];
#pragma unroll
        for (int u = 0; u < kEB; ++u) {
          const bool ok = u0 + u < cnt;
          const bool nv = ok && be[u] != 0.0;
#pragma unroll
          for (int k = 0; k < NP; ++k) {
            const int j = lane + 32 * k;
            po[u][k] = (ok && j < h) ? __ldg(P2 + static_cast<int64_t>(lo[u]) * h + j) : make_double2(0.0, 0.0);
            vv[u][k] = (nv && j < h) ? __ldcs(V2 + static_cast<int64_t>(le[u]) * h + j) : make_double2(0.0, 0.0);
          }
        }
        double cu[kEB];
#pragma unroll
        for (int u = 0; u < kEB; ++u) {
          double c0 = 0.0, c1 = 0.0;
#pragma unroll
          for (int k = 0; k < NP; ++k) {
            c0 = __fma_rn(vv[u][k].x, pv[k].x - po[u][k].x, c0);
            c1 = __fma_rn(vv[u][k].y, pv[k].y - po[u][k].y, c1);
          }
          cu[u] = c0 + c1;
        }
#pragma unroll
        for (int o = 16; o > 0; o >>= 1)
#pragma unroll
          for (int u = 0; u < kEB; ++u) cu[u] += __shfl_xor_sync(kFull, cu[u], o);
#pragma unroll
        for (int u = 0; u < kEB; ++u) {
          if (u0 + u >= cnt) continue;
          if (be[u] != 0.0) {
            const double bc = be[u] * cu[u];
#pragma unroll
            for (int k = 0; k < NP; ++k) {
              acc[k].x = __fma_rn(ca[u], pv[k].x - po[u][k].x, __fma_rn(-bc, vv[u][k].x, acc[k].x));
              acc[k].y = __fma_rn(ca[u], pv[k].y - po[u][k].y, __fma_rn(-bc, vv[u][k].y, acc[k].y));
            }
          } else {
            dsum += ca[u];
#pragma unroll
            for (int k = 0; k < NP; ++k) {
              acc[k].x = __fma_rn(-ca[u], po[u][k].x, acc[k].x);
              acc[k].y = __fma_rn(-ca[u], po[u][k].y, acc[k].y);
            }
          }
        }
      }
    }
#pragma unroll
    for (int k = 0; k < NP; ++k) {
      const int j = lane + 32 * k;
      if (j >= h) continue;
      double2 o;
      o.x = pv[k].x + sigma * __fma_rn(dsum, pv[k].x, acc[k].x);
      o.y = pv[k].y + sigma * __fma_rn(dsum, pv[k].y, acc[k].y);
      reinterpret_cast<double2*>(Ap)[base + j] = o;
      s_a += pv[k].x * o.x + pv[k].y * o.y;
      s_b += pv[k].x * pv[k].x + pv[k].y * pv[k].y;
    }
  }
  s_a = block_sum(s_a, sh);
  s_b = block_sum(s_b, sh);
  if (threadIdx.x == 0) {
    part[2 * blockIdx.x] = s_a;
    part[2 * blockIdx.x + 1] = s_b;
  }
}

#define NF_DISPATCH(nf, KERNEL, ...)           \
  switch (nf) {                                \
    case 1: KERNEL<1> __VA_ARGS__; break;      \
    case 2: KERNEL<2> __VA_ARGS__; break;      \
    case 3: KERNEL<3> __VA_ARGS__; break;      \
    case 4: KERNEL<4> __VA_ARGS__; break;      \
    case 5: KERNEL<5> __VA_ARGS__; break;      \
    default: KERNEL<6> __VA_ARGS__; break;     \
  }

}  // namespace

NodeGeom node_geom(Ctx& c, int64_t n, int64_t d) {
  const ChunkGeom cg = chunk_geom(d);
  NodeGeom g;
  g.gx = 256;
  g.gy = cg.nch;  // chunks per node
  g.nf = cg.nf;
  const int64_t warps = n * cg.nch;
  g.grid = std::max(1, std::min(cdiv(warps, 8), c.sm_count * 8));
  return g;
}

#define GEOM                                 \
  NodeGeom ng = node_geom(c, g.n, d);        \
  const int di = static_cast<int>(d);        \
  const int nch = ng.gy;

// Partitioned PCG (c.own_v1 >= 0): the gather visits only this rank's nodes,
// in the graph's degree order; cached per (graph, range).
struct OwnOrder {
  uint64_t uid = 0;
  int64_t v0 = 0, v1 = -1, count = 0;
  DBuf<int> order;
};
const OwnOrder& own_order(Ctx& c, const Graph& g) {
  static thread_local std::vector<std::unique_ptr<OwnOrder>> cache;
  for (auto& o : cache)
    if (o->uid == g.uid && o->v0 == c.own_v0 && o->v1 == c.own_v1) return *o;
  auto o = std::make_unique<OwnOrder>();
  o->uid = g.uid, o->v0 = c.own_v0, o->v1 = c.own_v1;
  std::vector<int> all(static_cast<size_t>(g.n)), mine;
  if (g.n) d2h(c, all.data(), g.order.p, all.size() * sizeof(int));
  for (int v : all)
    if (v >= c.own_v0 && v < c.own_v1) mine.push_back(v);
  o->count = static_cast<int64_t>(mine.size());
  o->order.resize(mine.size() + 1);
  if (!mine.empty()) h2d(c, o->order.p, mine.data(), mine.size() * sizeof(int));
  c.sync();
  if (cache.size() > 8) cache.erase(cache.begin());
  cache.push_back(std::move(o));
  return *cache.back();
}

// Work items of the node gathers: every node, or this rank's in a partitioned solve.
struct Items {
  const int* order;
  int64_t count;
};
Items node_items(Ctx& c, const Graph& g) {
  if (c.own_v1 < 0) return {g.order.p, g.n};
  const OwnOrder& o = own_order(c, g);
  return {o.order.p, o.count};
}

const HaloPlan& halo_plan(Ctx& c, const Graph& g) {
  static thread_local std::vector<std::unique_ptr<HaloPlan>> cache;
  const int P = c.comm ? c.comm->nranks : 1;
  for (auto& h : cache)
    if (h->uid == g.uid && h->v0 == c.own_v0 && h->v1 == c.own_v1 && h->nranks == P) return *h;
  auto h = std::make_unique<HaloPlan>();
  h->uid = g.uid, h->v0 = c.own_v0, h->v1 = c.own_v1, h->nranks = P;
  const int64_t n = g.n, chunk = (n + P - 1) / P;
  auto owner = [&](int v) { return static_cast<int>(v / chunk); };
  std::vector<int> off(static_cast<size_t>(n) + 1), adj(static_cast<size_t>(2 * g.E));
  d2h(c, off.data(), g.off.p, off.size() * sizeof(int));
  if (g.E) d2h(c, adj.data(), g.adj_o.p, adj.size() * sizeof(int));
  const int me = c.comm ? c.comm->rank : 0;
  std::vector<std::vector<int>> send(static_cast<size_t>(P)), recv(static_cast<size_t>(P));
  for (int64_t v = c.own_v0; v < c.own_v1; ++v)
    for (int e = off[v]; e < off[v + 1]; ++e) {
      const int o = adj[static_cast<size_t>(e)], s = owner(o);
      if (s == me) continue;
      send[static_cast<size_t>(s)].push_back(static_cast<int>(v));  // s gathers v
      recv[static_cast<size_t>(s)].push_back(o);                     // this rank gathers o
    }
  std::vector<int> si, ri;
  h->send_off.push_back(0);
  h->recv_off.push_back(0);
  for (int s = 0; s < P; ++s) {
    auto& a = send[static_cast<size_t>(s)];
    auto& b = recv[static_cast<size_t>(s)];
    std::sort(a.begin(), a.end());
    a.erase(std::unique(a.begin(), a.end()), a.end());
    std::sort(b.begin(), b.end());
    b.erase(std::unique(b.begin(), b.end()), b.end());
    si.insert(si.end(), a.begin(), a.end());
    ri.insert(ri.end(), b.begin(), b.end());
    h->send_off.push_back(static_cast<int64_t>(si.size()));
    h->recv_off.push_back(static_cast<int64_t>(ri.size()));
  }
  h->nsend = static_cast<int64_t>(si.size());
  h->nrecv = static_cast<int64_t>(ri.size());
  h->send_idx.resize(si.size() + 1);
  h->recv_idx.resize(ri.size() + 1);
  if (!si.empty()) h2d(c, h->send_idx.p, si.data(), si.size() * sizeof(int));
  if (!ri.empty()) h2d(c, h->recv_idx.p, ri.data(), ri.size() * sizeof(int));
  c.sync();
  if (cache.size() > 8) cache.erase(cache.begin());
  cache.push_back(std::move(h));
  return *cache.back();
}

__global__ void k_rows_pack(const double* __restrict__ src, const int* __restrict__ idx, int64_t rows, int d,
                            double* __restrict__ dst) {
  const int64_t total = rows * d;
  for (int64_t t = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; t < total;
       t += static_cast<int64_t>(gridDim.x) * blockDim.x) {
    const int64_t r = t / d, f = t % d;
    dst[t] = src[static_cast<int64_t>(idx[r]) * d + f];
  }
}
__global__ void k_rows_unpack(const double* __restrict__ src, const int* __restrict__ idx, int64_t rows, int d,
                              double* __restrict__ dst) {
  const int64_t total = rows * d;
  for (int64_t t = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; t < total;
       t += static_cast<int64_t>(gridDim.x) * blockDim.x) {
    const int64_t r = t / d, f = t % d;
    dst[static_cast<int64_t>(idx[r]) * d + f] = src[t];
  }
}

void halo_exchange(Ctx& c, const Graph& g, double* p, int64_t d) {
  if (!c.comm || c.comm->nranks == 1) return;
  const HaloPlan& h = halo_plan(c, g);
  double* sbuf = c.buf<double>("halo.send", static_cast<size_t>(h.nsend * d) + 1);
  double* rbuf = c.buf<double>("halo.recv", static_cast<size_t>(h.nrecv * d) + 1);
  if (h.nsend) {
    k_rows_pack<<<std::max(1, std::min(cdiv(h.nsend * d, 256), c.sm_count * 8)), 256, 0, c.s>>>(
        p, h.send_idx.p, h.nsend, static_cast<int>(d), sbuf);
    CPB_LAUNCH_CHECK();
  }
  comm_exchange(c, sbuf, h.send_off, rbuf, h.recv_off, d);
  if (h.nrecv) {
    k_rows_unpack<<<std::max(1, std::min(cdiv(h.nrecv * d, 256), c.sm_count * 8)), 256, 0, c.s>>>(
        rbuf, h.recv_idx.p, h.nrecv, static_cast<int>(d), p);
    CPB_LAUNCH_CHECK();
  }
}

const EdgePart& edge_part(Ctx& c, const Graph& g) {
  static thread_local std::vector<std::unique_ptr<EdgePart>> cache;
  const int P = c.comm ? c.comm->nranks : 1;
  for (auto& e : cache)
    if (e->uid == g.uid && e->v0 == c.own_v0 && e->v1 == c.own_v1 && e->nranks == P) return *e;
  auto e = std::make_unique<EdgePart>();
  e->uid = g.uid, e->v0 = c.own_v0, e->v1 = c.own_v1, e->nranks = P;
  std::vector<int> ei(static_cast<size_t>(g.E)), ej(static_cast<size_t>(g.E));
  if (g.E) {
    d2h(c, ei.data(), g.ei.p, ei.size() * sizeof(int));
    d2h(c, ej.data(), g.ej.p, ej.size() * sizeof(int));
  }
  auto first_at_least = [&](int64_t v) {  // edges are sorted by (i, j): the owned ones are contiguous
    return static_cast<int64_t>(std::lower_bound(ei.begin(), ei.end(), static_cast<int>(std::min<int64_t>(v, g.n))) -
                                ei.begin());
  };
  const int64_t chunk = (g.n + P - 1) / P;
  for (int q = 0; q < P; ++q) {
    const int64_t a = first_at_least(std::min<int64_t>(g.n, chunk * q));
    const int64_t b = first_at_least(std::min<int64_t>(g.n, chunk * (q + 1)));
    e->row0.push_back(a);
    e->rows.push_back(b - a);
  }
  e->e0 = first_at_least(c.own_v0);
  e->e1 = first_at_least(c.own_v1);
  std::vector<int> ghost;  // edges into an owned node from a lower-id node of another rank
  for (int64_t l = 0; l < e->e0; ++l)
    if (ej[static_cast<size_t>(l)] >= c.own_v0 && ej[static_cast<size_t>(l)] < c.own_v1)
      ghost.push_back(static_cast<int>(l));
  e->nghost = static_cast<int64_t>(ghost.size());
  e->ghost.resize(ghost.size() + 1);
  if (!ghost.empty()) h2d(c, e->ghost.p, ghost.data(), ghost.size() * sizeof(int));
  c.sync();
  if (cache.size() > 8) cache.erase(cache.begin());
  cache.push_back(std::move(e));
  return *cache.back();
}

void gather_bt(Ctx& c, const Graph& g, const double* Z, int64_t d, double* out) {
  if (g.n == 0 || d == 0) return;
  GEOM
  NF_DISPATCH(ng.nf, k_g_bt, <<<ng.grid, 256, 0, c.s>>>(Z, nullptr, nullptr, 0.0, g.off.p, g.adj_e.p, g.adj_o.p,
                                                         g.order.p, g.n, di, nch, 0, out));
  CPB_LAUNCH_CHECK();
}

void gather_a_minus_bt(Ctx& c, const Graph& g, const double* A, const double* Zh, int64_t d, double* Xh) {
  if (g.n == 0 || d == 0) return;
  GEOM
  NF_DISPATCH(ng.nf, k_g_bt, <<<ng.grid, 256, 0, c.s>>>(Zh, nullptr, A, 0.0, g.off.p, g.adj_e.p, g.adj_o.p,
                                                         g.order.p, g.n, di, nch, 1, Xh));
  CPB_LAUNCH_CHECK();
}

void gather_admm_rhs(Ctx& c, const Graph& g, const double* A, const double* U, const double* L, double rho,
                     int64_t d, double* R) {
  if (g.n == 0 || d == 0) return;
  GEOM
  NF_DISPATCH(ng.nf, k_g_bt, <<<ng.grid, 256, 0, c.s>>>(U, L, A, rho, g.off.p, g.adj_e.p, g.adj_o.p, g.order.p, g.n,
                                                         di, nch, 2, R));
  CPB_LAUNCH_CHECK();
}

int gather_lap(Ctx& c, const Graph& g, const double* y, double rho, int64_t d, double* out, double* part,
               const int* active) {
  GEOM
  NF_DISPATCH(ng.nf, k_g_lap, <<<ng.grid, 256, 0, c.s>>>(y, rho, g.off.p, g.adj_o.p, g.order.p, g.n, di, nch, out,
                                                          part, active));
  CPB_LAUNCH_CHECK();
  return ng.grid;
}

int gather_gap(Ctx& c, const Graph& g, const double* X, const double* A, const double* Z, int64_t d, double* part) {
  GEOM
  const Items it = node_items(c, g);
  NF_DISPATCH(ng.nf, k_g_gap, <<<ng.grid, 256, 0, c.s>>>(X, A, Z, g.off.p, g.adj_e.p, g.adj_o.p, it.order, it.count,
                                                          di, nch, part));
  CPB_LAUNCH_CHECK();
  return ng.grid;
}

int gather_grad_diag(Ctx& c, const Graph& g, const double* X, const double* A, const double* V, const double* ps,
                     const double* jal, const double* jbe, const double* thr, int64_t d, double sigma, int q,
                     bool want_diag, double* G, double* diag, double* part) {
  GEOM
  const Items it = node_items(c, g);
  NF_DISPATCH(ng.nf, k_g_grad, <<<ng.grid, 256, 0, c.s>>>(X, A, V, ps, jal, jbe, thr, g.off.p, g.adj_e.p, g.adj_o.p,
                                                           it.order, it.count, di, nch, sigma, q, want_diag ? 1 : 0,
                                                           G, diag, part));
  CPB_LAUNCH_CHECK();
  return ng.grid;
}

// Per-edge feature bits of the q = 1 / q = inf generalized Jacobian, built once per
// Newton system from V (one coalesced pass, warp ballots): mask bit f = [|v_f| > t]
// (q = 1) or [|v_f| > theta] (q = inf), sgn bit f = [v_f > 0].  The Hessian's gathers
// then read 2 bits per feature instead of the 8-byte V element (same decisions, bitwise).
__global__ void __launch_bounds__(256) k_edge_masks(const double* __restrict__ V, const double* __restrict__ thr,
                                                    int64_t E, int d, int q, unsigned* __restrict__ mask,
                                                    unsigned* __restrict__ sgn) {
  const int lane = threadIdx.x & 31, W = (d + 31) >> 5;
  for (int64_t l = (blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x) >> 5; l < E;
       l += (static_cast<int64_t>(gridDim.x) * blockDim.x) >> 5) {
    const double t = thr[l];
    const double* v = V + l * d;
    for (int k = 0; k < W; ++k) {
      const int f = 32 * k + lane;
      const double vf = f < d ? __ldcs(v + f) : 0.0;
      const unsigned m = __ballot_sync(kFull, f < d && fabs(vf) > t);
      const unsigned sg = __ballot_sync(kFull, f < d && vf > 0.0);
      if (lane == 0) {
        mask[l * W + k] = m;
        sgn[l * W + k] = sg;
      }
    }
  }
}

void edge_masks(Ctx& c, const Graph& g, const double* V, const double* thr, int64_t d, int q, unsigned* mask,
                unsigned* sgn) {
  if (g.E == 0) return;
  const int grid = std::max(1, std::min(cdiv(g.E, 8), c.sm_count * 8));
  Ctx::Timer tm(&c, "edge_masks", (static_cast<double>(g.E) * d + g.E) * 8.0 + 2.0 * g.E * ((d + 31) / 32) * 4.0);
  k_edge_masks<<<grid, 256, 0, c.s>>>(V, thr, g.E, static_cast<int>(d), q, mask, sgn);
  CPB_LAUNCH_CHECK();
}

int hess_two_pass(Ctx& c, const Graph& g, const double* P, const double* V, const double* jal, const double* jbe,
                  const double* thr, int64_t d, double sigma, int q, double* bc, double* Ap, double* part,
                  const int* active, const unsigned* mask, const unsigned* sgn) {
  if (q == 2 && g.E > 0 && hess_tma_supported(d)) return hess_tma(c, g, P, V, jal, jbe, d, sigma, Ap, part, active);
  if (q == 2 && g.E > 0 && d % 2 == 0 && d <= 192) {
    const int np = static_cast<int>((d / 2 + 31) / 32);
    const int* ord = g.order.p;
    int64_t items = g.n;
    int grid = std::max(1, std::min(cdiv(g.n, 8), c.sm_count * 8));
    if (c.own_v1 >= 0) {  // partitioned PCG: this rank's nodes, the same grid on every rank
      const OwnOrder& o = own_order(c, g);
      ord = o.order.p, items = o.count, grid = c.sm_count * 8;
    }
    const int* wl = nullptr;  // degree-descending grid-stride walk (node lists measured 1.5-2x slower at C5)
    const int di = static_cast<int>(d);
    switch (np) {
      case 1: k_hess_warp<1><<<grid, 256, 0, c.s>>>(P, V, jal, jbe, g.off.p, g.adj_e.p, g.adj_o.p, ord, items, di,
                                                   sigma, Ap, part, active, wl); break;
      case 2: k_hess_warp<2><<<grid, 256, 0, c.s>>>(P, V, jal, jbe, g.off.p, g.adj_e.p, g.adj_o.p, ord, items, di,
                                                   sigma, Ap, part, active, wl); break;
      default: k_hess_warp<3><<<grid, 256, 0, c.s>>>(P, V, jal, jbe, g.off.p, g.adj_e.p, g.adj_o.p, ord, items, di,
                                                    sigma, Ap, part, active, wl); break;
    }
    CPB_LAUNCH_CHECK();
    return grid;
  }
  if ((q == 2 || q == 0) && g.E > 0) {
    // per-edge dots: every edge, or in a partitioned solve this rank's owned + ghost edges
    auto dots = [&](const int* list, int64_t e0, int64_t cnt) {
      if (cnt == 0) return;
      const int grid = std::max(1, std::min(cdiv(cnt, 8), c.sm_count * 8));
      if (q == 2)
        k_edge_dot<<<grid, 256, 0, c.s>>>(P, V, jbe, g.ei.p, g.ej.p, list, e0, cnt, static_cast<int>(d), bc, active);
      else
        k_edge_dot_inf<<<grid, 256, 0, c.s>>>(P, V, jal, jbe, g.ei.p, g.ej.p, list, e0, cnt, static_cast<int>(d), bc,
                                              active, mask, sgn);
      CPB_LAUNCH_CHECK();
    };
    if (c.comm && c.own_v1 >= 0) {
      const EdgePart& ep = edge_part(c, g);
      dots(nullptr, ep.e0, ep.e1 - ep.e0);
      dots(ep.ghost.p, 0, ep.nghost);
    } else {
      dots(nullptr, 0, g.E);
    }
  }
  GEOM
  const int* ord = g.order.p;
  int64_t items = g.n;
  int grid = ng.grid;
  if (c.own_v1 >= 0) {  // partitioned PCG: this rank's nodes, the same grid on every rank
    const OwnOrder& o = own_order(c, g);
    ord = o.order.p, items = o.count, grid = c.sm_count * 8;
  }
  if (q != 2 && !mask) invalid("hessian: q = 1 / inf needs the edge_masks bits");
  if (q == 2) {
    NF_DISPATCH(ng.nf, k_g_hess2, <<<grid, 256, 0, c.s>>>(P, V, jal, bc, thr, g.off.p, g.adj_e.p, g.adj_o.p, ord,
                                                           items, di, nch, sigma, q, Ap, part, active, nullptr,
                                                           nullptr));
  } else if (q == 1) {
    NF_DISPATCH(ng.nf, k_g_hess1, <<<grid, 256, 0, c.s>>>(P, V, jal, bc, thr, g.off.p, g.adj_e.p, g.adj_o.p, ord,
                                                           items, di, nch, sigma, q, Ap, part, active, mask, sgn));
  } else {
    NF_DISPATCH(ng.nf, k_g_hess0, <<<grid, 256, 0, c.s>>>(P, V, jal, bc, thr, g.off.p, g.adj_e.p, g.adj_o.p, ord,
                                                           items, di, nch, sigma, q, Ap, part, active, mask, sgn));
  }
  CPB_LAUNCH_CHECK();
  return grid;
}

}  // namespace cpb
