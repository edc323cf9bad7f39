// Register-resident edge-row kernels for d <= 1024: one warp per edge, the
// edge's whole row held in registers (lane l owns features l + 32 k, k < NK),
// so every multi-pass per-edge computation (norm first, then the scaled
// outputs) reads HBM once.  Same arithmetic as the generic kernels in ops.cu;
// per-edge reductions are warp trees, block partials fixed-order.
//
//  * k_phi_edge_r: V = X B + Z / sigma, ||V_l||, envelope (ssnal.cpp:24-39)
//  * k_mult_r:     Z <- Pi(Z + sigma X B), self-check, feasibility and the
//                  gap's edge terms at the new Z (ssnal.cpp:183-206,
//                  objective.cpp:63-113)
#include <cstdlib>

#include "edge.cuh"

namespace cpb {

namespace {

__device__ __forceinline__ double softr(double v, double t) {
  return static_cast<double>((v > 0.0) - (v < 0.0)) * fmax(fabs(v) - t, 0.0);
}

#define EDGE_WARPS(E)                                                                                \
  const int lane = threadIdx.x & 31;                                                                 \
  for (int64_t l = (blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x) >> 5; l < (E); \
       l += (static_cast<int64_t>(gridDim.x) * blockDim.x) >> 5)

template <int NK>
__global__ void __launch_bounds__(256) k_phi_edge_r(const double* __restrict__ X, const double* __restrict__ Z,
                                                    const int* __restrict__ ei, const int* __restrict__ ej,
                                                    const double* __restrict__ thr, const double* __restrict__ rad,
                                                    int64_t E, int d, double sigma, int q, double* __restrict__ V,
                                                    double* __restrict__ nv, double* part) {
  __shared__ double sh[32];
  double acc = 0.0;
  EDGE_WARPS(E) {
    const double* xa = X + static_cast<int64_t>(ei[l]) * d;
    const double* xb = X + static_cast<int64_t>(ej[l]) * d;
    const double* z = Z + l * d;
    double* v = V + l * d;
    const double t = thr[l];
    double x[NK];
#pragma unroll
    for (int k = 0; k < NK; ++k) {
      const int f = lane + 32 * k;
      x[k] = f < d ? (xa[f] - xb[f]) + __ldcs(z + f) / sigma : 0.0;
    }
#pragma unroll
    for (int k = 0; k < NK; ++k) {
      const int f = lane + 32 * k;
      if (f < d) __stcs(v + f, x[k]);
    }
    double env;
    if (q == 2) {
      double ss = 0.0;
#pragma unroll
      for (int k = 0; k < NK; ++k) ss += x[k] * x[k];
      ss = warp_sum(ss);
      const double nvl = sqrt(ss);
      double pn = 0.0, sq = ss;
      if (!(nvl <= t)) {
        const double s = 1.0 - t / nvl;
        double a = 0.0, b = 0.0;
#pragma unroll
        for (int k = 0; k < NK; ++k) {
          const double p = s * x[k];
          a += p * p;
          b += (p - x[k]) * (p - x[k]);
        }
        pn = sqrt(warp_sum(a));
        sq = warp_sum(b);
      }
      env = rad[l] * pn + (0.5 * sigma) * sq;
      if (lane == 0) nv[l] = nvl;
    } else {
      double a = 0.0, b = 0.0;
#pragma unroll
      for (int k = 0; k < NK; ++k) {
        const int f = lane + 32 * k;
        if (f >= d) continue;
        const double p = softr(x[k], t);
        a += fabs(p);
        b += (p - x[k]) * (p - x[k]);
      }
      env = rad[l] * warp_sum(a) + (0.5 * sigma) * warp_sum(b);
      if (lane == 0) nv[l] = 0.0;
    }
    if (lane == 0) acc += env;
  }
  acc = block_sum(acc, sh);
  if (threadIdx.x == 0) part[blockIdx.x] = acc;
}

// part per block: [0] sum w||XB||_q, [1] ||XB - prox(XB + Z)||^2, [2] ||XB||^2, [3] ||Z||^2,
// [4] ||XB - PV||^2, [5] unused, [6] max|Z + sigma XB|, [7] max|Zenv - Zsum|, [8] dual excess
template <int NK>
__global__ void __launch_bounds__(256) k_mult_r(const double* __restrict__ X, double* __restrict__ Z,
                                                const double* __restrict__ V, const double* __restrict__ ps,
                                                const double* __restrict__ thr, const double* __restrict__ rad,
                                                const double* __restrict__ w, const int* __restrict__ ei,
                                                const int* __restrict__ ej, int64_t E, int d, double sigma, int q,
                                                double* part) {
  __shared__ double sh[32];
  double s[5] = {0, 0, 0, 0, 0}, mx = 0.0, err = 0.0, excess = -1.0;
  EDGE_WARPS(E) {
    const double* xa = X + static_cast<int64_t>(ei[l]) * d;
    const double* xb = X + static_cast<int64_t>(ej[l]) * d;
    double* z = Z + l * d;
    const double* vr = V + l * d;
    const double rl = rad[l], tl = thr[l], sl = ps[l];
    double x[NK], zp[NK];
    double nn = 0.0, m = 0.0;
#pragma unroll
    for (int k = 0; k < NK; ++k) {
      const int f = lane + 32 * k;
      x[k] = f < d ? xa[f] - xb[f] : 0.0;
      zp[k] = f < d ? z[f] + sigma * x[k] : 0.0;  // Zsum
      nn += zp[k] * zp[k];
      m = fmax(m, fabs(zp[k]));
    }
    mx = fmax(mx, m);
    const double nz = sqrt(warp_sum(nn));
    const double sc = rl / nz;
    double fr = 0.0, e = 0.0, xb2 = 0.0, zz = 0.0, uu = 0.0, l1 = 0.0, zmax = 0.0;
#pragma unroll
    for (int k = 0; k < NK; ++k) {
      const int f = lane + 32 * k;
      if (f >= d) continue;
      const double zs = zp[k];
      zp[k] = (q == 2) ? ((nz <= rl) ? zs : sc * zs) : fmax(fmin(zs, rl), -rl);
      const double vv = __ldcs(vr + f);
      const double pv = (q == 2) ? sl * vv : softr(vv, tl);
      const double zenv = sigma * (vv - pv);
      e = fmax(e, fabs(zenv - zp[k]));
      z[f] = zp[k];
      fr += (x[k] - pv) * (x[k] - pv);
      const double u = x[k] + zp[k];
      xb2 += x[k] * x[k];
      zz += zp[k] * zp[k];
      uu += u * u;
      l1 += fabs(x[k]);
      zmax = fmax(zmax, fabs(zp[k]));
    }
    err = fmax(err, e);
    fr = warp_sum(fr);
    xb2 = warp_sum(xb2);
    zz = warp_sum(zz);
    double al = 0.0, pen, ex;
    if (q == 2) {
      const double nu = sqrt(warp_sum(uu));
      if (nu <= rl) {
        al = xb2;
      } else {
        const double s2 = 1.0 - rl / nu;
#pragma unroll
        for (int k = 0; k < NK; ++k) {
          const double t = x[k] - s2 * (x[k] + zp[k]);
          al += t * t;
        }
        al = warp_sum(al);
      }
      pen = w[l] * sqrt(xb2);
      ex = sqrt(zz) - (rl + 1e-9);
    } else {
#pragma unroll
      for (int k = 0; k < NK; ++k) {
        const int f = lane + 32 * k;
        if (f >= d) continue;
        const double t = x[k] - softr(x[k] + zp[k], rl);
        al += t * t;
      }
      al = warp_sum(al);
      pen = w[l] * warp_sum(l1);
      ex = warp_max(zmax) - (rl + 1e-9);
    }
    excess = fmax(excess, ex);
    if (lane == 0) {
      s[0] += pen;
      s[1] += al;
      s[2] += xb2;
      s[3] += zz;
      s[4] += fr;
    }
  }
#pragma unroll
  for (int k = 0; k < 5; ++k) {
    const double r = block_sum(s[k], sh);
    if (threadIdx.x == 0) part[9 * blockIdx.x + k] = r;
  }
  const double a = block_max(mx, sh);
  const double b = block_max(err, sh);
  const double cmax = block_max(excess, sh);
  if (threadIdx.x == 0) {
    part[9 * blockIdx.x + 5] = 0.0;
    part[9 * blockIdx.x + 6] = a;
    part[9 * blockIdx.x + 7] = b;
    part[9 * blockIdx.x + 8] = cmax;
  }
}

int nk_of(int64_t d) {
  const int need = static_cast<int>((d + 31) / 32);
  for (int b : {1, 2, 4, 8, 16, 25, 32})
    if (need <= b) return b;
  return 0;
}

#define NKR_DISPATCH(nk, KERNEL, ...)         \
  switch (nk) {                               \
    case 1: KERNEL<1> __VA_ARGS__; break;     \
    case 2: KERNEL<2> __VA_ARGS__; break;     \
    case 4: KERNEL<4> __VA_ARGS__; break;     \
    case 8: KERNEL<8> __VA_ARGS__; break;     \
    case 16: KERNEL<16> __VA_ARGS__; break;   \
    case 25: KERNEL<25> __VA_ARGS__; break;   \
    default: KERNEL<32> __VA_ARGS__; break;   \
  }

}  // namespace

// Opt-in (CPB_EDGE_REG=1): at d = 784 the register-resident rows cost 126-168
// registers (8 warps/SM) and measured slower than the generic group kernels
// (multiplier 1.63 vs 1.15 ms, phi 0.62 vs 0.44 ms at C2), whose second pass
// re-reads the row from L1/L2 at full occupancy.
bool edge_reg_supported(int64_t d) {
  static const bool enabled = std::getenv("CPB_EDGE_REG") != nullptr;
  return enabled && d >= 1 && nk_of(d) > 0;
}

int edge_grid(Ctx& c, int64_t E) { return std::max(1, std::min(cdiv(E, 8), c.sm_count * 8)); }

int phi_edge_reg(Ctx& c, const Graph& g, const double* X, const double* Z, const double* thr, const double* rad,
                 int64_t d, double sigma, int q, double* V, double* nv, double* part) {
  const int grid = edge_grid(c, g.E);
  NKR_DISPATCH(nk_of(d), k_phi_edge_r, <<<grid, 256, 0, c.s>>>(X, Z, g.ei.p, g.ej.p, thr, rad, g.E,
                                                                static_cast<int>(d), sigma, q, V, nv, part));
  CPB_LAUNCH_CHECK();
  return grid;
}

int mult_reg(Ctx& c, const Graph& g, const double* X, double* Z, const double* V, const double* ps, const double* thr,
             const double* rad, int64_t d, double sigma, int q, double* part) {
  const int grid = edge_grid(c, g.E);
  NKR_DISPATCH(nk_of(d), k_mult_r, <<<grid, 256, 0, c.s>>>(X, Z, V, ps, thr, rad, g.w.p, g.ei.p, g.ej.p, g.E,
                                                            static_cast<int>(d), sigma, q, part));
  CPB_LAUNCH_CHECK();
  return grid;
}

}  // namespace cpb
