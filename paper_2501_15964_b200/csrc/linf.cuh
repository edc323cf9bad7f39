// q = infinity building blocks (no reference counterpart: prox.cpp:17-21
// accepts q in {1, 2} only; the math is SURVEY.md §8(c), restated in
// oracle/prox_linalg.cpp l1_theta):
//   prox_{t||.||inf}(v) = clamp(v, -theta, theta)        (0 when ||v||_1 <= t)
//   Pi_{B1(r)}(z)       = sign(z) max(|z| - theta_r, 0)  (z when ||z||_1 <= r)
//   (I - M)             = diag(1_S) - s_S s_S^T / |S|    (I inside the ball)
// with theta the l1-ball projection threshold and S = {|v_f| > theta}.
#pragma once

#include "common.cuh"

namespace cpb {

// theta >= 0 with sum_f max(|v_f| - theta, 0) = t when ||v||_1 > t, else -1;
// *cnt = |S|.  Michelot's fixed point: theta_0 = (||v||_1 - t) / d on the full
// support, then theta <- (sum_{|v| > theta} |v| - t) / #{|v| > theta} while the
// support shrinks (a handful of passes in practice).  Sums run over lane-strided
// partials (element f -> lane f mod 32 in increasing f) met by an xor butterfly,
// the order oracle/prox_linalg.cpp l1_theta reproduces, so theta is bitwise
// the oracle's.  For t = 0 the support empties at theta = max |v| (prox = v).
// `val(f)` yields element f; one pass over the row per iteration by the
// group's lanes (group_sum over blockDim.x <= 32 lanes, see common.cuh).
template <class F>
__device__ __forceinline__ double linf_theta(F val, int d, double t, unsigned gm, int* cnt) {
  double s1 = 0.0;
  for (int f = threadIdx.x; f < d; f += blockDim.x) s1 += fabs(val(f));
  s1 = group_sum(s1, gm);
  if (!(s1 > t)) {
    *cnt = 0;
    return -1.0;
  }
  double theta = (s1 - t) / static_cast<double>(d);
  int support = d;
  // the support shrinks strictly on every pass that continues (at most d
  // passes); a pass whose support does not shrink — the fixed point, or a
  // rounding-induced regrowth that would otherwise cycle — keeps theta
  for (;;) {
    double s = 0.0, c = 0.0;
    for (int f = threadIdx.x; f < d; f += blockDim.x) {
      const double a = fabs(val(f));
      if (a > theta) {
        s += a;
        c += 1.0;
      }
    }
    s = group_sum(s, gm);
    c = group_sum(c, gm);
    const int ci = static_cast<int>(c);
    if (ci == 0) {
      support = 0;
      break;
    }
    if (ci >= support) break;
    theta = (s - t) / c;
    support = ci;
  }
  *cnt = support;
  return theta;
}

__device__ __forceinline__ double clampd(double v, double th) { return fmax(fmin(v, th), -th); }

}  // namespace cpb

namespace cpb {

// linf_theta for a warp-owned row (blockDim.x = 32) whose values val(f) are
// cheap to re-read (staged in shared memory), d <= 32 * 32 * kLinfWords:
// after the first counting pass each lane keeps its candidates {|v_f| >
// threshold} as a bit set and later passes visit only those.  Exactly the
// passes of linf_theta (same elements in the same per-lane order, so the same
// partial sums and theta): an element dropped by one pass can only come back
// if theta decreased, and linf_theta stops on exactly that pass (the support
// does not shrink), as this loop does when the candidate count stops shrinking.
constexpr int kLinfWords = 4;  // up to 128 elements per lane (d <= 4096)
template <class F>
__device__ __forceinline__ double linf_theta_bits(F val, int d, double t, int* cnt) {
  const int lane = threadIdx.x & 31;
  double s1 = 0.0;
  for (int f = lane; f < d; f += 32) s1 += fabs(val(f));
  s1 = warp_sum(s1);
  if (!(s1 > t)) {
    *cnt = 0;
    return -1.0;
  }
  double theta = (s1 - t) / static_cast<double>(d);
  int support = d;
  unsigned m[kLinfWords];
  bool first = true;
  for (;;) {
    double s = 0.0, c = 0.0;
    if (first) {  // full pass: build the candidate bits
#pragma unroll
      for (int w = 0; w < kLinfWords; ++w) {
        unsigned bits = 0u;
        for (int b = 0; b < 32; ++b) {
          const int f = lane + 32 * (32 * w + b);
          if (f >= d) break;
          const double a = fabs(val(f));
          if (a > theta) {
            s += a;
            c += 1.0;
            bits |= 1u << b;
          }
        }
        m[w] = bits;
      }
      first = false;
    } else {
#pragma unroll
      for (int w = 0; w < kLinfWords; ++w) {
        unsigned bits = m[w], keep = 0u;
        while (bits) {
          const int b = __ffs(bits) - 1;
          bits &= bits - 1;
          const double a = fabs(val(lane + 32 * (32 * w + b)));
          if (a > theta) {
            s += a;
            c += 1.0;
            keep |= 1u << b;
          }
        }
        m[w] = keep;
      }
    }
    s = warp_sum(s);
    c = warp_sum(c);
    const int ci = static_cast<int>(c);
    if (ci == 0) {
      support = 0;
      break;
    }
    if (ci >= support) break;
    theta = (s - t) / c;
    support = ci;
  }
  *cnt = support;
  return theta;
}

}  // namespace cpb
