// Graph construction and graph-level kernels (graph.cpp of the reference).
//
//  * knn_graph: compute_knn_weights (graph.cpp:75-114).  The pairwise squared
//    distances are computed in FP64 in exactly the order Eigen 3.4's SSE2
//    squaredNorm adds them (four interleaved chains, then the packet tail), so
//    every distance — and therefore every (dist, j) ranking, the edge set and
//    the edge order — is bit-identical to the reference.  A fused per-row
//    top-k (lexicographic (dist, j), ties to the smaller index, graph.cpp:97-98)
//    keeps only k candidates per row: the n x n matrix is never materialised.
//  * graph_from_edges: WeightedGraph(n, edges) (graph.cpp:25-45) on device.
//  * finalize_graph: node CSR (incident edges ascending), degree order.
//  * incidence operator B / Bᵀ (graph.cpp:122-152): Bᵀ is an atomic-free
//    node-CSR gather accumulating in ascending edge id, hence bitwise equal to
//    the reference's scatter loop.
//  * components_dev: min-label hooking + pointer jumping; labels ranked by
//    each component's smallest node = DFS first-appearance order (graph.cpp:169-196).
//  * laplacian_lambda_max: power_iteration on B Bᵀ (linalg.cpp:194-242).
#include <cub/cub.cuh>
#include <math_constants.h>

#include <algorithm>
#include <cmath>
#include <queue>
#include <random>
#include <vector>

#include "comm.cuh"
#include "gather.cuh"
#include "graph.cuh"

namespace cpb {

namespace {

// ---- row-kernel geometry -----------------------------------------------------
// Rows (nodes or edges) of length d are processed by dx threads (features)
// times dy rows per 256-thread block.
struct RowGeom {
  int dx, dy;
};
inline RowGeom row_geom(int64_t d) {
  int dx = 32;
  while (dx < d && dx < 256) dx <<= 1;
  return {dx, 256 / dx};
}
inline int row_grid(Ctx& c, int64_t rows, RowGeom g) {
  return std::max(1, std::min(cdiv(rows, g.dy), c.sm_count * 16));
}

// ---- kNN: exact FP64 tiled distances + fused top-k -----------------------------
constexpr int KB_M = 32, KB_N = 64, KB_K = 16, KB_LIST = 32;

__device__ __forceinline__ bool lex_less(double a, int ja, double b, int jb) {
  return a < b || (a == b && ja < jb);
}

__device__ __forceinline__ double sqdiff(double a, double b) {
  const double t = __dsub_rn(a, b);
  return __dmul_rn(t, t);
}

// Finish one Eigen-order squared norm from the four chain sums and the packet
// tail (Redux.h LinearVectorizedTraversal; see oracle/oracle.hpp esum).
__device__ __forceinline__ double eigen_finish(double c0, double c1, double c2, double c3, const double* __restrict__ x,
                                               const double* __restrict__ y, int d, int e2) {
  if (d < 4) {
    double r = sqdiff(x[0], y[0]);
    if (d >= 2) r = __dadd_rn(r, sqdiff(x[1], y[1]));
    if (d == 3) r = __dadd_rn(r, sqdiff(x[2], y[2]));
    return r;
  }
  double p0 = __dadd_rn(c0, c2), p1 = __dadd_rn(c1, c3);
  if (d - e2 >= 2) {
    p0 = __dadd_rn(p0, sqdiff(x[e2], y[e2]));
    p1 = __dadd_rn(p1, sqdiff(x[e2 + 1], y[e2 + 1]));
  }
  double r = __dadd_rn(p0, p1);
  if (d & 1) r = __dadd_rn(r, sqdiff(x[d - 1], y[d - 1]));
  return r;
}

// One block: KB_M query rows against all n samples, KB_N columns at a time.
// Thread (tx, ty) of 16 x 16 owns rows {ty, ty+16} x cols {tx + 16 tn}.
// With `rows` set, block b handles query rows rows[32 b ..] (nq of them):
// the exact pass for the rows the tensor-core path could not settle.
__global__ void __launch_bounds__(256) k_knn_topk(const double* __restrict__ A, int n, int d, int e2, int k,
                                                  const int* __restrict__ rows, int row_base, int nq,
                                                  double* __restrict__ out_d, int* __restrict__ out_j) {
  __shared__ double sA[KB_K][KB_M];
  __shared__ double sB[KB_K][KB_N];
  __shared__ double sD[KB_M][KB_N + 1];
  __shared__ double sLd[KB_M][KB_LIST];
  __shared__ int sLj[KB_M][KB_LIST];

  const int tid = threadIdx.x, tx = tid & 15, ty = tid >> 4;
  const int lane = tid & 31, warp = tid >> 5;
  const int row0 = blockIdx.x * KB_M;
  auto qrow = [&](int rr) { return row0 + rr < nq ? (rows ? rows[row0 + rr] : row_base + row0 + rr) : n; };

  for (int p = tid; p < KB_M * KB_LIST; p += 256) {
    sLd[p / KB_LIST][p % KB_LIST] = CUDART_INF;
    sLj[p / KB_LIST][p % KB_LIST] = 0x7fffffff;
  }

  for (int col0 = 0; col0 < n; col0 += KB_N) {
    double acc[2][4][4];
#pragma unroll
    for (int a = 0; a < 2; ++a)
#pragma unroll
      for (int b = 0; b < 4; ++b)
#pragma unroll
        for (int q = 0; q < 4; ++q) acc[a][b][q] = 0.0;

    for (int k0 = 0; k0 < e2; k0 += KB_K) {
      __syncthreads();
      for (int p = tid; p < KB_M * KB_K; p += 256) {
        const int r = p / KB_K, kk = p % KB_K, gr = qrow(r), gk = k0 + kk;
        sA[kk][r] = (gr < n && gk < e2) ? A[static_cast<int64_t>(gr) * d + gk] : 0.0;
      }
      for (int p = tid; p < KB_N * KB_K; p += 256) {
        const int r = p / KB_K, kk = p % KB_K, gr = col0 + r, gk = k0 + kk;
        sB[kk][r] = (gr < n && gk < e2) ? A[static_cast<int64_t>(gr) * d + gk] : 0.0;
      }
      __syncthreads();
#pragma unroll
      for (int kk = 0; kk < KB_K; kk += 4) {
#pragma unroll
        for (int q = 0; q < 4; ++q) {
          const double a0 = sA[kk + q][ty], a1 = sA[kk + q][ty + 16];
          double b[4];
#pragma unroll
          for (int tn = 0; tn < 4; ++tn) b[tn] = sB[kk + q][tx + 16 * tn];
#pragma unroll
          for (int tn = 0; tn < 4; ++tn) {
            acc[0][tn][q] = __dadd_rn(acc[0][tn][q], sqdiff(a0, b[tn]));
            acc[1][tn][q] = __dadd_rn(acc[1][tn][q], sqdiff(a1, b[tn]));
          }
        }
      }
    }
    __syncthreads();
#pragma unroll
    for (int tm = 0; tm < 2; ++tm)
#pragma unroll
      for (int tn = 0; tn < 4; ++tn) {
        const int r = qrow(ty + 16 * tm), cidx = col0 + tx + 16 * tn;
        double dist = CUDART_INF;
        if (r < n && cidx < n)
          dist = eigen_finish(acc[tm][tn][0], acc[tm][tn][1], acc[tm][tn][2], acc[tm][tn][3],
                              A + static_cast<int64_t>(r) * d, A + static_cast<int64_t>(cidx) * d, d, e2);
        sD[ty + 16 * tm][tx + 16 * tn] = dist;
      }
    __syncthreads();
    // merge: warp w owns rows 4w..4w+3
    for (int rr = warp * 4; rr < warp * 4 + 4; ++rr) {
      const int r = qrow(rr);
      if (r >= n) continue;
      for (int half = 0; half < 2; ++half) {
        const int cl = lane + 32 * half, j = col0 + cl;
        const double dd = sD[rr][cl];
        const double td = sLd[rr][k - 1];
        const int tj = sLj[rr][k - 1];
        const bool cand = j < n && j != r && lex_less(dd, j, td, tj);
        unsigned mask = __ballot_sync(0xffffffffu, cand);
        while (mask) {
          const int src = __ffs(mask) - 1;
          mask &= mask - 1;
          const double cd = __shfl_sync(0xffffffffu, dd, src);
          const int cj = __shfl_sync(0xffffffffu, j, src);
          const double kd = sLd[rr][k - 1];
          const int kj = sLj[rr][k - 1];
          if (!lex_less(cd, cj, kd, kj)) continue;  // list tightened meanwhile (warp-uniform)
          double ed = CUDART_INF;
          int ej = 0x7fffffff;
          if (lane < k) {
            ed = sLd[rr][lane];
            ej = sLj[rr][lane];
          }
          const unsigned lt = __ballot_sync(0xffffffffu, lane < k && lex_less(ed, ej, cd, cj));
          const int pos = __popc(lt);
          double pd = __shfl_up_sync(0xffffffffu, ed, 1);
          int pj = __shfl_up_sync(0xffffffffu, ej, 1);
          __syncwarp();
          if (lane < k) {
            if (lane == pos) {
              sLd[rr][lane] = cd;
              sLj[rr][lane] = cj;
            } else if (lane > pos) {
              sLd[rr][lane] = pd;
              sLj[rr][lane] = pj;
            }
          }
          __syncwarp();
        }
      }
    }
  }
  __syncthreads();
  for (int p = tid; p < KB_M * k; p += 256) {
    const int rr = p / k, m = p % k, r = qrow(rr);
    if (r < n) {
      out_d[static_cast<int64_t>(r) * k + m] = sLd[rr][m];
      out_j[static_cast<int64_t>(r) * k + m] = sLj[rr][m];
    }
  }
}

// Fallback for k > 32: full distance rows (Eigen order, one thread per pair),
// then a stable segmented radix sort per row.
__global__ void k_knn_rows(const double* __restrict__ A, int n, int d, int e2, int r0, int rows,
                           unsigned long long* __restrict__ keys, int* __restrict__ vals) {
  const int64_t total = static_cast<int64_t>(rows) * n;
  for (int64_t p = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; p < total;
       p += static_cast<int64_t>(gridDim.x) * blockDim.x) {
    const int rr = static_cast<int>(p / n), j = static_cast<int>(p % n), i = r0 + rr;
    const double* x = A + static_cast<int64_t>(i) * d;
    const double* y = A + static_cast<int64_t>(j) * d;
    double c0 = 0, c1 = 0, c2 = 0, c3 = 0;
    for (int q = 0; q < e2; q += 4) {
      c0 = __dadd_rn(c0, sqdiff(x[q], y[q]));
      c1 = __dadd_rn(c1, sqdiff(x[q + 1], y[q + 1]));
      c2 = __dadd_rn(c2, sqdiff(x[q + 2], y[q + 2]));
      c3 = __dadd_rn(c3, sqdiff(x[q + 3], y[q + 3]));
    }
    const double dist = eigen_finish(c0, c1, c2, c3, x, y, d, e2);
    keys[p] = (j == i) ? ~0ull : static_cast<unsigned long long>(__double_as_longlong(dist));
    vals[p] = j;
  }
}
__global__ void k_knn_take(const unsigned long long* __restrict__ keys, const int* __restrict__ vals, int n, int r0,
                           int rows, int k, double* __restrict__ out_d, int* __restrict__ out_j) {
  const int64_t total = static_cast<int64_t>(rows) * k;
  for (int64_t p = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; p < total;
       p += static_cast<int64_t>(gridDim.x) * blockDim.x) {
    const int rr = static_cast<int>(p / k), m = static_cast<int>(p % k);
    const int64_t src = static_cast<int64_t>(rr) * n + m;
    out_d[static_cast<int64_t>(r0 + rr) * k + m] = __longlong_as_double(static_cast<long long>(keys[src]));
    out_j[static_cast<int64_t>(r0 + rr) * k + m] = vals[src];
  }
}
__global__ void k_seg_offsets(int* off, int rows, int n) {
  const int t = blockIdx.x * blockDim.x + threadIdx.x;
  if (t <= rows) off[t] = t * n;
}

__global__ void k_check_lists(const double* __restrict__ kd, const int* __restrict__ kj, int n, int k, int* bad) {
  const int64_t total = static_cast<int64_t>(n) * k;
  for (int64_t p = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; p < total;
       p += static_cast<int64_t>(gridDim.x) * blockDim.x) {
    const int j = kj[p], i = static_cast<int>(p / k);
    const double v = kd[p];
    if (j < 0 || j >= n || j == i || !(v >= 0.0) || !isfinite(v)) *bad = 1;
  }
}

// (min, max) pair keys carrying the squared distance.
__global__ void k_pair_keys(const double* __restrict__ kd, const int* __restrict__ kj, int n, int k,
                            unsigned long long* __restrict__ key, double* __restrict__ val) {
  const int64_t total = static_cast<int64_t>(n) * k;
  for (int64_t p = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; p < total;
       p += static_cast<int64_t>(gridDim.x) * blockDim.x) {
    const int i = static_cast<int>(p / k), j = kj[p];
    const unsigned long long a = static_cast<unsigned long long>(min(i, j)), b = static_cast<unsigned long long>(max(i, j));
    key[p] = a * static_cast<unsigned long long>(n) + b;
    val[p] = kd[p];
  }
}
// Keep the first of each run of equal keys whose weight does not underflow
// (graph.cpp:104-111); w = exp(-phi * d2).
__global__ void k_pair_flags(const unsigned long long* __restrict__ key, const double* __restrict__ d2, int64_t m,
                             double phi, unsigned char* __restrict__ flag, double* __restrict__ w) {
  for (int64_t p = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; p < m;
       p += static_cast<int64_t>(gridDim.x) * blockDim.x) {
    const double wt = exp(__dmul_rn(-phi, d2[p]));
    w[p] = wt;
    flag[p] = (p == 0 || key[p] != key[p - 1]) && wt > 0.0;
  }
}
__global__ void k_decode_pairs(const unsigned long long* __restrict__ key, int64_t E, int n, int* ei, int* ej) {
  for (int64_t p = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; p < E;
       p += static_cast<int64_t>(gridDim.x) * blockDim.x) {
    ei[p] = static_cast<int>(key[p] / static_cast<unsigned long long>(n));
    ej[p] = static_cast<int>(key[p] % static_cast<unsigned long long>(n));
  }
}

// ---- WeightedGraph(n, edges) ----------------------------------------------------
__global__ void k_validate_edges(const long long* __restrict__ i, const long long* __restrict__ j,
                                 const double* __restrict__ w, int64_t E, long long n, int* err) {
  for (int64_t p = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; p < E;
       p += static_cast<int64_t>(gridDim.x) * blockDim.x) {
    const long long a = i[p], b = j[p];
    const double x = w[p];
    if (a < 0 || b < 0 || a >= n || b >= n) atomicOr(err, 1);
    else if (a >= b) atomicOr(err, 2);
    else if (!(x > 0.0) || !isfinite(x)) atomicOr(err, 4);
  }
}
__global__ void k_edge_keys(const long long* __restrict__ i, const long long* __restrict__ j, int64_t E,
                            long long n, unsigned long long* key, int* idx) {
  for (int64_t p = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; p < E;
       p += static_cast<int64_t>(gridDim.x) * blockDim.x) {
    key[p] = static_cast<unsigned long long>(i[p]) * static_cast<unsigned long long>(n) +
             static_cast<unsigned long long>(j[p]);
    idx[p] = static_cast<int>(p);
  }
}
__global__ void k_gather_edges(const unsigned long long* __restrict__ key, const int* __restrict__ idx,
                               const double* __restrict__ win, int64_t E, long long n, int* ei, int* ej, double* w,
                               double* d2, int* dup) {
  for (int64_t p = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; p < E;
       p += static_cast<int64_t>(gridDim.x) * blockDim.x) {
    ei[p] = static_cast<int>(key[p] / static_cast<unsigned long long>(n));
    ej[p] = static_cast<int>(key[p] % static_cast<unsigned long long>(n));
    w[p] = win[idx[p]];
    d2[p] = CUDART_NAN;
    if (p > 0 && key[p] == key[p - 1]) atomicOr(dup, 1);
  }
}

// ---- CSR -------------------------------------------------------------------------
__global__ void k_csr_entries(const int* __restrict__ ei, const int* __restrict__ ej, int E, int* key, int* val,
                              int* deg) {
  for (int p = blockIdx.x * blockDim.x + threadIdx.x; p < E; p += gridDim.x * blockDim.x) {
    key[p] = ej[p];
    val[p] = p;
    key[E + p] = ei[p];
    val[E + p] = p;
    atomicAdd(deg + ei[p], 1);
    atomicAdd(deg + ej[p], 1);
  }
}
__global__ void k_csr_other(const int* __restrict__ key, const int* __restrict__ adj_e, const int* __restrict__ ei,
                            const int* __restrict__ ej, int m, int* adj_o) {
  for (int p = blockIdx.x * blockDim.x + threadIdx.x; p < m; p += gridDim.x * blockDim.x) {
    const int v = key[p], l = adj_e[p];
    adj_o[p] = (ei[l] == v) ? ej[l] : ei[l];
  }
}
__global__ void k_iota(int* p, int n) {
  for (int t = blockIdx.x * blockDim.x + threadIdx.x; t < n; t += gridDim.x * blockDim.x) p[t] = t;
}

// ---- incidence operator -----------------------------------------------------------
__global__ void k_incidence(const double* __restrict__ X, const int* __restrict__ ei, const int* __restrict__ ej,
                            int64_t E, int d, double* __restrict__ out) {
  for (int64_t l = blockIdx.x * static_cast<int64_t>(blockDim.y) + threadIdx.y; l < E;
       l += static_cast<int64_t>(gridDim.x) * blockDim.y) {
    const double* a = X + static_cast<int64_t>(ei[l]) * d;
    const double* b = X + static_cast<int64_t>(ej[l]) * d;
    double* o = out + l * d;
    for (int f = threadIdx.x; f < d; f += blockDim.x) o[f] = __dsub_rn(a[f], b[f]);
  }
}
// ---- connected components ------------------------------------------------------------
// Lock-free union-find over the flagged edges in one pass (ECL-CC style):
// find with path halving, then link the larger root under the smaller with
// CAS, retrying on contention.  A root is only ever linked under a smaller
// root, so each component ends rooted at its smallest node whatever the
// interleaving: the labels are deterministic.
__device__ __forceinline__ int cc_find(int* L, int x) {
  int y = __ldcg(L + x);  // L2 (coherent) reads: other threads relink concurrently
  while (y != x) {
    const int z = __ldcg(L + y);
    if (z != y) L[x] = z;  // path halving (benign race: z is an ancestor)
    x = y;
    y = z;
  }
  return x;
}
__global__ void k_cc_union(const int* __restrict__ ei, const int* __restrict__ ej,
                           const unsigned char* __restrict__ flag, int E, int* L) {
  for (int l = blockIdx.x * blockDim.x + threadIdx.x; l < E; l += gridDim.x * blockDim.x) {
    if (flag && !flag[l]) continue;
    int u = cc_find(L, ei[l]), v = cc_find(L, ej[l]);
    while (u != v) {
      if (u > v) {
        const int t = u;
        u = v;
        v = t;
      }
      const int old = atomicCAS(L + v, v, u);  // v is (was) a root: hang it under u
      if (old == v) break;
      v = cc_find(L, old);
      u = cc_find(L, u);
    }
  }
}
__global__ void k_cc_jump(int* L, int n) {
  for (int v = blockIdx.x * blockDim.x + threadIdx.x; v < n; v += gridDim.x * blockDim.x) {
    int x = L[v];
    while (true) {
      const int y = L[x];
      if (y == x) break;
      x = y;
    }
    L[v] = x;
  }
}
__global__ void k_cc_roots(const int* __restrict__ L, int n, int* root) {
  for (int v = blockIdx.x * blockDim.x + threadIdx.x; v < n; v += gridDim.x * blockDim.x) root[v] = (L[v] == v);
}
__global__ void k_cc_label(const int* __restrict__ L, const int* __restrict__ rank, int n, int* labels) {
  for (int v = blockIdx.x * blockDim.x + threadIdx.x; v < n; v += gridDim.x * blockDim.x) labels[v] = rank[L[v]];
}

// ---- Laplacian power iteration -------------------------------------------------------------
// w = L v in the column order of L's column-major CSC (SparseDenseProduct.h): neighbours
// ascending with the degree term at position v (fused into k_power below).
// Sums of a[k] * b[k] in Eigen 3.4's SSE2 reduction order (Redux.h, LinearVectorizedTraversal
// with Packet2d; the oracle's esum): four stride-4 chains, P0 += P1, the leftover packet,
// predux, the odd tail.  Chains c = 0..3 run on four threads (sequential by nature); `slot`
// selects a 4-double area of `sh`; thread `lead` returns the result, all others 0.  Bitwise
// the reference's norm / dot, so lambda_max (and AMA's step 0.99 / lambda_max) is too.
__device__ double eigen_dot(const double* a, const double* b, int n, double* sh, int lead) {
  const int c = threadIdx.x - lead;
  const int e2 = (n / 4) * 4;
  if (c >= 0 && c < 4 && n >= 4) {
    double p = __dmul_rn(a[c], b[c]);
#pragma unroll 8
    for (int k = c + 4; k < e2; k += 4) p = __dadd_rn(p, __dmul_rn(a[k], b[k]));
    sh[c] = p;
  }
  __syncthreads();
  double res = 0.0;
  if (c == 0) {
    auto f = [&](int k) { return __dmul_rn(a[k], b[k]); };
    if (n < 2) {
      res = n == 1 ? f(0) : 0.0;
    } else {
      double p00 = f(0), p01 = f(1);
      if (n >= 4) {
        p00 = __dadd_rn(sh[0], sh[2]);
        p01 = __dadd_rn(sh[1], sh[3]);
        if ((n / 2) * 2 > e2) {
          p00 = __dadd_rn(p00, f(e2));
          p01 = __dadd_rn(p01, f(e2 + 1));
        }
      }
      res = __dadd_rn(p00, p01);
      if (n & 1) res = __dadd_rn(res, f(n - 1));
    }
  }
  return res;
}
// <w, w> and <v, w> at once: the two dots' chains run concurrently on lanes 0-3 of warps 0
// and 1, then lanes 0 of those warps finish them (two block barriers per iteration).
__device__ __forceinline__ void eigen_dots2(const double* v, const double* w, int n, double* sh /* 64 */,
                                            double& sww, double& svw) {
  const int lane = threadIdx.x & 31, wp = threadIdx.x >> 5;
  const int e2 = (n / 4) * 4;
  const double* a = wp == 0 ? w : v;  // warp 0: <w, w>, warp 1: <v, w>
  if (wp < 2 && lane < 4 && n >= 4) {
    double p = __dmul_rn(a[lane], w[lane]);
#pragma unroll 8
    for (int k = lane + 4; k < e2; k += 4) p = __dadd_rn(p, __dmul_rn(a[k], w[k]));
    sh[wp * 4 + lane] = p;
  }
  __syncthreads();
  if (wp < 2 && lane == 0) {
    auto f = [&](int k) { return __dmul_rn(a[k], w[k]); };
    double res;
    if (n < 2) {
      res = n == 1 ? f(0) : 0.0;
    } else {
      double p00 = f(0), p01 = f(1);
      if (n >= 4) {
        p00 = __dadd_rn(sh[wp * 4 + 0], sh[wp * 4 + 2]);
        p01 = __dadd_rn(sh[wp * 4 + 1], sh[wp * 4 + 3]);
        if ((n / 2) * 2 > e2) {
          p00 = __dadd_rn(p00, f(e2));
          p01 = __dadd_rn(p01, f(e2 + 1));
        }
      }
      res = __dadd_rn(p00, p01);
      if (n & 1) res = __dadd_rn(res, f(n - 1));
    }
    sh[8 + wp] = res;
  }
  __syncthreads();
  sww = sh[8];
  svw = sh[9];
}
// power_iteration (linalg.cpp:194-242) for one probe per block: w = L v in the column order of
// L's column-major CSC (SparseDenseProduct.h: neighbours ascending with the degree term at
// position v), then the two dots in Eigen's order.
__global__ void __launch_bounds__(1024) k_power(const int* __restrict__ off, const int* __restrict__ adj_o,
                                                const double* __restrict__ start, int n, double tol, long long max_iter,
                                                double* v, double* w, double* out, int in_smem) {
  // one block per probe (linalg.cpp:206-216 runs them one after another; they are independent)
  extern __shared__ double smvw[];
  start += static_cast<int64_t>(blockIdx.x) * n;
  if (in_smem) {  // small graphs: the iterate and L v live in shared memory
    v = smvw;
    w = smvw + n;
  } else {
    v += static_cast<int64_t>(blockIdx.x) * n;
    w += static_cast<int64_t>(blockIdx.x) * n;
  }
  out += 2 * blockIdx.x;
  __shared__ double sh[64];
  const double ns0 = eigen_dot(start, start, n, sh, 0);
  if (threadIdx.x == 0) sh[8] = ns0;
  __syncthreads();
  const double ns = sqrt(sh[8]);
  __syncthreads();
  for (int t = threadIdx.x; t < n; t += blockDim.x) v[t] = __ddiv_rn(start[t], ns);
  __syncthreads();
  double prev = 0.0, est = 0.0;
  int dead = 0;
  for (long long it = 1; it <= max_iter; ++it) {
    for (int t = threadIdx.x; t < n; t += blockDim.x) {
      const int p0 = off[t], p1 = off[t + 1];
      const double deg = static_cast<double>(p1 - p0);
      const double xv = v[t];
      double acc = 0.0;
      bool diag_done = (p1 == p0);
#pragma unroll 4
      for (int p = p0; p < p1; ++p) {
        const int u = adj_o[p];
        if (!diag_done && u > t) {
          acc = __dadd_rn(acc, __dmul_rn(deg, xv));
          diag_done = true;
        }
        acc = __dsub_rn(acc, v[u]);
      }
      if (!diag_done) acc = __dadd_rn(acc, __dmul_rn(deg, xv));
      w[t] = acc;
    }
    __syncthreads();
    double sww, svw;
    eigen_dots2(v, w, n, sh, sww, svw);
    const double nw = sqrt(sww);
    if (nw <= 1e-300) {
      dead = 1;
      break;
    }
    const double lam = svw;
    est = lam;
    for (int t = threadIdx.x; t < n; t += blockDim.x) v[t] = __ddiv_rn(w[t], nw);
    __syncthreads();
    if (it > 1 && fabs(lam - prev) <= tol * fmax(fabs(lam), 1e-300)) break;
    prev = lam;
  }
  if (threadIdx.x == 0) {
    out[0] = est;
    out[1] = dead;
  }
}

// ---- data norms --------------------------------------------------------------------------------
__global__ void k_sumsq(const double* __restrict__ x, int64_t count, double* partial) {
  __shared__ double sh[32];
  double s = 0.0;
  for (int64_t p = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; p < count;
       p += static_cast<int64_t>(gridDim.x) * blockDim.x)
    s = __dadd_rn(s, __dmul_rn(x[p], x[p]));
  s = block_sum(s, sh);
  if (threadIdx.x == 0) partial[blockIdx.x] = s;
}

template <class F>
void cub_call(Ctx& c, const char* tag, F f) {
  size_t bytes = 0;
  CPB_CUDA(f(nullptr, bytes));
  void* tmp = c.buf<char>(std::string("cub.") + tag, bytes + 16);
  CPB_CUDA(f(tmp, bytes));
}

uint64_t next_uid() {
  static uint64_t u = 0;
  return ++u;
}

}  // namespace

// ===========================================================================================
void finalize_graph(Ctx& c, Graph& g) {
  const int n = static_cast<int>(g.n), E = static_cast<int>(g.E);
  g.uid = next_uid();
  g.off.resize(n + 1);
  g.adj_e.resize(2 * static_cast<size_t>(E));
  g.adj_o.resize(2 * static_cast<size_t>(E));
  g.order.resize(n);
  int* deg = c.buf<int>("csr.deg", n + 1);
  CPB_CUDA(cudaMemsetAsync(deg, 0, (n + 1) * sizeof(int), c.s));
  if (E > 0) {
    int* key = c.buf<int>("csr.key", 2 * static_cast<size_t>(E));
    int* val = c.buf<int>("csr.val", 2 * static_cast<size_t>(E));
    int* key2 = c.buf<int>("csr.key2", 2 * static_cast<size_t>(E));
    k_csr_entries<<<std::min(cdiv(E, 256), c.sm_count * 8), 256, 0, c.s>>>(g.ei.p, g.ej.p, E, key, val, deg);
    CPB_LAUNCH_CHECK();
    int bits = 1;
    while ((1ll << bits) < n) ++bits;
    const int m = 2 * E;
    cub_call(c, "csr.sort", [&](void* t, size_t& b) {
      return cub::DeviceRadixSort::SortPairs(t, b, key, key2, val, g.adj_e.p, m, 0, bits, c.s);
    });
    k_csr_other<<<std::min(cdiv(m, 256), c.sm_count * 8), 256, 0, c.s>>>(key2, g.adj_e.p, g.ei.p, g.ej.p, m,
                                                                          g.adj_o.p);
    CPB_LAUNCH_CHECK();
  }
  cub_call(c, "csr.scan", [&](void* t, size_t& b) {
    return cub::DeviceScan::ExclusiveSum(t, b, deg, g.off.p, n + 1, c.s);
  });
  // max degree and descending-degree node order
  int* node = c.buf<int>("csr.node", n);
  int* degs = c.buf<int>("csr.degs", n);
  k_iota<<<std::max(1, std::min(cdiv(n, 256), c.sm_count * 8)), 256, 0, c.s>>>(node, n);
  CPB_LAUNCH_CHECK();
  if (n > 0) {
    cub_call(c, "csr.order", [&](void* t, size_t& b) {
      return cub::DeviceRadixSort::SortPairsDescending(t, b, deg, degs, node, g.order.p, n, 0, 32, c.s);
    });
    int md = 0;
    CPB_CUDA(cudaMemcpyAsync(&md, degs, sizeof(int), cudaMemcpyDeviceToHost, c.s));
    c.sync();
    g.max_degree = md;
  }
}

// Breadth-first node sequence over all components (lowest unvisited id
// starts the next one), with the CSR offsets copied to the host on the way.
std::vector<int> bfs_sequence(Ctx& c, const Graph& g, std::vector<int>* off_out) {
  const int n = static_cast<int>(g.n);
  std::vector<int> off(static_cast<size_t>(n) + 1), adj(static_cast<size_t>(2 * g.E));
  d2h(c, off.data(), g.off.p, off.size() * sizeof(int));
  if (g.E > 0) d2h(c, adj.data(), g.adj_o.p, adj.size() * sizeof(int));
  std::vector<int> seq(static_cast<size_t>(n));
  std::vector<char> seen(static_cast<size_t>(n), 0);
  size_t head = 0, tail = 0;
  for (int s0 = 0; s0 < n; ++s0) {
    if (seen[s0]) continue;
    seen[s0] = 1;
    seq[tail++] = s0;
    while (head < tail) {
      const int v = seq[head++];
      for (int e = off[v]; e < off[v + 1]; ++e) {
        const int o = adj[static_cast<size_t>(e)];
        if (!seen[o]) seen[o] = 1, seq[tail++] = o;
      }
    }
  }
  if (off_out) *off_out = std::move(off);
  return seq;
}

// Windowed longest-processing-time assignment: items (in the given order) are
// cut into windows of `win` consecutive items; inside each window the largest
// items go to the least-loaded of the nw warps.  Returns nw + 1 offsets
// followed by every warp's item list (items keep their window order).
std::vector<int> lpt_lists(const std::vector<int64_t>& cost, int nw, int win) {
  const int m = static_cast<int>(cost.size());
  std::vector<std::vector<int>> lists(static_cast<size_t>(nw));
  using Load = std::pair<int64_t, int>;
  std::priority_queue<Load, std::vector<Load>, std::greater<Load>> heap;
  for (int w = 0; w < nw; ++w) heap.push({0, w});
  std::vector<int> wv;
  for (int w0 = 0; w0 < m; w0 += win) {
    const int w1 = std::min(m, w0 + win);
    wv.clear();
    for (int it = w0; it < w1; ++it) wv.push_back(it);
    std::stable_sort(wv.begin(), wv.end(), [&](int a, int b) { return cost[a] > cost[b]; });
    for (int it : wv) {
      Load l = heap.top();
      heap.pop();
      lists[static_cast<size_t>(l.second)].push_back(it);
      heap.push({l.first + cost[it], l.second});
    }
  }
  std::vector<int> flat(static_cast<size_t>(nw) + 1 + m);
  int pos = nw + 1;
  for (int w = 0; w < nw; ++w) {
    flat[static_cast<size_t>(w)] = pos;
    for (int it : lists[static_cast<size_t>(w)]) flat[static_cast<size_t>(pos++)] = it;
  }
  flat[static_cast<size_t>(nw)] = pos;
  return flat;
}

std::unique_ptr<Graph> graph_from_edges(Ctx& c, int64_t n, const int64_t* i, const int64_t* j, const double* w,
                                        int64_t E) {
  if (n < 0) invalid("graph node count must be nonnegative");
  if (n >= (1ll << 31) - 1 || 2 * E >= (1ll << 31) - 1) invalid("graph too large for 32-bit indices");
  auto g = std::make_unique<Graph>();
  g->n = n;
  g->E = E;
  g->ei.resize(E);
  trace("graph buffers allocated");
  g->ej.resize(E);
  g->w.resize(E);
  g->d2.resize(E);
  if (E > 0) {
    long long* di = c.buf<long long>("fe.i", E);
    long long* dj = c.buf<long long>("fe.j", E);
    double* dw = c.buf<double>("fe.w", E);
    int* err = c.buf<int>("fe.err", 2);
    h2d(c, di, i, E * sizeof(long long));
    h2d(c, dj, j, E * sizeof(long long));
    h2d(c, dw, w, E * sizeof(double));
    CPB_CUDA(cudaMemsetAsync(err, 0, 2 * sizeof(int), c.s));
    const int grid = std::min(cdiv(E, 256), c.sm_count * 8);
    k_validate_edges<<<grid, 256, 0, c.s>>>(di, dj, dw, E, n, err);
    CPB_LAUNCH_CHECK();
    int herr[2] = {0, 0};
    d2h(c, herr, err, 2 * sizeof(int));
    if (herr[0] & 1) invalid("edge endpoint out of range");
    if (herr[0] & 2) invalid("edges must satisfy i < j");
    if (herr[0] & 4) invalid("edge weights must be positive and finite");
    auto* key = c.buf<unsigned long long>("fe.key", E);
    auto* key2 = c.buf<unsigned long long>("fe.key2", E);
    int* idx = c.buf<int>("fe.idx", E);
    int* idx2 = c.buf<int>("fe.idx2", E);
    k_edge_keys<<<grid, 256, 0, c.s>>>(di, dj, E, n, key, idx);
    CPB_LAUNCH_CHECK();
    int bits = 1;
    while (bits < 64 && (1ull << bits) < static_cast<unsigned long long>(n) * static_cast<unsigned long long>(n)) ++bits;
    cub_call(c, "fe.sort", [&](void* t, size_t& b) {
      return cub::DeviceRadixSort::SortPairs(t, b, key, key2, idx, idx2, static_cast<int>(E), 0, bits, c.s);
    });
    k_gather_edges<<<grid, 256, 0, c.s>>>(key2, idx2, dw, E, n, g->ei.p, g->ej.p, g->w.p, g->d2.p, err + 1);
    CPB_LAUNCH_CHECK();
    d2h(c, herr, err, 2 * sizeof(int));
    if (herr[1]) invalid("duplicate edge");
  }
  finalize_graph(c, *g);
  return g;
}

void knn_validate(const Data& A, int64_t k, double phi) {
  const int64_t n = A.n;
  if (k < 1 || k > n - 1)
    invalid("compute_knn_weights: k must satisfy 1 <= k <= n-1, got k=" + std::to_string(k) +
            " with n=" + std::to_string(n));
  if (!(phi >= 0.0) || !std::isfinite(phi)) invalid("compute_knn_weights: phi must be finite and nonnegative");
  if (n >= (1ll << 31) - 1 || n * k >= (1ll << 31) - 1) invalid("compute_knn_weights: problem too large");
}

// The k nearest (d2, j) of every query row in [r0, r1), ascending (graph.cpp:79-88),
// into kd/kj at the global row positions (n x k arrays).
void knn_rows_dev(Ctx& c, const Data& A, int64_t k, int64_t r0, int64_t r1, double* kd, int* kj) {
  const int64_t n = A.n, d = A.d;
  if (r0 < 0 || r1 > n || r0 > r1) invalid("knn rows: row range out of bounds");
  if (r0 == r1) return;
  const int e2 = d >= 4 ? static_cast<int>((d / 4) * 4) : 0;
  Ctx::Timer tm(&c, "knn_topk", 0.0);
  if (knn_tc_enabled(c, n, d, k)) {
    int* ovf = c.buf<int>("knn.ovf", n);
    const int64_t nov = knn_tc(c, A, k, r0, r1, kd, kj, ovf);
    if (nov > 0) {
      k_knn_topk<<<cdiv(nov, KB_M), 256, 0, c.s>>>(A.A.p, static_cast<int>(n), static_cast<int>(d), e2,
                                                    static_cast<int>(k), ovf, 0, static_cast<int>(nov), kd, kj);
      CPB_LAUNCH_CHECK();
    }
  } else if (k <= KB_LIST) {
    c.knn_last = {0, 0.0, 0, 0};
    c.knn_band_rows = 0;
    k_knn_topk<<<cdiv(r1 - r0, KB_M), 256, 0, c.s>>>(A.A.p, static_cast<int>(n), static_cast<int>(d), e2,
                                                      static_cast<int>(k), nullptr, static_cast<int>(r0),
                                                      static_cast<int>(r1 - r0), kd, kj);
    CPB_LAUNCH_CHECK();
  } else {
    c.knn_last = {0, 0.0, 0, 0};
    c.knn_band_rows = 0;
    const int64_t rows = std::max<int64_t>(1, std::min<int64_t>(n, (int64_t(1) << 26) / n));
    auto* keys = c.buf<unsigned long long>("knnf.k", rows * n);
    auto* keys2 = c.buf<unsigned long long>("knnf.k2", rows * n);
    int* vals = c.buf<int>("knnf.v", rows * n);
    int* vals2 = c.buf<int>("knnf.v2", rows * n);
    int* segoff = c.buf<int>("knnf.off", rows + 1);
    for (int64_t q0 = r0; q0 < r1; q0 += rows) {
      const int rr = static_cast<int>(std::min(rows, r1 - q0));
      const int64_t m = static_cast<int64_t>(rr) * n;
      k_knn_rows<<<std::min(cdiv(m, 256), c.sm_count * 16), 256, 0, c.s>>>(
          A.A.p, static_cast<int>(n), static_cast<int>(d), e2, static_cast<int>(q0), rr, keys, vals);
      CPB_LAUNCH_CHECK();
      k_seg_offsets<<<cdiv(rr + 1, 256), 256, 0, c.s>>>(segoff, rr, static_cast<int>(n));
      CPB_LAUNCH_CHECK();
      cub_call(c, "knnf.sort", [&](void* t, size_t& b) {
        return cub::DeviceSegmentedRadixSort::SortPairs(t, b, keys, keys2, vals, vals2, static_cast<int>(m), rr,
                                                        segoff, segoff + 1, 0, 64, c.s);
      });
      k_knn_take<<<std::min(cdiv(static_cast<int64_t>(rr) * k, 256), c.sm_count * 8), 256, 0, c.s>>>(
          keys2, vals2, static_cast<int>(n), static_cast<int>(q0), rr, static_cast<int>(k), kd, kj);
      CPB_LAUNCH_CHECK();
    }
  }
}

std::unique_ptr<Graph> knn_graph(Ctx& c, const Data& A, int64_t k, double phi) {
  knn_validate(A, k, phi);
  const int64_t n = A.n, NK = n * k;
  trace("knn_graph begin");
  if (c.comm && c.comm->nranks > 1) {
    // Row-sharded: this rank's query rows, then an in-place
    // all-gather of the padded n x k lists; every rank builds the same graph.
    const int64_t chunk = c.comm->chunk(n), P = c.comm->nranks;
    double* kd = c.buf<double>("knn.d", chunk * P * k);
    int* kj = c.buf<int>("knn.j", chunk * P * k);
    knn_rows_dev(c, A, k, c.comm->v0(n), c.comm->v1(n), kd, kj);
    comm_allgather_bytes(c, kd, static_cast<size_t>(chunk * k) * sizeof(double));
    comm_allgather_bytes(c, kj, static_cast<size_t>(chunk * k) * sizeof(int));
    return graph_from_knn_dev(c, n, k, phi, kd, kj);
  }
  double* kd = c.buf<double>("knn.d", NK);
  int* kj = c.buf<int>("knn.j", NK);
  knn_rows_dev(c, A, k, 0, n, kd, kj);
  trace("knn rows enqueued");
  auto g = graph_from_knn_dev(c, n, k, phi, kd, kj);
  trace("knn graph built");
  return g;
}

// Union of the per-row lists as (min, max) pairs, sorted and unique, with
// w = exp(-phi d2), dropping underflowed weights (graph.cpp:89-111).
std::unique_ptr<Graph> graph_from_knn_dev(Ctx& c, int64_t n, int64_t k, double phi, const double* kd, const int* kj) {
  if (!(phi >= 0.0) || !std::isfinite(phi)) invalid("compute_knn_weights: phi must be finite and nonnegative");
  if (k < 1 || k > n - 1 || n >= (1ll << 31) - 1 || n * k >= (1ll << 31) - 1)
    invalid("compute_knn_weights: bad list shape");
  const int64_t NK = n * k;
  {  // every entry must be a neighbour id != its row with a finite d2 >= 0
    int* bad = c.buf<int>("knn.bad", 1);
    CPB_CUDA(cudaMemsetAsync(bad, 0, sizeof(int), c.s));
    k_check_lists<<<std::min(cdiv(NK, 256), c.sm_count * 8), 256, 0, c.s>>>(kd, kj, static_cast<int>(n),
                                                                             static_cast<int>(k), bad);
    CPB_LAUNCH_CHECK();
    int hb = 0;
    d2h(c, &hb, bad, sizeof(int));
    if (hb) invalid("graph from kNN lists: entry out of range, self-loop or non-finite distance");
  }
  // union of (min, max) pairs, sorted and unique, with weights
  auto* key = c.buf<unsigned long long>("knn.key", NK);
  auto* key2 = c.buf<unsigned long long>("knn.key2", NK);
  double* val = c.buf<double>("knn.val", NK);
  double* val2 = c.buf<double>("knn.val2", NK);
  double* wv = c.buf<double>("knn.w", NK);
  auto* flag = c.buf<unsigned char>("knn.flag", NK);
  const int grid = std::min(cdiv(NK, 256), c.sm_count * 8);
  k_pair_keys<<<grid, 256, 0, c.s>>>(kd, kj, static_cast<int>(n), static_cast<int>(k), key, val);
  CPB_LAUNCH_CHECK();
  int bits = 1;
  while (bits < 64 && (1ull << bits) < static_cast<unsigned long long>(n) * static_cast<unsigned long long>(n)) ++bits;
  cub_call(c, "knn.sort", [&](void* t, size_t& b) {
    return cub::DeviceRadixSort::SortPairs(t, b, key, key2, val, val2, static_cast<int>(NK), 0, bits, c.s);
  });
  k_pair_flags<<<grid, 256, 0, c.s>>>(key2, val2, NK, phi, flag, wv);
  CPB_LAUNCH_CHECK();
  int* nsel = c.buf<int>("knn.nsel", 1);
  // compact keys, d2 and w
  cub_call(c, "knn.selk", [&](void* t, size_t& b) {
    return cub::DeviceSelect::Flagged(t, b, key2, flag, key, nsel, static_cast<int>(NK), c.s);
  });
  int E = 0;
  d2h(c, &E, nsel, sizeof(int));
  trace("knn pairs selected (synced)");
  auto g = std::make_unique<Graph>();
  g->n = n;
  g->E = E;
  g->ei.resize(E);
  g->ej.resize(E);
  g->w.resize(E);
  g->d2.resize(E);
  cub_call(c, "knn.seld", [&](void* t, size_t& b) {
    return cub::DeviceSelect::Flagged(t, b, val2, flag, g->d2.p, nsel, static_cast<int>(NK), c.s);
  });
  cub_call(c, "knn.selw", [&](void* t, size_t& b) {
    return cub::DeviceSelect::Flagged(t, b, wv, flag, g->w.p, nsel, static_cast<int>(NK), c.s);
  });
  if (E > 0) {
    k_decode_pairs<<<std::min(cdiv(E, 256), c.sm_count * 8), 256, 0, c.s>>>(key, E, static_cast<int>(n), g->ei.p,
                                                                             g->ej.p);
    CPB_LAUNCH_CHECK();
  }
  finalize_graph(c, *g);
  return g;
}

void incidence_apply_dev(Ctx& c, const Graph& g, const double* X, int64_t d, double* out) {
  if (g.E == 0) return;
  RowGeom rg = row_geom(d);
  k_incidence<<<row_grid(c, g.E, rg), dim3(rg.dx, rg.dy), 0, c.s>>>(X, g.ei.p, g.ej.p, g.E, static_cast<int>(d), out);
  CPB_LAUNCH_CHECK();
}

void incidence_apply_t_dev(Ctx& c, const Graph& g, const double* Z, int64_t d, double* out) {
  gather_bt(c, g, Z, d, out);
}

int64_t components_dev(Ctx& c, const Graph& g, const unsigned char* flag, int* labels) {
  const int n = static_cast<int>(g.n), E = static_cast<int>(g.E);
  if (n == 0) return 0;
  int* L = c.buf<int>("cc.L", n);
  int* root = c.buf<int>("cc.root", n + 1);
  int* rank = c.buf<int>("cc.rank", n + 1);
  const int gn = std::max(1, std::min(cdiv(n, 256), c.sm_count * 8));
  const int ge = std::max(1, std::min(cdiv(E, 256), c.sm_count * 8));
  k_iota<<<gn, 256, 0, c.s>>>(L, n);
  CPB_LAUNCH_CHECK();
  if (E > 0) {
    k_cc_union<<<ge, 256, 0, c.s>>>(g.ei.p, g.ej.p, flag, E, L);
    CPB_LAUNCH_CHECK();
    k_cc_jump<<<gn, 256, 0, c.s>>>(L, n);
    CPB_LAUNCH_CHECK();
  }
  k_cc_roots<<<gn, 256, 0, c.s>>>(L, n, root);
  CPB_CUDA(cudaMemsetAsync(root + n, 0, sizeof(int), c.s));
  CPB_LAUNCH_CHECK();
  cub_call(c, "cc.scan", [&](void* t, size_t& b) { return cub::DeviceScan::ExclusiveSum(t, b, root, rank, n + 1, c.s); });
  k_cc_label<<<gn, 256, 0, c.s>>>(L, rank, n, labels);
  CPB_LAUNCH_CHECK();
  int K = 0;
  d2h(c, &K, rank + n, sizeof(int));
  return K;
}

// IncidenceOperator::laplacian (graph.cpp:154-167): B B^T, unweighted, in
// compressed-column form.  Column v holds the neighbours below v (-1), the
// degree on the diagonal, then the neighbours above v (-1): the CSR's
// incident edges are in ascending edge id = ascending neighbour order.
// Isolated nodes have an empty column (the reference adds no triplet).
__global__ void k_lap_colcount(const int* __restrict__ off, int n, long long* __restrict__ cnt) {
  for (int v = blockIdx.x * blockDim.x + threadIdx.x; v < n; v += gridDim.x * blockDim.x) {
    const int deg = off[v + 1] - off[v];
    cnt[v] = deg + (deg > 0 ? 1 : 0);
  }
}
__global__ void k_lap_fill(const int* __restrict__ off, const int* __restrict__ adj_o, int n,
                           const long long* __restrict__ colptr, long long* __restrict__ row,
                           double* __restrict__ val) {
  for (int v = blockIdx.x * blockDim.x + threadIdx.x; v < n; v += gridDim.x * blockDim.x) {
    const int a = off[v], b = off[v + 1];
    if (a == b) continue;
    long long q = colptr[v];
    bool diag = false;
    for (int e = a; e < b; ++e) {
      const int o = adj_o[e];
      if (!diag && o > v) {
        row[q] = v, val[q] = static_cast<double>(b - a), ++q;
        diag = true;
      }
      row[q] = o, val[q] = -1.0, ++q;
    }
    if (!diag) row[q] = v, val[q] = static_cast<double>(b - a);
  }
}

int64_t laplacian_csc(Ctx& c, const Graph& g, int64_t* colptr, int64_t* rowidx, double* values) {
  const int n = static_cast<int>(g.n);
  long long* cnt = c.buf<long long>("lap.cnt", n + 1);
  long long* cp = c.buf<long long>("lap.cp", n + 1);
  CPB_CUDA(cudaMemsetAsync(cnt + n, 0, sizeof(long long), c.s));
  const int gn = std::max(1, std::min(cdiv(n, 256), c.sm_count * 8));
  if (n > 0) {
    k_lap_colcount<<<gn, 256, 0, c.s>>>(g.off.p, n, cnt);
    CPB_LAUNCH_CHECK();
  }
  cub_call(c, "lap.scan", [&](void* t, size_t& b) { return cub::DeviceScan::ExclusiveSum(t, b, cnt, cp, n + 1, c.s); });
  long long nnz = 0;
  d2h(c, &nnz, cp + n, sizeof(long long));
  if (!colptr) return nnz;
  long long* row = c.buf<long long>("lap.row", static_cast<size_t>(nnz) + 1);
  double* val = c.buf<double>("lap.val", static_cast<size_t>(nnz) + 1);
  if (n > 0) {
    k_lap_fill<<<gn, 256, 0, c.s>>>(g.off.p, g.adj_o.p, n, cp, row, val);
    CPB_LAUNCH_CHECK();
  }
  static_assert(sizeof(long long) == sizeof(int64_t), "int64");
  d2h(c, colptr, cp, (n + 1) * sizeof(int64_t));
  if (nnz) {
    if (rowidx) d2h(c, rowidx, row, nnz * sizeof(int64_t));
    if (values) d2h(c, values, val, nnz * sizeof(double));
  }
  return nnz;
}

double laplacian_lambda_max(Ctx& c, const Graph& g, double tol, int64_t max_iter) {
  if (!(tol > 0.0)) invalid("power_iteration: tol must be positive");
  if (max_iter < 1) invalid("power_iteration: max_iter must be >= 1");
  const int64_t n = g.n;
  if (n == 0) return 0.0;
  // Probes exactly as linalg.cpp:206-216: two fixed-seed libstdc++ Gaussian draws, then e_0.
  std::vector<double> starts(3 * static_cast<size_t>(n), 0.0);
  const uint64_t seeds[2] = {0x5851f42d4c957f2dULL, 0x14057b7ef767814fULL};
  for (int s = 0; s < 2; ++s) {
    std::mt19937_64 rng(seeds[s]);
    std::normal_distribution<double> gauss;
    for (int64_t v = 0; v < n; ++v) starts[s * n + v] = gauss(rng);
  }
  starts[2 * n] = 1.0;
  double* ds = c.buf<double>("pw.start", 3 * n);
  double* v = c.buf<double>("pw.v", 3 * n);
  double* w = c.buf<double>("pw.w", 3 * n);
  h2d(c, ds, starts.data(), starts.size() * sizeof(double));
  // the three probes run concurrently, one block each
  const size_t smem = 2 * static_cast<size_t>(n) * sizeof(double);
  const int in_smem = smem <= 200 * 1024;
  if (in_smem && first_on_device("k_power.smem"))
    CPB_CUDA(cudaFuncSetAttribute(k_power, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024));
  k_power<<<3, 1024, in_smem ? smem : 0, c.s>>>(g.off.p, g.adj_o.p, ds, static_cast<int>(n), tol, max_iter, v, w,
                                                c.dscal, in_smem);
  CPB_LAUNCH_CHECK();
  double out[6];
  c.fetch(0, 6, out);
  double best = 0.0;
  bool any = false;
  for (int s = 0; s < 3; ++s) {
    if (out[2 * s + 1] == 0.0) {
      any = true;
      best = std::max(best, out[2 * s]);
    }
  }
  return any ? best : 0.0;
}

double data_fro_norm(Ctx& c, Data& A) {
  if (A.normA >= 0.0) return A.normA;
  const int64_t m = A.d * A.n;
  const int grid = std::max(1, std::min(cdiv(m, 256), c.sm_count * 4));
  double* part = c.buf<double>("norm.part", grid);
  k_sumsq<<<grid, 256, 0, c.s>>>(A.A.p, m, part);
  CPB_LAUNCH_CHECK();
  reduce_sum(c, part, grid, c.dscal);
  double s;
  c.fetch(0, 1, &s);
  A.normA = std::sqrt(s);
  return A.normA;
}

}  // namespace cpb
