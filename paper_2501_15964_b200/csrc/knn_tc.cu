// kNN candidate search on the 5th-generation tensor cores, followed by an
// exact FP64 re-check: compute_knn_weights (graph.cpp:75-114), north-star
// subsystem (1).
//
//   1. k_knn_split: A (FP64, n x d) -> A_hi, A_lo (TF32 values in FP32
//      containers, row stride dp = d rounded up to 4) with A ~ A_hi + A_lo,
//      plus squared row norms.
//   2. k_knn_tc: the pairwise dot products A Aᵀ as a 3xTF32 GEMM
//      (hi.hi + hi.lo + lo.hi) with tcgen05.mma kind::tf32, M = 128 query rows
//      x N = 256 points per MMA tile, FP32 accumulators in TMEM (two 256-column
//      buffers so the epilogue of tile t overlaps the MMAs of tile t+1),
//      operands staged by TMA (128-byte swizzle, two-stage mbarrier ring).
//      Warp roles: warp 4 = TMA producer, warp 5 = TMEM allocator + single-
//      thread MMA issuer, warps 0-3 = epilogue.  The epilogue reads each
//      accumulator row with tcgen05.ld, forms d2~ = |a_i|^2 + |a_j|^2 - 2 a_i.a_j
//      and keeps, per query row and per column segment, the KC = 32 smallest
//      d2~ in shared memory.  The n x n matrix never reaches HBM.
//   3. k_knn_recheck: per row, tau = k-th smallest d2~ over the segment
//      lists; with a rigorous per-row bound |d2~ - d2| <= delta_i every true
//      k-nearest neighbour has d2~ <= tau + 2 delta_i, so those candidates are
//      re-evaluated in FP64 in exactly Eigen's SSE2 squaredNorm order
//      (graph.cpp:95; four chains + packet tail, see graph.cu) and the top k by
//      (d2, j) are kept (graph.cpp:97-98).  Rows whose band might extend past a
//      full segment list (duplicates, very dense shells) are listed for the
//      exact FP64 tile kernel, so the result is always bit-identical to the
//      reference.
//
// delta_i = (3 d + 64) 2^-22 |a_i| M + 2^-21 (|a_i| + M)^2 with M = max_j |a_j|:
// it covers the FP64->FP32 rounding and the TF32 split (<= 4 2^-22 |a_i||a_j|),
// FP32 accumulation of the 3d products even if every addition truncated
// (3 d 2^-23 sum_r |a_ir a_jr|, doubled for margin), and the FP32 evaluation of
// d2~.  The re-check also verifies |d2~ - d2| <= delta_i on every candidate it
// evaluates and sends the row to the exact kernel if it ever fails.
#include <cuda.h>
#include <math_constants.h>

#include <cstdlib>

#include "graph.cuh"
#include "ptx.cuh"

namespace cpb {

namespace {

constexpr int TM = 128, TN = 256, TK = 32, KC = 32, STAGES = 2, MAXSEG = 8;
constexpr unsigned A_BYTES = TM * TK * 4;  // 16 KB: 128 rows x 128 B
constexpr unsigned B_BYTES = TN * TK * 4;  // 32 KB
constexpr unsigned STAGE_BYTES = 2 * A_BYTES + 2 * B_BYTES;
constexpr unsigned LIST_BYTES = 2u * KC * TM * 4;
constexpr unsigned SMEM_BYTES = STAGES * STAGE_BYTES + LIST_BYTES + 128 + 1024;
constexpr uint32_t TMEM_COLS = 2 * TN;

// ---- PTX wrappers --------------------------------------------------------------
__device__ __forceinline__ void tma_load_2d(void* dst, const CUtensorMap* map, int c0, int c1, uint64_t* bar) {
  asm volatile(
      "cp.async.bulk.tensor.2d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3}], [%4];" ::"r"(
          smem_u32(dst)),
      "l"(map), "r"(c0), "r"(c1), "r"(smem_u32(bar))
      : "memory");
}
// UMMA shared-memory descriptor, K-major, 128-byte swizzle: 8-row x 128-byte
// atoms 1024 B apart (SBO), LBO unused (1), descriptor version 1 (sm_100).
__device__ __forceinline__ uint64_t sw128_desc(const void* p) {
  const uint64_t a = (smem_u32(p) >> 4) & 0x3FFFu;
  return a | (1ull << 16) | (64ull << 32) | (1ull << 46) | (2ull << 61);
}
__device__ __forceinline__ void mma_tf32(uint32_t tmem, uint64_t a, uint64_t b, uint32_t idesc, uint32_t acc) {
  asm volatile(
      "{\n"
      ".reg .pred p;\n"
      "setp.ne.b32 p, %4, 0;\n"
      "tcgen05.mma.cta_group::1.kind::tf32 [%0], %1, %2, %3, p;\n"
      "}\n" ::"r"(tmem),
      "l"(a), "l"(b), "r"(idesc), "r"(acc));
}
__device__ __forceinline__ void mma_commit(uint64_t* bar) {
  asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(smem_u32(bar))
               : "memory");
}
__device__ __forceinline__ void tc_fence_before() { asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory"); }
__device__ __forceinline__ void tc_fence_after() { asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory"); }
// tcgen05.ld without the wait (the caller issues tmem_wait_ld before use).
__device__ __forceinline__ void tmem_ld32_nowait(uint32_t taddr, uint32_t (&r)[32]) {
  asm volatile(
      "tcgen05.ld.sync.aligned.32x32b.x32.b32 {%0, %1, %2, %3, %4, %5, %6, %7, %8, %9, %10, %11, %12, %13, %14, %15, "
      "%16, %17, %18, %19, %20, %21, %22, %23, %24, %25, %26, %27, %28, %29, %30, %31}, [%32];"
      : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7]), "=r"(r[8]),
        "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]), "=r"(r[14]), "=r"(r[15]), "=r"(r[16]),
        "=r"(r[17]), "=r"(r[18]), "=r"(r[19]), "=r"(r[20]), "=r"(r[21]), "=r"(r[22]), "=r"(r[23]), "=r"(r[24]),
        "=r"(r[25]), "=r"(r[26]), "=r"(r[27]), "=r"(r[28]), "=r"(r[29]), "=r"(r[30]), "=r"(r[31])
      : "r"(taddr));
}
__device__ __forceinline__ void tmem_wait_ld() { asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory"); }
__device__ __forceinline__ void tmem_ld32(uint32_t taddr, uint32_t (&r)[32]) {
  asm volatile(
      "tcgen05.ld.sync.aligned.32x32b.x32.b32 {%0, %1, %2, %3, %4, %5, %6, %7, %8, %9, %10, %11, %12, %13, %14, %15, "
      "%16, %17, %18, %19, %20, %21, %22, %23, %24, %25, %26, %27, %28, %29, %30, %31}, [%32];"
      : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7]), "=r"(r[8]),
        "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]), "=r"(r[14]), "=r"(r[15]), "=r"(r[16]),
        "=r"(r[17]), "=r"(r[18]), "=r"(r[19]), "=r"(r[20]), "=r"(r[21]), "=r"(r[22]), "=r"(r[23]), "=r"(r[24]),
        "=r"(r[25]), "=r"(r[26]), "=r"(r[27]), "=r"(r[28]), "=r"(r[29]), "=r"(r[30]), "=r"(r[31])
      : "r"(taddr));
  asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
}
__device__ __forceinline__ float tf32_rna(float x) {
  uint32_t u;
  asm("cvt.rna.tf32.f32 %0, %1;" : "=r"(u) : "f"(x));
  return __uint_as_float(u);
}

// ---- 1. split -------------------------------------------------------------------
// One warp per row (rows >= n only write the +inf norm padding).
__global__ void k_knn_split(const double* __restrict__ A, int n, int d, int dp, int npad, float* __restrict__ hi,
                            float* __restrict__ lo, double* __restrict__ n64, float* __restrict__ n32) {
  const int lane = threadIdx.x & 31;
  for (int r = (blockIdx.x * blockDim.x + threadIdx.x) >> 5; r < npad; r += (gridDim.x * blockDim.x) >> 5) {
    if (r >= n) {
      if (lane == 0) n32[r] = CUDART_INF_F;
      continue;
    }
    double ss = 0.0;
    for (int f = lane; f < dp; f += 32) {
      const double a = f < d ? A[static_cast<int64_t>(r) * d + f] : 0.0;
      const float a32 = static_cast<float>(a);
      const float h = tf32_rna(a32);
      hi[static_cast<int64_t>(r) * dp + f] = h;
      lo[static_cast<int64_t>(r) * dp + f] = tf32_rna(a32 - h);
      ss += a * a;
    }
    ss = warp_sum(ss);
    if (lane == 0) {
      n64[r] = ss;
      n32[r] = static_cast<float>(ss);
    }
  }
}

// ---- 2. tensor-core candidate pass ---------------------------------------------
// LIST mode: per (row, segment) the KC smallest d2~ (shared-memory list).
// THRESH mode: the A operand is a compacted set of nq query rows (qrows[] =
// their ids), and every column with d2~ <= qlim[row] is appended to that
// row's (row, segment) bucket of `caps` entries; ccount gets the full count
// (> caps means the bucket overflowed).
template <bool THRESH>
__global__ void __launch_bounds__(192, 1)
    k_knn_tc(const __grid_constant__ CUtensorMap ta_hi, const __grid_constant__ CUtensorMap ta_lo,
             const __grid_constant__ CUtensorMap tb_hi, const __grid_constant__ CUtensorMap tb_lo,
             const float* __restrict__ n32, int rbase, int n, int kblocks, int ntiles, int nseg, float* __restrict__ cd,
             int* __restrict__ cj, const int* __restrict__ qrows, const float* __restrict__ qlim, int nq, int caps,
             int* __restrict__ ccount) {
  extern __shared__ unsigned char smem_raw[];
  unsigned char* sm = smem_raw + ((1024u - (smem_u32(smem_raw) & 1023u)) & 1023u);
  float* Ld = reinterpret_cast<float*>(sm + STAGES * STAGE_BYTES);
  int* Lj = reinterpret_cast<int*>(Ld + KC * TM);
  uint64_t* bars = reinterpret_cast<uint64_t*>(Lj + KC * TM);
  uint64_t *full = bars, *empty = bars + 2, *tfull = bars + 4, *tempty = bars + 6;
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(bars + 8);

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int row0 = rbase + blockIdx.x * TM, seg = blockIdx.y;
  const int t0 = static_cast<int>(static_cast<int64_t>(ntiles) * seg / nseg);
  const int t1 = static_cast<int>(static_cast<int64_t>(ntiles) * (seg + 1) / nseg);

  if (threadIdx.x == 128) {
    for (int s = 0; s < 2; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&empty[s], 1);
      mbar_init(&tfull[s], 1);
      mbar_init(&tempty[s], 128);
    }
    fence_mbar_init();
  }
  if (warp == 5) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(tmem_slot)),
                 "r"(TMEM_COLS));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = *tmem_slot;

  if (warp == 4) {
    // ===== TMA producer =====
    if (lane == 0) {
      int it = 0;
      for (int t = t0; t < t1; ++t)
        for (int kb = 0; kb < kblocks; ++kb, ++it) {
          const int s = it % STAGES;
          mbar_wait(&empty[s], ((it / STAGES) & 1) ^ 1);
          unsigned char* st = sm + s * STAGE_BYTES;
          mbar_expect_tx(&full[s], STAGE_BYTES);
          const int k0 = kb * TK;
          tma_load_2d(st, &ta_hi, k0, row0, &full[s]);
          tma_load_2d(st + A_BYTES, &ta_lo, k0, row0, &full[s]);
          tma_load_2d(st + 2 * A_BYTES, &tb_hi, k0, t * TN, &full[s]);
          tma_load_2d(st + 2 * A_BYTES + B_BYTES / 2, &tb_hi, k0, t * TN + TN / 2, &full[s]);
          tma_load_2d(st + 2 * A_BYTES + B_BYTES, &tb_lo, k0, t * TN, &full[s]);
          tma_load_2d(st + 2 * A_BYTES + B_BYTES + B_BYTES / 2, &tb_lo, k0, t * TN + TN / 2, &full[s]);
        }
    }
  } else if (warp == 5) {
    // ===== MMA issuer (one thread) =====
    if (lane == 0) {
      // kind::tf32 instruction descriptor: D f32, A/B tf32, both K-major, N = 256, M = 128.
      const uint32_t idesc = (1u << 4) | (2u << 7) | (2u << 10) | (static_cast<uint32_t>(TN >> 3) << 17) |
                             (static_cast<uint32_t>(TM >> 4) << 24);
      int it = 0;
      for (int t = t0, lt = 0; t < t1; ++t, ++lt) {
        const int b = lt & 1;
        mbar_wait(&tempty[b], ((lt >> 1) & 1) ^ 1);
        tc_fence_after();
        const uint32_t acc = tmem + static_cast<uint32_t>(b * TN);
        for (int kb = 0; kb < kblocks; ++kb, ++it) {
          const int s = it % STAGES;
          mbar_wait(&full[s], (it / STAGES) & 1);
          tc_fence_after();
          const unsigned char* st = sm + s * STAGE_BYTES;
#pragma unroll
          for (int k = 0; k < TK / 8; ++k) {  // UMMA_K = 8 tf32 = 32 bytes
            const uint64_t ah = sw128_desc(st + 32 * k), al = sw128_desc(st + A_BYTES + 32 * k);
            const uint64_t bh = sw128_desc(st + 2 * A_BYTES + 32 * k);
            const uint64_t bl = sw128_desc(st + 2 * A_BYTES + B_BYTES + 32 * k);
            mma_tf32(acc, al, bh, idesc, (kb | k) != 0 ? 1u : 0u);
            mma_tf32(acc, ah, bl, idesc, 1u);
            mma_tf32(acc, ah, bh, idesc, 1u);
          }
          mma_commit(&empty[s]);  // frees the smem stage once these MMAs retire
        }
        mma_commit(&tfull[b]);  // accumulator buffer b is complete
      }
    }
  } else {
    // ===== epilogue: thread t owns query row row0 + t (TMEM lane t); LIST mode
    // rows are [rbase, n), THRESH mode local rows index qrows =====
    const int t = threadIdx.x, lr = row0 + t;
    int row;
    float lim = CUDART_INF_F;
    if (THRESH) {
      row = lr < nq ? qrows[lr] : -1;
      lim = lr < nq ? qlim[lr] : -CUDART_INF_F;
    } else {
      row = lr < n ? lr : -1;
    }
    const float ni = row >= 0 ? n32[row] : CUDART_INF_F;
    int cnt = 0, maxpos = 0;
    float thr = CUDART_INF_F;
    const int64_t tbase = (static_cast<int64_t>(lr) * nseg + seg) * caps;
    for (int tt = t0, lt = 0; tt < t1; ++tt, ++lt) {
      const int b = lt & 1;
      mbar_wait(&tfull[b], (lt >> 1) & 1);
      tc_fence_after();
      const uint32_t tbuf = tmem + (static_cast<uint32_t>(warp * 32) << 16) + static_cast<uint32_t>(b * TN);
      uint32_t rn[32];
      tmem_ld32(tbuf, rn);
#pragma unroll 1
      for (int ch = 0; ch < TN / 32; ++ch) {
        uint32_t r[32];
#pragma unroll
        for (int v = 0; v < 32; ++v) r[v] = rn[v];
        // the next chunk's accumulator load overlaps this chunk's processing
        if (ch + 1 < TN / 32) tmem_ld32_nowait(tbuf + static_cast<uint32_t>((ch + 1) * 32), rn);
        const int cb = tt * TN + ch * 32;
        // branch-free common path: the chunk's 32 column norms as 8 broadcast
        // float4 loads, 32 d2~ values, one candidate bit mask; the (rare)
        // insertions then run over the set bits with static register indices
        const float4* nj4 = reinterpret_cast<const float4*>(n32 + cb);
        float d2v[32];
#pragma unroll
        for (int u = 0; u < 8; ++u) {
          const float4 q4 = __ldg(nj4 + u);
          d2v[4 * u + 0] = (ni + q4.x) - 2.0f * __uint_as_float(r[4 * u + 0]);
          d2v[4 * u + 1] = (ni + q4.y) - 2.0f * __uint_as_float(r[4 * u + 1]);
          d2v[4 * u + 2] = (ni + q4.z) - 2.0f * __uint_as_float(r[4 * u + 2]);
          d2v[4 * u + 3] = (ni + q4.w) - 2.0f * __uint_as_float(r[4 * u + 3]);
        }
        unsigned m = 0;
#pragma unroll
        for (int v = 0; v < 32; ++v) m |= ((THRESH ? d2v[v] <= lim : d2v[v] < thr) ? 1u : 0u) << v;
        const int self = row - cb;
        if (self >= 0 && self < 32) m &= ~(1u << self);
        if (m) {
          // rare path, kept small for the instruction cache: spill the chunk
          // to a local array once and walk the set bits
          float dl[32];
#pragma unroll
          for (int v = 0; v < 32; ++v) dl[v] = d2v[v];
          while (m) {
            const int v = __ffs(m) - 1;
            m &= m - 1;
            const float d2 = dl[v];
            const int col = cb + v;
            if (THRESH) {
              if (cnt < caps) {
                cd[tbase + cnt] = d2;
                cj[tbase + cnt] = col;
              }
              ++cnt;
            } else if (d2 < thr) {  // thr may have dropped since the mask was taken
              const int pos = cnt < KC ? cnt++ : maxpos;
              Ld[pos * TM + t] = d2;
              Lj[pos * TM + t] = col;
              if (cnt == KC) {
                thr = Ld[t];
                maxpos = 0;
                for (int q = 1; q < KC; ++q) {
                  const float x = Ld[q * TM + t];
                  if (x > thr) thr = x, maxpos = q;
                }
              }
            }
          }
        }
        tmem_wait_ld();  // the prefetched chunk is in rn
      }
      tc_fence_before();
      mbar_arrive(&tempty[b]);
    }
    if (THRESH) {
      if (row >= 0) ccount[static_cast<int64_t>(lr) * nseg + seg] = cnt;
    } else if (row >= 0) {
      const int64_t base = (static_cast<int64_t>(row) * nseg + seg) * KC;
      for (int q = 0; q < KC; ++q) {
        cd[base + q] = q < cnt ? Ld[q * TM + t] : CUDART_INF_F;
        cj[base + q] = q < cnt ? Lj[q * TM + t] : -1;
      }
    }
  }
  tc_fence_before();
  __syncthreads();
  if (warp == 5) {
    tc_fence_after();
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem), "r"(TMEM_COLS));
  }
}

// ---- 3. exact re-check ----------------------------------------------------------
__device__ __forceinline__ double sqdiff(double a, double b) {
  const double t = __dsub_rn(a, b);
  return __dmul_rn(t, t);
}
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

// Warp argmin over (key, pos) pairs; ties to the smaller pos.
template <class K>
__device__ __forceinline__ void warp_argmin(K& key, int& pos) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) {
    const K ok = __shfl_xor_sync(0xffffffffu, key, o);
    const int op = __shfl_xor_sync(0xffffffffu, pos, o);
    if (ok < key || (ok == key && op < pos)) key = ok, pos = op;
  }
}

constexpr int RC_WARPS = 8, RC_MAX = MAXSEG * KC;  // candidates per row handled by one warp

__device__ __forceinline__ double row_delta(double n2, double M, int d) {
  const double na = sqrt(n2);
  return (3.0 * d + 64.0) * 0x1p-22 * na * M + 0x1p-21 * (na + M) * (na + M);
}

// Exact Eigen-order d2 of the nc candidates s_j (approximations s_a) of `row`,
// then the top k by (d2, j) into kd/kj.  One quad of lanes per candidate
// (lane c of the quad sums chain c).  Returns false (nothing written) if some
// |d2~ - d2| exceeded delta.
__device__ bool exact_topk(const double* __restrict__ A, int row, int nc, int d, int e2, int k, double delta,
                           double* s_d, const int* s_j, const float* s_a, double* __restrict__ kd,
                           int* __restrict__ kj, float& wmax) {
  const int lane = threadIdx.x & 31, quad = lane >> 2, ch = lane & 3;
  const double* x = A + static_cast<int64_t>(row) * d;
  bool bad = false;
  for (int b0 = 0; b0 < nc; b0 += 8) {
    const int ci = min(b0 + quad, nc - 1);
    const double* y = A + static_cast<int64_t>(s_j[ci]) * d;
    double acc = 0.0;
    for (int q = ch; q < e2; q += 4) acc = __dadd_rn(acc, sqdiff(x[q], y[q]));
    const int qb = lane & ~3;
    const double c0 = __shfl_sync(0xffffffffu, acc, qb), c1 = __shfl_sync(0xffffffffu, acc, qb + 1);
    const double c2 = __shfl_sync(0xffffffffu, acc, qb + 2), c3 = __shfl_sync(0xffffffffu, acc, qb + 3);
    if (ch == 0 && b0 + quad < nc) {
      const double ex = eigen_finish(c0, c1, c2, c3, x, y, d, e2);
      s_d[b0 + quad] = ex;
      const double err = fabs(static_cast<double>(s_a[b0 + quad]) - ex);
      wmax = fmaxf(wmax, static_cast<float>(err / delta));
      if (err > delta) bad = true;
    }
  }
  if (__any_sync(0xffffffffu, bad)) return false;
  __syncwarp();
  unsigned tk = 0;
  for (int r = 0; r < k; ++r) {
    double key = CUDART_INF;
    int kjv = 0x7fffffff, pos = 0x7fffffff;
    for (int m = 0; m * 32 + lane < nc; ++m) {
      const int p = m * 32 + lane;
      if ((tk >> m) & 1u) continue;
      const double dv = s_d[p];
      const int jv = s_j[p];
      if (dv < key || (dv == key && jv < kjv)) key = dv, kjv = jv, pos = p;
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
      const double ok = __shfl_xor_sync(0xffffffffu, key, o);
      const int oj = __shfl_xor_sync(0xffffffffu, kjv, o);
      const int op = __shfl_xor_sync(0xffffffffu, pos, o);
      if (ok < key || (ok == key && oj < kjv)) key = ok, kjv = oj, pos = op;
    }
    if (lane == 0) {
      kd[static_cast<int64_t>(row) * k + r] = key;
      kj[static_cast<int64_t>(row) * k + r] = kjv;
    }
    if ((pos & 31) == lane) tk |= 1u << (pos >> 5);
  }
  return true;
}

__device__ __forceinline__ void flush_worst(float wmax, float* worst) {
  wmax = static_cast<float>(warp_max(static_cast<double>(wmax)));
  if ((threadIdx.x & 31) == 0 && worst) atomicMax(reinterpret_cast<int*>(worst), __float_as_int(wmax));  // >= 0
}

// LIST-mode re-check, one warp per row.  Entry e = lane + 32 m of the row's
// nseg * KC list entries belongs to segment m (KC == 32).  Rows whose band
// reaches past a full segment list go to the threshold pass (ovf, with their
// band limit); rows without k finite candidates or with a bound violation go
// to the exact tile kernel (hard).
__global__ void __launch_bounds__(RC_WARPS * 32)
    k_knn_recheck(const double* __restrict__ A, const float* __restrict__ cd, const int* __restrict__ cj,
                  const double* __restrict__ n64, const double* __restrict__ max_n2, int r0, int n, int d, int e2,
                  int k, int nseg, double* __restrict__ kd, int* __restrict__ kj, int* __restrict__ cnts,
                  int* __restrict__ ovf, float* __restrict__ ovf_lim, int* __restrict__ hard,
                  float* __restrict__ worst) {
  static_assert(KC == 32, "one list entry per lane and segment");
  __shared__ double s_d[RC_WARPS][RC_MAX];
  __shared__ int s_j[RC_WARPS][RC_MAX];
  __shared__ float s_a[RC_WARPS][RC_MAX];
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  const double M = sqrt(*max_n2);
  float wmax = 0.0f;
  for (int row = r0 + blockIdx.x * RC_WARPS + w; row < n; row += gridDim.x * RC_WARPS) {
    float v[MAXSEG];
    int j[MAXSEG];
#pragma unroll
    for (int m = 0; m < MAXSEG; ++m) {
      v[m] = CUDART_INF_F;
      j[m] = -1;
      if (m < nseg) {
        const int64_t e = (static_cast<int64_t>(row) * nseg + m) * KC + lane;
        v[m] = cd[e];
        j[m] = cj[e];
        if (j[m] < 0) v[m] = CUDART_INF_F;
      }
    }
    // tau = k-th smallest candidate value
    unsigned taken = 0;
    float tau = CUDART_INF_F;
    bool short_list = false;
    for (int r = 0; r < k; ++r) {
      float key = CUDART_INF_F;
      int pos = 0x7fffffff;
#pragma unroll
      for (int m = 0; m < MAXSEG; ++m)
        if (!((taken >> m) & 1u) && j[m] >= 0 && v[m] < key) key = v[m], pos = m * 32 + lane;
      warp_argmin(key, pos);
      if (pos == 0x7fffffff) {
        short_list = true;
        break;
      }
      tau = key;
      if ((pos & 31) == lane) taken |= 1u << (pos >> 5);
    }
    const double delta = row_delta(n64[row], M, d);
    const double lim = static_cast<double>(tau) + 2.0 * delta;
    bool overflow = false;
#pragma unroll
    for (int m = 0; m < MAXSEG; ++m) {
      if (m >= nseg) break;
      const bool fullseg = __all_sync(0xffffffffu, j[m] >= 0);
      const double mx = warp_max(static_cast<double>(v[m]));
      if (fullseg && mx <= lim) overflow = true;
    }
    bool ok = false;
    if (!short_list && !overflow) {
      int nc = 0;
#pragma unroll
      for (int m = 0; m < MAXSEG; ++m) {
        const bool cand = j[m] >= 0 && static_cast<double>(v[m]) <= lim;
        const unsigned bm = __ballot_sync(0xffffffffu, cand);
        if (cand) {
          const int p = nc + __popc(bm & ((1u << lane) - 1u));
          s_j[w][p] = j[m];
          s_a[w][p] = v[m];
        }
        nc += __popc(bm);
      }
      __syncwarp();
      ok = exact_topk(A, row, nc, d, e2, k, delta, s_d[w], s_j[w], s_a[w], kd, kj, wmax);
    }
    if (!ok && lane == 0) {
      if (overflow && !short_list) {
        const int p = atomicAdd(&cnts[0], 1);
        ovf[p] = row;
        ovf_lim[p] = __double2float_ru(lim);
      } else {
        hard[atomicAdd(&cnts[1], 1)] = row;
      }
    }
    __syncwarp();
  }
  flush_worst(wmax, worst);
}

// THRESH-mode re-check: local row lr (global id qrows[lr]) owns nseg buckets
// of `caps` candidates, all with d2~ inside the band.
__global__ void __launch_bounds__(RC_WARPS * 32)
    k_knn_recheck_t(const double* __restrict__ A, const float* __restrict__ cd, const int* __restrict__ cj,
                    const int* __restrict__ ccount, const int* __restrict__ qrows, const double* __restrict__ n64,
                    const double* __restrict__ max_n2, int nq, int d, int e2, int k, int nseg, int caps,
                    double* __restrict__ kd, int* __restrict__ kj, int* __restrict__ cnts, int* __restrict__ hard,
                    float* __restrict__ worst) {
  __shared__ double s_d[RC_WARPS][RC_MAX];
  __shared__ int s_j[RC_WARPS][RC_MAX];
  __shared__ float s_a[RC_WARPS][RC_MAX];
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  const double M = sqrt(*max_n2);
  float wmax = 0.0f;
  for (int lr = blockIdx.x * RC_WARPS + w; lr < nq; lr += gridDim.x * RC_WARPS) {
    const int row = qrows[lr];
    int nc = 0;
    bool over = false;
    for (int s = 0; s < nseg; ++s) {
      const int c = ccount[static_cast<int64_t>(lr) * nseg + s];
      if (c > caps) over = true;
      const int cc = min(c, caps);
      const int64_t base = (static_cast<int64_t>(lr) * nseg + s) * caps;
      for (int q = lane; q < cc; q += 32)
        if (nc + q < RC_MAX) {
          s_j[w][nc + q] = cj[base + q];
          s_a[w][nc + q] = cd[base + q];
        }
      nc += cc;
    }
    if (nc > RC_MAX || nc < k) over = true;
    __syncwarp();
    bool ok = false;
    if (!over) ok = exact_topk(A, row, nc, d, e2, k, row_delta(n64[row], M, d), s_d[w], s_j[w], s_a[w], kd, kj, wmax);
    if (!ok && lane == 0) hard[atomicAdd(&cnts[1], 1)] = row;
    __syncwarp();
  }
  flush_worst(wmax, worst);
}

__global__ void k_gather_rows(const float* __restrict__ hi, const float* __restrict__ lo, const int* __restrict__ rows,
                              int nq, int dp, float* __restrict__ qhi, float* __restrict__ qlo) {
  const int64_t total = static_cast<int64_t>(nq) * dp;
  for (int64_t p = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; p < total;
       p += static_cast<int64_t>(gridDim.x) * blockDim.x) {
    const int64_t r = p / dp, f = p % dp;
    const int64_t src = static_cast<int64_t>(rows[r]) * dp + f;
    qhi[p] = hi[src];
    qlo[p] = lo[src];
  }
}

using EncodeTiled = CUresult (*)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*,
                                 const cuuint64_t*, const cuuint32_t*, const cuuint32_t*, CUtensorMapInterleave,
                                 CUtensorMapSwizzle, CUtensorMapL2promotion, CUtensorMapFloatOOBfill);

EncodeTiled encode_fn() {
  static EncodeTiled fn = [] {
    void* p = nullptr;
    cudaDriverEntryPointQueryResult q{};
    CPB_CUDA(cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q));
    if (q != cudaDriverEntryPointSuccess || !p) runtime("kNN: cuTensorMapEncodeTiled is unavailable");
    return reinterpret_cast<EncodeTiled>(p);
  }();
  return fn;
}

void make_map(CUtensorMap* m, const float* base, int64_t dp, int64_t rows) {
  const cuuint64_t dims[2] = {static_cast<cuuint64_t>(dp), static_cast<cuuint64_t>(rows)};
  const cuuint64_t strides[1] = {static_cast<cuuint64_t>(dp) * 4};
  const cuuint32_t box[2] = {static_cast<cuuint32_t>(TK), static_cast<cuuint32_t>(TM)};
  const cuuint32_t es[2] = {1, 1};
  const CUresult r = encode_fn()(m, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 2, const_cast<float*>(base), dims, strides, box,
                                 es, CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B,
                                 CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (r != CUDA_SUCCESS) runtime("kNN: cuTensorMapEncodeTiled failed (" + std::to_string(static_cast<int>(r)) + ")");
}

}  // namespace

bool knn_tc_enabled(Ctx& c, int64_t n, int64_t d, int64_t k) {
  const char* env = std::getenv("CPB_KNN_TC");
  if (env && env[0] == '0') return false;
  return c.sm_major == 10 && d >= 16 && n >= 2048 && k <= KC - 8 && n < (int64_t(1) << 30) / MAXSEG;
}

int64_t knn_tc(Ctx& c, const Data& A, int64_t k, int64_t r0_, int64_t r1_, double* kd, int* kj, int* hard) {
  const int n = static_cast<int>(A.n), d = static_cast<int>(A.d);
  const int r0 = static_cast<int>(r0_), r1 = static_cast<int>(r1_);
  const int dp = (d + 3) & ~3, e2 = (d / 4) * 4;
  const int ntiles = cdiv(n, TN), nrb = cdiv(r1 - r0, TM), kblocks = cdiv(dp, TK);
  const int npad = ntiles * TN;
  // column segments so that blocks * nseg fills the SMs (one CTA per SM)
  auto pick_seg = [&](int blocks0) {
    int ns = 1;
    double best = 0.0;
    for (int s = 1; s <= MAXSEG && s <= ntiles; ++s) {
      const double blocks = static_cast<double>(blocks0) * s;
      const double eff = blocks / (std::ceil(blocks / c.sm_count) * c.sm_count);
      if (eff > best + 0.05) best = eff, ns = s;
    }
    return ns;
  };
  const int nseg = pick_seg(nrb);
  float* hi = c.buf<float>("knntc.hi", static_cast<size_t>(n) * dp);
  float* lo = c.buf<float>("knntc.lo", static_cast<size_t>(n) * dp);
  double* n64 = c.buf<double>("knntc.n64", n);
  float* n32 = c.buf<float>("knntc.n32", npad);
  double* mx = c.buf<double>("knntc.max", 1);
  float* cd = c.buf<float>("knntc.cd", static_cast<size_t>(n) * nseg * KC);
  int* cj = c.buf<int>("knntc.cj", static_cast<size_t>(n) * nseg * KC);
  int* cnts = c.buf<int>("knntc.cnts", 2);
  float* worst = c.buf<float>("knntc.worst", 1);
  int* ovf = c.buf<int>("knntc.ovf", n);
  float* ovf_lim = c.buf<float>("knntc.ovflim", n);
  {
    Ctx::Timer tm(&c, "knn_split", static_cast<double>(n) * d * 8 + 2.0 * n * dp * 4);
    k_knn_split<<<std::min(cdiv(npad, 8), c.sm_count * 16), 256, 0, c.s>>>(A.A.p, n, d, dp, npad, hi, lo, n64, n32);
    CPB_LAUNCH_CHECK();
    reduce_max(c, n64, n, mx);
  }
  CUtensorMap mhi, mlo;
  make_map(&mhi, hi, dp, n);
  make_map(&mlo, lo, dp, n);
  if (first_on_device("k_knn_tc.smem")) {
    CPB_CUDA(cudaFuncSetAttribute(k_knn_tc<false>, cudaFuncAttributeMaxDynamicSharedMemorySize, SMEM_BYTES));
    CPB_CUDA(cudaFuncSetAttribute(k_knn_tc<true>, cudaFuncAttributeMaxDynamicSharedMemorySize, SMEM_BYTES));
  }
  {
    // "bytes" of the dense contraction = its algorithmic flops 2 n^2 d (reported as TFLOP/s)
    Ctx::Timer tm(&c, "knn_gemm", 2.0 * static_cast<double>(r1 - r0) * n * d);
    k_knn_tc<false><<<dim3(nrb, nseg), 192, SMEM_BYTES, c.s>>>(mhi, mlo, mhi, mlo, n32, r0, r1, kblocks, ntiles, nseg, cd,
                                                               cj, nullptr, nullptr, 0, KC, nullptr);
    CPB_LAUNCH_CHECK();
  }
  CPB_CUDA(cudaMemsetAsync(cnts, 0, 2 * sizeof(int), c.s));
  CPB_CUDA(cudaMemsetAsync(worst, 0, sizeof(float), c.s));
  {
    Ctx::Timer tm(&c, "knn_recheck", 0.0);
    k_knn_recheck<<<std::min(cdiv(r1 - r0, RC_WARPS), c.sm_count * 8), RC_WARPS * 32, 0, c.s>>>(
        A.A.p, cd, cj, n64, mx, r0, r1, d, e2, static_cast<int>(k), nseg, kd, kj, cnts, ovf, ovf_lim, hard, worst);
    CPB_LAUNCH_CHECK();
  }
  int h[2] = {0, 0};
  trace("knn_tc enqueued");
  d2h(c, h, cnts, 2 * sizeof(int));
  trace("knn_tc recheck synced");
  const int nq = h[0];
  if (nq > 0) {
    // threshold pass over the rows whose band outgrew a list
    // few rows: spread the column sweep over all MAXSEG segments (one CTA each)
    const int qrb = cdiv(nq, TM), qseg = qrb * 4 <= c.sm_count ? std::min(MAXSEG, ntiles) : pick_seg(qrb);
    const int caps = RC_MAX;  // per segment; the re-check also caps the row total at RC_MAX
    float* qhi = c.buf<float>("knntc.qhi", static_cast<size_t>(nq) * dp);
    float* qlo = c.buf<float>("knntc.qlo", static_cast<size_t>(nq) * dp);
    float* td = c.buf<float>("knntc.td", static_cast<size_t>(qrb) * TM * qseg * caps);
    int* tj = c.buf<int>("knntc.tj", static_cast<size_t>(qrb) * TM * qseg * caps);
    int* tc = c.buf<int>("knntc.tc", static_cast<size_t>(nq) * qseg);
    Ctx::Timer tm(&c, "knn_band", 2.0 * static_cast<double>(nq) * n * d);
    k_gather_rows<<<std::min(cdiv(static_cast<int64_t>(nq) * dp, 256), c.sm_count * 16), 256, 0, c.s>>>(
        hi, lo, ovf, nq, dp, qhi, qlo);
    CPB_LAUNCH_CHECK();
    CUtensorMap qmh, qml;
    make_map(&qmh, qhi, dp, nq);
    make_map(&qml, qlo, dp, nq);
    k_knn_tc<true><<<dim3(qrb, qseg), 192, SMEM_BYTES, c.s>>>(qmh, qml, mhi, mlo, n32, 0, n, kblocks, ntiles, qseg, td,
                                                              tj, ovf, ovf_lim, nq, caps, tc);
    CPB_LAUNCH_CHECK();
    k_knn_recheck_t<<<std::min(cdiv(nq, RC_WARPS), c.sm_count * 8), RC_WARPS * 32, 0, c.s>>>(
        A.A.p, td, tj, tc, ovf, n64, mx, nq, d, e2, static_cast<int>(k), qseg, caps, kd, kj, cnts, hard, worst);
    CPB_LAUNCH_CHECK();
    d2h(c, h, cnts, 2 * sizeof(int));
  }
  float wr = 0.0f;
  d2h(c, &wr, worst, sizeof(float));
  c.knn_last = {static_cast<int64_t>(h[1]), static_cast<double>(wr), nseg, 1};
  c.knn_band_rows = nq;
  return h[1];
}

}  // namespace cpb
