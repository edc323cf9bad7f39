// Preconditioned CG on node-shaped d x n blocks (linalg.cpp:143-192), with
// the loop control on the device.
//
// One iteration = operator (Hessian / Laplacian: Ap and <p,Ap>, <p,p> block
// partials) -> k_cg_b -> k_cg_s2 -> k_cg_c.  Every kernel no-ops once the
// state's `active` flag drops, so the host enqueues iterations in batches
// and reads the 80-byte state only between batches.
//
//   k_cg_b : every block reduces the operator partials itself (fixed order,
//            identical in all blocks) to alpha = rz / pAp, then r -= alpha Ap
//            and the per-feature ||r_f||^2 and <r, r/diag> partials.
//   k_cg_s2: worst relative feature-row residual (linalg.cpp:128-139) and
//            beta; decides convergence / max_iter.
//   k_cg_c : x += alpha p; p = r/diag + beta p.
//
// The vector kernels tile (32 features) x (a chunk of rows): per-feature
// partial sums need no atomics, loads stay coalesced along the feature axis.
#include <cstdlib>

#include "comm.cuh"
#include "gather.cuh"
#include "ops.cuh"

namespace cpb {

namespace {

struct CgState {
  double rz, pAp, alpha, beta, relres, tol, pp, rz_next;
  long long it, maxit;
  int active, stepped, phaseC, upd_p, status, pad;
};

struct Tile {
  int R, F;           // row chunks, feature chunks (32 wide)
  int64_t rows_per;   // rows per chunk
  int blocks() const { return R * F; }
};
// R row chunks x F feature chunks, with R x F at most one wave of resident
// blocks (`cap`): the tiles are equal, so a second, partial wave would leave
// most SMs idle for a whole tile (k_cg_b ran at 4.6 TB/s with 1.35 waves).
Tile tile_geom(int64_t n, int64_t d, int cap) {
  Tile t;
  t.F = static_cast<int>((d + 31) / 32);
  t.R = static_cast<int>(std::max<int64_t>(1, std::min<int64_t>(cap / t.F, n / 16)));
  t.rows_per = (n + t.R - 1) / t.R;
  return t;
}

// Fixed-order sum over the linear thread id (1-D or 2-D blocks).
__device__ __forceinline__ double sum_part(const double* part, int nb, int stride, double* sh) {
  const int tid = threadIdx.y * blockDim.x + threadIdx.x, nt = blockDim.x * blockDim.y;
  double s = 0.0;
  for (int b = tid; b < nb; b += nt) s += part[static_cast<int64_t>(b) * stride];
  return block_sum(s, sh);
}

// Reduce the 8 row-lanes of a (32 x 8) tile column-wise through shared memory.
__device__ __forceinline__ double tile_col_sum(double v, double* s8) {
  s8[threadIdx.y * 32 + threadIdx.x] = v;
  __syncthreads();
  double r = 0.0;
  if (threadIdx.y == 0)
    for (int y = 0; y < 8; ++y) r += s8[y * 32 + threadIdx.x];
  __syncthreads();
  return r;
}

// neg: the right-hand side is -rhs (SSNAL passes its gradient G for b = -G: no separate negation pass)
__global__ void __launch_bounds__(256) k_cg_init(const double* __restrict__ rhs, int neg, const double* __restrict__ Mx,
                                                 const double* __restrict__ diag, int64_t n, int d, int F,
                                                 int64_t rows_per, double* __restrict__ x, double* __restrict__ r,
                                                 double* __restrict__ p, double* part_rz, double* part_bb) {
  __shared__ double sh[32];
  __shared__ double s8[256];
  const int fc = blockIdx.x % F, rc = blockIdx.x / F;
  const int f = fc * 32 + threadIdx.x;
  const int64_t r0 = rc * rows_per, r1 = min(n, r0 + rows_per);
  double rz = 0.0, bb = 0.0;
  auto row = [&](int64_t i, double bin, double mx, double dg) {
    const double b = neg ? -bin : bin;
    const double rv = Mx ? b - mx : b;
    if (!Mx) x[i] = 0.0;
    r[i] = rv;
    const double z = rv / dg;
    p[i] = z;
    rz += rv * z;
    bb += b * b;
  };
  if (f < d) {
    // batches of 8 rows with the loads first (see k_cg_b); sums in ascending row order
    int64_t v = r0 + threadIdx.y;
    for (; v + 56 < r1; v += 64) {
      double bi[8], mi[8], dg[8];
#pragma unroll
      for (int u = 0; u < 8; ++u) {
        const int64_t i = (v + 8 * u) * d + f;
        bi[u] = rhs[i];
        mi[u] = Mx ? Mx[i] : 0.0;
        dg[u] = diag[i];
      }
#pragma unroll
      for (int u = 0; u < 8; ++u) row((v + 8 * u) * d + f, bi[u], mi[u], dg[u]);
    }
    for (; v < r1; v += 8) {
      const int64_t i = v * d + f;
      row(i, rhs[i], Mx ? Mx[i] : 0.0, diag[i]);
    }
  }
  const double cb = tile_col_sum(bb, s8);
  if (threadIdx.y == 0 && f < d) part_bb[static_cast<int64_t>(rc) * d + f] = cb;
  rz = block_sum(rz, sh);
  if (threadIdx.x == 0 && threadIdx.y == 0) part_rz[blockIdx.x] = rz;
}

// Worst relative feature-row residual from R x d column partials.
__device__ double relres_cols(const double* part, int R, int d, const double* bn, double* sh) {
  double worst = 0.0;
  for (int f = threadIdx.x; f < d; f += blockDim.x) {
    double s = 0.0;
    for (int rc = 0; rc < R; ++rc) s += part[static_cast<int64_t>(rc) * d + f];
    const double b = bn[f];
    worst = fmax(worst, sqrt(s) / (b > 0.0 ? b : 1.0));
  }
  return block_max(worst, sh);
}

__global__ void k_cg_s0(CgState* st, const double* part_rz, int nblk, const double* part_bb, int R, int d,
                        double tol, long long maxit, double* bn, int warm) {
  __shared__ double sh[32];
  for (int f = threadIdx.x; f < d; f += blockDim.x) {
    double s = 0.0;
    for (int rc = 0; rc < R; ++rc) s += part_bb[static_cast<int64_t>(rc) * d + f];
    bn[f] = sqrt(s);
  }
  __syncthreads();
  const double rel = relres_cols(part_bb, R, d, bn, sh);
  const double rz = sum_part(part_rz, nblk, 1, sh);
  if (threadIdx.x == 0) {
    st->rz = rz;
    st->relres = rel;
    st->tol = tol;
    st->it = 0;
    st->maxit = maxit;
    st->active = (!warm && rel <= tol) ? 0 : 1;
    st->stepped = st->phaseC = st->upd_p = 0;
    st->status = 0;
  }
}

__global__ void __launch_bounds__(256) k_cg_b(CgState* st, const double* __restrict__ part_h, int hb,
                                              const double* __restrict__ Ap, const double* __restrict__ diag,
                                              int64_t n, int d, int F, int64_t rows_per, double* __restrict__ r,
                                              double* part_rz, double* part_rr) {
  __shared__ double sh[32];
  __shared__ double s8[256];
  const bool lead = blockIdx.x == 0 && threadIdx.x == 0 && threadIdx.y == 0;
  if (lead) st->phaseC = 0;
  if (!st->active) return;
  const double pAp = sum_part(part_h, hb, 2, sh);
  const double pp = sum_part(part_h + 1, hb, 2, sh);
  if (pAp <= 0.0) {  // linalg.cpp:172-176: stop (p = 0) or throw (not PD)
    if (lead) {
      st->active = 0;
      st->stepped = 0;
      if (pp != 0.0) st->status = 1;
    }
    return;
  }
  const double alpha = st->rz / pAp;
  if (lead) {
    st->it += 1;
    st->pAp = pAp;
    st->pp = pp;
    st->alpha = alpha;
    st->stepped = 1;
  }
  const int fc = blockIdx.x % F, rc = blockIdx.x / F;
  const int f = fc * 32 + threadIdx.x;
  const int64_t r0 = rc * rows_per, r1 = min(n, r0 + rows_per);
  double rz = 0.0, rr = 0.0;
  if (f < d) {
    // batches of 8 rows: all 24 loads issued before the divisions (the z = r / diag division's
    // latency otherwise sits between consecutive loads); sums in ascending row order as before
    int64_t v = r0 + threadIdx.y;
    for (; v + 56 < r1; v += 64) {
      double rv[8], ap[8], dg[8];
#pragma unroll
      for (int u = 0; u < 8; ++u) {
        const int64_t i = (v + 8 * u) * d + f;
        rv[u] = r[i];
        ap[u] = Ap[i];
        dg[u] = diag[i];
      }
#pragma unroll
      for (int u = 0; u < 8; ++u) {
        const double x = rv[u] - alpha * ap[u];
        r[(v + 8 * u) * d + f] = x;
        rz += x * (x / dg[u]);
        rr += x * x;
      }
    }
    for (; v < r1; v += 8) {
      const int64_t i = v * d + f;
      const double rv = r[i] - alpha * Ap[i];
      r[i] = rv;
      rz += rv * (rv / diag[i]);
      rr += rv * rv;
    }
  }
  const double cr = tile_col_sum(rr, s8);
  if (threadIdx.y == 0 && f < d) part_rr[static_cast<int64_t>(rc) * d + f] = cr;
  rz = block_sum(rz, sh);
  if (threadIdx.x == 0 && threadIdx.y == 0) part_rz[blockIdx.x] = rz;
}

__global__ void k_cg_s2(CgState* st, const double* part_rz, int nblk, const double* part_rr, int R, int d,
                        const double* bn) {
  __shared__ double sh[32];
  if (!st->stepped) return;
  const double rel = relres_cols(part_rr, R, d, bn, sh);
  const double rzn = sum_part(part_rz, nblk, 1, sh);
  if (threadIdx.x == 0) {
    st->stepped = 0;
    st->phaseC = 1;
    st->relres = rel;
    if (rel <= st->tol || st->it >= st->maxit) {
      st->active = 0;
      st->upd_p = 0;
    } else {
      st->rz_next = rzn;
      st->beta = rzn / st->rz;
      st->rz = rzn;
      st->upd_p = 1;
    }
  }
}

// x += alpha p; p = r/diag + beta p (when continuing)
__global__ void k_cg_c(const CgState* __restrict__ st, const double* __restrict__ r, const double* __restrict__ diag,
                       int64_t m, double* __restrict__ x, double* __restrict__ p) {
  if (!st->phaseC) return;
  const double alpha = st->alpha, beta = st->beta;
  const bool upd = st->upd_p != 0;
  for (int64_t i = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; i < m;
       i += static_cast<int64_t>(gridDim.x) * blockDim.x) {
    const double pv = p[i];
    x[i] = x[i] + alpha * pv;
    if (upd) p[i] = r[i] / diag[i] + beta * pv;
  }
}

}  // namespace

const int* cg_active_ptr(const void* st) { return st ? &static_cast<const CgState*>(st)->active : nullptr; }

PcgOut pcg_dev(Ctx& c, int64_t n, int64_t d, const PcgOp& op, double op_bytes, const char* op_name,
               const double* rhs, PcgWork w, double tol, int64_t max_iter, bool warm, bool dist,
               const Graph* halo, bool neg_rhs) {
  if (!(tol > 0.0)) invalid("pcg: tol must be positive");
  if (max_iter < 1) invalid("pcg: max_iter must be >= 1");
  dist = dist && c.comm != nullptr;
  // this rank's rows [v0, v0 + nown) (all of them without a communicator)
  const int64_t chunk = dist ? c.comm->chunk(n) : n;
  const int64_t v0 = dist ? c.comm->v0(n) : 0;
  const int64_t nown = dist ? c.comm->v1(n) - v0 : n;
  const int64_t m = d * nown, off = v0 * d;
  struct OwnScope {  // the operator covers this rank's nodes while the PCG runs
    Ctx& c;
    int64_t p0, p1;
    OwnScope(Ctx& c_, bool on, int64_t a, int64_t b) : c(c_), p0(c_.own_v0), p1(c_.own_v1) {
      if (on) c.own_v0 = a, c.own_v1 = b;
    }
    ~OwnScope() { c.own_v0 = p0, c.own_v1 = p1; }
  } own(c, dist, v0, v0 + nown);
  int cap = 0;  // resident 256-thread blocks of the vector kernels per wave
  {
    int per_sm = 0;
    CPB_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, k_cg_b, 256, 0));
    cap = std::max(1, per_sm) * c.sm_count;
  }
  const Tile tg = tile_geom(chunk, d, cap);  // identical on every rank: partial tables line up
  // p rows other ranks own: only the halo the operator gathers (ascending-id
  // plans both sides derive from the replicated graph), or the whole chunk
  auto refresh_p = [&] {
    if (halo)
      halo_exchange(c, *halo, w.p, d);
    else
      comm_allgather(c, w.p, static_cast<size_t>(chunk * d));
  };
  const int nblk = tg.blocks();
  double* part_rz = c.buf<double>("pcg.rz", nblk + 8);
  double* part_rr = c.buf<double>("pcg.rr", static_cast<size_t>(tg.R) * d + 8);
  double* part_h = c.buf<double>("pcg.h", 2 * static_cast<size_t>(c.sm_count) * 16 + 8);
  double* bn = c.buf<double>("pcg.bn", d + 8);
  CgState* st = reinterpret_cast<CgState*>(c.dscal + 64);
  const double* Mx = nullptr;
  if (warm) {
    op(w.x, w.Ap, part_h, nullptr);
    Mx = w.Ap;
  }
  const int di = static_cast<int>(d);
  const dim3 tb(32, 8);
  k_cg_init<<<nblk, tb, 0, c.s>>>(rhs + off, neg_rhs ? 1 : 0, Mx ? Mx + off : nullptr, w.diag + off, nown, di, tg.F, tg.rows_per,
                                  w.x + off, w.r + off, w.p + off, part_rz, part_rr);
  CPB_LAUNCH_CHECK();
  if (dist) {
    comm_allreduce_sum(c, part_rz, nblk);
    comm_allreduce_sum(c, part_rr, static_cast<size_t>(tg.R) * d);
    refresh_p();
  }
  k_cg_s0<<<1, 1024, 0, c.s>>>(st, part_rz, nblk, part_rr, tg.R, di, tol, max_iter, bn, Mx != nullptr);
  CPB_LAUNCH_CHECK();
  const int fg = std::max(1, std::min(cdiv(m, 256), c.sm_count * 4));
  // Batch sizing: the first batch is the previous solve's iteration count
  // (consecutive Newton systems need similar counts), then small top-ups, so
  // few no-op iterations are launched past convergence.
  int& hint = c.cg_hint[op_name];
  int batch = hint > 0 ? std::max(2, std::min(hint - 1, 64)) : 4;
  long long it_before = 0;
  PcgOut out;
  for (;;) {
    for (int b = 0; b < batch; ++b) {
      int hb;
      {
        Ctx::Timer tm(&c, op_name, op_bytes);
        hb = op(w.p, w.Ap, part_h, st);
      }
      if (dist) comm_allreduce_sum(c, part_h, 2 * static_cast<size_t>(hb));
      {
        Ctx::Timer tm(&c, "pcg_update_b", 4.0 * m * 8.0);
        k_cg_b<<<nblk, tb, 0, c.s>>>(st, part_h, hb, w.Ap + off, w.diag + off, nown, di, tg.F, tg.rows_per,
                                      w.r + off, part_rz, part_rr);
        CPB_LAUNCH_CHECK();
      }
      if (dist) {
        comm_allreduce_sum(c, part_rz, nblk);
        comm_allreduce_sum(c, part_rr, static_cast<size_t>(tg.R) * d);
      }
      {
        Ctx::Timer tm(&c, "pcg_s2", 0.0);
        k_cg_s2<<<1, 1024, 0, c.s>>>(st, part_rz, nblk, part_rr, tg.R, di, bn);
        CPB_LAUNCH_CHECK();
      }
      {
        Ctx::Timer tm(&c, "pcg_update_c", 6.0 * m * 8.0);
        k_cg_c<<<fg, 256, 0, c.s>>>(st, w.r + off, w.diag + off, m, w.x + off, w.p + off);
        CPB_LAUNCH_CHECK();
      }
      if (dist) refresh_p();
    }
    CgState h;
    CPB_CUDA(cudaMemcpyAsync(c.hscal, st, sizeof(CgState), cudaMemcpyDeviceToHost, c.s));
    c.sync();
    std::memcpy(&h, c.hscal, sizeof(CgState));
    // launches after the loop ended were no-ops: drop them from the statistics
    const int wasted = batch - static_cast<int>(h.it - it_before);
    if (wasted > 0) {
      c.discard_pending(op_name, wasted);
      c.discard_pending("pcg_update_b", wasted);
      c.discard_pending("pcg_s2", wasted);
      c.discard_pending("pcg_update_c", wasted);
    }
    it_before = h.it;
    if (h.status == 1) runtime("pcg: operator is not positive definite (p'Ap <= 0)");
    if (!h.active) {
      out.iterations = h.it;
      out.converged = h.relres <= tol;
      break;
    }
    batch = h.it < 8 ? 4 : 2 + static_cast<int>(h.it / 8);
  }
  if (dist) {
    comm_allgather(c, w.x, static_cast<size_t>(chunk * d));
    c.sync();
  }
  hint = static_cast<int>(out.iterations);
  return out;
}

}  // namespace cpb
