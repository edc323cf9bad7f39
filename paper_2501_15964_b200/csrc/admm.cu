// ADMM (admm.cpp:16-87).  The reference factors I + rho L once with a sparse
// Cholesky (SimplicialLLT + AMD, linalg.cpp:32-54) and back-solves d
// right-hand sides per iteration.  On B200 the X-update is instead a
// warm-started Jacobi-PCG on the matrix-free Laplacian operator (node-CSR
// gathers, no factor, no fill), solved to a relative feature-row residual of
// 1e-13 — the same linear system, solved to rounding-level accuracy.
#include <chrono>
#include <cmath>
#include <limits>

#include "gather.cuh"
#include "solve.cuh"
#include "linf.cuh"

namespace cpb {

namespace {
using Clock = std::chrono::steady_clock;
double since(Clock::time_point t0) { return std::chrono::duration<double>(Clock::now() - t0).count(); }

#define ROWS_BEGIN(rows)                                                                               \
  for (int64_t row_ = blockIdx.x * static_cast<int64_t>(blockDim.y) + threadIdx.y; row_ < (rows); \
       row_ += static_cast<int64_t>(gridDim.x) * blockDim.y)

struct GG {
  int gx, gy, grid;
};
GG geom(Ctx& c, int64_t rows, int64_t d) {
  int gx = 1;
  while (gx < d && gx < 32) gx <<= 1;
  const int gy = 256 / gx;
  return {gx, gy, std::max(1, std::min(cdiv(rows, gy), c.sm_count * 8))};
}
__device__ __forceinline__ double soft(double v, double t) {
  return static_cast<double>((v > 0.0) - (v < 0.0)) * fmax(fabs(v) - t, 0.0);
}

__global__ void k_lap_diag(const int* __restrict__ off, int64_t n, int d, double rho, double* __restrict__ diag) {
  const int64_t m = n * d;
  for (int64_t p = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; p < m;
       p += static_cast<int64_t>(gridDim.x) * blockDim.x) {
    const int64_t v = p / d;
    diag[p] = 1.0 + rho * static_cast<double>(off[v + 1] - off[v]);
  }
}

// XB; V = XB + Lam/rho; U = prox(V, r/rho); Lam += rho (XB - U); Zc = Pi_r(Lam)  (admm.cpp:63-70)
__global__ void k_admm_edge(const double* __restrict__ X, double* __restrict__ U, double* __restrict__ L,
                            double* __restrict__ Zc, const double* __restrict__ rad, const int* __restrict__ ei,
                            const int* __restrict__ ej, int64_t E, int d, double rho, int q) {
  const unsigned gm = group_mask();
  ROWS_BEGIN(E) {
    const double* xa = X + static_cast<int64_t>(ei[row_]) * d;
    const double* xb = X + static_cast<int64_t>(ej[row_]) * d;
    double* u = U + row_ * d;
    double* lam = L + row_ * d;
    double* zc = Zc + row_ * d;
    const double rl = rad[row_], tl = rl / rho;
    if (q == Q_L2) {
      double vv = 0.0;
      for (int f = threadIdx.x; f < d; f += blockDim.x) {
        const double v = (xa[f] - xb[f]) + lam[f] / rho;
        vv += v * v;
      }
      const double nv = sqrt(group_sum(vv, gm));
      const double s = 1.0 - tl / nv;
      double ll = 0.0;
      for (int f = threadIdx.x; f < d; f += blockDim.x) {
        const double x = xa[f] - xb[f];
        const double v = x + lam[f] / rho;
        const double un = (nv <= tl) ? 0.0 : s * v;
        u[f] = un;
        const double ln = lam[f] + rho * (x - un);
        lam[f] = ln;
        ll += ln * ln;
      }
      const double nl = sqrt(group_sum(ll, gm));
      const double sc = rl / nl;
      for (int f = threadIdx.x; f < d; f += blockDim.x) zc[f] = (nl <= rl) ? lam[f] : sc * lam[f];
    } else if (q == Q_LINF) {
      int cnt;
      const double thv = linf_theta([&](int f) { return (xa[f] - xb[f]) + lam[f] / rho; }, d, tl, gm, &cnt);
      for (int f = threadIdx.x; f < d; f += blockDim.x) {
        const double x = xa[f] - xb[f];
        const double un = thv < 0.0 ? 0.0 : clampd(x + lam[f] / rho, thv);
        u[f] = un;
        lam[f] = lam[f] + rho * (x - un);
      }
      const double thl = linf_theta([&](int f) { return lam[f]; }, d, rl, gm, &cnt);
      for (int f = threadIdx.x; f < d; f += blockDim.x) zc[f] = thl < 0.0 ? lam[f] : soft(lam[f], thl);
    } else {
      for (int f = threadIdx.x; f < d; f += blockDim.x) {
        const double x = xa[f] - xb[f];
        const double un = soft(x + lam[f] / rho, tl);
        u[f] = un;
        const double ln = lam[f] + rho * (x - un);
        lam[f] = ln;
        zc[f] = fmax(fmin(ln, rl), -rl);
      }
    }
  }
}
}  // namespace

cp_termination admm_solve(Prob& P, const cp_solver_config& cfg, bool warm, double* Xout, double* Zout,
                          SolveCache& cache) {
  (void)cache;
  Ctx& c = *P.c;
  const auto t0 = Clock::now();
  const int64_t d = P.d(), n = P.n(), E = P.E(), m = d * n, me = d * E;
  auto fin = [&](const GapOut& s, int64_t it, bool conv) {
    cp_termination t;
    std::memset(&t, 0, sizeof(t));
    t.f_primal = s.fp, t.f_dual = s.fd, t.gap = s.gap, t.iterations = it, t.converged = conv ? 1 : 0;
    t.wall_time = since(t0);
    return t;
  };
  // initial_point: X, Lambda (solver_util.hpp:56-68)
  if (warm) {
    project_columns_dev(c, P.q, Zout, P.rad, d, E, Zout);
  } else {
    copy_dev(c, Xout, P.A->A.p, m);
    CPB_CUDA(cudaMemsetAsync(Zout, 0, me * sizeof(double), c.s));
  }
  {
    GapOut s0 = eval_gap(P, Xout, Zout);
    trace_gap(c, cfg, 0, s0, since(t0));
    if (s0.gap <= cfg.epsilon && s0.kkt <= cfg.kkt_factor * cfg.epsilon) return fin(s0, 0, true);
  }
  const double rho = cfg.admm_rho;
  double* X = Xout;
  double* Lam = c.buf<double>("ad.L", me);
  double* U = c.buf<double>("ad.U", me);
  double* Zc = c.buf<double>("ad.Zc", me);
  double* R = c.buf<double>("ad.R", m);
  double* Xb = c.buf<double>("ad.Xb", m);
  double* Zb = c.buf<double>("ad.Zb", me);
  PcgWork w{X, c.buf<double>("ad.r", m), c.buf<double>("ad.p", m), c.buf<double>("ad.Ap", m),
            c.buf<double>("ad.diag", m)};
  copy_dev(c, Lam, Zout, me);
  incidence_apply_dev(c, *P.g, X, d, U);  // U = X B (admm.cpp:56-57)
  {
    const int fg = std::max(1, std::min(cdiv(m, 256), c.sm_count * 4));
    k_lap_diag<<<fg, 256, 0, c.s>>>(P.g->off.p, n, static_cast<int>(d), rho, w.diag);
    CPB_LAUNCH_CHECK();
  }
  GG ge = geom(c, E, d);
  const Graph& g = *P.g;
  PcgOp op = [&](const double* p, double* Ap, double* part, const void* st) {
    return gather_lap(c, g, p, rho, d, Ap, part, cg_active_ptr(st));
  };
  double best_gap = std::numeric_limits<double>::infinity();
  GapOut best_s;
  const int64_t max_iter = resolved_max_iter(cfg);
  for (int64_t k = 1; k <= max_iter; ++k) {
    gather_admm_rhs(c, g, P.A->A.p, U, Lam, rho, d, R);
    pcg_dev(c, n, d, op, (2.0 * m + 2.0 * E) * 8.0, "lap_apply", R, w, 1e-13, 100000, true);
    k_admm_edge<<<ge.grid, dim3(ge.gx, ge.gy), 0, c.s>>>(X, U, Lam, Zc, P.rad, g.ei.p, g.ej.p, E,
                                                         static_cast<int>(d), rho, P.q);
    CPB_LAUNCH_CHECK();
    GapOut s = eval_gap(P, X, Zc);
    trace_gap(c, cfg, k, s, since(t0));
    if (s.gap <= cfg.epsilon && s.kkt <= cfg.kkt_factor * cfg.epsilon) {
      copy_dev(c, Zout, Zc, me);
      return fin(s, k, true);
    }
    if (s.gap < best_gap) {
      best_gap = s.gap;
      best_s = s;
      copy_dev(c, Xb, X, m);
      copy_dev(c, Zb, Zc, me);
    }
    if ((cfg.time_limit > 0.0 && since(t0) > cfg.time_limit) || k == max_iter) {
      copy_dev(c, Xout, Xb, m);
      copy_dev(c, Zout, Zb, me);
      return fin(best_s, k, false);
    }
  }
  return fin(best_s, max_iter, false);
}

}  // namespace cpb
