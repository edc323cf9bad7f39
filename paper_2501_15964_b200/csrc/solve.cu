// Solver drivers and the path engine (see solve.cuh).
#include <sched.h>

#include <algorithm>
#include <atomic>
#include <chrono>
#include <condition_variable>
#include <deque>
#include <exception>
#include <mutex>
#include <cstring>
#include <thread>
#include <tuple>
#include <utility>
#include <vector>
#include <cstdlib>
#include <cmath>
#include <limits>
#include <string>

#include <cub/cub.cuh>

#include "comm.cuh"
#include "gather.cuh"
#include "solve.cuh"

namespace cpb {

namespace {
using Clock = std::chrono::steady_clock;
double since(Clock::time_point t0) { return std::chrono::duration<double>(Clock::now() - t0).count(); }

bool accepts(const GapOut& g, const cp_solver_config& c) {
  return g.gap <= c.epsilon && g.kkt <= c.kkt_factor * c.epsilon;  // solver_util.hpp:28-30
}

cp_termination finish(const GapOut& s, int64_t it, bool conv, double wall) {
  cp_termination t;
  std::memset(&t, 0, sizeof(t));
  t.f_primal = s.fp;
  t.f_dual = s.fd;
  t.gap = s.gap;
  t.iterations = it;
  t.converged = conv ? 1 : 0;
  t.wall_time = wall;
  return t;
}

// BestIterate (solver_util.hpp:72-85): device copies of the best-gap pair.
struct Best {
  double gap = std::numeric_limits<double>::infinity();
  GapOut s;
  bool have = false;
  void offer(Ctx& c, const GapOut& g, const double* X, const double* Z, double* Xb, double* Zb, int64_t m,
             int64_t me) {
    if (g.gap < gap) {
      gap = g.gap;
      s = g;
      have = true;
      copy_dev(c, Xb, X, m);
      copy_dev(c, Zb, Z, me);
    }
  }
};

// initial_point (solver_util.hpp:56-68)
void initial_point(Prob& P, bool warm, double* X, double* Z) {
  Ctx& c = *P.c;
  const int64_t m = P.d() * P.n(), me = P.d() * P.E();
  if (warm) {
    project_columns_dev(c, P.q, Z, P.rad, P.d(), P.E(), Z);
  } else {
    copy_dev(c, X, P.A->A.p, m);
    if (me) CPB_CUDA(cudaMemsetAsync(Z, 0, me * sizeof(double), c.s));
  }
}

// ---- SSNAL (ssnal.cpp:113-215) ------------------------------------------------------
cp_termination ssnal(Prob& P, const cp_solver_config& cfg, bool warm, double* Xout, double* Zout) {
  Ctx& c = *P.c;
  const auto t0 = Clock::now();
  const int64_t d = P.d(), n = P.n(), E = P.E(), m = d * n, me = d * E;
  // With a communicator the solve is node-partitioned: this
  // rank owns nodes [v0, v1) and the edges whose smaller endpoint it owns; node
  // arrays X, D stay full (replicated / all-gathered), edge passes and node
  // gathers cover the owned part (+ ghost edges), sums are all-reduced.
  struct PartScope {
    Ctx& c;
    PartScope(Ctx& c_, int64_t n_) : c(c_) {
      if (c.comm) c.own_v0 = c.comm->v0(n_), c.own_v1 = c.comm->v1(n_);
    }
    ~PartScope() { c.own_v0 = 0, c.own_v1 = -1; }
  } part_scope(c, n);
  const bool parted = c.comm != nullptr;
  const int64_t ov0 = parted ? c.own_v0 * d : 0, om = parted ? (c.own_v1 - c.own_v0) * d : m;
  auto pdot = [&](const double* a, const double* b) {  // <a, b> over the owned rows, all-reduced
    double v = dot_dev(c, a + ov0, b + ov0, om);
    if (parted) {
      std::vector<double> t{v};
      comm_allreduce_host(c, t);
      v = t[0];
    }
    return v;
  };
  auto assemble_z = [&](double* Zfull) {  // every rank's owned edge rows -> full Z on every rank
    if (!parted || E == 0) return;
    const EdgePart& ep = edge_part(c, *P.g);
    comm_allgatherv_rows(c, Zfull, ep.row0, ep.rows, d);
  };
  initial_point(P, warm, Xout, Zout);
  {
    GapOut s0 = eval_gap(P, Xout, Zout);
    trace_gap(c, cfg, 0, s0, since(t0));
    if (accepts(s0, cfg)) return finish(s0, 0, true, since(t0));
  }
  double* X = c.buf<double>("s.X", m);
  double* Xt = c.buf<double>("s.Xt", m);
  double* Z = Zout;
  double* V = c.buf<double>("s.V", me);
  double* Vt = c.buf<double>("s.Vt", me);
  double* nv = c.buf<double>("s.nv", 2 * E);  // q = inf keeps (theta, |S|) per edge
  double* nvt = c.buf<double>("s.nvt", 2 * E);
  double* thr = c.buf<double>("s.thr", E);
  double* ps = c.buf<double>("s.ps", E);
  double* jal = c.buf<double>("s.jal", E);
  double* jbe = c.buf<double>("s.jbe", E);
  double* G = c.buf<double>("s.G", m);
  // PCG work arrays hold P * ceil(n / P) rows when the Newton systems are
  // node-partitioned (in-place all-gathers of each rank's chunk)
  const int64_t mpad = c.comm ? c.comm->chunk(n) * c.comm->nranks * d : m;
  PcgWork w{c.buf<double>("s.D", mpad), c.buf<double>("s.r", mpad), c.buf<double>("s.p", mpad),
            c.buf<double>("s.Ap", mpad), c.buf<double>("s.diag", mpad)};
  double* Xb = c.buf<double>("s.Xb", m);
  double* Zb = c.buf<double>("s.Zb", me);
  copy_dev(c, X, Xout, m);

  const double eps = cfg.epsilon;
  double sigma = cfg.ssnal_sigma0;
  double feas_prev = std::numeric_limits<double>::infinity();
  double zz = dot_dev(c, Z, Z, me);
  Best best;
  cp_termination cnt;
  std::memset(&cnt, 0, sizeof(cnt));
  int64_t done = 0;
  const int64_t max_outer = resolved_max_iter(cfg);
  for (int64_t k = 1; k <= max_outer; ++k) {
    const double eps_k = std::max(eps / 10.0, std::pow(0.5, static_cast<double>(k)));
    make_thr(c, E, P.rad, sigma, thr);
    double phi = eval_phi(P, X, nullptr, 0.0, nullptr, Z, sigma, thr, zz, V, nv);
    bool v_at_x = true;  // V = X B + Z / sigma at the current X (false after a failed line search)
    for (int64_t j = 0; j < cfg.ssnal_newton_max; ++j) {
      const int64_t n_active = jac_params(P, nv, thr, ps, jal, jbe);
      if (trace_on()) trace(("newton active edges " + std::to_string(n_active) + " / " + std::to_string(E)).c_str());
      const double gnorm = std::sqrt(grad_diag(P, X, V, ps, jal, jbe, thr, sigma, G, w.diag, true));
      if (gnorm <= eps_k) break;
      ++cnt.newton;
      const double cg_tol = std::max(std::min(0.1, std::sqrt(gnorm)), 1e-12);
      PcgOut dir = pcg_newton(P, V, jal, jbe, thr, sigma, G, w, cg_tol, cfg.pcg_max_iter, n_active);
      cnt.cg += dir.iterations;
      cnt.hess_apply += dir.iterations;
      double* D = w.x;
      double descent = pdot(G, D);
      if (!(descent < 0.0)) {  // inexact CG returned a non-descent direction (ssnal.cpp:166-170)
        neg_dev(c, D + ov0, G + ov0, om);
        if (parted) comm_allgather(c, D, static_cast<size_t>(c.comm->chunk(n) * d));
        descent = -gnorm * gnorm;
      }
      double alpha = 1.0, trial = 0.0;
      bool ok = false;
      for (int bt = 0; bt < 60; ++bt) {
        trial = eval_phi(P, X, D, alpha, Xt, Z, sigma, thr, zz, Vt, nvt);
        ++cnt.armijo;
        if (trial <= phi + cfg.armijo_mu * alpha * descent) {
          ok = true;
          break;
        }
        alpha *= cfg.backtrack_beta;
      }
      if (ok) {
        std::swap(X, Xt);  // X + alpha D, bit-identical to the trial point
      } else {
        axpy_dev(c, X, X, alpha, D, m);  // reference quirk: alpha halved a 60th time (ssnal.cpp:172-179)
      }
      v_at_x = ok;
      std::swap(V, Vt);
      std::swap(nv, nvt);
      phi = trial;
    }
    jac_params(P, nv, thr, ps, jal, jbe);  // prox scale at the last accepted V
    MultOut mo = ssnal_multiplier(P, X, Z, V, ps, thr, sigma, v_at_x);
    zz = mo.zz;
    trace_gap(c, cfg, k, mo.gap, since(t0));
    if (accepts(mo.gap, cfg)) {
      copy_dev(c, Xout, X, m);
      assemble_z(Zout);
      cp_termination t = finish(mo.gap, k, true, since(t0));
      t.newton = cnt.newton, t.cg = cnt.cg, t.armijo = cnt.armijo, t.hess_apply = cnt.hess_apply;
      return t;
    }
    best.offer(c, mo.gap, X, Z, Xb, Zb, m, me);
    if (mo.feas > 0.5 * feas_prev) sigma = std::min(10.0 * sigma, 1e6);
    feas_prev = mo.feas;
    done = k;
    if (cfg.time_limit > 0.0 && since(t0) > cfg.time_limit) break;
  }
  copy_dev(c, Xout, Xb, m);
  copy_dev(c, Zout, Zb, me);
  assemble_z(Zout);
  cp_termination t = finish(best.s, done, false, since(t0));
  t.newton = cnt.newton, t.cg = cnt.cg, t.armijo = cnt.armijo, t.hess_apply = cnt.hess_apply;
  return t;
}

// Device -> host copy by the SMs through mapped pinned memory.  The path's
// per-gamma snapshots (4.4 GB at C3) used to go through the D2H copy engine,
// whose FIFO then held every small state read of the next solve (PCG state,
// gap partials, labels) behind the big copy, so the solve and the copies
// serialised (C3: 2.24 s solve + 1.63 s copies).  A few CTAs on the copy
// stream stream the snapshot over the host link instead, leaving the copy
// engine to the solver's reads.
__global__ void __launch_bounds__(256) k_to_host(const double* __restrict__ src, double* dst, int64_t n) {
  const int64_t stride = static_cast<int64_t>(gridDim.x) * blockDim.x;
  int64_t i = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x;
  for (; i + 3 * stride < n; i += 4 * stride) {
    const double a = __ldcs(src + i), b = __ldcs(src + i + stride), c = __ldcs(src + i + 2 * stride),
                 d = __ldcs(src + i + 3 * stride);
    dst[i] = a, dst[i + stride] = b, dst[i + 2 * stride] = c, dst[i + 3 * stride] = d;
  }
  for (; i < n; i += stride) dst[i] = __ldcs(src + i);
}

// ---- fast AMA (ama.cpp:17-89) ---------------------------------------------------------
// One captured CUDA graph (instantiated once, relaunched); counts its kernels into g_launches
// per launch so gpu_launches stays the number of kernels that ran.
struct GraphExec {
  cudaGraphExec_t exec = nullptr;
  unsigned long long kernels = 0;
  template <class F>
  void capture(cudaStream_t s, F&& body) {
    cudaGraph_t g = nullptr;
    const unsigned long long l0 = g_launches;
    CPB_CUDA(cudaStreamBeginCapture(s, cudaStreamCaptureModeThreadLocal));
    try {
      body();
    } catch (...) {
      cudaStreamEndCapture(s, &g);
      if (g) cudaGraphDestroy(g);
      throw;
    }
    CPB_CUDA(cudaStreamEndCapture(s, &g));
    kernels = g_launches - l0;
    g_launches = l0;
    const cudaError_t e = cudaGraphInstantiate(&exec, g, 0);
    cudaGraphDestroy(g);
    CPB_CUDA(e);
  }
  void launch(cudaStream_t s) {
    CPB_CUDA(cudaGraphLaunch(exec, s));
    g_launches += kernels;
  }
  GraphExec() = default;
  GraphExec(const GraphExec&) = delete;
  GraphExec& operator=(const GraphExec&) = delete;
  ~GraphExec() {
    if (exec) cudaGraphExecDestroy(exec);
  }
};

cp_termination fast_ama(Prob& P, const cp_solver_config& cfg, bool warm, double* Xout, double* Zout,
                        SolveCache& cache) {
  Ctx& c = *P.c;
  const auto t0 = Clock::now();
  const int64_t d = P.d(), n = P.n(), E = P.E(), m = d * n, me = d * E;
  initial_point(P, warm, Xout, Zout);
  {
    GapOut s0 = eval_gap(P, Xout, Zout);
    trace_gap(c, cfg, 0, s0, since(t0));
    if (accepts(s0, cfg)) return finish(s0, 0, true, since(t0));
  }
  double lmax;
  auto it = cache.lambda_max.find(P.g->uid);
  if (it != cache.lambda_max.end() && it->second > 0.0) {
    lmax = it->second;
  } else {
    lmax = laplacian_lambda_max(c, *P.g, 1e-9, 10000);
    cache.lambda_max[P.g->uid] = lmax;
  }
  if (!(lmax > 0.0)) runtime("fast AMA: spectral bound of B B^T is not positive");
  const double step = cfg.ama_step_safety / lmax;
  double* Zh = c.buf<double>("a.Zh", me);
  double* Zp = c.buf<double>("a.Zp", me);
  double* Xh = c.buf<double>("a.Xh", m);
  double* Xb = c.buf<double>("a.Xb", m);
  double* Zb = c.buf<double>("a.Zb", me);
  copy_dev(c, Zh, Zout, me);
  copy_dev(c, Zp, Zout, me);
  double t = 1.0;
  Best best;
  const int64_t max_iter = resolved_max_iter(cfg);
  int64_t k = 0;
  // Between two gap checks: small problems run the block as one cooperative kernel
  // (k_ama_block); otherwise every full 10-iteration block is one CUDA graph launch
  // (k_ama_mom + 10 x (B^T gather, edge step)) with the momenta computed on the device bitwise
  // like the host's, its t seeded once (graph blocks are consecutive).  Time limit checked
  // per block.
  constexpr int kBlk = 10;
  double* tm = c.buf<double>("a.tm", kBlk + 1);
  GraphExec blk;
  while (k < max_iter) {
    // the iterations up to the next gap check (ama.cpp: k == 1, every 10th, the last)
    const int64_t next = (k == 0) ? 1 : std::min<int64_t>((k / kBlk + 1) * kBlk, max_iter);
    const int cnt = static_cast<int>(next - k);
    double* parts = nullptr;
    const int fg = ama_block_fused(P, Xh, Zh, Zp, Xout, step, t, cnt, &parts);  // small problems: one kernel
    if (fg > 0) {
      for (int j = 0; j < cnt; ++j) t = 0.5 * (1.0 + std::sqrt(1.0 + 4.0 * t * t));  // host copy of t
    } else if (cnt == kBlk) {
      if (!blk.exec) {
        ama_set_t(P, tm, kBlk, t);
        blk.capture(c.s, [&] {
          ama_momenta(P, tm, kBlk);
          for (int j = 0; j < kBlk; ++j) {
            ama_primal(P, Zh, Xh);
            ama_dual_step(P, Xh, Zh, Zp, step, 0.0, tm + j);
          }
        });
      }
      blk.launch(c.s);
      for (int j = 0; j < kBlk; ++j) t = 0.5 * (1.0 + std::sqrt(1.0 + 4.0 * t * t));  // host copy of t
      ama_primal(P, Zp, Xout);  // X = A - Znew B^T (recover_primal)
    } else {
      for (int j = 0; j < cnt; ++j) {
        ama_primal(P, Zh, Xh);
        const double tn = 0.5 * (1.0 + std::sqrt(1.0 + 4.0 * t * t));
        ama_dual_step(P, Xh, Zh, Zp, step, (t - 1.0) / tn);
        t = tn;
      }
      ama_primal(P, Zp, Xout);  // X = A - Znew B^T (recover_primal)
    }
    k = next;
    GapOut s = fg > 0 ? gap_from_partials(P, parts, fg, fg) : eval_gap(P, Xout, Zp);
    trace_gap(c, cfg, k, s, since(t0));
    if (accepts(s, cfg)) {
      copy_dev(c, Zout, Zp, me);
      return finish(s, k, true, since(t0));
    }
    best.offer(c, s, Xout, Zp, Xb, Zb, m, me);
    if (cfg.time_limit > 0.0 && since(t0) > cfg.time_limit) break;
  }
  copy_dev(c, Xout, Xb, m);
  copy_dev(c, Zout, Zb, me);
  return finish(best.s, k, false, since(t0));
}

}  // namespace

// objective.cpp:38-61
int64_t resolved_max_iter(const cp_solver_config& c) {
  if (c.max_iter > 0) return c.max_iter;
  return c.algorithm == 2 ? 100 : 20000;
}
void validate_config(const cp_solver_config& c) {
  if (c.algorithm < 0 || c.algorithm > 2) invalid("solve: unknown algorithm");
  if (!(c.epsilon > 0.0) || !std::isfinite(c.epsilon)) invalid("config: epsilon must be positive and finite");
  if (!(c.kkt_factor > 0.0) || !std::isfinite(c.kkt_factor)) invalid("config: kkt_factor must be positive and finite");
  if (c.max_iter < 0) invalid("config: max_iter must be >= 0");
  if (!(c.admm_rho > 0.0)) invalid("config: admm_rho must be positive");
  if (!(c.ama_step_safety > 0.0) || c.ama_step_safety >= 1.0) invalid("config: ama_step_safety must lie in (0, 1)");
  if (!(c.ssnal_sigma0 > 0.0)) invalid("config: ssnal_sigma0 must be positive");
  if (!(c.armijo_mu > 0.0) || c.armijo_mu >= 0.5) invalid("config: armijo_mu must lie in (0, 0.5)");
  if (!(c.backtrack_beta > 0.0) || c.backtrack_beta >= 1.0) invalid("config: backtrack_beta must lie in (0, 1)");
  if (c.ssnal_newton_max < 1) invalid("config: ssnal_newton_max must be >= 1");
  if (c.pcg_max_iter < 1) invalid("config: pcg_max_iter must be >= 1");
}

cp_termination admm_solve(Prob& P, const cp_solver_config& cfg, bool warm, double* X, double* Z, SolveCache& cache);

cp_termination solve_dev(Prob& P, const cp_solver_config& cfg, bool warm, double* X, double* Z, SolveCache& cache) {
  validate_config(cfg);
  Ctx& c = *P.c;
  c.trace.clear();
  const int64_t m = P.d() * P.n();
  // trivial_solution (solver_util.hpp:44-51)
  if (!(P.gamma > 0.0) || P.E() == 0) {
    copy_dev(c, X, P.A->A.p, m);
    if (P.E()) CPB_CUDA(cudaMemsetAsync(Z, 0, P.E() * P.d() * sizeof(double), c.s));
    cp_termination t;
    std::memset(&t, 0, sizeof(t));
    t.converged = 1;
    return t;
  }
  switch (cfg.algorithm) {
    case 0: return admm_solve(P, cfg, warm, X, Z, cache);
    case 1: return fast_ama(P, cfg, warm, X, Z, cache);
    default: return ssnal(P, cfg, warm, X, Z);
  }
}

// ---- clusters (path.cpp:60-89) --------------------------------------------------------
namespace {
// Eigen-order squared norm of a row (or a row difference) by a quad of lanes,
// one lane per packet chain (esum in oracle/oracle.hpp).
__device__ double quad_sqnorm(const double* x, const double* y, int d, int sub, unsigned qm) {
  auto val = [&](int k) {
    const double t = y ? x[k] - y[k] : x[k];
    return t * t;
  };
  if (d < 4) {
    double r = val(0);
    if (d >= 2) r = r + val(1);
    if (d == 3) r = r + val(2);
    return r;
  }
  const int e2 = (d / 4) * 4;
  double acc = 0.0;
  for (int k = sub; k < e2; k += 4) acc = acc + val(k);
  const double c0 = __shfl_sync(qm, acc, 0, 4), c1 = __shfl_sync(qm, acc, 1, 4);
  const double c2 = __shfl_sync(qm, acc, 2, 4), c3 = __shfl_sync(qm, acc, 3, 4);
  double p0 = c0 + c2, p1 = c1 + c3;
  if (d - e2 >= 2) {
    p0 = p0 + val(e2);
    p1 = p1 + val(e2 + 1);
  }
  double r = p0 + p1;
  if (d & 1) r = r + val(d - 1);
  return r;
}
__device__ __forceinline__ unsigned quad_mask() { return 0xfu << ((threadIdx.x & 31u) & ~3u); }

__global__ void k_row_norm_max(const double* __restrict__ X, int64_t n, int d, double* part) {
  __shared__ double sh[32];
  const int sub = threadIdx.x & 3;
  const unsigned qm = quad_mask();
  double mx = 0.0;
  for (int64_t v = (blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x) >> 2; v < n;
       v += (static_cast<int64_t>(gridDim.x) * blockDim.x) >> 2)
    mx = fmax(mx, sqrt(quad_sqnorm(X + v * d, nullptr, d, sub, qm)));
  mx = block_max(mx, sh);
  if (threadIdx.x == 0) part[blockIdx.x] = mx;
}
__global__ void k_fused_edges(const double* __restrict__ X, const int* __restrict__ ei, const int* __restrict__ ej,
                              int64_t E, int d, const double* thr, unsigned char* flag) {
  const int sub = threadIdx.x & 3;
  const unsigned qm = quad_mask();
  const double t = *thr;
  for (int64_t l = (blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x) >> 2; l < E;
       l += (static_cast<int64_t>(gridDim.x) * blockDim.x) >> 2) {
    const double s = sqrt(quad_sqnorm(X + static_cast<int64_t>(ei[l]) * d, X + static_cast<int64_t>(ej[l]) * d, d,
                                      sub, qm));
    if (sub == 0) flag[l] = s <= t;
  }
}
__global__ void k_fuse_thr(const double* mx, double fuse_tol, double* thr) { *thr = fuse_tol * (1.0 + *mx); }
__global__ void k_count(const int* labels, int n, int* cnt) {
  for (int v = blockIdx.x * blockDim.x + threadIdx.x; v < n; v += gridDim.x * blockDim.x) atomicAdd(cnt + labels[v], 1);
}
// centroid(c, f) = (sum over members in ascending node order) / size (path.cpp:80-87)
__global__ void k_centroids(const double* __restrict__ X, const int* __restrict__ members, const int* __restrict__ coff,
                            int64_t K, int d, double* __restrict__ cent) {
  const int64_t total = K * d;
  for (int64_t p = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; p < total;
       p += static_cast<int64_t>(gridDim.x) * blockDim.x) {
    const int64_t cl = p / d;
    const int f = static_cast<int>(p % d);
    const int a = coff[cl], b = coff[cl + 1];
    double s = 0.0;
    for (int q = a; q < b; ++q) s = s + X[static_cast<int64_t>(members[q]) * d + f];
    cent[cl * d + f] = s / static_cast<double>(b - a);
  }
}
__global__ void k_iota2(int* p, int n) {
  for (int t = blockIdx.x * blockDim.x + threadIdx.x; t < n; t += gridDim.x * blockDim.x) p[t] = t;
}
}  // namespace

int64_t extract_clusters_dev(Ctx& c, const Graph& g, const double* X, int64_t d, double fuse_tol, int* labels,
                             double* centroids) {
  if (!(fuse_tol > 0.0)) invalid("extract_clusters: fuse_tol must be positive");
  const int64_t n = g.n, E = g.E;
  Ctx::Timer tm(&c, "extract_clusters", static_cast<double>(n) * d * 8.0 + 2.0 * E * 4.0);  // X once, the edge list
  const int grid = std::max(1, std::min(cdiv(4 * n, 256), c.sm_count * 4));
  double* part = c.buf<double>("cl.part", grid + 2);
  double* thr = c.buf<double>("cl.thr", 2);
  k_row_norm_max<<<grid, 256, 0, c.s>>>(X, n, static_cast<int>(d), part);
  CPB_LAUNCH_CHECK();
  reduce_max(c, part, grid, thr + 1);
  k_fuse_thr<<<1, 1, 0, c.s>>>(thr + 1, fuse_tol, thr);
  CPB_LAUNCH_CHECK();
  unsigned char* flag = c.buf<unsigned char>("cl.flag", E + 1);
  if (E > 0) {
    const int ge = std::max(1, std::min(cdiv(4 * E, 256), c.sm_count * 8));
    k_fused_edges<<<ge, 256, 0, c.s>>>(X, g.ei.p, g.ej.p, E, static_cast<int>(d), thr, flag);
    CPB_LAUNCH_CHECK();
  }
  const int64_t K = components_dev(c, g, flag, labels);
  if (centroids && n > 0) {
    int* cnt = c.buf<int>("cl.cnt", K + 1);
    int* coff = c.buf<int>("cl.coff", K + 1);
    int* node = c.buf<int>("cl.node", n);
    int* lab2 = c.buf<int>("cl.lab2", n);
    int* members = c.buf<int>("cl.members", n);
    CPB_CUDA(cudaMemsetAsync(cnt, 0, (K + 1) * sizeof(int), c.s));
    const int gn = std::max(1, std::min(cdiv(n, 256), c.sm_count * 4));
    k_count<<<gn, 256, 0, c.s>>>(labels, static_cast<int>(n), cnt);
    CPB_LAUNCH_CHECK();
    k_iota2<<<gn, 256, 0, c.s>>>(node, static_cast<int>(n));
    CPB_LAUNCH_CHECK();
    size_t bytes = 0;
    CPB_CUDA(cub::DeviceScan::ExclusiveSum(nullptr, bytes, cnt, coff, static_cast<int>(K + 1), c.s));
    void* tmp = c.buf<char>("cl.cub1", bytes + 16);
    CPB_CUDA(cub::DeviceScan::ExclusiveSum(tmp, bytes, cnt, coff, static_cast<int>(K + 1), c.s));
    int bits = 1;
    while ((1ll << bits) < K) ++bits;
    bytes = 0;
    CPB_CUDA(cub::DeviceRadixSort::SortPairs(nullptr, bytes, labels, lab2, node, members, static_cast<int>(n), 0, bits,
                                             c.s));
    tmp = c.buf<char>("cl.cub2", bytes + 16);
    CPB_CUDA(cub::DeviceRadixSort::SortPairs(tmp, bytes, labels, lab2, node, members, static_cast<int>(n), 0, bits,
                                             c.s));
    const int gc = std::max(1, std::min(cdiv(K * d, 256), c.sm_count * 8));
    k_centroids<<<gc, 256, 0, c.s>>>(X, members, coff, K, static_cast<int>(d), centroids);
    CPB_LAUNCH_CHECK();
  }
  return K;
}

// Host copies of whole output blocks, split over the process's CPUs (pinned outputs of a C3 path
// are GBs: one thread copies ~10 GB/s).
void host_copy_parallel(const std::vector<std::tuple<void*, const void*, size_t>>& segs, int spare = 0) {
  constexpr size_t kPiece = size_t(32) << 20;
  std::vector<std::tuple<char*, const char*, size_t>> pieces;
  for (const auto& sg : segs)
    for (size_t o = 0; o < std::get<2>(sg); o += kPiece)
      pieces.emplace_back(static_cast<char*>(std::get<0>(sg)) + o, static_cast<const char*>(std::get<1>(sg)) + o,
                          std::min(kPiece, std::get<2>(sg) - o));
  if (pieces.empty()) return;
  cpu_set_t cs;
  int cpus = 1;
  if (sched_getaffinity(0, sizeof(cs), &cs) == 0) cpus = CPU_COUNT(&cs);
  const int nt = std::max(1, std::min<int>({cpus - spare, 32, static_cast<int>(pieces.size())}));
  std::atomic<size_t> next{0};
  auto work = [&] {
    for (size_t i = next++; i < pieces.size(); i = next++)
      std::memcpy(std::get<0>(pieces[i]), std::get<1>(pieces[i]), std::get<2>(pieces[i]));
  };
  std::vector<std::thread> th;
  for (int i = 1; i < nt; ++i) th.emplace_back(work);
  work();
  for (auto& x : th) x.join();
}

// Host copies that wait for device work: a worker thread takes (event, blocks) items in order,
// waits for the event (the source blocks' device-to-host copy) and copies, while the path's
// solves go on.  The destructor drains the queue and joins.
class HostCopier {
 public:
  using Segs = std::vector<std::tuple<void*, const void*, size_t>>;
  explicit HostCopier(int dev) : dev_(dev) {}
  ~HostCopier() {
    join();
    for (auto e : events_) cudaEventDestroy(e);
  }
  cudaEvent_t record(cudaStream_t s) {  // an event owned by the copier, recorded on s
    cudaEvent_t e;
    CPB_CUDA(cudaEventCreateWithFlags(&e, cudaEventDisableTiming));
    events_.push_back(e);
    CPB_CUDA(cudaEventRecord(e, s));
    return e;
  }
  void push(cudaEvent_t after, Segs segs) {
    if (!th_.joinable()) th_ = std::thread([this] { loop(); });
    {
      std::lock_guard<std::mutex> lk(mu_);
      q_.emplace_back(after, std::move(segs));
    }
    cv_.notify_one();
  }
  void finish() {  // waits for every queued copy; rethrows the worker's error
    join();
    if (err_) std::rethrow_exception(std::exchange(err_, nullptr));
  }

 private:
  void join() {
    if (!th_.joinable()) return;
    {
      std::lock_guard<std::mutex> lk(mu_);
      done_ = true;
    }
    cv_.notify_one();
    th_.join();
  }
  void loop() {
    cudaSetDevice(dev_);
    for (;;) {
      std::pair<cudaEvent_t, Segs> it;
      {
        std::unique_lock<std::mutex> lk(mu_);
        cv_.wait(lk, [&] { return done_ || !q_.empty(); });
        if (q_.empty()) return;
        it = std::move(q_.front());
        q_.pop_front();
      }
      try {
        CPB_CUDA(cudaEventSynchronize(it.first));
        const auto t0 = std::chrono::steady_clock::now();
        host_copy_parallel(it.second, 2);  // two CPUs stay with the thread driving the solves
        if (trace_on()) {
          size_t b = 0;
          for (const auto& sg : it.second) b += std::get<2>(sg);
          const double ms = std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now() - t0).count();
          trace(("host copy " + std::to_string(b >> 20) + " MB in " + std::to_string(ms) + " ms").c_str());
        }
      } catch (...) {
        if (!err_) err_ = std::current_exception();
      }
    }
  }
  int dev_;
  std::thread th_;
  std::mutex mu_;
  std::condition_variable cv_;
  std::deque<std::pair<cudaEvent_t, Segs>> q_;
  bool done_ = false;
  std::exception_ptr err_;
  std::vector<cudaEvent_t> events_;
};

void run_path_dev(Ctx& c, Data& A, const Graph& g, int q, const double* gammas, int64_t T,
                  const cp_solver_config& cfg, const cp_path_options& opt, double* X_out, double* Z_out,
                  int64_t* labels_out, int64_t* K_out, cp_termination* terms_out, const cp_path_sink* sink) {
  if (T < 1) invalid("run_path: empty schedule");
  if (A.n != g.n) invalid("run_path: graph size does not match the data");
  if (q != 0 && q != 1 && q != 2) invalid("penalty norm exponent must be 1, 2 or 0 (infinity), got " + std::to_string(q));
  validate_config(cfg);
  // every gamma is validated before any work starts (ProblemInstance, objective.cpp:26-33), so
  // a bad value never leaves the caller's outputs half written
  for (int64_t t = 0; t < T; ++t)
    if (!(gammas[t] >= 0.0) || !std::isfinite(gammas[t])) invalid("instance: gamma must be finite and >= 0");
  if (opt.require_connected) {
    int* lab = c.buf<int>("path.lab0", g.n + 1);
    const int64_t comps = components_dev(c, g, nullptr, lab);
    if (comps > 1)
      runtime("run_path: graph has " + std::to_string(comps) + " connected components; full fusion is unreachable");
  }
  const int64_t d = A.d, n = A.n, E = g.E, m = d * n, me = d * E;
  double* X = c.buf<double>("path.X", m);
  double* Z = c.buf<double>("path.Z", me);
  double* rad = c.buf<double>("path.rad", E + 1);
  int* lab = c.buf<int>("path.lab", n + 1);
  std::vector<int> hl(static_cast<size_t>(n));
  SolveCache cache;
  bool warm = false;
  // Outputs in page-locked host memory (cp_host_alloc / cudaHostRegister)
  // are filled asynchronously, overlapped with the next gamma's solve.
  auto pinned = [](const void* p) {
    if (!p) return true;
    cudaPointerAttributes at;
    if (cudaPointerGetAttributes(&at, p) != cudaSuccess) {
      cudaGetLastError();
      return false;
    }
    return at.type == cudaMemoryTypeHost;
  };
  const bool async_out = (X_out || Z_out) && pinned(X_out) && pinned(Z_out) && c.copy_stream() != nullptr;
  cudaStream_t cs = async_out ? c.copy_stream() : nullptr;
  // device views of mapped pinned outputs (cp_host_alloc maps them): the SMs ship the snapshots
  auto mapped = [&](double* h) -> double* {
    if (!h || !async_out) return nullptr;
    void* dp = nullptr;
    if (cudaHostGetDevicePointer(&dp, h, 0) != cudaSuccess) {
      cudaGetLastError();
      return nullptr;
    }
    return static_cast<double*>(dp);
  };
  // mapped pinned outputs are written by a copy kernel; other host buffers go
  // through cudaMemcpyAsync on the copy engine
  double* mX = mapped(X_out);
  double* mZ = mapped(Z_out);
  // CTAs of the copy kernel: enough to fill the ~57 GB/s link, few enough to
  // leave the SMs to the solver (C3 e2e: 2 -> 4.53 s, 4 -> 3.24, 6 -> 3.26,
  // 8 -> 3.28, 16 -> 3.48, 32 -> 3.69; copy engine 3.88 s)
  const int d2h_ctas = 6;
  double* snapX[2] = {nullptr, nullptr};
  double* snapZ[2] = {nullptr, nullptr};
  // The copy stream may still be writing the caller's buffers when a solve
  // throws: drain it and release the events on every exit.
  struct AsyncGuard {
    cudaStream_t cs = nullptr;
    cudaEvent_t snap_ready[2] = {nullptr, nullptr}, copy_done[2] = {nullptr, nullptr};
    ~AsyncGuard() {
      if (cs) cudaStreamSynchronize(cs);
      for (int s = 0; s < 2; ++s) {
        if (snap_ready[s]) cudaEventDestroy(snap_ready[s]);
        if (copy_done[s]) cudaEventDestroy(copy_done[s]);
      }
    }
  } ag;
  ag.cs = cs;
  cudaEvent_t* snap_ready = ag.snap_ready;
  cudaEvent_t* copy_done = ag.copy_done;
  double* cent = nullptr;
  std::vector<double> hcent;
  if (sink && sink->centroids) cent = c.buf<double>("path.cent", m + 1);
  if (async_out) {
    for (int s = 0; s < 2; ++s) {
      snapX[s] = c.buf<double>(s ? "path.sX1" : "path.sX0", m + 1);
      if (Z_out) snapZ[s] = c.buf<double>(s ? "path.sZ1" : "path.sZ0", me + 1);
      CPB_CUDA(cudaEventCreateWithFlags(&snap_ready[s], cudaEventDisableTiming));
      CPB_CUDA(cudaEventCreateWithFlags(&copy_done[s], cudaEventDisableTiming));
      CPB_CUDA(cudaEventRecord(copy_done[s], cs));
    }
  }
  int64_t K_prev = -1;
  // A gamma whose warm start the solver accepted as is (X unchanged) after a projection that moved
  // nothing (Z unchanged) has the last shipped gamma's outputs bit for bit: its blocks are not
  // snapshotted or sent over the link again but copied on the host from that gamma's blocks.
  int64_t shipped = -1;
  cudaEvent_t shipped_done = nullptr;  // the last shipped gamma's device-to-host copy (async outputs)
  int dev = 0;
  CPB_CUDA(cudaGetDevice(&dev));
  HostCopier copier(dev);
  auto dup_segs = [&](int64_t t, int64_t src) {
    HostCopier::Segs segs;
    if (X_out) segs.emplace_back(X_out + t * m, X_out + src * m, m * sizeof(double));
    if (Z_out && me) segs.emplace_back(Z_out + t * me, Z_out + src * me, me * sizeof(double));
    return segs;
  };
  for (int64_t t = 0; t < T; ++t) {
    const double gamma = gammas[t];
    Prob P;
    P.c = &c;
    P.A = &A;
    P.g = &g;
    P.gamma = gamma;
    P.q = q;
    P.rad = rad;
    make_radii(c, g, gamma, rad);
    cp_termination term = solve_dev(P, cfg, warm, X, Z, cache);
    if (sink && sink->trace) sink->trace(sink->user, t, c.trace.data(), static_cast<int64_t>(c.trace.size()));
    // a warm start the solver accepted as is (0 iterations, gamma > 0, edges present) leaves X
    // bitwise unchanged, so the previous gamma's labels, K and centroids are this gamma's
    const bool x_unchanged = warm && term.iterations == 0 && gamma > 0.0 && E > 0 && K_prev >= 0;
    const int64_t K = x_unchanged ? K_prev : extract_clusters_dev(c, g, X, d, opt.fuse_tol, lab, cent);
    K_prev = K;
    if (cent && !(sink->skip_identity && K == n)) {  // ClusterAssignment::centroids (path.cpp:135)
      if (!x_unchanged) {
        hcent.resize(static_cast<size_t>(K * d));
        d2h(c, hcent.data(), cent, K * d * sizeof(double));
      }
      sink->centroids(sink->user, t, K, d, hcent.data());
    }
    if (terms_out) terms_out[t] = term;
    if (K_out) K_out[t] = K;
    if (labels_out) {
      if (!x_unchanged) d2h(c, hl.data(), lab, n * sizeof(int));
      for (int64_t i = 0; i < n; ++i) labels_out[t * n + i] = hl[static_cast<size_t>(i)];
    }
    const bool same_out = x_unchanged && shipped >= 0 && !c.comm && (X_out || Z_out) &&
                          (!Z_out || me == 0 || !last_projection_changed(c));
    if (same_out) {
      if (async_out)
        copier.push(shipped_done, dup_segs(t, shipped));  // after the source's copy, off this thread
      else
        host_copy_parallel(dup_segs(t, shipped));  // the source blocks are complete
    } else if (async_out) {
      shipped = t;
      // Snapshot the solution (D2D) and ship it to pinned host memory on the
      // copy stream while the next gamma is solved (double-buffered).
      const int s = static_cast<int>(t & 1);
      CPB_CUDA(cudaStreamWaitEvent(c.s, copy_done[s], 0));
      if (X_out) copy_dev(c, snapX[s], X, m);
      if (Z_out && me) copy_dev(c, snapZ[s], Z, me);
      CPB_CUDA(cudaEventRecord(snap_ready[s], c.s));
      CPB_CUDA(cudaStreamWaitEvent(cs, snap_ready[s], 0));
      auto ship = [&](double* host, double* mapped, const double* snap, int64_t cnt) {
        if (mapped) {
          k_to_host<<<d2h_ctas, 256, 0, cs>>>(snap, mapped, cnt);
          CPB_LAUNCH_CHECK();
        } else {
          CPB_CUDA(cudaMemcpyAsync(host, snap, cnt * sizeof(double), cudaMemcpyDeviceToHost, cs));
        }
      };
      if (X_out) ship(X_out + t * m, mX ? mX + t * m : nullptr, snapX[s], m);
      if (Z_out && me) ship(Z_out + t * me, mZ ? mZ + t * me : nullptr, snapZ[s], me);
      CPB_CUDA(cudaEventRecord(copy_done[s], cs));
      shipped_done = copier.record(cs);
    } else {
      shipped = t;
      if (X_out) d2h(c, X_out + t * m, X, m * sizeof(double));
      if (Z_out && me) d2h(c, Z_out + t * me, Z, me * sizeof(double));
    }
    warm = opt.warm_start != 0;
    trace("path gamma done");
  }
  if (async_out) CPB_CUDA(cudaStreamSynchronize(cs));
  copier.finish();
  c.sync();
}

}  // namespace cpb
