// TEST INFRASTRUCTURE ONLY (see oracle.hpp).  A flat C surface over the
// oracle so pytest (ctypes) and bench.py's CPU-baseline leg can drive it.
// Return codes follow the product C-ABI: 0 ok, 1 invalid_argument,
// 2 runtime_error; the message is kept per thread.
#include "oracle.hpp"

#include <chrono>
#include <cstring>

using namespace oracle;

namespace {
thread_local std::string g_err;

template <class F>
int guard(F f) {
  try {
    f();
    return 0;
  } catch (const std::invalid_argument& e) {
    g_err = e.what();
    return 1;
  } catch (const std::exception& e) {
    g_err = e.what();
    return 2;
  }
}

struct OGraph {
  Graph g;
  std::vector<double> d2;
};

Mat wrap(const double* p, Index r, Index c) {
  Mat m(r, c);
  if (r > 0 && c > 0) std::memcpy(m.v.data(), p, sizeof(double) * static_cast<size_t>(r * c));
  return m;
}
void put(const Mat& m, double* p) {
  if (m.size()) std::memcpy(p, m.v.data(), sizeof(double) * static_cast<size_t>(m.size()));
}
Norm nq(int q) {  // 0 encodes q = infinity (no reference counterpart)
  if (q == 0) return Norm::linf;
  if (q == 1) return Norm::l1;
  if (q == 2) return Norm::l2;
  throw std::invalid_argument("penalty norm exponent must be 1, 2 or 0 (infinity), got " + std::to_string(q));
}

}  // namespace

extern "C" {

// Layout-identical to cp_solver_config / cp_termination in include/cluspath_b200.h.
struct orc_config {
  int32_t algorithm, collect_trace;
  double epsilon, kkt_factor;
  int64_t max_iter;
  double time_limit, admm_rho, ama_step_safety, ssnal_sigma0, armijo_mu, backtrack_beta;
  int64_t ssnal_newton_max, pcg_max_iter;
};
struct orc_term {
  double f_primal, f_dual, gap;
  int64_t iterations;
  int32_t converged, pad;
  double wall_time;
  int64_t newton, cg, armijo, hess_apply;
};

static Config to_cfg(const orc_config* c) {
  Config k;
  if (!c) return k;
  if (c->algorithm < 0 || c->algorithm > 2) throw std::invalid_argument("solve: unknown algorithm");
  k.algorithm = static_cast<Algo>(c->algorithm);
  k.collect_trace = c->collect_trace != 0;
  k.epsilon = c->epsilon;
  k.kkt_factor = c->kkt_factor;
  k.max_iter = c->max_iter;
  k.time_limit = c->time_limit;
  k.admm_rho = c->admm_rho;
  k.ama_step_safety = c->ama_step_safety;
  k.ssnal_sigma0 = c->ssnal_sigma0;
  k.armijo_mu = c->armijo_mu;
  k.backtrack_beta = c->backtrack_beta;
  k.ssnal_newton_max = c->ssnal_newton_max;
  k.pcg_max_iter = c->pcg_max_iter;
  return k;
}
static void to_term(const Solution& s, orc_term* t) {
  if (!t) return;
  std::memset(t, 0, sizeof(*t));
  t->f_primal = s.term.f_primal;
  t->f_dual = s.term.f_dual;
  t->gap = s.term.gap;
  t->iterations = s.term.iterations;
  t->converged = s.term.converged ? 1 : 0;
  t->wall_time = s.term.wall_time;
  t->newton = s.counters.newton;
  t->cg = s.counters.cg;
  t->armijo = s.counters.armijo;
  t->hess_apply = s.counters.hess_apply;
}

const char* orc_error() { return g_err.c_str(); }

int orc_graph_new(int64_t n, const int64_t* i, const int64_t* j, const double* w, int64_t E, void** out) {
  return guard([&] {
    std::vector<Edge> e(static_cast<size_t>(E));
    for (int64_t l = 0; l < E; ++l) e[static_cast<size_t>(l)] = Edge{i[l], j[l], w[l]};
    *out = new OGraph{Graph(n, std::move(e)), {}};
  });
}
void orc_graph_free(void* g) { delete static_cast<OGraph*>(g); }
int64_t orc_graph_E(void* g) { return static_cast<OGraph*>(g)->g.E(); }
int64_t orc_graph_n(void* g) { return static_cast<OGraph*>(g)->g.n; }
void orc_graph_export(void* gp, int64_t* i, int64_t* j, double* w, double* d2) {
  auto* G = static_cast<OGraph*>(gp);
  for (int64_t l = 0; l < G->g.E(); ++l) {
    const Edge& e = G->g.edges[static_cast<size_t>(l)];
    if (i) i[l] = e.i;
    if (j) j[l] = e.j;
    if (w) w[l] = e.w;
    if (d2 && !G->d2.empty()) d2[l] = G->d2[static_cast<size_t>(l)];
  }
}
void orc_graph_degree(void* gp, int64_t* deg) {
  auto* G = static_cast<OGraph*>(gp);
  for (int64_t v = 0; v < G->g.n; ++v) deg[v] = G->g.degree[static_cast<size_t>(v)];
}
int64_t orc_graph_find(void* gp, int64_t i, int64_t j) {
  auto r = static_cast<OGraph*>(gp)->g.find_edge(i, j);
  return r ? *r : -1;
}

int orc_validate_data(const double* A, int64_t d, int64_t n) {
  return guard([&] { validate_data(wrap(A, d, n)); });
}

int orc_knn(const double* A, int64_t d, int64_t n, int64_t k, double phi, void** out) {
  return guard([&] {
    auto* G = new OGraph;
    try {
      G->g = knn_weights(wrap(A, d, n), k, phi, &G->d2);
    } catch (...) {
      delete G;
      throw;
    }
    *out = G;
  });
}

int orc_B(void* gp, const double* X, int64_t d, int64_t n, double* out) {
  return guard([&] {
    Mat o;
    incidence_apply(static_cast<OGraph*>(gp)->g, wrap(X, d, n), o);
    put(o, out);
  });
}
int orc_Bt(void* gp, const double* Z, int64_t d, int64_t E, double* out) {
  return guard([&] {
    Mat o;
    incidence_apply_t(static_cast<OGraph*>(gp)->g, wrap(Z, d, E), o);
    put(o, out);
  });
}
int orc_laplacian_dense(void* gp, double* out) {
  return guard([&] {
    const Graph& g = static_cast<OGraph*>(gp)->g;
    Csc L = laplacian(g);
    std::memset(out, 0, sizeof(double) * static_cast<size_t>(g.n * g.n));
    for (Index c = 0; c < g.n; ++c)
      for (Index p = L.colptr[static_cast<size_t>(c)]; p < L.colptr[static_cast<size_t>(c + 1)]; ++p)
        out[c * g.n + L.row[static_cast<size_t>(p)]] = L.val[static_cast<size_t>(p)];
  });
}
int orc_cc(void* gp, int64_t* labels, int64_t* K) {
  return guard([&] {
    auto l = connected_components(static_cast<OGraph*>(gp)->g);
    for (size_t v = 0; v < l.size(); ++v) labels[v] = l[v];
    *K = component_count(l);
  });
}

int orc_prox_columns(int q, const double* V, const double* t, int64_t d, int64_t E, double* out) {
  return guard([&] {
    Mat o;
    prox_columns_into(wrap(V, d, E), std::vector<double>(t, t + E), nq(q), o);
    put(o, out);
  });
}
int orc_project_columns(int q, const double* Z, const double* r, int64_t d, int64_t E, double* out) {
  return guard([&] {
    Mat o = wrap(Z, d, E);
    project_columns_inplace(o, std::vector<double>(r, r + E), nq(q));
    put(o, out);
  });
}
// Dense d x d matrix of the Jacobian element plus its (alpha, beta).
int orc_prox_jacobian(int q, const double* v, int64_t d, double t, double* J, double* alpha, double* beta) {
  return guard([&] {
    ProxJac P = prox_jacobian(v, d, t, nq(q));
    std::vector<double> e(static_cast<size_t>(d), 0.0);
    for (int64_t c = 0; c < d; ++c) {
      e.assign(static_cast<size_t>(d), 0.0);
      e[static_cast<size_t>(c)] = 1.0;
      P.apply(e.data(), d, J + c * d);
    }
    if (alpha) *alpha = P.alpha;
    if (beta) *beta = P.beta;
  });
}
int orc_prox_jacobian_diag(int q, const double* v, int64_t d, double t, double* diag) {
  return guard([&] {
    ProxJac P = prox_jacobian(v, d, t, nq(q));
    for (int64_t r = 0; r < d; ++r) diag[r] = P.diag(r);
  });
}
int orc_moreau(int q, const double* v, int64_t d, double t, double* res) {
  return guard([&] { *res = moreau_check(v, d, t, nq(q)); });
}
int orc_norms(int q, const double* v, int64_t d, double* nrm, double* dual) {
  return guard([&] {
    *nrm = norm_value(v, d, nq(q));
    *dual = dual_norm_value(v, d, nq(q));
  });
}

// PCG on a dense SPD matrix (optionally Jacobi with a per-row diagonal).
int orc_pcg_dense(const double* M, int64_t n, const double* rhs, int64_t m, const double* pdiag, double tol,
                  int64_t maxit, double* x, int64_t* iters, double* residual, int* converged) {
  return guard([&] {
    LinOp op = op_dense(wrap(M, n, n));
    LinOp pre;
    if (pdiag) pre = op_jacobi_vec(std::vector<double>(pdiag, pdiag + n));
    PcgOut r = pcg(op, wrap(rhs, n, m), pdiag ? &pre : nullptr, tol, maxit);
    put(r.x, x);
    *iters = r.iterations;
    *residual = r.residual;
    *converged = r.converged ? 1 : 0;
  });
}
int orc_power_dense(const double* M, int64_t n, double tol, int64_t maxit, double* out) {
  return guard([&] { *out = power_iteration(op_dense(wrap(M, n, n)), tol, maxit); });
}
int orc_power_laplacian(void* gp, double tol, int64_t maxit, double* out) {
  return guard([&] { *out = power_iteration(op_csc(laplacian(static_cast<OGraph*>(gp)->g)), tol, maxit); });
}
int orc_cholesky_solve(void* gp, double rho, const double* rhs, int64_t m, double* out) {
  return guard([&] {
    const Graph& g = static_cast<OGraph*>(gp)->g;
    Cholesky f(laplacian(g), rho);
    put(f.solve(wrap(rhs, g.n, m)), out);
  });
}

#define ORC_INST                                        \
  Mat Am = wrap(A, d, n);                               \
  const Graph& g = static_cast<OGraph*>(gp)->g;         \
  Instance in(Am, g, gamma, nq(q));

int orc_primal(const double* A, int64_t d, int64_t n, void* gp, double gamma, int q, const double* X, double* out) {
  return guard([&] {
    ORC_INST
    *out = primal_objective(in, wrap(X, d, n));
  });
}
int orc_dual(const double* A, int64_t d, int64_t n, void* gp, double gamma, int q, const double* Z, double* out) {
  return guard([&] {
    ORC_INST
    *out = dual_objective(in, wrap(Z, d, g.E()));
  });
}
int orc_kkt(const double* A, int64_t d, int64_t n, void* gp, double gamma, int q, const double* X, const double* Z,
            double* out) {
  return guard([&] {
    ORC_INST
    *out = kkt_residual(in, wrap(X, d, n), wrap(Z, d, g.E()));
  });
}
int orc_phi(const double* A, int64_t d, int64_t n, void* gp, double gamma, int q, const double* Z, double sigma,
            const double* X, double* out) {
  return guard([&] {
    ORC_INST
    *out = ssnal_phi_value(in, wrap(Z, d, g.E()), sigma, wrap(X, d, n));
  });
}
int orc_phi_grad(const double* A, int64_t d, int64_t n, void* gp, double gamma, int q, const double* Z, double sigma,
                 const double* X, double* out) {
  return guard([&] {
    ORC_INST
    put(ssnal_phi_gradient(in, wrap(Z, d, g.E()), sigma, wrap(X, d, n)), out);
  });
}
int orc_hess_apply(const double* A, int64_t d, int64_t n, void* gp, double gamma, int q, const double* Z,
                   double sigma, const double* X, const double* D, double* out) {
  return guard([&] {
    ORC_INST
    put(ssnal_hessian_apply(in, wrap(Z, d, g.E()), sigma, wrap(X, d, n), wrap(D, d, n)), out);
  });
}
int orc_solve(const double* A, int64_t d, int64_t n, void* gp, double gamma, int q, const orc_config* cfg,
              const double* warmX, int64_t wxd, int64_t wxn, const double* warmZ, int64_t wzd, int64_t wzE, double* X,
              double* Z, orc_term* term) {
  return guard([&] {
    ORC_INST
    Config c = to_cfg(cfg);
    Solution warm;
    if (warmX && warmZ) {
      warm.X = wrap(warmX, wxd, wxn);
      warm.Z = wrap(warmZ, wzd, wzE);
    }
    Solution s = solve(in, c, (warmX && warmZ) ? &warm : nullptr, nullptr);
    put(s.X, X);
    put(s.Z, Z);
    to_term(s, term);
  });
}
// Full path.  X: T x (d x n), Z: T x (d x E), labels: T x n, K: T.
int orc_run_path(const double* A, int64_t d, int64_t n, void* gp, int q, const double* gammas, int64_t T,
                 const orc_config* cfg, int warm_start, int require_connected, double fuse_tol, double* X, double* Z,
                 int64_t* labels, int64_t* K, orc_term* terms) {
  return guard([&] {
    Mat Am = wrap(A, d, n);
    const Graph& g = static_cast<OGraph*>(gp)->g;
    PathOut p = run_path(Am, g, nq(q), std::vector<double>(gammas, gammas + T), to_cfg(cfg), warm_start != 0,
                         require_connected != 0, fuse_tol);
    for (int64_t t = 0; t < T; ++t) {
      if (X) put(p.sols[static_cast<size_t>(t)].X, X + t * d * n);
      if (Z) put(p.sols[static_cast<size_t>(t)].Z, Z + t * d * g.E());
      if (labels)
        for (int64_t i = 0; i < n; ++i) labels[t * n + i] = p.clusters[static_cast<size_t>(t)].labels[static_cast<size_t>(i)];
      if (K) K[t] = p.clusters[static_cast<size_t>(t)].K;
      if (terms) to_term(p.sols[static_cast<size_t>(t)], terms + t);
    }
  });
}
int orc_extract_clusters(const double* X, int64_t d, int64_t n, void* gp, double fuse_tol, int64_t* labels,
                         int64_t* K, double* centroids) {
  return guard([&] {
    Clusters c = extract_clusters(wrap(X, d, n), static_cast<OGraph*>(gp)->g, fuse_tol);
    for (int64_t i = 0; i < n; ++i) labels[i] = c.labels[static_cast<size_t>(i)];
    *K = c.K;
    if (centroids) put(c.centroids, centroids);
  });
}
int orc_make_schedule(double start, double end, int64_t count, int geometric, double* out) {
  return guard([&] {
    auto v = make_schedule(start, end, count, geometric != 0);
    std::memcpy(out, v.data(), sizeof(double) * v.size());
  });
}
// centers: d x m column-major.
int orc_mixture(const double* centers, int64_t d, int64_t m, double spread, int64_t per_center, uint64_t seed,
                double* out) {
  return guard([&] {
    std::vector<std::vector<double>> c(static_cast<size_t>(m));
    for (int64_t k = 0; k < m; ++k) c[static_cast<size_t>(k)].assign(centers + k * d, centers + (k + 1) * d);
    put(gaussian_mixture(c, spread, per_center, seed), out);
  });
}
// Per-row k nearest (d2, j) lists of rows [r0, r1) (graph.cpp:79-88): all j != i,
// partial_sort of (dist, j) pairs; kd/kj are (r1 - r0) x k, row-major.
int orc_knn_rows(const double* A, int64_t d, int64_t n, int64_t k, int64_t r0, int64_t r1, double* kd,
                 int64_t* kj) {
  return guard([&] {
    if (k < 1 || k > n - 1 || r0 < 0 || r1 > n || r0 > r1) throw std::invalid_argument("orc_knn_rows: bad range");
    Mat Am = wrap(A, d, n);
    std::vector<std::pair<double, Index>> cand;
    for (Index i = r0; i < r1; ++i) {
      cand.clear();
      for (Index j = 0; j < n; ++j) {
        if (j == i) continue;
        const double* x = Am.col(i);
        const double* y = Am.col(j);
        cand.emplace_back(esum(d, [&](Index r) {
                            const double t = x[r] - y[r];
                            return t * t;
                          }),
                          j);
      }
      std::partial_sort(cand.begin(), cand.begin() + k, cand.end());
      for (Index m = 0; m < k; ++m) {
        kd[(i - r0) * k + m] = cand[static_cast<size_t>(m)].first;
        kj[(i - r0) * k + m] = cand[static_cast<size_t>(m)].second;
      }
    }
  });
}
// ---- CPU-baseline unit costs (bench.py cpu_baseline / --impl reference) ----------
// Seconds for the kNN of the first `rows` samples against all n (graph.cpp:90-103).
int orc_time_knn_rows(const double* A, int64_t d, int64_t n, int64_t k, int64_t rows, double* seconds) {
  return guard([&] {
    Mat Am = wrap(A, d, n);
    auto t0 = std::chrono::steady_clock::now();
    std::vector<std::pair<double, Index>> cand;
    volatile double sink = 0.0;
    for (Index i = 0; i < rows && i < n; ++i) {
      cand.clear();
      for (Index j = 0; j < n; ++j) {
        if (j == i) continue;
        const double* x = Am.col(i);
        const double* y = Am.col(j);
        cand.emplace_back(esum(d, [&](Index r) {
                            const double t = x[r] - y[r];
                            return t * t;
                          }),
                          j);
      }
      std::partial_sort(cand.begin(), cand.begin() + k, cand.end());
      sink = sink + cand[0].first;
    }
    *seconds = std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
  });
}
// Seconds per call of the SSNAL building blocks at (gamma, sigma), X = A, Z = 0:
// out[0] eval_phi, [1] gradient, [2] jacobians + Jacobi diagonal, [3] Hessian
// apply, [4] one PCG vector update (x, r, z, p, dots, row norms), [5] gap
// (primal + dual + KKT), [6] multiplier step (B X, envelope, projection).
int orc_time_ssnal_units(const double* A, int64_t d, int64_t n, void* gp, double gamma, int q, double sigma,
                         int reps, double* out) {
  return guard([&] {
    Mat Am = wrap(A, d, n);
    const Graph& g = static_cast<OGraph*>(gp)->g;
    Instance in(Am, g, gamma, nq(q));
    Mat Z(d, g.E(), 0.0), X = Am;
    const Index E = g.E();
    using C = std::chrono::steady_clock;
    auto secs = [](C::time_point a) { return std::chrono::duration<double>(C::now() - a).count(); };
    std::vector<double> thr = in.radii();
    for (double& x : thr) x /= sigma;
    double t[7] = {0, 0, 0, 0, 0, 0, 0};
    volatile double sink = 0.0;
    for (int r = 0; r < reps; ++r) {
      auto t0 = C::now();
      // eval_phi (ssnal.cpp:24-39)
      Mat V, PV;
      incidence_apply(g, X, V);
      for (Index k = 0; k < V.size(); ++k) V.v[static_cast<size_t>(k)] += Z.v[static_cast<size_t>(k)] / sigma;
      prox_columns_into(V, thr, in.q, PV);
      double env = 0.0;
      std::vector<double> diff(static_cast<size_t>(d));
      for (Index l = 0; l < E; ++l) {
        for (Index rr = 0; rr < d; ++rr) diff[static_cast<size_t>(rr)] = PV(rr, l) - V(rr, l);
        env += in.gamma * g.edges[static_cast<size_t>(l)].w * norm_value(PV.col(l), d, in.q) + 0.5 * sigma * sq_norm(diff.data(), d);
      }
      sink = sink + env;
      t[0] += secs(t0);
      t0 = C::now();
      Mat U(d, E), T;
      for (Index k = 0; k < U.size(); ++k) U.v[static_cast<size_t>(k)] = V.v[static_cast<size_t>(k)] - PV.v[static_cast<size_t>(k)];
      incidence_apply_t(g, U, T);
      Mat G(d, n);
      for (Index k = 0; k < G.size(); ++k) G.v[static_cast<size_t>(k)] = X.v[static_cast<size_t>(k)] - Am.v[static_cast<size_t>(k)] + sigma * T.v[static_cast<size_t>(k)];
      sink = sink + sq_norm(G.v.data(), G.size());
      t[1] += secs(t0);
      t0 = C::now();
      std::vector<ProxJac> J;
      J.reserve(static_cast<size_t>(E));
      for (Index l = 0; l < E; ++l) J.push_back(prox_jacobian(V.col(l), d, thr[static_cast<size_t>(l)], in.q));
      Mat dg(d, n, 1.0);
      for (Index l = 0; l < E; ++l) {
        const Edge& e = g.edges[static_cast<size_t>(l)];
        for (Index rr = 0; rr < d; ++rr) {
          const double c = sigma * (1.0 - J[static_cast<size_t>(l)].diag(rr));
          dg(rr, e.i) += c;
          dg(rr, e.j) += c;
        }
      }
      t[2] += secs(t0);
      t0 = C::now();
      Mat W;
      incidence_apply(g, G, W);
      std::vector<double> jw(static_cast<size_t>(d));
      for (Index l = 0; l < E; ++l) {
        J[static_cast<size_t>(l)].apply(W.col(l), d, jw.data());
        for (Index rr = 0; rr < d; ++rr) W(rr, l) = W(rr, l) - jw[static_cast<size_t>(rr)];
      }
      Mat T2;
      incidence_apply_t(g, W, T2);
      Mat H(d, n);
      for (Index k = 0; k < H.size(); ++k) H.v[static_cast<size_t>(k)] = G.v[static_cast<size_t>(k)] + sigma * T2.v[static_cast<size_t>(k)];
      t[3] += secs(t0);
      t0 = C::now();
      {
        Mat x(d, n, 0.0), rr = G, p = G;
        const double alpha = 0.5;
        for (Index k = 0; k < x.size(); ++k) x.v[static_cast<size_t>(k)] += alpha * p.v[static_cast<size_t>(k)];
        for (Index k = 0; k < rr.size(); ++k) rr.v[static_cast<size_t>(k)] -= alpha * H.v[static_cast<size_t>(k)];
        double worst = 0.0;
        for (Index i = 0; i < d; ++i) worst = std::max(worst, std::sqrt(ssum(n, [&](Index c) { return rr(i, c) * rr(i, c); })));
        Mat z(d, n);
        for (Index k = 0; k < z.size(); ++k) z.v[static_cast<size_t>(k)] = rr.v[static_cast<size_t>(k)] / dg.v[static_cast<size_t>(k)];
        const double rz = dotp(rr.v.data(), z.v.data(), rr.size());
        const double pAp = dotp(p.v.data(), H.v.data(), p.size());
        for (Index k = 0; k < p.size(); ++k) p.v[static_cast<size_t>(k)] = z.v[static_cast<size_t>(k)] + 0.3 * p.v[static_cast<size_t>(k)];
        sink = sink + worst + rz + pAp;
      }
      t[4] += secs(t0);
      t0 = C::now();
      sink = sink + primal_objective(in, X) + dual_objective(in, Z) + kkt_residual(in, X, Z);
      t[5] += secs(t0);
      t0 = C::now();
      {
        Mat XB;
        incidence_apply(g, X, XB);
        Mat Zenv(d, E), Zsum(d, E);
        for (Index k = 0; k < Zenv.size(); ++k) {
          Zenv.v[static_cast<size_t>(k)] = sigma * (V.v[static_cast<size_t>(k)] - PV.v[static_cast<size_t>(k)]);
          Zsum.v[static_cast<size_t>(k)] = Z.v[static_cast<size_t>(k)] + sigma * XB.v[static_cast<size_t>(k)];
        }
        project_columns_inplace(Zsum, in.radii(), in.q);
        sink = sink + max_abs(Zenv.v.data(), Zenv.size()) + max_abs(Zsum.v.data(), Zsum.size());
      }
      t[6] += secs(t0);
    }
    for (int k = 0; k < 7; ++k) out[k] = t[k] / reps;
  });
}

// N(0,1) draws of libstdc++ normal_distribution over mt19937_64(seed).
void orc_normals(uint64_t seed, int64_t count, double* out) {
  std::mt19937_64 rng(seed);
  std::normal_distribution<double> g(0.0, 1.0);
  for (int64_t k = 0; k < count; ++k) out[k] = g(rng);
}

}  // extern "C"
