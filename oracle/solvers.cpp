// TEST INFRASTRUCTURE ONLY (see oracle.hpp).  Restates objective.cpp,
// solver_util.hpp, ssnal.cpp, admm.cpp, ama.cpp, path.cpp and the Gaussian
// mixture generator of io.cpp.
#include "oracle.hpp"

#include <chrono>
#include <limits>

namespace oracle {

using Clock = std::chrono::steady_clock;
static double since(Clock::time_point t0) { return std::chrono::duration<double>(Clock::now() - t0).count(); }

// objective.cpp:43-61
void Config::validate() const {
  if (!(epsilon > 0.0) || !std::isfinite(epsilon)) throw std::invalid_argument("config: epsilon must be positive and finite");
  if (!(kkt_factor > 0.0) || !std::isfinite(kkt_factor)) throw std::invalid_argument("config: kkt_factor must be positive and finite");
  if (max_iter < 0) throw std::invalid_argument("config: max_iter must be >= 0");
  if (!(admm_rho > 0.0)) throw std::invalid_argument("config: admm_rho must be positive");
  if (!(ama_step_safety > 0.0) || ama_step_safety >= 1.0) throw std::invalid_argument("config: ama_step_safety must lie in (0, 1)");
  if (!(ssnal_sigma0 > 0.0)) throw std::invalid_argument("config: ssnal_sigma0 must be positive");
  if (!(armijo_mu > 0.0) || armijo_mu >= 0.5) throw std::invalid_argument("config: armijo_mu must lie in (0, 0.5)");
  if (!(backtrack_beta > 0.0) || backtrack_beta >= 1.0) throw std::invalid_argument("config: backtrack_beta must lie in (0, 1)");
  if (ssnal_newton_max < 1) throw std::invalid_argument("config: ssnal_newton_max must be >= 1");
  if (pcg_max_iter < 1) throw std::invalid_argument("config: pcg_max_iter must be >= 1");
}

// objective.cpp:26-36
Instance::Instance(const Mat& A_, const Graph& g_, double gamma_, Norm q_) : A(&A_), g(&g_), gamma(gamma_), q(q_) {
  if (A_.cols != g_.n) throw std::invalid_argument("instance: graph node count does not match the sample count");
  if (!(gamma >= 0.0) || !std::isfinite(gamma)) throw std::invalid_argument("instance: gamma must be finite and >= 0");
}
std::vector<double> Instance::radii() const {
  std::vector<double> r(static_cast<size_t>(E()));
  for (Index l = 0; l < E(); ++l) r[static_cast<size_t>(l)] = gamma * g->edges[static_cast<size_t>(l)].w;
  return r;
}

namespace {
Mat sub(const Mat& a, const Mat& b) {
  Mat o(a.rows, a.cols);
  par_for(a.size(), [&](Index k) { o.v[static_cast<size_t>(k)] = a.v[static_cast<size_t>(k)] - b.v[static_cast<size_t>(k)]; });
  return o;
}
double sqn(const Mat& a) { return sq_norm(a.v.data(), a.size()); }
double fro(const Mat& a) { return std::sqrt(sqn(a)); }
// max is exact in any order
double maxabs(const Mat& a) {
  const Index T = threads();
  std::vector<double> part(static_cast<size_t>(T), 0.0);
  par_ranges(a.size(), [&](Index lo, Index hi) {
    const Index t = a.size() ? lo * T / a.size() : 0;
    part[static_cast<size_t>(std::min(t, T - 1))] = max_abs(a.v.data() + lo, hi - lo);
  });
  double m = 0.0;
  for (double x : part) m = std::max(m, x);
  return m;
}
// per-column terms in parallel, summed sequentially in ascending l
template <class F>
double colsum(Index E, F term) {
  std::vector<double> t(static_cast<size_t>(E));
  par_for(E, [&](Index l) { t[static_cast<size_t>(l)] = term(l); });
  double acc = 0.0;
  for (double x : t) acc += x;
  return acc;
}
}  // namespace

// objective.cpp:63-74
double primal_objective(const Instance& in, const Mat& X) {
  if (X.rows != in.d() || X.cols != in.n()) throw std::invalid_argument("primal_objective: X has the wrong shape");
  const double value = 0.5 * sqn(sub(X, *in.A));
  if (in.E() == 0 || in.gamma == 0.0) return value;
  Mat D;
  incidence_apply(*in.g, X, D);
  const double pen = colsum(D.cols, [&](Index l) { return in.g->edges[static_cast<size_t>(l)].w * norm_value(D.col(l), D.rows, in.q); });
  return value + in.gamma * pen;
}

// objective.cpp:76-88
double dual_objective(const Instance& in, const Mat& Z) {
  if (Z.rows != in.d() || Z.cols != in.E()) throw std::invalid_argument("dual_objective: Z has the wrong shape");
  std::vector<char> bad(static_cast<size_t>(Z.cols), 0);
  par_for(Z.cols, [&](Index l) {
    const double radius = in.gamma * in.g->edges[static_cast<size_t>(l)].w;
    bad[static_cast<size_t>(l)] = dual_norm_value(Z.col(l), Z.rows, in.q) > radius + 1e-9;
  });
  for (Index l = 0; l < Z.cols; ++l)
    if (bad[static_cast<size_t>(l)])
      throw std::invalid_argument("dual_objective: Z violates the dual-ball constraint on edge " + std::to_string(l));
  Mat ZBt;
  incidence_apply_t(*in.g, Z, ZBt);
  return -0.5 * sqn(ZBt) + dotp(ZBt.v.data(), in.A->v.data(), ZBt.size());
}

double duality_gap(double fp, double fd) { return std::abs(fp - fd) / (1.0 + std::abs(fp) + std::abs(fd)); }

Mat recover_primal(const Instance& in, const Mat& Z) {
  if (Z.rows != in.d() || Z.cols != in.E()) throw std::invalid_argument("recover_primal: Z has the wrong shape");
  Mat ZBt;
  incidence_apply_t(*in.g, Z, ZBt);
  return sub(*in.A, ZBt);
}

// objective.cpp:100-113
double kkt_residual(const Instance& in, const Mat& X, const Mat& Z) {
  if (X.rows != in.d() || X.cols != in.n()) throw std::invalid_argument("kkt_residual: X has the wrong shape");
  if (Z.rows != in.d() || Z.cols != in.E()) throw std::invalid_argument("kkt_residual: Z has the wrong shape");
  Mat ZBt;
  incidence_apply_t(*in.g, Z, ZBt);
  Mat S(X.rows, X.cols);
  par_for(S.size(), [&](Index k) {
    S.v[static_cast<size_t>(k)] = X.v[static_cast<size_t>(k)] - in.A->v[static_cast<size_t>(k)] + ZBt.v[static_cast<size_t>(k)];
  });
  const double stat = fro(S) / (1.0 + fro(*in.A));
  if (in.E() == 0 || in.gamma == 0.0) return stat;
  Mat XB, P;
  incidence_apply(*in.g, X, XB);
  Mat W(XB.rows, XB.cols);
  par_for(W.size(), [&](Index k) { W.v[static_cast<size_t>(k)] = XB.v[static_cast<size_t>(k)] + Z.v[static_cast<size_t>(k)]; });
  prox_columns_into(W, in.radii(), in.q, P);
  const double align = fro(sub(XB, P)) / (1.0 + fro(XB) + fro(Z));
  return std::max(stat, align);
}

// ---- solver_util.hpp -------------------------------------------------------
namespace {
struct Gap {
  double fp = 0, fd = 0, gap = 0, kkt = 0;
  bool accepts(const Config& c) const { return gap <= c.epsilon && kkt <= c.kkt_factor * c.epsilon; }
};
Gap evaluate_gap(const Instance& in, const Mat& X, const Mat& Z) {
  Gap g;
  g.fp = primal_objective(in, X);
  g.fd = dual_objective(in, Z);
  g.gap = duality_gap(g.fp, g.fd);
  g.kkt = kkt_residual(in, X, Z);
  return g;
}
bool trivial(const Instance& in, Solution& sol) {
  if (in.gamma > 0.0 && in.E() > 0) return false;
  sol.X = *in.A;
  sol.Z = Mat(in.d(), in.E(), 0.0);
  sol.term.converged = true;
  return true;
}
void initial_point(const Instance& in, const Solution* warm, Mat& X, Mat& Z) {
  if (warm) {
    if (warm->X.rows != in.d() || warm->X.cols != in.n() || warm->Z.rows != in.d() || warm->Z.cols != in.E())
      throw std::invalid_argument("warm start does not match the instance shapes");
    X = warm->X;
    Z = warm->Z;
    project_columns_inplace(Z, in.radii(), in.q);
  } else {
    X = *in.A;
    Z = Mat(in.d(), in.E(), 0.0);
  }
}
struct Best {
  Mat X, Z;
  Gap s;
  double best = std::numeric_limits<double>::infinity();
  void offer(const Mat& X_, const Mat& Z_, const Gap& g) {
    if (g.gap < best) {
      best = g.gap;
      X = X_;
      Z = Z_;
      s = g;
    }
  }
};
Solution finish(Mat X, Mat Z, const Gap& s, Index it, bool conv, double wall, const Counters& cnt) {
  Solution sol;
  sol.X = std::move(X);
  sol.Z = std::move(Z);
  sol.term.f_primal = s.fp;
  sol.term.f_dual = s.fd;
  sol.term.gap = s.gap;
  sol.term.iterations = it;
  sol.term.converged = conv;
  sol.term.wall_time = wall;
  sol.counters = cnt;
  return sol;
}
bool over_time(const Config& c, Clock::time_point t0) { return c.time_limit > 0.0 && since(t0) > c.time_limit; }

// ---- ssnal.cpp:24-82 --------------------------------------------------------
struct Phi {
  Mat V, PV;
  double value = 0.0;
};
Phi eval_phi(const Instance& in, const Mat& Z, double sigma, const std::vector<double>& thr, const Mat& X) {
  Phi e;
  incidence_apply(*in.g, X, e.V);
  par_for(e.V.size(), [&](Index k) { e.V.v[static_cast<size_t>(k)] += Z.v[static_cast<size_t>(k)] / sigma; });
  prox_columns_into(e.V, thr, in.q, e.PV);
  const Index d = e.V.rows;
  const double env = colsum(e.V.cols, [&](Index l) {
    std::vector<double> diff(static_cast<size_t>(d));
    const double w = in.g->edges[static_cast<size_t>(l)].w;
    for (Index r = 0; r < d; ++r) diff[static_cast<size_t>(r)] = e.PV(r, l) - e.V(r, l);
    return in.gamma * w * norm_value(e.PV.col(l), d, in.q) + 0.5 * sigma * sq_norm(diff.data(), d);
  });
  e.value = 0.5 * sqn(sub(X, *in.A)) + env - sqn(Z) / (2.0 * sigma);
  return e;
}
Mat phi_grad(const Instance& in, double sigma, const Mat& X, const Phi& e) {
  Mat T, U = sub(e.V, e.PV);
  incidence_apply_t(*in.g, U, T);
  Mat G(X.rows, X.cols);
  par_for(G.size(), [&](Index k) {
    G.v[static_cast<size_t>(k)] = X.v[static_cast<size_t>(k)] - in.A->v[static_cast<size_t>(k)] + sigma * T.v[static_cast<size_t>(k)];
  });
  return G;
}
std::vector<ProxJac> edge_jacobians(const Instance& in, const Mat& V, const std::vector<double>& thr) {
  std::vector<ProxJac> J(static_cast<size_t>(V.cols));
  par_for(V.cols, [&](Index l) { J[static_cast<size_t>(l)] = prox_jacobian(V.col(l), V.rows, thr[static_cast<size_t>(l)], in.q); });
  return J;
}
Mat hess_apply(const Instance& in, double sigma, const Mat& D, const std::vector<ProxJac>& J) {
  Mat W;
  incidence_apply(*in.g, D, W);
  par_ranges(W.cols, [&](Index lo, Index hi) {
    std::vector<double> jw(static_cast<size_t>(W.rows));
    for (Index l = lo; l < hi; ++l) {
      J[static_cast<size_t>(l)].apply(W.col(l), W.rows, jw.data());
      for (Index r = 0; r < W.rows; ++r) W(r, l) = W(r, l) - jw[static_cast<size_t>(r)];
    }
  });
  Mat T;
  incidence_apply_t(*in.g, W, T);
  Mat H(D.rows, D.cols);
  par_for(H.size(), [&](Index k) { H.v[static_cast<size_t>(k)] = D.v[static_cast<size_t>(k)] + sigma * T.v[static_cast<size_t>(k)]; });
  return H;
}
Mat hess_diag(const Instance& in, double sigma, const std::vector<ProxJac>& J) {
  Mat g(in.d(), in.n(), 1.0);
  // node ranges per thread, ascending l within each (the sequential order per node)
  par_ranges(in.n(), [&](Index lo, Index hi) {
    for (Index l = 0; l < in.E(); ++l) {
      const Edge& e = in.g->edges[static_cast<size_t>(l)];
      const bool in_i = e.i >= lo && e.i < hi, in_j = e.j >= lo && e.j < hi;
      if (!in_i && !in_j) continue;
      for (Index r = 0; r < in.d(); ++r) {
        const double c = sigma * (1.0 - J[static_cast<size_t>(l)].diag(r));
        if (in_i) g(r, e.i) += c;
        if (in_j) g(r, e.j) += c;
      }
    }
  });
  return g;
}
std::vector<double> thresholds(const Instance& in, double sigma) {
  std::vector<double> t = in.radii();
  for (double& x : t) x /= sigma;
  return t;
}
}  // namespace

double ssnal_phi_value(const Instance& in, const Mat& Z, double sigma, const Mat& X) {
  return eval_phi(in, Z, sigma, thresholds(in, sigma), X).value;
}
Mat ssnal_phi_gradient(const Instance& in, const Mat& Z, double sigma, const Mat& X) {
  Phi e = eval_phi(in, Z, sigma, thresholds(in, sigma), X);
  return phi_grad(in, sigma, X, e);
}
Mat ssnal_hessian_apply(const Instance& in, const Mat& Z, double sigma, const Mat& X, const Mat& D) {
  auto t = thresholds(in, sigma);
  Phi e = eval_phi(in, Z, sigma, t, X);
  return hess_apply(in, sigma, D, edge_jacobians(in, e.V, t));
}

// ssnal.cpp:113-215
Solution solve_ssnal(const Instance& in, const Config& c, const Solution* warm, Cache*) {
  c.validate();
  const auto t0 = Clock::now();
  Solution triv;
  if (trivial(in, triv)) return triv;
  Mat X, Z;
  initial_point(in, warm, X, Z);
  Counters cnt;
  const double eps = c.epsilon;
  {
    Gap s0 = evaluate_gap(in, X, Z);
    if (s0.accepts(c)) return finish(std::move(X), std::move(Z), s0, 0, true, since(t0), cnt);
  }
  const std::vector<double> radii = in.radii();
  const Index d = in.d(), n = in.n();
  double sigma = c.ssnal_sigma0;
  double feas_prev = std::numeric_limits<double>::infinity();
  Best best;
  Index done = 0;
  const Index max_outer = c.resolved_max_iter();
  for (Index k = 1; k <= max_outer; ++k) {
    const double eps_k = std::max(eps / 10.0, std::pow(0.5, static_cast<double>(k)));
    const std::vector<double> thr = thresholds(in, sigma);
    Phi e = eval_phi(in, Z, sigma, thr, X);
    for (Index j = 0; j < c.ssnal_newton_max; ++j) {
      Mat G = phi_grad(in, sigma, X, e);
      const double gnorm = fro(G);
      if (gnorm <= eps_k) break;
      ++cnt.newton;
      auto J = edge_jacobians(in, e.V, thr);
      LinOp H;
      H.rows = d;
      H.fn = [&](const Mat& Dm) {
        ++cnt.hess_apply;
        return hess_apply(in, sigma, Dm, J);
      };
      LinOp pre = op_jacobi(hess_diag(in, sigma, J));
      const double cg_tol = std::min(0.1, std::sqrt(gnorm));
      Mat rhs(G.rows, G.cols);
      par_for(G.size(), [&](Index q) { rhs.v[static_cast<size_t>(q)] = -G.v[static_cast<size_t>(q)]; });
      PcgOut dir = pcg(H, rhs, &pre, std::max(cg_tol, 1e-12), c.pcg_max_iter);
      cnt.cg += dir.iterations;
      Mat D = std::move(dir.x);
      double descent = dotp(G.v.data(), D.v.data(), G.size());
      if (!(descent < 0.0)) {
        D = rhs;
        descent = -gnorm * gnorm;
      }
      double alpha = 1.0;
      Phi trial;
      Mat Xt(d, n);
      for (int bt = 0; bt < 60; ++bt) {
        par_for(X.size(), [&](Index q) { Xt.v[static_cast<size_t>(q)] = X.v[static_cast<size_t>(q)] + alpha * D.v[static_cast<size_t>(q)]; });
        trial = eval_phi(in, Z, sigma, thr, Xt);
        ++cnt.armijo;
        if (trial.value <= e.value + c.armijo_mu * alpha * descent) break;
        alpha *= c.backtrack_beta;
      }
      par_for(X.size(), [&](Index q) { X.v[static_cast<size_t>(q)] += alpha * D.v[static_cast<size_t>(q)]; });
      e = std::move(trial);
    }
    Mat XB;
    incidence_apply(*in.g, X, XB);
    {
      Mat Zenv(d, in.E()), Zsum(d, in.E());
      par_for(Zenv.size(), [&](Index q) {
        Zenv.v[static_cast<size_t>(q)] = sigma * (e.V.v[static_cast<size_t>(q)] - e.PV.v[static_cast<size_t>(q)]);
        Zsum.v[static_cast<size_t>(q)] = Z.v[static_cast<size_t>(q)] + sigma * XB.v[static_cast<size_t>(q)];
      });
      const double scale = 1.0 + maxabs(Zsum);
      project_columns_inplace(Zsum, radii, in.q);
      if (maxabs(sub(Zenv, Zsum)) > 1e-10 * scale) throw std::runtime_error("ssnal: multiplier self-check failed");
      Z = std::move(Zsum);
    }
    Gap s = evaluate_gap(in, X, Z);
    if (s.accepts(c)) return finish(std::move(X), std::move(Z), s, k, true, since(t0), cnt);
    best.offer(X, Z, s);
    const double feas = fro(sub(XB, e.PV)) / (1.0 + fro(XB));
    if (feas > 0.5 * feas_prev) sigma = std::min(10.0 * sigma, 1e6);
    feas_prev = feas;
    done = k;
    if (over_time(c, t0)) break;
  }
  return finish(std::move(best.X), std::move(best.Z), best.s, done, false, since(t0), cnt);
}

// admm.cpp:16-87
Solution solve_admm(const Instance& in, const Config& c, const Solution* warm, Cache* cache) {
  c.validate();
  const auto t0 = Clock::now();
  Solution triv;
  if (trivial(in, triv)) return triv;
  Mat X, Lam;
  initial_point(in, warm, X, Lam);
  Counters cnt;
  {
    Gap s0 = evaluate_gap(in, X, Lam);
    if (s0.accepts(c)) return finish(std::move(X), std::move(Lam), s0, 0, true, since(t0), cnt);
  }
  const double rho = c.admm_rho;
  std::shared_ptr<const Cholesky> fac;
  if (cache && cache->factor && cache->factor_rho == rho && cache->factor->n == in.n()) {
    fac = cache->factor;
  } else {
    fac = std::make_shared<Cholesky>(laplacian(*in.g), rho);
    if (cache) {
      cache->factor = fac;
      cache->factor_rho = rho;
    }
  }
  const std::vector<double> radii = in.radii();
  std::vector<double> thr = radii;
  for (double& x : thr) x /= rho;
  const Index d = in.d(), n = in.n(), E = in.E();
  Mat XB;
  incidence_apply(*in.g, X, XB);
  Mat U = XB, V(d, E), W(d, E), T, Zc;
  Best best;
  const Index max_iter = c.resolved_max_iter();
  for (Index k = 1; k <= max_iter; ++k) {
    for (Index q = 0; q < W.size(); ++q) W.v[static_cast<size_t>(q)] = rho * U.v[static_cast<size_t>(q)] - Lam.v[static_cast<size_t>(q)];
    incidence_apply_t(*in.g, W, T);
    Mat RHS(n, d);  // transposed right-hand side: d columns of length n
    for (Index i = 0; i < n; ++i)
      for (Index r = 0; r < d; ++r) RHS(i, r) = (*in.A)(r, i) + T(r, i);
    Mat sol = fac->solve(RHS);
    for (Index i = 0; i < n; ++i)
      for (Index r = 0; r < d; ++r) X(r, i) = sol(i, r);
    incidence_apply(*in.g, X, XB);
    for (Index q = 0; q < V.size(); ++q) V.v[static_cast<size_t>(q)] = XB.v[static_cast<size_t>(q)] + Lam.v[static_cast<size_t>(q)] / rho;
    prox_columns_into(V, thr, in.q, U);
    for (Index q = 0; q < Lam.size(); ++q) Lam.v[static_cast<size_t>(q)] += rho * (XB.v[static_cast<size_t>(q)] - U.v[static_cast<size_t>(q)]);
    Zc = Lam;
    project_columns_inplace(Zc, radii, in.q);
    Gap s = evaluate_gap(in, X, Zc);
    if (s.accepts(c)) return finish(std::move(X), std::move(Zc), s, k, true, since(t0), cnt);
    best.offer(X, Zc, s);
    if (over_time(c, t0)) return finish(std::move(best.X), std::move(best.Z), best.s, k, false, since(t0), cnt);
  }
  return finish(std::move(best.X), std::move(best.Z), best.s, max_iter, false, since(t0), cnt);
}

// ama.cpp:17-89
Solution solve_ama(const Instance& in, const Config& c, const Solution* warm, Cache* cache) {
  c.validate();
  const auto t0 = Clock::now();
  Solution triv;
  if (trivial(in, triv)) return triv;
  Mat X, Z;
  initial_point(in, warm, X, Z);
  Counters cnt;
  {
    Gap s0 = evaluate_gap(in, X, Z);
    if (s0.accepts(c)) return finish(std::move(X), std::move(Z), s0, 0, true, since(t0), cnt);
  }
  double lmax;
  if (cache && cache->lambda_max > 0.0) {
    lmax = cache->lambda_max;
  } else {
    lmax = power_iteration(op_csc(laplacian(*in.g)));
    if (cache) cache->lambda_max = lmax;
  }
  if (!(lmax > 0.0)) throw std::runtime_error("fast AMA: spectral bound of B B^T is not positive");
  const double step = c.ama_step_safety / lmax;
  const std::vector<double> radii = in.radii();
  Mat Zhat = Z, Zprev = Z, T, G, Znew(Z.rows, Z.cols);
  double t = 1.0;
  Best best;
  const Index max_iter = c.resolved_max_iter();
  Index k = 0;
  while (k < max_iter) {
    ++k;
    incidence_apply_t(*in.g, Zhat, T);
    for (Index q = 0; q < T.size(); ++q) T.v[static_cast<size_t>(q)] = in.A->v[static_cast<size_t>(q)] - T.v[static_cast<size_t>(q)];
    incidence_apply(*in.g, T, G);
    for (Index q = 0; q < Znew.size(); ++q) Znew.v[static_cast<size_t>(q)] = Zhat.v[static_cast<size_t>(q)] + step * G.v[static_cast<size_t>(q)];
    project_columns_inplace(Znew, radii, in.q);
    const double tn = 0.5 * (1.0 + std::sqrt(1.0 + 4.0 * t * t));
    const double mom = (t - 1.0) / tn;
    for (Index q = 0; q < Zhat.size(); ++q)
      Zhat.v[static_cast<size_t>(q)] = Znew.v[static_cast<size_t>(q)] + mom * (Znew.v[static_cast<size_t>(q)] - Zprev.v[static_cast<size_t>(q)]);
    Zprev = Znew;
    t = tn;
    if (k == 1 || k % 10 == 0 || k == max_iter) {
      X = recover_primal(in, Znew);
      Gap s = evaluate_gap(in, X, Znew);
      if (s.accepts(c)) return finish(std::move(X), Znew, s, k, true, since(t0), cnt);
      best.offer(X, Znew, s);
    }
    if (over_time(c, t0)) break;
  }
  return finish(std::move(best.X), std::move(best.Z), best.s, k, false, since(t0), cnt);
}

Solution solve(const Instance& in, const Config& c, const Solution* warm, Cache* cache) {
  switch (c.algorithm) {
    case Algo::ADMM: return solve_admm(in, c, warm, cache);
    case Algo::AMA: return solve_ama(in, c, warm, cache);
    case Algo::SSNAL: return solve_ssnal(in, c, warm, cache);
  }
  throw std::invalid_argument("solve: unknown algorithm");
}

// ---- path.cpp --------------------------------------------------------------
std::vector<double> make_schedule(double start, double end, Index count, bool geometric) {
  if (!(start > 0.0) || !(end > 0.0) || !std::isfinite(start) || !std::isfinite(end))
    throw std::invalid_argument("schedule endpoints must be positive and finite");
  if (count < 1) throw std::invalid_argument("schedule count must be >= 1");
  if (count > 1 && start == end) throw std::invalid_argument("schedule with count > 1 needs distinct endpoints");
  if (count == 1) return {start};
  const double lo = std::min(start, end), hi = std::max(start, end);
  std::vector<double> v(static_cast<size_t>(count));
  if (!geometric) {
    for (Index t = 0; t < count; ++t) v[static_cast<size_t>(t)] = lo + (hi - lo) * static_cast<double>(t) / static_cast<double>(count - 1);
  } else {
    const double lr = std::log(hi / lo) / static_cast<double>(count - 1);
    for (Index t = 0; t < count; ++t) v[static_cast<size_t>(t)] = lo * std::exp(static_cast<double>(t) * lr);
  }
  v.front() = lo;
  v.back() = hi;
  for (size_t t = 1; t < v.size(); ++t)
    if (!(v[t] > v[t - 1])) throw std::invalid_argument("schedule endpoints too close: values are not strictly increasing");
  return v;
}

// path.cpp:60-89
Clusters extract_clusters(const Mat& X, const Graph& g, double fuse_tol) {
  if (X.cols != g.n) throw std::invalid_argument("extract_clusters: X column count != node count");
  if (!(fuse_tol > 0.0)) throw std::invalid_argument("extract_clusters: fuse_tol must be positive");
  double mx = 0.0;
  for (Index i = 0; i < X.cols; ++i) mx = std::max(mx, norm2(X.col(i), X.rows));
  const double thr = fuse_tol * (1.0 + mx);
  std::vector<Edge> fused;
  std::vector<double> diff(static_cast<size_t>(X.rows));
  for (const Edge& e : g.edges) {
    for (Index r = 0; r < X.rows; ++r) diff[static_cast<size_t>(r)] = X(r, e.i) - X(r, e.j);
    if (norm2(diff.data(), X.rows) <= thr) fused.push_back(Edge{e.i, e.j, 1.0});
  }
  Graph sub(g.n, std::move(fused));
  Clusters out;
  out.labels = connected_components(sub);
  out.K = component_count(out.labels);
  out.centroids = Mat(X.rows, out.K, 0.0);
  std::vector<Index> sizes(static_cast<size_t>(out.K), 0);
  for (Index i = 0; i < X.cols; ++i) {
    const Index L = out.labels[static_cast<size_t>(i)];
    for (Index r = 0; r < X.rows; ++r) out.centroids(r, L) += X(r, i);
    ++sizes[static_cast<size_t>(L)];
  }
  for (Index L = 0; L < out.K; ++L)
    for (Index r = 0; r < X.rows; ++r) out.centroids(r, L) /= static_cast<double>(sizes[static_cast<size_t>(L)]);
  return out;
}

// path.cpp:110-142
PathOut run_path(const Mat& A, const Graph& g, Norm q, const std::vector<double>& gammas, const Config& c,
                 bool warm_start, bool require_connected, double fuse_tol) {
  if (gammas.empty()) throw std::invalid_argument("run_path: empty schedule");
  if (A.cols != g.n) throw std::invalid_argument("run_path: graph size does not match the data");
  if (require_connected) {
    const Index comps = component_count(connected_components(g));
    if (comps > 1) throw std::runtime_error("run_path: graph has " + std::to_string(comps) + " connected components; full fusion is unreachable");
  }
  PathOut out;
  out.gammas = gammas;
  out.sols.reserve(gammas.size());
  Cache cache;
  const Solution* warm = nullptr;
  for (double gamma : gammas) {
    Instance in(A, g, gamma, q);
    Solution sol = solve(in, c, warm, &cache);
    out.clusters.push_back(extract_clusters(sol.X, g, fuse_tol));
    out.sols.push_back(std::move(sol));
    warm = warm_start ? &out.sols.back() : nullptr;
  }
  return out;
}

// io.cpp:142-165: mt19937_64(seed), N(0,1) draws, column by column, row inner.
Mat gaussian_mixture(const std::vector<std::vector<double>>& centers, double spread, Index per_center,
                     std::uint64_t seed) {
  if (centers.empty()) throw std::invalid_argument("mixture needs at least one center");
  if (per_center < 1) throw std::invalid_argument("mixture needs per_center >= 1");
  if (!(spread >= 0.0)) throw std::invalid_argument("mixture spread must be >= 0");
  const Index d = static_cast<Index>(centers.front().size());
  for (const auto& cc : centers)
    if (static_cast<Index>(cc.size()) != d) throw std::invalid_argument("mixture centers differ in dimension");
  std::mt19937_64 rng(seed);
  std::normal_distribution<double> gauss(0.0, 1.0);
  const Index n = static_cast<Index>(centers.size()) * per_center;
  Mat A(d, n);
  Index col = 0;
  for (size_t m = 0; m < centers.size(); ++m)
    for (Index s = 0; s < per_center; ++s, ++col)
      for (Index r = 0; r < d; ++r) A(r, col) = centers[m][static_cast<size_t>(r)] + spread * gauss(rng);
  validate_data(A);
  return A;
}

}  // namespace oracle
