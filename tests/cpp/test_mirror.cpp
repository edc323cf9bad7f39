// C++ parity tests of the drop-in boundary: the reference's own unit-test
// cases (tests/test_graph.cpp, test_prox.cpp, test_solvers.cpp, test_path.cpp
// under /root/reference/proj), restated against the C++ mirror
// include/cluspath/*.hpp, which calls libcluspath_b200.so (sm_100a) through
// the C-ABI.  Run by tests/test_cpp_mirror.py on a GPU box.
#include <cmath>
#include <cstdio>
#include <functional>
#include <random>
#include <string>
#include <vector>

#include "cluspath/bench.hpp"
#include "cluspath/graph.hpp"
#include "cluspath/linalg.hpp"
#include "cluspath/path.hpp"
#include "cluspath/prox.hpp"
#include "cluspath/solvers.hpp"

using namespace cluspath;

// ---- a very small doctest-like harness ----------------------------------------
static int g_fail = 0, g_checks = 0;
static std::vector<std::pair<std::string, std::function<void()>>>& registry() {
  static std::vector<std::pair<std::string, std::function<void()>>> r;
  return r;
}
struct Reg {
  Reg(const char* n, std::function<void()> f) { registry().emplace_back(n, std::move(f)); }
};
#define CAT2(a, b) a##b
#define CAT(a, b) CAT2(a, b)
#define TEST_CASE(name)                                 \
  static void CAT(tc_, __LINE__)();                     \
  static Reg CAT(reg_, __LINE__)(name, CAT(tc_, __LINE__)); \
  static void CAT(tc_, __LINE__)()
#define CHECK(cond)                                                           \
  do {                                                                        \
    ++g_checks;                                                               \
    if (!(cond)) {                                                            \
      ++g_fail;                                                               \
      std::printf("  CHECK failed %s:%d: %s\n", __FILE__, __LINE__, #cond); \
    }                                                                         \
  } while (0)
#define CHECK_THROWS_AS(expr, exc)                                                        \
  do {                                                                                    \
    ++g_checks;                                                                           \
    bool ok_ = false;                                                                     \
    try {                                                                                 \
      (void)(expr);                                                                       \
    } catch (const exc&) {                                                                \
      ok_ = true;                                                                         \
    } catch (...) {                                                                       \
    }                                                                                     \
    if (!ok_) {                                                                           \
      ++g_fail;                                                                           \
      std::printf("  CHECK_THROWS_AS failed %s:%d: %s\n", __FILE__, __LINE__, #expr);   \
    }                                                                                     \
  } while (0)
static bool approx(double a, double b, double rel = 1e-12) { return std::abs(a - b) <= rel * std::max(1.0, std::abs(b)); }

static DataMatrix line_data(std::initializer_list<double> xs) {
  Matrix A(1, static_cast<Index>(xs.size()));
  Index c = 0;
  for (double x : xs) A(0, c++) = x;
  return make_data_matrix(A);
}
static double maxabs_diff(const Matrix& a, const Matrix& b) {
  double m = 0.0;
  for (Index k = 0; k < a.size(); ++k) m = std::max(m, std::abs(a.data()[k] - b.data()[k]));
  return m;
}

// ---- graph (test_graph.cpp) -----------------------------------------------------------
TEST_CASE("weighted graph sorts and validates edges") {  // test_graph.cpp:51-77
  WeightedGraph g(4, {{2, 3, 0.5}, {0, 1, 1.0}, {1, 3, 2.0}});
  CHECK(g.nodes() == 4 && g.edge_count() == 3);
  CHECK(g.edge(0).i == 0 && g.edge(0).j == 1 && g.edge(1).i == 1 && g.edge(2).i == 2);
  CHECK(g.degree(3) == 2 && g.max_degree() == 2);
  CHECK(g.find_edge(3, 1).has_value() && *g.find_edge(3, 1) == 1);
  CHECK(!g.find_edge(0, 2).has_value());
  Vector w = g.weights();
  CHECK(w[0] == 1.0 && w[1] == 2.0 && w[2] == 0.5);
  CHECK_THROWS_AS(WeightedGraph(4, {{1, 1, 1.0}}), std::invalid_argument);
  CHECK_THROWS_AS(WeightedGraph(4, {{3, 1, 1.0}}), std::invalid_argument);
  CHECK_THROWS_AS(WeightedGraph(4, {{0, 4, 1.0}}), std::invalid_argument);
  CHECK_THROWS_AS(WeightedGraph(4, {{0, 1, 0.0}}), std::invalid_argument);
  CHECK_THROWS_AS(WeightedGraph(4, {{0, 1, -2.0}}), std::invalid_argument);
  CHECK_THROWS_AS(WeightedGraph(4, {{0, 1, 1.0}, {0, 1, 2.0}}), std::invalid_argument);
}

TEST_CASE("knn graph on a 1-D line, weights, ties, range, underflow") {  // test_graph.cpp:91-138
  WeightedGraph g = compute_knn_weights(line_data({0.0, 1.0, 3.0}), 1, 0.0);
  CHECK(g.edge_count() == 2 && g.edge(0).i == 0 && g.edge(0).j == 1 && g.edge(1).i == 1 && g.edge(1).j == 2);
  CHECK(g.edge(0).w == 1.0 && g.edge(1).w == 1.0);
  WeightedGraph h = compute_knn_weights(line_data({0.0, 1.0, 3.0}), 1, 0.5);
  CHECK(approx(h.edge(0).w, 0.6065306597126334, 1e-14) && approx(h.edge(1).w, 0.1353352832366127, 1e-14));
  Matrix A(2, 5);
  const double xs[5] = {0.0, 5.0, -5.0, 5.1, -5.1};
  for (int c = 0; c < 5; ++c) A(0, c) = xs[c];
  WeightedGraph t = compute_knn_weights(make_data_matrix(A), 1, 0.0);
  CHECK(t.find_edge(0, 1).has_value() && !t.find_edge(0, 2).has_value());
  CHECK(t.find_edge(1, 3).has_value() && t.find_edge(2, 4).has_value() && t.edge_count() == 3);
  CHECK_THROWS_AS(compute_knn_weights(line_data({0.0, 1.0, 3.0}), 0, 0.5), std::invalid_argument);
  CHECK_THROWS_AS(compute_knn_weights(line_data({0.0, 1.0, 3.0}), 3, 0.5), std::invalid_argument);
  CHECK(compute_knn_weights(line_data({0.0, 1.0, 3.0}), 2, 0.5).edge_count() == 3);
  CHECK(compute_knn_weights(line_data({0.0, 1.0}), 1, 1.0).edge_count() == 1);
  CHECK(compute_knn_weights(line_data({0.0, 1.0}), 1, 1e10).edge_count() == 0);
}

TEST_CASE("incidence operator and its transpose") {  // test_graph.cpp:140-171
  WeightedGraph g(3, {{0, 1, 1.0}, {1, 2, 1.0}});
  IncidenceOperator B(g);
  Matrix X(1, 3);
  X(0, 0) = 5, X(0, 1) = 2, X(0, 2) = 9;
  Matrix XB = B.apply(X);
  CHECK(XB.rows() == 1 && XB.cols() == 2 && XB(0, 0) == 3.0 && XB(0, 1) == -7.0);
  std::mt19937_64 rng(11);
  std::normal_distribution<double> gauss;
  WeightedGraph g5(5, {{0, 1, 1.0}, {0, 3, 1.0}, {1, 2, 1.0}, {2, 4, 1.0}, {3, 4, 1.0}});
  IncidenceOperator B5(g5);
  Matrix X5(3, 5), Z5(3, 5);
  for (Index k = 0; k < 15; ++k) X5.data()[k] = gauss(rng), Z5.data()[k] = gauss(rng);
  Matrix xb = B5.apply(X5), zbt = B5.apply_transpose(Z5);
  double lhs = 0, rhs = 0;
  for (Index k = 0; k < 15; ++k) lhs += xb.data()[k] * Z5.data()[k], rhs += X5.data()[k] * zbt.data()[k];
  CHECK(approx(lhs, rhs, 1e-12));
  for (Index l = 0; l < g5.edge_count(); ++l)
    for (Index r = 0; r < 3; ++r) CHECK(xb(r, l) == X5(r, g5.edge(l).i) - X5(r, g5.edge(l).j));
  CHECK_THROWS_AS(B.apply(Matrix(1, 4)), std::invalid_argument);
}

TEST_CASE("connected components label by first appearance") {  // test_graph.cpp:214-232
  auto l = connected_components(WeightedGraph(5, {{0, 1, 1.0}, {2, 3, 1.0}}));
  CHECK((l == std::vector<Index>{0, 0, 1, 1, 2}) && component_count(l) == 3);
  CHECK((connected_components(WeightedGraph(4, {{2, 3, 1.0}})) == std::vector<Index>{0, 1, 2, 2}));
  CHECK(component_count(connected_components(WeightedGraph(3, {{0, 1, 1.0}, {1, 2, 1.0}}))) == 1);
}

// ---- prox (test_prox.cpp) ------------------------------------------------------------------
TEST_CASE("soft thresholds and projections") {  // test_prox.cpp:45-76
  Vector p = prox_norm({3, 4}, 1.0, PenaltyNorm::l2);
  CHECK(approx(p[0], 2.4, 1e-14) && approx(p[1], 3.2, 1e-14));
  CHECK(prox_norm({3, 4}, 5.0, PenaltyNorm::l2)[0] == 0.0);
  CHECK((prox_norm({3, -4}, 1.0, PenaltyNorm::l1) == Vector{2.0, -3.0}));
  Vector q = prox_norm({0.5, -4}, 1.0, PenaltyNorm::l1);
  CHECK(q[0] == 0.0 && q[1] == -3.0);
  Vector z = project_dual_ball({6, 8}, 5.0, PenaltyNorm::l2);
  CHECK(approx(z[0], 3.0, 1e-14) && approx(z[1], 4.0, 1e-14));
  CHECK((project_dual_ball({3, -4}, 2.0, PenaltyNorm::l1) == Vector{2.0, -2.0}));
  CHECK_THROWS_AS(prox_norm({1, 1}, -0.5, PenaltyNorm::l2), std::invalid_argument);
  CHECK_THROWS_AS(penalty_norm_from_q(3), std::invalid_argument);
}

TEST_CASE("moreau identity holds to machine precision") {  // test_prox.cpp:78-87
  std::mt19937_64 rng(42);
  std::uniform_real_distribution<double> tdist(0.0, 3.0);
  std::normal_distribution<double> g(0.0, 2.0);
  for (PenaltyNorm norm : {PenaltyNorm::l2, PenaltyNorm::l1})
    for (int trial = 0; trial < 100; ++trial) {
      Vector v(1 + rng() % 6);
      for (double& x : v) x = g(rng);
      CHECK(moreau_check(v, tdist(rng), norm) <= 1e-12);
    }
}

// ---- solvers (test_solvers.cpp) --------------------------------------------------------------
static DataMatrix five_point() {
  Matrix A(2, 5);
  const double a[2][5] = {{0.0, 1.0, -0.8, 0.3, -0.2}, {0.0, 0.2, 0.6, -0.9, 0.5}};
  for (int r = 0; r < 2; ++r)
    for (int c = 0; c < 5; ++c) A(r, c) = a[r][c];
  return make_data_matrix(A);
}
static WeightedGraph five_graph() {
  return WeightedGraph(5, {{0, 1, 1.0}, {0, 2, 0.7}, {0, 3, 0.9}, {0, 4, 1.1}, {1, 2, 0.6}, {1, 3, 0.8}, {1, 4, 1.2},
                           {2, 3, 0.5}, {2, 4, 0.95}, {3, 4, 0.65}});
}

TEST_CASE("objectives on the two-point example") {  // test_solvers.cpp:108-136
  DataMatrix data = line_data({0.0, 2.0});
  WeightedGraph g(2, {{0, 1, 1.0}});
  ProblemInstance inst(data, g, 0.5, PenaltyNorm::l2);
  Matrix X(1, 2);
  X(0, 0) = 0.5, X(0, 1) = 1.5;
  CHECK(approx(primal_objective(inst, X), 0.75, 1e-14));
  Matrix Z(1, 1);
  Z(0, 0) = -0.5;
  CHECK(approx(dual_objective(inst, Z), 0.75, 1e-14));
  Matrix rec = recover_primal(inst, Z);
  CHECK(approx(rec(0, 0), 0.5, 1e-14) && approx(rec(0, 1), 1.5, 1e-14));
  Matrix Zbad(1, 1);
  Zbad(0, 0) = -0.6;
  CHECK_THROWS_AS(dual_objective(inst, Zbad), std::invalid_argument);
  CHECK_THROWS_AS(ProblemInstance(data, WeightedGraph(3, {{0, 1, 1.0}}), 0.5, PenaltyNorm::l2), std::invalid_argument);
  CHECK_THROWS_AS(ProblemInstance(data, g, -0.5, PenaltyNorm::l2), std::invalid_argument);
}

TEST_CASE("every solver reproduces the two-point closed form") {  // test_solvers.cpp:164-197
  std::mt19937_64 rng(77);
  std::uniform_real_distribution<double> coord(-2.0, 2.0), wdist(0.5, 2.0), gdist(0.05, 1.5);
  for (int trial = 0; trial < 6; ++trial) {
    const Index d = 1 + trial % 3;
    Vector a1(d), a2(d);
    for (Index r = 0; r < d; ++r) a1[r] = coord(rng), a2[r] = coord(rng);
    const double w = wdist(rng), gamma = gdist(rng);
    Matrix A(d, 2);
    for (Index r = 0; r < d; ++r) A(r, 0) = a1[r], A(r, 1) = a2[r];
    DataMatrix data = make_data_matrix(A);
    WeightedGraph g(2, {{0, 1, w}});
    ProblemInstance inst(data, g, gamma, PenaltyNorm::l2);
    auto [x1, x2] = two_point_closed_form(a1, a2, w, gamma);
    for (Algorithm algo : {Algorithm::ADMM, Algorithm::FastAMA, Algorithm::SSNAL}) {
      SolverConfig config;
      config.algorithm = algo;
      config.epsilon = 1e-8;
      Solution sol = solve(inst, config);
      CHECK(sol.termination.converged);
      for (Index r = 0; r < d; ++r) CHECK(std::abs(sol.X(r, 0) - x1[r]) <= 1e-6 && std::abs(sol.X(r, 1) - x2[r]) <= 1e-6);
    }
  }
}

TEST_CASE("trivial problems, warm starts and shape checks") {  // test_solvers.cpp:199-242
  DataMatrix data = line_data({1.0, -3.0});
  WeightedGraph g(2, {{0, 1, 1.0}}), empty(2, {});
  for (Algorithm algo : {Algorithm::ADMM, Algorithm::FastAMA, Algorithm::SSNAL}) {
    SolverConfig config;
    config.algorithm = algo;
    for (auto* inst : {new ProblemInstance(data, g, 0.0, PenaltyNorm::l2), new ProblemInstance(data, empty, 1.0, PenaltyNorm::l2)}) {
      Solution sol = solve(*inst, config);
      CHECK(sol.termination.converged && sol.termination.iterations == 0 && sol.termination.gap == 0.0);
      CHECK(maxabs_diff(sol.X, data.values) == 0.0);
      delete inst;
    }
    DataMatrix fp = five_point();
    WeightedGraph fg = five_graph();
    ProblemInstance inst(fp, fg, 0.15, PenaltyNorm::l2);
    config.epsilon = 1e-7;
    Solution cold = solve(inst, config);
    Solution warm = solve(inst, config, &cold);
    CHECK(cold.termination.converged && warm.termination.converged && warm.termination.iterations == 0);
    CHECK(maxabs_diff(warm.X, cold.X) == 0.0);
    Solution bogus;
    bogus.X = Matrix(2, 4);
    bogus.Z = Matrix(2, 10);
    CHECK_THROWS_AS(solve(inst, config, &bogus), std::invalid_argument);
  }
}

TEST_CASE("q = 1 and q = 2 solves agree across solvers (five-point instance)") {  // test_solvers.cpp:244-263, 399-414
  DataMatrix fp = five_point();
  WeightedGraph fg = five_graph();
  for (PenaltyNorm norm : {PenaltyNorm::l2, PenaltyNorm::l1})
    for (double gamma : {0.05, 0.15, 0.25}) {
      ProblemInstance inst(fp, fg, gamma, norm);
      std::vector<double> f;
      for (Algorithm algo : {Algorithm::ADMM, Algorithm::FastAMA, Algorithm::SSNAL}) {
        SolverConfig config;
        config.algorithm = algo;
        config.epsilon = 1e-9;
        Solution sol = solve(inst, config);
        CHECK(sol.termination.converged);
        const double fp_ = primal_objective(inst, sol.X), fd_ = dual_objective(inst, sol.Z);
        CHECK(fd_ <= fp_ + 1e-10 * (1.0 + std::abs(fp_)));
        CHECK(duality_gap(fp_, fd_) <= 1e-9 * (1.0 + 1e-9));
        CHECK(kkt_residual(inst, sol.X, sol.Z) <= 10 * 1e-9 * (1.0 + 1e-9));
        f.push_back(fp_);
      }
      CHECK(std::abs(f[1] - f[0]) <= 1e-7 * (1 + std::abs(f[0])) && std::abs(f[2] - f[0]) <= 1e-7 * (1 + std::abs(f[0])));
    }
}

TEST_CASE("iteration caps and determinism") {  // test_solvers.cpp:318-365
  DataMatrix fp = five_point();
  WeightedGraph fg = five_graph();
  ProblemInstance inst(fp, fg, 0.2, PenaltyNorm::l2);
  SolverConfig config;
  config.algorithm = Algorithm::ADMM;
  config.epsilon = 1e-12;
  config.max_iter = 3;
  Solution sol = solve(inst, config);
  CHECK(!sol.termination.converged && sol.termination.iterations == 3 && sol.termination.gap > 0.0);
  for (Algorithm algo : {Algorithm::ADMM, Algorithm::FastAMA, Algorithm::SSNAL}) {
    SolverConfig c;
    c.algorithm = algo;
    Solution s1 = solve(inst, c), s2 = solve(inst, c);
    CHECK(maxabs_diff(s1.X, s2.X) == 0.0 && maxabs_diff(s1.Z, s2.Z) == 0.0);
    CHECK(s1.termination.iterations == s2.termination.iterations && s1.termination.gap == s2.termination.gap);
  }
}

TEST_CASE("augmented lagrangian derivatives match finite differences") {  // test_solvers.cpp:367-397
  DataMatrix fp = five_point();
  WeightedGraph fg = five_graph();
  ProblemInstance inst(fp, fg, 0.3, PenaltyNorm::l2);
  const double sigma = 1.7, h = 1e-6;
  std::mt19937_64 rng(55);
  std::normal_distribution<double> gauss;
  Matrix Z(2, 10), X(2, 5), D(2, 5);
  for (Index k = 0; k < 20; ++k) Z.data()[k] = 0.1 * gauss(rng);
  double dn = 0;
  for (Index k = 0; k < 10; ++k) X.data()[k] = fp.values.data()[k] + 0.3 * gauss(rng), D.data()[k] = gauss(rng), dn += D.data()[k] * D.data()[k];
  for (Index k = 0; k < 10; ++k) D.data()[k] /= std::sqrt(dn);
  Matrix Xp = X, Xm = X;
  for (Index k = 0; k < 10; ++k) Xp.data()[k] += h * D.data()[k], Xm.data()[k] -= h * D.data()[k];
  const double fd = (ssnal_phi_value(inst, Z, sigma, Xp) - ssnal_phi_value(inst, Z, sigma, Xm)) / (2 * h);
  Matrix G = ssnal_phi_gradient(inst, Z, sigma, X);
  double dir = 0;
  for (Index k = 0; k < 10; ++k) dir += G.data()[k] * D.data()[k];
  CHECK(std::abs(fd - dir) <= 1e-5 * std::abs(dir));
  Matrix Gp = ssnal_phi_gradient(inst, Z, sigma, Xp), Gm = ssnal_phi_gradient(inst, Z, sigma, Xm);
  Matrix HD = ssnal_hessian_apply(inst, Z, sigma, X, D);
  double err = 0, nh = 0;
  for (Index k = 0; k < 10; ++k) {
    const double e = HD.data()[k] - (Gp.data()[k] - Gm.data()[k]) / (2 * h);
    err += e * e, nh += HD.data()[k] * HD.data()[k];
  }
  CHECK(std::sqrt(err) <= 1e-5 * (1.0 + std::sqrt(nh)));
}

// ---- path (test_path.cpp) ---------------------------------------------------------------
TEST_CASE("schedules and cluster extraction") {  // test_path.cpp:32-146
  GammaSchedule s = make_schedule(1.0, 100.0, 3, Spacing::geometric);
  CHECK(s.values.size() == 3 && approx(s.values[1], 10.0, 1e-14));
  CHECK_THROWS_AS(make_schedule(0.5, 0.5, 2, Spacing::linear), std::invalid_argument);
  CHECK_THROWS_AS(spacing_from_name("log"), std::invalid_argument);
  WeightedGraph chain(4, {{0, 1, 1.0}, {1, 2, 1.0}, {2, 3, 1.0}});
  Matrix X(1, 4);
  X(0, 0) = 0, X(0, 1) = 1, X(0, 2) = 1, X(0, 3) = 3;
  ClusterAssignment c = extract_clusters(X, chain);
  CHECK(c.K == 3 && (c.labels == std::vector<Index>{0, 1, 1, 2}) && c.centroids(0, 1) == 1.0);
  Matrix Y(1, 2);
  Y(0, 0) = 1000.0, Y(0, 1) = 1000.5;
  WeightedGraph pair(2, {{0, 1, 1.0}});
  CHECK(extract_clusters(Y, pair).K == 1 && extract_clusters(Y, pair, 1e-5).K == 2);
  CHECK_THROWS_AS(extract_clusters(Matrix(1, 3), chain), std::invalid_argument);
}

TEST_CASE("a two-point path crosses the fusion threshold at the predicted gamma") {  // test_path.cpp:148-170
  DataMatrix data = line_data({0.0, 2.0});
  WeightedGraph g(2, {{0, 1, 1.0}});
  GammaSchedule schedule = make_schedule(0.1, 10.0, 9, Spacing::geometric);
  SolverConfig config;
  config.epsilon = 1e-8;
  PathResult result = run_path(data, g, PenaltyNorm::l2, schedule, config);
  CHECK(result.solutions.size() == 9 && result.all_converged());
  for (size_t t = 0; t < 9; ++t) {
    const double gamma = result.schedule.values[t];
    CHECK(result.assignments[t].K == (gamma < 1.0 ? 2 : 1));
    auto [x1, x2] = two_point_closed_form({0.0}, {2.0}, 1.0, gamma);
    CHECK(std::abs(result.solutions[t].X(0, 0) - x1[0]) <= 1e-6 && std::abs(result.solutions[t].X(0, 1) - x2[0]) <= 1e-6);
  }
}

TEST_CASE("warm starts reuse the previous solution; disconnected graphs") {  // test_path.cpp:172-245
  SyntheticData synth = generate_gaussian_mixture({{-2.0, 0.0}, {2.0, 0.0}}, 0.4, 15, 7);
  WeightedGraph graph = compute_knn_weights(synth.data, 4, 0.5);
  GammaSchedule schedule = make_schedule(0.05, 5.0, 12, Spacing::geometric);
  SolverConfig config;
  PathOptions cold;
  cold.warm_start = false;
  PathResult with = run_path(synth.data, graph, PenaltyNorm::l2, schedule, config);
  PathResult without = run_path(synth.data, graph, PenaltyNorm::l2, schedule, config, cold);
  CHECK(with.all_converged() && without.all_converged());
  Index wt = 0, ct = 0;
  for (size_t t = 0; t < 12; ++t) wt += with.stats[t].iterations, ct += without.stats[t].iterations;
  CHECK(wt <= ct);
  for (size_t t = 0; t < 12; ++t) CHECK(maxabs_diff(with.solutions[t].X, without.solutions[t].X) <= 1e-3);
  DataMatrix data = line_data({0.0, 1.0, 10.0, 11.0});
  WeightedGraph g(4, {{0, 1, 1.0}, {2, 3, 1.0}});
  GammaSchedule s2 = make_schedule(0.5, 1.0, 2, Spacing::geometric);
  PathOptions opts;
  opts.require_connected = true;
  CHECK_THROWS_AS(run_path(data, g, PenaltyNorm::l2, s2, SolverConfig{}, opts), std::runtime_error);
  opts.require_connected = false;
  PathResult r = run_path(data, g, PenaltyNorm::l2, s2, SolverConfig{}, opts);
  CHECK(r.all_converged() && r.assignments.back().K >= 2);
}

TEST_CASE("path JSON and CSV outputs") {  // test_path.cpp:243-270, test_io.cpp:197-203
  DataMatrix data = line_data({0.0, 2.0});
  WeightedGraph g(2, {{0, 1, 1.0}});
  GammaSchedule s = make_schedule(0.5, 2.0, 3, Spacing::geometric);
  SolverConfig cfg;
  cfg.epsilon = 1e-8;
  PathResult r = run_path(data, g, PenaltyNorm::l2, s, cfg);
  const std::string j = path_result_to_json(r);
  CHECK(j.find("\"spacing\": \"geometric\"") != std::string::npos);
  CHECK(j.find("\"algorithm\": \"ssnal\"") != std::string::npos);
  CHECK(j.find("\"epsilon\": 1e-08") != std::string::npos);
  CHECK(j.find("\"max_iter\": 100") != std::string::npos);
  CHECK(j.find("\"wall_time_s\"") != std::string::npos && j.find("\"f_p\"") != std::string::npos);
  std::FILE* f = std::fopen("_build/path.json", "wb");
  if (f) {
    std::fputs(j.c_str(), f);
    std::fclose(f);
  }
  WeightedGraph h(3, {{0, 1, 0.5}, {1, 2, 2.0}});
  export_graph_csv("_build/g.csv", h);
  std::FILE* in = std::fopen("_build/g.csv", "rb");
  char buf[64] = {0};
  const size_t got = in ? std::fread(buf, 1, sizeof(buf) - 1, in) : 0;
  if (in) std::fclose(in);
  CHECK(std::string(buf, got) == "i,j,w\n0,1,0.5\n1,2,2\n");
  CHECK(format_double(1e5) == "1e+05" && format_double(2.0) == "2" && format_double(0.001) == "0.001");
}

TEST_CASE("laplacian of the path and complete graphs") {  // test_graph.cpp:173-185
  WeightedGraph path3(3, {{0, 1, 0.7}, {1, 2, 0.2}});
  Matrix Lp = IncidenceOperator(path3).laplacian().toDense();
  const double ep[9] = {1, -1, 0, -1, 2, -1, 0, -1, 1};
  bool ok = true;
  for (Index r = 0; r < 3; ++r)
    for (Index c = 0; c < 3; ++c) ok = ok && Lp(r, c) == ep[r * 3 + c];
  CHECK(ok);
  WeightedGraph k3(3, {{0, 1, 1.0}, {0, 2, 1.0}, {1, 2, 1.0}});
  SparseMatrix Lc = IncidenceOperator(k3).laplacian();
  CHECK(Lc.nonZeros() == 9 && Lc.toDense()(0, 0) == 2.0 && Lc.toDense()(2, 1) == -1.0);
  WeightedGraph iso(4, {{0, 2, 1.0}});
  SparseMatrix Li = IncidenceOperator(iso).laplacian();
  CHECK(Li.nonZeros() == 4 && Li.colptr[1] == Li.colptr[2]);  // node 1 isolated: empty column
}

TEST_CASE("prox jacobian structure") {  // test_prox.cpp:146-170
  ProxJacobian J = prox_jacobian(Vector{3.0, 4.0}, 1.0, PenaltyNorm::l2);
  CHECK(approx(J.diag(0), 0.8 + 9.0 / 125.0, 1e-14));
  Vector y = J.apply(Vector{1.0, 0.0});
  CHECK(approx(y[0], 0.8 + 9.0 / 125.0, 1e-14) && approx(y[1], 12.0 / 125.0, 1e-14));
  Vector z = prox_jacobian(Vector{3.0, 4.0}, 5.0, PenaltyNorm::l2).apply(Vector{1.0, 2.0});
  CHECK(z[0] == 0.0 && z[1] == 0.0);
  CHECK_THROWS_AS(prox_jacobian(Vector{1.0}, -1.0, PenaltyNorm::l1), std::invalid_argument);
}

TEST_CASE("q = infinity through the mirror") {  // no reference counterpart
  Matrix V(3, 1);
  V(0, 0) = 3.0;
  V(1, 0) = -1.0;
  V(2, 0) = 0.5;
  Matrix P;
  prox_columns_into(V, {1.0}, PenaltyNorm::linf, P);
  CHECK(P(0, 0) == 2.0 && P(1, 0) == -1.0 && P(2, 0) == 0.5);
  Matrix Zp = project_columns(V, {1.0}, PenaltyNorm::linf);
  CHECK(Zp(0, 0) == 1.0 && Zp(1, 0) == 0.0 && Zp(2, 0) == 0.0);
}

// ---- linalg (test_linalg.cpp) ------------------------------------------------------------
// Small dense helpers standing in for the Eigen calls of the reference tests.
static Matrix matmul(const Matrix& A, const Matrix& B) {
  Matrix C(A.rows(), B.cols());
  for (Index c = 0; c < B.cols(); ++c)
    for (Index k = 0; k < A.cols(); ++k)
      for (Index r = 0; r < A.rows(); ++r) C(r, c) += A(r, k) * B(k, c);
  return C;
}
static Matrix dense_solve(Matrix M, Matrix B) {  // Gaussian elimination with partial pivoting
  const Index n = M.rows();
  for (Index k = 0; k < n; ++k) {
    Index p = k;
    for (Index r = k + 1; r < n; ++r)
      if (std::abs(M(r, k)) > std::abs(M(p, k))) p = r;
    for (Index c = 0; c < n; ++c) std::swap(M(k, c), M(p, c));
    for (Index c = 0; c < B.cols(); ++c) std::swap(B(k, c), B(p, c));
    for (Index r = k + 1; r < n; ++r) {
      const double f = M(r, k) / M(k, k);
      for (Index c = k; c < n; ++c) M(r, c) -= f * M(k, c);
      for (Index c = 0; c < B.cols(); ++c) B(r, c) -= f * B(k, c);
    }
  }
  for (Index k = n - 1; k >= 0; --k)
    for (Index c = 0; c < B.cols(); ++c) {
      double s = B(k, c);
      for (Index j = k + 1; j < n; ++j) s -= M(k, j) * B(j, c);
      B(k, c) = s / M(k, k);
    }
  return B;
}
static double sym_lambda_max(Matrix A) {  // cyclic Jacobi eigenvalue sweeps
  const Index n = A.rows();
  for (int sweep = 0; sweep < 100; ++sweep) {
    double off = 0.0;
    for (Index p = 0; p < n; ++p)
      for (Index q = p + 1; q < n; ++q) off += A(p, q) * A(p, q);
    if (off < 1e-30) break;
    for (Index p = 0; p < n; ++p)
      for (Index q = p + 1; q < n; ++q) {
        if (std::abs(A(p, q)) < 1e-300) continue;
        const double th = 0.5 * std::atan2(2.0 * A(p, q), A(q, q) - A(p, p));
        const double c = std::cos(th), s = std::sin(th);
        for (Index k = 0; k < n; ++k) {
          const double akp = A(k, p), akq = A(k, q);
          A(k, p) = c * akp - s * akq;
          A(k, q) = s * akp + c * akq;
        }
        for (Index k = 0; k < n; ++k) {
          const double apk = A(p, k), aqk = A(q, k);
          A(p, k) = c * apk - s * aqk;
          A(q, k) = s * apk + c * aqk;
        }
      }
  }
  double m = A(0, 0);
  for (Index k = 1; k < n; ++k) m = std::max(m, A(k, k));
  return m;
}
static Matrix random_spd(std::mt19937_64& rng, Index n) {  // test_linalg.cpp:23-31
  std::normal_distribution<double> gauss;
  Matrix G(n, n);
  for (Index r = 0; r < n; ++r)
    for (Index c = 0; c < n; ++c) G(r, c) = gauss(rng);
  Matrix M(n, n);
  for (Index r = 0; r < n; ++r)
    for (Index c = 0; c < n; ++c) {
      double s = 0.0;
      for (Index k = 0; k < n; ++k) s += G(r, k) * G(c, k);
      M(r, c) = s;
    }
  for (Index k = 0; k < n; ++k) M(k, k) += 0.5;
  return M;
}
static SparseMatrix path3_laplacian() {
  WeightedGraph g(3, {{0, 1, 1.0}, {1, 2, 1.0}});
  return IncidenceOperator(g).laplacian();
}
static double maxabs(const Matrix& a) {
  double m = 0.0;
  for (Index k = 0; k < a.size(); ++k) m = std::max(m, std::abs(a.data()[k]));
  return m;
}

TEST_CASE("cholesky factor of I + rho L on the 3-path") {  // test_linalg.cpp:35-45
  CholeskyFactor factor(path3_laplacian(), 1.0);
  CHECK(factor.size() == 3);
  CHECK(factor.rho() == 1.0);
  Matrix rhs = Matrix::Zero(3, 1);
  rhs(0, 0) = 1.0;
  Matrix x = factor.solve(rhs);
  CHECK(approx(x(0, 0), 0.625, 1e-14));
  CHECK(approx(x(1, 0), 0.25, 1e-14));
  CHECK(approx(x(2, 0), 0.125, 1e-14));
}

TEST_CASE("cholesky solve residual on random laplacians") {  // test_linalg.cpp:47-70
  std::mt19937_64 rng(17);
  std::uniform_real_distribution<double> unif(0.2, 3.0);
  for (int trial = 0; trial < 10; ++trial) {
    const Index n = 4 + static_cast<Index>(rng() % 12);
    std::vector<Edge> edges;
    for (Index i = 0; i + 1 < n; ++i) edges.push_back({i, i + 1, 1.0});
    for (Index i = 0; i < n; ++i)
      for (Index j = i + 2; j < n; ++j)
        if ((rng() & 3u) == 0u) edges.push_back({i, j, 1.0});
    WeightedGraph g(n, edges);
    const double rho = unif(rng);
    CholeskyFactor factor(IncidenceOperator(g).laplacian(), rho);
    Matrix M = IncidenceOperator(g).laplacian().toDense();
    for (Index k = 0; k < M.size(); ++k) M.data()[k] *= rho;
    for (Index k = 0; k < n; ++k) M(k, k) += 1.0;
    Matrix rhs(n, 3);
    std::normal_distribution<double> gauss;
    for (Index r = 0; r < n; ++r)
      for (Index c = 0; c < 3; ++c) rhs(r, c) = gauss(rng);
    Matrix x = factor.solve(rhs);
    Matrix res = matmul(M, x);
    for (Index k = 0; k < res.size(); ++k) res.data()[k] -= rhs.data()[k];
    CHECK(maxabs(res) <= 1e-10 * (1.0 + maxabs(rhs)));
  }
}

TEST_CASE("cholesky rejects invalid input") {  // test_linalg.cpp:72-78
  CHECK_THROWS_AS(CholeskyFactor(path3_laplacian(), -1.0), std::invalid_argument);
  SparseMatrix asym;
  asym.rows_ = asym.cols_ = 2;
  asym.colptr = {0, 0, 1};
  asym.rowidx = {0};
  asym.values = {1.0};  // (0, 1) only: not symmetric
  CHECK_THROWS_AS(CholeskyFactor(asym, 1.0), std::invalid_argument);
}

TEST_CASE("linear operator factories agree with dense arithmetic") {  // test_linalg.cpp:80-110
  std::mt19937_64 rng(3);
  Matrix M = random_spd(rng, 5);
  LinearOperator dense = LinearOperator::dense(M, true);
  CHECK(dense.rows() == 5);
  CHECK(dense.symmetric());
  CHECK(dense.positive_definite());
  SparseMatrix S;
  S.rows_ = S.cols_ = 5;
  S.colptr.push_back(0);
  for (Index c = 0; c < 5; ++c) {
    for (Index r = 0; r < 5; ++r)
      if (M(r, c) != 0.0) S.rowidx.push_back(r), S.values.push_back(M(r, c));
    S.colptr.push_back(static_cast<int64_t>(S.values.size()));
  }
  LinearOperator sparse = LinearOperator::sparse(S, true);
  Matrix X(5, 2);
  std::normal_distribution<double> gauss;
  for (Index r = 0; r < 5; ++r)
    for (Index c = 0; c < 2; ++c) X(r, c) = gauss(rng);
  const Matrix MX = matmul(M, X);
  CHECK(maxabs_diff(dense.apply(X), MX) <= 1e-14);
  CHECK(maxabs_diff(sparse.apply(X), MX) <= 1e-14);
  CHECK(maxabs_diff(LinearOperator::identity(5).apply(X), X) == 0.0);
  Vector d{1, 2, 4, 8, 16};
  Matrix Z = LinearOperator::jacobi(d).apply(X);
  for (Index r = 0; r < 5; ++r)
    for (Index c = 0; c < 2; ++c) CHECK(approx(Z(r, c), X(r, c) / d[static_cast<size_t>(r)]));
  CHECK_THROWS_AS(LinearOperator::jacobi(Vector(3, 0.0)), std::invalid_argument);
  CHECK_THROWS_AS(dense.apply(Matrix::Zero(4, 1)), std::invalid_argument);
  CHECK_THROWS_AS(LinearOperator::dense(Matrix(2, 3)), std::invalid_argument);
}

TEST_CASE("pcg solves a frozen 2x2 system") {  // test_linalg.cpp:112-118
  Matrix M(2, 2);
  M(0, 0) = 4, M(0, 1) = 1, M(1, 0) = 1, M(1, 1) = 3;
  PcgResult res = pcg(LinearOperator::dense(M, true), Vector{1, 2}, nullptr, 1e-12, 50);
  CHECK(res.converged);
  CHECK(approx(res.x(0, 0), 1.0 / 11.0, 1e-10));
  CHECK(approx(res.x(1, 0), 7.0 / 11.0, 1e-10));
  CHECK(res.residual <= 1e-12);
}

TEST_CASE("pcg on the identity converges in one iteration") {  // test_linalg.cpp:120-127
  Vector b{1, -2, 3, -4};
  PcgResult res = pcg(LinearOperator::identity(4), b, nullptr, 1e-10, 10);
  CHECK(res.converged);
  CHECK(res.iterations == 1);
  double e = 0.0;
  for (Index k = 0; k < 4; ++k) e = std::max(e, std::abs(res.x(k, 0) - b[static_cast<size_t>(k)]));
  CHECK(e <= 1e-14);
}

TEST_CASE("pcg matches dense solves on random SPD systems") {  // test_linalg.cpp:129-144
  std::mt19937_64 rng(29);
  std::normal_distribution<double> gauss;
  for (int trial = 0; trial < 8; ++trial) {
    const Index n = 20;
    Matrix M = random_spd(rng, n);
    Matrix b(n, 1);
    for (Index i = 0; i < n; ++i) b(i, 0) = gauss(rng);
    LinearOperator op = LinearOperator::dense(M, true);
    Vector dg(static_cast<size_t>(n));
    for (Index i = 0; i < n; ++i) dg[static_cast<size_t>(i)] = M(i, i);
    LinearOperator precond = LinearOperator::jacobi(dg);
    PcgResult res = pcg(op, b, &precond, 1e-12, 400);
    Matrix exact = dense_solve(M, b);
    CHECK(res.converged);
    double e = 0.0, ne = 0.0;
    for (Index i = 0; i < n; ++i) e += std::pow(res.x(i, 0) - exact(i, 0), 2), ne += exact(i, 0) * exact(i, 0);
    CHECK(std::sqrt(e) <= 1e-8 * (1.0 + std::sqrt(ne)));
  }
}

TEST_CASE("pcg handles matrix-block right-hand sides") {  // test_linalg.cpp:146-160
  std::mt19937_64 rng(31);
  std::normal_distribution<double> gauss;
  const Index n = 12;
  Matrix M = random_spd(rng, n);
  Matrix B(n, 3);
  for (Index r = 0; r < n; ++r)
    for (Index c = 0; c < 3; ++c) B(r, c) = gauss(rng);
  PcgResult res = pcg(LinearOperator::dense(M, true), B, nullptr, 1e-11, 600);
  Matrix exact = dense_solve(M, B);
  CHECK(res.converged);
  CHECK(maxabs_diff(res.x, exact) <= 1e-7 * (1.0 + maxabs(exact)));
}

TEST_CASE("pcg rejects indefinite operators and zero rhs is immediate") {  // test_linalg.cpp:162-174
  Matrix Mneg(3, 3);
  for (Index k = 0; k < 3; ++k) Mneg(k, k) = -1.0;
  CHECK_THROWS_AS(pcg(LinearOperator::dense(Mneg, false), Vector{1, 1, 1}, nullptr, 1e-10, 10), std::runtime_error);
  PcgResult res = pcg(LinearOperator::identity(3), Vector(3, 0.0), nullptr, 1e-10, 10);
  CHECK(res.converged);
  CHECK(res.iterations == 0);
  CHECK(maxabs(res.x) == 0.0);
}

TEST_CASE("pcg and power iteration on a host functor operator") {  // LinearOperator(rows, fn) (linalg.hpp:45)
  Matrix M(2, 2);
  M(0, 0) = 4, M(0, 1) = 1, M(1, 0) = 1, M(1, 1) = 3;
  int calls = 0;
  LinearOperator op(2, [&](const Matrix& x) {
    ++calls;
    return matmul(M, x);
  }, true, true);
  PcgResult res = pcg(op, Vector{1, 2}, nullptr, 1e-12, 50);
  CHECK(res.converged && calls >= 2);
  CHECK(approx(res.x(0, 0), 1.0 / 11.0, 1e-10) && approx(res.x(1, 0), 7.0 / 11.0, 1e-10));
  CHECK(approx(power_iteration(op), 3.5 + std::sqrt(1.25), 1e-8));
  LinearOperator bad(2, [](const Matrix&) -> Matrix { throw std::invalid_argument("functor says no"); });
  CHECK_THROWS_AS(pcg(bad, Vector{1, 2}, nullptr, 1e-12, 5), std::invalid_argument);
}

TEST_CASE("power iteration finds the top eigenvalue") {  // test_linalg.cpp:176-195
  Matrix D = Matrix::Zero(2, 2);
  D(0, 0) = 1.0;
  D(1, 1) = 5.0;
  CHECK(approx(power_iteration(LinearOperator::dense(D, true)), 5.0, 1e-8));
  WeightedGraph g(2, {{0, 1, 1.0}});
  CHECK(approx(power_iteration(LinearOperator::sparse(IncidenceOperator(g).laplacian(), false)), 2.0, 1e-8));
  CHECK(power_iteration(LinearOperator::dense(Matrix::Zero(3, 3), false)) == 0.0);
  SparseMatrix L = path3_laplacian();
  CHECK(approx(power_iteration(LinearOperator::sparse(L, false)), sym_lambda_max(L.toDense()), 1e-8));
}

TEST_CASE("power iteration on random laplacians matches dense spectra") {  // test_linalg.cpp:197-212
  std::mt19937_64 rng(41);
  for (int trial = 0; trial < 6; ++trial) {
    const Index n = 5 + static_cast<Index>(rng() % 10);
    std::vector<Edge> edges;
    for (Index i = 0; i + 1 < n; ++i) edges.push_back({i, i + 1, 1.0});
    for (Index i = 0; i < n; ++i)
      for (Index j = i + 2; j < n; ++j)
        if ((rng() & 1u) == 0u) edges.push_back({i, j, 1.0});
    WeightedGraph g(n, edges);
    SparseMatrix L = IncidenceOperator(g).laplacian();
    const double lmax = power_iteration(LinearOperator::sparse(L, false), 1e-12, 20000);
    CHECK(approx(lmax, sym_lambda_max(L.toDense()), 1e-6));
  }
}

TEST_CASE("norm values, prox_norm_into and project_dual_ball_into") {  // prox.hpp:14-26 (test_prox.cpp:28-60)
  CHECK(approx(norm_value(Vector{3.0, -4.0}, PenaltyNorm::l2), 5.0, 1e-15));
  CHECK(approx(norm_value(Vector{3.0, -4.0}, PenaltyNorm::l1), 7.0, 1e-15));
  CHECK(approx(dual_norm_value(Vector{3.0, -4.0}, PenaltyNorm::l1), 4.0, 1e-15));
  CHECK(approx(dual_norm_value(Vector{3.0, -4.0}, PenaltyNorm::l2), 5.0, 1e-15));
  Vector out;
  prox_norm_into(Vector{3.0, 4.0}, 2.5, PenaltyNorm::l2, out);
  CHECK(approx(out[0], 1.5, 1e-15) && approx(out[1], 2.0, 1e-15));
  project_dual_ball_into(Vector{3.0, -0.5}, 1.0, PenaltyNorm::l1, out);
  CHECK(out[0] == 1.0 && out[1] == -0.5);
  CHECK_THROWS_AS(prox_norm_into(Vector{1.0}, -1.0, PenaltyNorm::l2, out), std::invalid_argument);
}

TEST_CASE("solver trace rows and per-gamma centroids") {  // solvers.hpp:54-66, path.cpp:135
  Matrix A(2, 6);
  const double pts[6][2] = {{0, 0}, {0.1, 0}, {0, 0.1}, {3, 3}, {3.1, 3}, {3, 3.1}};
  for (Index c = 0; c < 6; ++c) A(0, c) = pts[c][0], A(1, c) = pts[c][1];
  DataMatrix data = make_data_matrix(A);
  WeightedGraph g = compute_knn_weights(data, 2, 0.5);
  SolverConfig cfg;
  cfg.collect_trace = true;
  ProblemInstance inst(data, g, 0.3, PenaltyNorm::l2);
  Solution sol = solve(inst, cfg);
  CHECK(!sol.trace.empty() && sol.trace.front().iter == 0);
  CHECK(approx(sol.trace.back().gap, sol.termination.gap, 0.0));
  GammaSchedule sched = make_schedule(0.01, 5.0, 5, Spacing::geometric);
  PathResult r = run_path(data, g, PenaltyNorm::l2, sched, cfg);
  for (size_t t = 0; t < r.assignments.size(); ++t) {
    const ClusterAssignment& a = r.assignments[t];
    ClusterAssignment e = extract_clusters(r.solutions[t].X, g);
    CHECK(a.K == e.K && a.labels == e.labels);
    CHECK(a.centroids.rows() == 2 && a.centroids.cols() == a.K);
    CHECK(maxabs_diff(a.centroids, e.centroids) == 0.0);
    CHECK(!r.solutions[t].trace.empty());
  }
  Matrix Xcopy = r.solutions[0].X;  // deep copy out of the path's shared host slab
  Xcopy(0, 0) += 1.0;
  CHECK(Xcopy(0, 0) != r.solutions[0].X(0, 0));
}

// ---- bench (test_bench.cpp) -----------------------------------------------------------------
struct BenchFixture {  // test_bench.cpp:14-30
  SyntheticData synth;
  WeightedGraph graph;
  GammaSchedule schedule;
  BenchFixture()
      : synth(generate_gaussian_mixture({Vector{-2.0, 0.0}, Vector{2.0, 0.0}}, 0.4, 10, 11)),
        graph(compute_knn_weights(synth.data, 4, 0.5)),
        schedule(make_schedule(0.1, 2.0, 5, Spacing::geometric)) {}
  BenchTask task() const { return BenchTask{&synth.data, &graph, PenaltyNorm::l2, schedule}; }
};

TEST_CASE("a single method is its own baseline and solves everything at tau = 1") {  // test_bench.cpp:34-52
  BenchFixture f;
  BenchOptions options;
  PerfProfile profile = run_bench({f.task()}, {Algorithm::SSNAL}, options);
  CHECK(profile.problem_count == 5 && profile.baseline_T > 0.0 && profile.curves.size() == 1);
  const MethodCurve& curve = profile.curves[0];
  CHECK(curve.method == Algorithm::SSNAL && curve.solved_total == 5);
  CHECK(approx(curve.full_time, profile.baseline_T));
  CHECK(curve.points.size() == 10 && curve.points[0].first == 1.0 && curve.points[0].second == 5);
  for (const auto& [tau, solved] : curve.points) CHECK(solved == 5);
}

TEST_CASE("curves are nondecreasing in tau and bounded by the problem count") {  // test_bench.cpp:54-78
  BenchFixture f;
  BenchOptions options;
  PerfProfile profile = run_bench({f.task()}, {Algorithm::SSNAL, Algorithm::ADMM, Algorithm::FastAMA}, options);
  CHECK(profile.problem_count == 5 && profile.curves.size() == 3);
  for (const MethodCurve& curve : profile.curves) {
    Index prev = 0;
    for (const auto& [tau, solved] : curve.points) {
      CHECK(solved >= prev && solved <= profile.problem_count);
      prev = solved;
    }
    CHECK(curve.points.back().second == curve.solved_total);
    if (curve.solved_total == profile.problem_count) CHECK(curve.full_time >= profile.baseline_T);
  }
}

TEST_CASE("a zero cutoff override leaves every curve at zero; bench validates inputs") {  // test_bench.cpp:80-116
  BenchFixture f;
  BenchOptions options;
  options.cutoff_override = 0.0;
  PerfProfile profile = run_bench({f.task()}, {Algorithm::SSNAL, Algorithm::ADMM}, options);
  for (const MethodCurve& curve : profile.curves) {
    CHECK(curve.solved_total == 0 && curve.full_time > 0.0);
    for (const auto& [tau, solved] : curve.points) CHECK(solved == 0);
  }
  BenchOptions hard;
  hard.epsilon = 1e-14;
  hard.base_config.max_iter = 1;
  CHECK_THROWS_AS(run_bench({f.task()}, {Algorithm::ADMM, Algorithm::FastAMA}, hard), std::runtime_error);
  BenchOptions plain;
  CHECK_THROWS_AS(run_bench({}, {Algorithm::SSNAL}, plain), std::invalid_argument);
  CHECK_THROWS_AS(run_bench({f.task()}, {}, plain), std::invalid_argument);
  BenchTask broken = f.task();
  broken.data = nullptr;
  CHECK_THROWS_AS(run_bench({broken}, {Algorithm::SSNAL}, plain), std::invalid_argument);
  plain.tau_max = 0;
  CHECK_THROWS_AS(run_bench({f.task()}, {Algorithm::SSNAL}, plain), std::invalid_argument);
}

TEST_CASE("profile CSV has one labeled row per curve point") {  // test_bench.cpp:118-140
  BenchFixture f;
  BenchOptions options;
  options.tau_max = 3;
  const std::string csv = perf_profile_csv(run_bench({f.task()}, {Algorithm::SSNAL, Algorithm::ADMM}, options));
  CHECK(csv.rfind("method,tau,solved\n", 0) == 0);
  CHECK(csv.find("ssnal,1,") != std::string::npos && csv.find("admm,3,") != std::string::npos);
  int rows = 0;
  for (char ch : csv) rows += ch == '\n';
  CHECK(rows == 7);
}

int main() {
  int failed_cases = 0;
  for (auto& [name, fn] : registry()) {
    const int before = g_fail;
    try {
      fn();
    } catch (const std::exception& e) {
      ++g_fail;
      std::printf("  unexpected exception: %s\n", e.what());
    }
    const bool ok = g_fail == before;
    failed_cases += ok ? 0 : 1;
    std::printf("%s  %s\n", ok ? "PASS" : "FAIL", name.c_str());
  }
  std::printf("%zu test cases, %d failed; %d checks, %d failed\n", registry().size(), failed_cases, g_checks, g_fail);
  return g_fail == 0 ? 0 : 1;
}
