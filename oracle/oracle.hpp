// TEST INFRASTRUCTURE ONLY — the CPU oracle for the B200 convex-clustering path.
//
// This is a single-threaded C++ restatement of the reference solver
// (/root/reference/proj, "cluspath", C++20 on Eigen 3.4).  Only tests/,
// __graft_entry__.smoke() and bench.py's cpu_baseline / --impl reference legs
// may load it, and only as the checker or the timed CPU baseline — never as
// the product path.  The product (paper_2501_15964_b200/) never links it.
//
// Eigen 3.4 is absent in this image, so the reference itself cannot be built
// (SURVEY.md §8(c)).  This restatement therefore reproduces the arithmetic the
// reference performs, including the order Eigen's SSE2 (Packet2d, no -march,
// no FMA) LinearVectorizedTraversal reduction adds terms in (esum below), and
// is pinned against every known-answer test of the reference's own suite
// (tests/test_oracle_kat.py, citing test_*.cpp:line).
#pragma once

#include <algorithm>
#include <cmath>
#include <cstdint>
#include <functional>
#include <memory>
#include <optional>
#include <random>
#include <stdexcept>
#include <string>
#include <vector>

namespace oracle {

using Index = std::int64_t;

// Column-major dense matrix, the layout of Eigen::MatrixXd (types.hpp:12).
struct Mat {
  Index rows = 0, cols = 0;
  std::vector<double> v;
  Mat() = default;
  Mat(Index r, Index c, double fill = 0.0) : rows(r), cols(c), v(static_cast<size_t>(r * c), fill) {}
  double& operator()(Index r, Index c) { return v[static_cast<size_t>(c * rows + r)]; }
  double operator()(Index r, Index c) const { return v[static_cast<size_t>(c * rows + r)]; }
  double* col(Index c) { return v.data() + c * rows; }
  const double* col(Index c) const { return v.data() + c * rows; }
  Index size() const { return rows * cols; }
};

// ---- Eigen 3.4 reduction orders --------------------------------------------
// Redux.h, LinearVectorizedTraversal with Packet2d and alignedStart = 0 (the
// reduced expressions carry no DirectAccessBit): two packet accumulators over
// stride-4 blocks, P0 += P1, a leftover packet, predux, then the odd tail.
template <class F>
inline double esum(Index n, F f) {
  if (n <= 0) return 0.0;
  if (n < 2) return f(0);
  double p00 = f(0), p01 = f(1);
  if (n >= 4) {
    const Index e2 = (n / 4) * 4, e1 = (n / 2) * 2;
    double p10 = f(2), p11 = f(3);
    for (Index k = 4; k < e2; k += 4) {
      p00 += f(k);
      p01 += f(k + 1);
      p10 += f(k + 2);
      p11 += f(k + 3);
    }
    p00 += p10;
    p01 += p11;
    if (e1 > e2) {
      p00 += f(e2);
      p01 += f(e2 + 1);
    }
  }
  double res = p00 + p01;
  if (n & 1) res += f(n - 1);
  return res;
}
// DefaultTraversal (strided rows of a column-major matrix): left to right.
template <class F>
inline double ssum(Index n, F f) {
  if (n <= 0) return 0.0;
  double res = f(0);
  for (Index k = 1; k < n; ++k) res += f(k);
  return res;
}
inline double sq_norm(const double* x, Index n) { return esum(n, [&](Index k) { return x[k] * x[k]; }); }
inline double norm2(const double* x, Index n) { return std::sqrt(sq_norm(x, n)); }
inline double dotp(const double* x, const double* y, Index n) {
  return esum(n, [&](Index k) { return x[k] * y[k]; });
}
// ---- optional host threads (checker runs at C3-C5 sizes only) ---------------
// ORC_THREADS (default 1: the reference is single-threaded, and the CPU
// baselines time one thread).  par_ranges splits an index range whose
// iterations are independent into contiguous chunks; every output element is
// produced by exactly the sequential loop's arithmetic, and global reductions
// stay sequential in Eigen's order, so results are bitwise those of one thread
// (node-partitioned scatters keep the ascending-edge order per node).
int threads();
void par_ranges(Index n, const std::function<void(Index, Index)>& f);
template <class F>
inline void par_for(Index n, F f) {
  par_ranges(n, [&](Index lo, Index hi) {
    for (Index k = lo; k < hi; ++k) f(k);
  });
}
inline double max_abs(const double* x, Index n) {
  double m = 0.0;
  for (Index k = 0; k < n; ++k) m = std::max(m, std::abs(x[k]));
  return m;
}

// ---- graph (graph.hpp:14-92, graph.cpp) ------------------------------------
struct Edge {
  Index i = 0, j = 0;
  double w = 0.0;
};

struct Graph {
  Index n = 0;
  std::vector<Edge> edges;   // lexicographic (i, j)
  std::vector<Index> degree;
  Graph() = default;
  Graph(Index n, std::vector<Edge> e);  // sorts + validates (graph.cpp:25-45)
  Index E() const { return static_cast<Index>(edges.size()); }
  std::optional<Index> find_edge(Index i, Index j) const;
  Index max_degree() const;
};

void validate_data(const Mat& A);  // make_data_matrix (graph.cpp:10-23)
// compute_knn_weights (graph.cpp:75-114).  d2_out, when given, receives the
// squared distance of every kept edge (the quantity the GPU must match bitwise).
Graph knn_weights(const Mat& A, Index k, double phi, std::vector<double>* d2_out = nullptr);
void incidence_apply(const Graph& g, const Mat& X, Mat& out);      // graph.cpp:122-132
void incidence_apply_t(const Graph& g, const Mat& Z, Mat& out);    // graph.cpp:140-152
// CSC of B B^T exactly as Eigen's setFromTriplets builds it (graph.cpp:154-167).
struct Csc {
  Index n = 0;
  std::vector<Index> colptr, row;
  std::vector<double> val;
};
Csc laplacian(const Graph& g);
std::vector<Index> connected_components(const Graph& g);  // graph.cpp:169-196
Index component_count(const std::vector<Index>& labels);

// ---- prox (prox.hpp, prox.cpp) ---------------------------------------------
// linf (q = infinity) has no reference implementation (prox.cpp:17-21 rejects
// it): parity unpinned; the math restated here is SURVEY.md §8(c):
//   prox_{t||.||inf}(v) = v - Pi_{B1(t)}(v) = clamp(v, -theta, theta),
//   Pi_{B1(t)}(v)       = sign(v) max(|v| - theta, 0) when ||v||_1 > t,
// theta the l1-ball threshold (Michelot's fixed point in the device's 32-lane
// summation order, prox_linalg.cpp); outside the ball the Clarke
// Jacobian element of the projection is diag(1_S) - s_S s_S^T / |S|.
enum class Norm { linf = 0, l1 = 1, l2 = 2 };
// l1-ball projection threshold: theta >= 0 with sum max(|v| - theta, 0) = t
// when ||v||_1 > t, else -1; *count = |S| of the converged support.
double l1_theta(const double* v, Index n, double t, Index* count);
double norm_value(const double* v, Index n, Norm q);
double dual_norm_value(const double* v, Index n, Norm q);
void prox_norm_into(const double* v, Index n, double t, Norm q, double* out);
void project_dual_ball_into(const double* z, Index n, double r, Norm q, double* out);
void prox_columns_into(const Mat& V, const std::vector<double>& t, Norm q, Mat& out);
void project_columns_inplace(Mat& Z, const std::vector<double>& r, Norm q);
struct ProxJac {
  Norm q = Norm::l2;
  double alpha = 0.0, beta = 0.0;
  std::vector<double> dir;     // q=2 rank-one direction
  std::vector<char> active;    // q=1 mask; q=inf support S = {|v| > theta}
  double theta = -1.0;         // q=inf: l1-ball threshold (< 0: v inside the ball)
  Index support = 0;           // q=inf: |S|
  void apply(const double* w, Index n, double* out) const;
  double diag(Index r) const;
};
ProxJac prox_jacobian(const double* v, Index n, double t, Norm q);
double moreau_check(const double* v, Index n, double t, Norm q);

// ---- linalg (linalg.hpp, linalg.cpp) ---------------------------------------
struct LinOp {
  Index rows = 0;
  std::function<Mat(const Mat&)> fn;
  Mat apply(const Mat& x) const;
};
LinOp op_dense(const Mat& M);
LinOp op_csc(const Csc& L);
LinOp op_jacobi(const Mat& diag);        // entrywise (linalg.cpp:110-122)
LinOp op_jacobi_vec(const std::vector<double>& diag);
struct PcgOut {
  Mat x;
  Index iterations = 0;
  double residual = 0.0;
  bool converged = false;
};
PcgOut pcg(const LinOp& op, const Mat& rhs, const LinOp* pre, double tol, Index max_iter);
double power_iteration(const LinOp& op, double tol = 1e-9, Index max_iter = 10000);
// Factor-once solve of (I + rho L) X = RHS.  The reference uses Eigen's
// SimplicialLLT with AMD (linalg.cpp:32-54); this restatement uses an
// envelope Cholesky under reverse Cuthill-McKee — same matrix, same exact
// solution, different rounding.
struct Cholesky {
  Index n = 0;
  double rho = 0.0;
  std::vector<Index> perm, first;   // perm[new] = old
  std::vector<size_t> rowptr;
  std::vector<double> L;            // row i holds columns first[i]..i
  Cholesky(const Csc& L, double rho);
  Mat solve(const Mat& rhs) const;  // rhs n x m
};

// ---- solvers (solvers.hpp, objective.cpp, solver_util.hpp, ssnal/admm/ama) --
enum class Algo { ADMM = 0, AMA = 1, SSNAL = 2 };
struct Config {
  Algo algorithm = Algo::SSNAL;
  double epsilon = 1e-6, kkt_factor = 10.0;
  Index max_iter = 0;
  double time_limit = 0.0;  // <= 0: none
  double admm_rho = 1.0, ama_step_safety = 0.99;
  double ssnal_sigma0 = 1.0, armijo_mu = 1e-4, backtrack_beta = 0.5;
  Index ssnal_newton_max = 50, pcg_max_iter = 500;
  bool collect_trace = false;
  Index resolved_max_iter() const { return max_iter > 0 ? max_iter : (algorithm == Algo::SSNAL ? 100 : 20000); }
  void validate() const;
};
struct Instance {
  const Mat* A = nullptr;
  const Graph* g = nullptr;
  double gamma = 0.0;
  Norm q = Norm::l2;
  Instance(const Mat& A, const Graph& g, double gamma, Norm q);
  std::vector<double> radii() const;
  Index d() const { return A->rows; }
  Index n() const { return A->cols; }
  Index E() const { return g->E(); }
};
struct Termination {
  double f_primal = 0, f_dual = 0, gap = 0;
  Index iterations = 0;
  bool converged = false;
  double wall_time = 0;
};
struct Counters {  // work counters (not in the reference API; used for parity diagnostics)
  Index newton = 0, cg = 0, armijo = 0, hess_apply = 0;
};
struct Solution {
  Mat X, Z;
  Termination term;
  Counters counters;
};
struct Cache {
  std::shared_ptr<const Cholesky> factor;
  double factor_rho = -1.0;
  double lambda_max = -1.0;
};

double primal_objective(const Instance& in, const Mat& X);
double dual_objective(const Instance& in, const Mat& Z);
double duality_gap(double fp, double fd);
Mat recover_primal(const Instance& in, const Mat& Z);
double kkt_residual(const Instance& in, const Mat& X, const Mat& Z);
double ssnal_phi_value(const Instance& in, const Mat& Z, double sigma, const Mat& X);
Mat ssnal_phi_gradient(const Instance& in, const Mat& Z, double sigma, const Mat& X);
Mat ssnal_hessian_apply(const Instance& in, const Mat& Z, double sigma, const Mat& X, const Mat& D);

Solution solve_ssnal(const Instance& in, const Config& c, const Solution* warm, Cache* cache);
Solution solve_admm(const Instance& in, const Config& c, const Solution* warm, Cache* cache);
Solution solve_ama(const Instance& in, const Config& c, const Solution* warm, Cache* cache);
Solution solve(const Instance& in, const Config& c, const Solution* warm, Cache* cache);

// ---- path (path.hpp, path.cpp) ---------------------------------------------
std::vector<double> make_schedule(double start, double end, Index count, bool geometric);
struct Clusters {
  std::vector<Index> labels;
  Index K = 0;
  Mat centroids;
};
Clusters extract_clusters(const Mat& X, const Graph& g, double fuse_tol = 1e-3);
struct PathOut {
  std::vector<double> gammas;
  std::vector<Solution> sols;
  std::vector<Clusters> clusters;
};
PathOut run_path(const Mat& A, const Graph& g, Norm q, const std::vector<double>& gammas,
                 const Config& c, bool warm_start = true, bool require_connected = false,
                 double fuse_tol = 1e-3);

// ---- io (io.cpp:142-165) ---------------------------------------------------
Mat gaussian_mixture(const std::vector<std::vector<double>>& centers, double spread,
                     Index per_center, std::uint64_t seed);

}  // namespace oracle
