// cluspath/b200.hpp — C++ mirror of the reference `cluspath` API
// (/root/reference/proj/include/cluspath: types.hpp, graph.hpp, prox.hpp,
// solvers.hpp, path.hpp) implemented over the C-ABI of libcluspath_b200.so
// (include/cluspath_b200.h).  Same namespace, names, argument meaning and
// exception types (std::invalid_argument / std::runtime_error), so code written
// against the reference recompiles against this header; every numeric routine
// runs on the B200.
//
// Differences a caller can see:
//  * Eigen is not required: `Matrix` is a small owning column-major matrix with
//    the same memory layout as Eigen::MatrixXd (d x n, one sample per column).
//  * LinearOperator / pcg / power_iteration / CholeskyFactor (linalg.hpp) run
//    on the device: the factories hold device data; an operator built from a
//    user functor is applied on the host (one device round trip per apply).
//    CholeskyFactor solves I + rho L by device CG to 1e-14 relative residual
//    per column instead of a sparse LLT factor (same solution up to rounding).
//  * SparseMatrix is a compressed-column struct (Eigen::SparseMatrix layout).
//  * A thread-local device context is used (device 0 unless set_device()).
//  * run_path returns its matrices in page-locked host storage shared by the
//    path's solutions (the device streams each gamma's X and Z into it while
//    the next gamma is solved); copying a Matrix always deep-copies.
#pragma once

#include <charconv>
#include <cmath>
#include <exception>
#include <functional>
#include <fstream>
#include <cstdint>
#include <cstring>
#include <memory>
#include <optional>
#include <stdexcept>
#include <string>
#include <string_view>
#include <utility>
#include <vector>

#include "cluspath_b200.h"

namespace cluspath {

using Index = std::int64_t;

// ---- types.hpp ---------------------------------------------------------------
class Matrix {
 public:
  Matrix() = default;
  Matrix(Index rows, Index cols) : r_(rows), c_(cols), v_(static_cast<size_t>(rows * cols), 0.0), p_(v_.data()) {}
  Matrix(const Matrix& o) : r_(o.r_), c_(o.c_), v_(o.p_, o.p_ + o.size()), p_(v_.data()) {}
  Matrix(Matrix&& o) noexcept : r_(o.r_), c_(o.c_), v_(std::move(o.v_)), ext_(std::move(o.ext_)), p_(o.p_) {
    o.r_ = o.c_ = 0, o.p_ = nullptr;
  }
  Matrix& operator=(const Matrix& o) {
    if (this != &o) *this = Matrix(o);
    return *this;
  }
  Matrix& operator=(Matrix&& o) noexcept {
    r_ = o.r_, c_ = o.c_, v_ = std::move(o.v_), ext_ = std::move(o.ext_), p_ = o.p_;
    o.r_ = o.c_ = 0, o.p_ = nullptr;
    return *this;
  }
  // A rows x cols matrix stored at p inside `slab`, which it keeps alive
  // (run_path's page-locked output storage); copies are deep.
  static Matrix adopt(Index rows, Index cols, std::shared_ptr<double> slab, double* p) {
    Matrix m;
    m.r_ = rows, m.c_ = cols, m.ext_ = std::move(slab), m.p_ = p;
    return m;
  }
  static Matrix Zero(Index rows, Index cols) { return Matrix(rows, cols); }
  static Matrix Constant(Index rows, Index cols, double x) {
    Matrix m(rows, cols);
    for (auto& e : m.v_) e = x;
    return m;
  }
  Index rows() const { return r_; }
  Index cols() const { return c_; }
  Index size() const { return r_ * c_; }
  double* data() { return p_; }
  const double* data() const { return p_; }
  double& operator()(Index r, Index c) { return p_[c * r_ + r]; }
  double operator()(Index r, Index c) const { return p_[c * r_ + r]; }
  double* col(Index c) { return p_ + c * r_; }
  const double* col(Index c) const { return p_ + c * r_; }
  void resize(Index rows, Index cols) {
    r_ = rows, c_ = cols;
    ext_.reset();
    v_.assign(static_cast<size_t>(rows * cols), 0.0);
    p_ = v_.data();
  }
  bool allFinite() const {
    for (Index k = 0; k < size(); ++k)
      if (!std::isfinite(p_[k])) return false;
    return true;
  }

 private:
  Index r_ = 0, c_ = 0;
  std::vector<double> v_;
  std::shared_ptr<double> ext_;
  double* p_ = nullptr;
};
using Vector = std::vector<double>;

namespace detail {
inline void check(int rc) {
  if (rc == CP_OK) return;
  const std::string msg = cp_last_error();
  if (rc == CP_EINVAL) throw std::invalid_argument(msg);
  throw std::runtime_error(msg);
}
struct CtxHolder {
  cp_ctx* ctx = nullptr;
  int device = 0;
  ~CtxHolder() {
    if (ctx) cp_ctx_destroy(ctx);
  }
};
inline CtxHolder& holder() {
  thread_local CtxHolder h;
  return h;
}
inline cp_ctx* ctx() {
  auto& h = holder();
  if (!h.ctx) check(cp_ctx_create(h.device, &h.ctx));
  return h.ctx;
}
struct DataDeleter {
  void operator()(cp_data* p) const { cp_data_destroy(p); }
};
struct GraphDeleter {
  void operator()(cp_graph* p) const { cp_graph_destroy(p); }
};
}  // namespace detail

// Select the CUDA device for this thread's subsequent calls.
inline void set_device(int device) {
  auto& h = detail::holder();
  if (h.ctx && h.device != device) {
    cp_ctx_destroy(h.ctx);
    h.ctx = nullptr;
  }
  h.device = device;
}

struct DataMatrix {
  Matrix values;                           // d x n
  std::vector<std::string> feature_names;  // optional, size d when present
  Index d() const { return values.rows(); }
  Index n() const { return values.cols(); }
};

// make_data_matrix (types.hpp:25-26; graph.cpp:10-23)
inline DataMatrix make_data_matrix(Matrix values, std::vector<std::string> feature_names = {}) {
  if (values.rows() < 1 || values.cols() < 1)
    throw std::invalid_argument("data matrix must have at least one feature and one sample");
  if (!values.allFinite()) throw std::invalid_argument("data matrix contains non-finite entries");
  if (!feature_names.empty()) {
    if (static_cast<Index>(feature_names.size()) != values.rows())
      throw std::invalid_argument("feature_names size does not match feature count");
    for (const auto& s : feature_names)
      if (s.empty()) throw std::invalid_argument("feature_names entries must be non-empty");
  }
  return DataMatrix{std::move(values), std::move(feature_names)};
}

namespace detail {
inline std::shared_ptr<cp_data> upload(const DataMatrix& data) {
  cp_data* p = nullptr;
  check(cp_data_create(ctx(), data.values.data(), data.d(), data.n(), &p));
  return std::shared_ptr<cp_data>(p, DataDeleter{});
}
}  // namespace detail

// ---- graph.hpp ---------------------------------------------------------------
struct Edge {
  Index i = 0;
  Index j = 0;
  double w = 0.0;
};

class WeightedGraph {
 public:
  WeightedGraph() = default;
  // Sorts and validates on the device (graph.cpp:25-45).
  WeightedGraph(Index n, std::vector<Edge> edges) {
    std::vector<int64_t> i(edges.size()), j(edges.size());
    std::vector<double> w(edges.size());
    for (size_t l = 0; l < edges.size(); ++l) i[l] = edges[l].i, j[l] = edges[l].j, w[l] = edges[l].w;
    cp_graph* g = nullptr;
    detail::check(cp_graph_from_edges(detail::ctx(), n, i.data(), j.data(), w.data(),
                                      static_cast<int64_t>(edges.size()), &g));
    adopt(g);
  }
  static WeightedGraph from_handle(cp_graph* g) {
    WeightedGraph out;
    out.adopt(g);
    return out;
  }

  Index nodes() const { return n_; }
  Index edge_count() const { return static_cast<Index>(edges_.size()); }
  const std::vector<Edge>& edges() const { return edges_; }
  const Edge& edge(Index l) const { return edges_.at(static_cast<size_t>(l)); }
  std::optional<Index> find_edge(Index i, Index j) const {
    if (i > j) std::swap(i, j);
    size_t lo = 0, hi = edges_.size();
    while (lo < hi) {
      const size_t mid = (lo + hi) / 2;
      const Edge& e = edges_[mid];
      if (e.i < i || (e.i == i && e.j < j)) lo = mid + 1;
      else hi = mid;
    }
    if (lo < edges_.size() && edges_[lo].i == i && edges_[lo].j == j) return static_cast<Index>(lo);
    return std::nullopt;
  }
  Index degree(Index v) const {
    if (v < 0 || v >= n_) throw std::invalid_argument("node index out of range");
    return degree_[static_cast<size_t>(v)];
  }
  Index max_degree() const {
    Index m = 0;
    for (Index x : degree_) m = std::max(m, x);
    return m;
  }
  Vector weights() const {
    Vector w(edges_.size());
    for (size_t l = 0; l < edges_.size(); ++l) w[l] = edges_[l].w;
    return w;
  }
  // kNN squared distances of the edges (NaN for user edge lists).
  const Vector& squared_distances() const { return d2_; }
  cp_graph* handle() const { return h_.get(); }

 private:
  void adopt(cp_graph* g) {
    h_ = std::shared_ptr<cp_graph>(g, detail::GraphDeleter{});
    n_ = cp_graph_nodes(g);
    const Index E = cp_graph_edge_count(g);
    std::vector<int64_t> i(static_cast<size_t>(E)), j(static_cast<size_t>(E));
    Vector w(static_cast<size_t>(E));
    d2_.assign(static_cast<size_t>(E), 0.0);
    detail::check(cp_graph_export(detail::ctx(), g, i.data(), j.data(), w.data(), d2_.data()));
    edges_.resize(static_cast<size_t>(E));
    for (Index l = 0; l < E; ++l) edges_[static_cast<size_t>(l)] = Edge{i[static_cast<size_t>(l)], j[static_cast<size_t>(l)], w[static_cast<size_t>(l)]};
    std::vector<int64_t> deg(static_cast<size_t>(n_));
    detail::check(cp_graph_degrees(detail::ctx(), g, deg.data()));
    degree_.assign(deg.begin(), deg.end());
  }
  std::shared_ptr<cp_graph> h_;
  Index n_ = 0;
  std::vector<Edge> edges_;
  std::vector<Index> degree_;
  Vector d2_;
};

// compute_knn_weights (graph.hpp:58; graph.cpp:75-114)
inline WeightedGraph compute_knn_weights(const DataMatrix& data, Index k, double phi) {
  auto d = detail::upload(data);
  cp_graph* g = nullptr;
  detail::check(cp_knn_graph(detail::ctx(), d.get(), k, phi, &g));
  return WeightedGraph::from_handle(g);
}

// IncidenceOperator (graph.hpp:62-86)
// Compressed-column sparse matrix (the layout of Eigen::SparseMatrix<double>).
struct SparseMatrix {
  Index rows_ = 0, cols_ = 0;
  std::vector<int64_t> colptr, rowidx;
  std::vector<double> values;
  Index rows() const { return rows_; }
  Index cols() const { return cols_; }
  Index nonZeros() const { return static_cast<Index>(values.size()); }
  Matrix toDense() const {
    Matrix M(rows_, cols_);
    for (Index c = 0; c < cols_; ++c)
      for (int64_t q = colptr[static_cast<size_t>(c)]; q < colptr[static_cast<size_t>(c) + 1]; ++q)
        M(rowidx[static_cast<size_t>(q)], c) = values[static_cast<size_t>(q)];
    return M;
  }
};

class IncidenceOperator {
 public:
  explicit IncidenceOperator(const WeightedGraph& g) : graph_(&g) {}
  Index nodes() const { return graph_->nodes(); }
  Index edge_count() const { return graph_->edge_count(); }
  const WeightedGraph& graph() const { return *graph_; }
  Matrix apply(const Matrix& X) const {
    Matrix out;
    apply_into(X, out);
    return out;
  }
  void apply_into(const Matrix& X, Matrix& out) const {
    out.resize(X.rows(), edge_count());
    detail::check(cp_incidence_apply(detail::ctx(), graph_->handle(), X.data(), X.rows(), X.cols(), out.data()));
  }
  Matrix apply_transpose(const Matrix& Z) const {
    Matrix out;
    apply_transpose_into(Z, out);
    return out;
  }
  void apply_transpose_into(const Matrix& Z, Matrix& out) const {
    out.resize(Z.rows(), nodes());
    detail::check(cp_incidence_apply_t(detail::ctx(), graph_->handle(), Z.data(), Z.rows(), Z.cols(), out.data()));
  }
  // laplacian() (graph.hpp:82): B B^T in compressed columns, built on the device.
  SparseMatrix laplacian() const {
    SparseMatrix L;
    L.rows_ = L.cols_ = graph_->nodes();
    int64_t nnz = 0;
    detail::check(cp_graph_laplacian(detail::ctx(), graph_->handle(), nullptr, nullptr, nullptr, &nnz));
    L.colptr.resize(static_cast<size_t>(L.cols_ + 1));
    L.rowidx.resize(static_cast<size_t>(nnz));
    L.values.resize(static_cast<size_t>(nnz));
    detail::check(cp_graph_laplacian(detail::ctx(), graph_->handle(), L.colptr.data(), L.rowidx.data(),
                                     L.values.data(), &nnz));
    return L;
  }
  // power_iteration(LinearOperator::sparse(laplacian())) (linalg.cpp:194-242)
  double laplacian_lambda_max(double tol = 1e-9, Index max_iter = 10000) const {
    double lam = 0.0;
    detail::check(cp_laplacian_lambda_max(detail::ctx(), graph_->handle(), tol, max_iter, &lam));
    return lam;
  }

 private:
  const WeightedGraph* graph_;
};

// graph.hpp:90-92
inline std::vector<Index> connected_components(const WeightedGraph& g) {
  std::vector<int64_t> lab(static_cast<size_t>(g.nodes()));
  int64_t K = 0;
  detail::check(cp_connected_components(detail::ctx(), g.handle(), lab.data(), &K));
  return std::vector<Index>(lab.begin(), lab.end());
}
inline Index component_count(const std::vector<Index>& labels) {
  Index best = -1;
  for (Index l : labels) best = std::max(best, l);
  return best + 1;
}

// ---- prox.hpp ----------------------------------------------------------------
// prox.hpp:8 PenaltyNorm{l1, l2}, extended with linf (q = infinity; no
// reference counterpart, C-ABI code 0).  penalty_norm_from_q keeps the
// reference's q in {1, 2}; linf is selected by name.
enum class PenaltyNorm { l1, l2, linf };
inline PenaltyNorm penalty_norm_from_q(int q) {
  if (q == 1) return PenaltyNorm::l1;
  if (q == 2) return PenaltyNorm::l2;
  throw std::invalid_argument("penalty norm exponent must be 1 or 2, got " + std::to_string(q));
}
inline int penalty_q(PenaltyNorm norm) { return norm == PenaltyNorm::l1 ? 1 : (norm == PenaltyNorm::l2 ? 2 : 0); }

// Columnwise helpers (prox.hpp:28-33), on the device.
inline void prox_columns_into(const Matrix& V, const Vector& thresholds, PenaltyNorm norm, Matrix& out) {
  if (static_cast<Index>(thresholds.size()) != V.cols())
    throw std::invalid_argument("prox_columns: one threshold per column required");
  out.resize(V.rows(), V.cols());
  detail::check(cp_prox_columns(detail::ctx(), penalty_q(norm), V.data(), thresholds.data(), V.rows(), V.cols(),
                                out.data()));
}
inline void project_columns_inplace(Matrix& Z, const Vector& radii, PenaltyNorm norm) {
  if (static_cast<Index>(radii.size()) != Z.cols())
    throw std::invalid_argument("project_columns: one radius per column required");
  Matrix out(Z.rows(), Z.cols());
  detail::check(cp_project_columns(detail::ctx(), penalty_q(norm), Z.data(), radii.data(), Z.rows(), Z.cols(),
                                   out.data()));
  Z = std::move(out);
}
inline Matrix project_columns(const Matrix& Z, const Vector& radii, PenaltyNorm norm) {
  Matrix out = Z;
  project_columns_inplace(out, radii, norm);
  return out;
}
// Single-vector forms (prox.hpp:19-26): one-column device calls.
inline Vector prox_norm(const Vector& v, double t, PenaltyNorm norm) {
  Matrix V(static_cast<Index>(v.size()), 1), out;
  std::memcpy(V.data(), v.data(), v.size() * sizeof(double));
  prox_columns_into(V, Vector{t}, norm, out);
  return Vector(out.data(), out.data() + v.size());
}
inline Vector project_dual_ball(const Vector& z, double r, PenaltyNorm norm) {
  Matrix Z(static_cast<Index>(z.size()), 1);
  std::memcpy(Z.data(), z.data(), z.size() * sizeof(double));
  project_columns_inplace(Z, Vector{r}, norm);
  return Vector(Z.data(), Z.data() + z.size());
}
// ProxJacobian::diag per column (prox.hpp:38-49).
inline Matrix prox_jacobian_diag(const Matrix& V, const Vector& thresholds, PenaltyNorm norm) {
  Matrix out(V.rows(), V.cols());
  detail::check(cp_prox_jacobian_diag(detail::ctx(), penalty_q(norm), V.data(), thresholds.data(), V.rows(),
                                      V.cols(), out.data()));
  return out;
}
// prox_jacobian (prox.hpp:38-54): the structured Jacobian of prox_{t||.||} at v;
// apply / diag evaluate on the device (cp_prox_jacobian_apply / _diag).
struct ProxJacobian {
  Vector v;
  double t = 0.0;
  PenaltyNorm norm = PenaltyNorm::l2;
  Vector apply(const Vector& w) const {
    if (w.size() != v.size()) throw std::invalid_argument("ProxJacobian::apply: size mismatch");
    Vector out(v.size());
    const double tt[1] = {t};
    detail::check(cp_prox_jacobian_apply(detail::ctx(), penalty_q(norm), v.data(), tt, w.data(),
                                         static_cast<int64_t>(v.size()), 1, out.data()));
    return out;
  }
  double diag(Index r) const {
    Vector out(v.size());
    const double tt[1] = {t};
    detail::check(cp_prox_jacobian_diag(detail::ctx(), penalty_q(norm), v.data(), tt,
                                        static_cast<int64_t>(v.size()), 1, out.data()));
    return out[static_cast<size_t>(r)];
  }
};
inline ProxJacobian prox_jacobian(const Vector& v, double t, PenaltyNorm norm) {
  if (!(t >= 0.0) || !std::isfinite(t)) throw std::invalid_argument("prox_jacobian: threshold must be finite and >= 0");
  return ProxJacobian{v, t, norm};
}

// norm_value / dual_norm_value (prox.hpp:14-15; prox.cpp:25-31), on the device.
inline std::pair<double, double> norm_pair(const Vector& v, PenaltyNorm norm) {
  double a = 0.0, b = 0.0;
  detail::check(cp_norm_values(detail::ctx(), penalty_q(norm), v.data(), static_cast<int64_t>(v.size()), 1, &a, &b));
  return {a, b};
}
inline double norm_value(const Vector& v, PenaltyNorm norm) { return norm_pair(v, norm).first; }
inline double dual_norm_value(const Vector& v, PenaltyNorm norm) { return norm_pair(v, norm).second; }
// prox_norm_into / project_dual_ball_into (prox.hpp:20-26)
inline void prox_norm_into(const Vector& v, double t, PenaltyNorm norm, Vector& out) {
  if (!(t >= 0.0) || !std::isfinite(t)) throw std::invalid_argument("prox_norm: threshold must be finite and >= 0");
  out = prox_norm(v, t, norm);
}
inline void project_dual_ball_into(const Vector& z, double r, PenaltyNorm norm, Vector& out) {
  if (!(r >= 0.0) || !std::isfinite(r))
    throw std::invalid_argument("project_dual_ball: threshold must be finite and >= 0");
  out = project_dual_ball(z, r, norm);
}

inline double moreau_check(const Vector& v, double t, PenaltyNorm norm) {
  const Vector p = prox_norm(v, t, norm), q = project_dual_ball(v, t, norm);
  double m = 0.0;
  for (size_t k = 0; k < v.size(); ++k) m = std::max(m, std::abs(p[k] + q[k] - v[k]));
  return m;
}

// ---- linalg.hpp ----------------------------------------------------------------
// LinearOperator (linalg.hpp:38-65).  Factories hold device data; a functor
// operator is applied on the host through the C-ABI callback.
class LinearOperator {
 public:
  using ApplyFn = std::function<Matrix(const Matrix&)>;
  LinearOperator(Index rows, ApplyFn fn, bool symmetric = true, bool positive_definite = false)
      : fn_(std::make_shared<Functor>()) {
    if (rows < 0) throw std::invalid_argument("LinearOperator: negative dimension");
    if (!fn) throw std::invalid_argument("LinearOperator: empty apply function");
    fn_->fn = std::move(fn);
    cp_linop* h = nullptr;
    detail::check(cp_linop_callback(detail::ctx(), rows, &LinearOperator::trampoline, fn_.get(), symmetric ? 1 : 0,
                                    positive_definite ? 1 : 0, &h));
    h_.reset(h, cp_linop_destroy);
  }
  Index rows() const { return info().rows; }
  bool symmetric() const { return info().sym; }
  bool positive_definite() const { return info().pd; }
  Matrix apply(const Matrix& x) const {
    if (x.rows() != rows()) throw std::invalid_argument("LinearOperator::apply: operand has wrong row count");
    Matrix out(x.rows(), x.cols());
    rethrow(cp_linop_apply(detail::ctx(), h_.get(), x.data(), x.cols(), out.data()));
    return out;
  }
  static LinearOperator identity(Index n) { return make([&](cp_linop** h) { return cp_linop_identity(detail::ctx(), n, h); }); }
  static LinearOperator dense(const Matrix& M, bool positive_definite = false) {
    if (M.rows() != M.cols()) throw std::invalid_argument("LinearOperator::dense: matrix must be square");
    return make([&](cp_linop** h) {
      return cp_linop_dense(detail::ctx(), M.data(), M.rows(), positive_definite ? 1 : 0, h);
    });
  }
  static LinearOperator sparse(const SparseMatrix& M, bool positive_definite = false) {
    if (M.rows() != M.cols()) throw std::invalid_argument("LinearOperator::sparse: matrix must be square");
    return make([&](cp_linop** h) {
      return cp_linop_sparse(detail::ctx(), M.rows(), M.colptr.data(), M.rowidx.data(), M.values.data(),
                             positive_definite ? 1 : 0, h);
    });
  }
  static LinearOperator jacobi(const Vector& diag) {
    return make([&](cp_linop** h) {
      return cp_linop_jacobi(detail::ctx(), diag.data(), static_cast<int64_t>(diag.size()), 1, h);
    });
  }
  static LinearOperator jacobi(const Matrix& diag) {
    return make([&](cp_linop** h) {
      return cp_linop_jacobi(detail::ctx(), diag.data(), diag.rows(), diag.cols() > 0 ? diag.cols() : 1, h);
    });
  }
  const cp_linop* handle() const { return h_.get(); }
  // a user functor's exception (or a C-ABI error) after a device call
  void rethrow(int rc) const {
    if (fn_ && fn_->err) {
      std::exception_ptr e = fn_->err;
      fn_->err = nullptr;
      std::rethrow_exception(e);
    }
    detail::check(rc);
  }

 private:
  struct Functor {
    ApplyFn fn;
    std::exception_ptr err;
  };
  struct Info {
    Index rows;
    bool sym, pd;
  };
  LinearOperator() = default;
  template <class F>
  static LinearOperator make(F f) {
    cp_linop* h = nullptr;
    detail::check(f(&h));
    LinearOperator op;
    op.h_.reset(h, cp_linop_destroy);
    return op;
  }
  Info info() const {
    int64_t r = 0;
    int s = 0, p = 0;
    detail::check(cp_linop_info(h_.get(), &r, &s, &p));
    return {r, s != 0, p != 0};
  }
  static int trampoline(void* user, const double* in, double* out, int64_t rows, int64_t cols) {
    auto* f = static_cast<Functor*>(user);
    try {
      Matrix x(rows, cols);
      std::memcpy(x.data(), in, sizeof(double) * static_cast<size_t>(rows * cols));
      Matrix y = f->fn(x);
      if (y.rows() != rows || y.cols() != cols)
        throw std::runtime_error("LinearOperator::apply: image shape mismatch");
      std::memcpy(out, y.data(), sizeof(double) * static_cast<size_t>(rows * cols));
      return 0;
    } catch (...) {
      f->err = std::current_exception();
      return 1;
    }
  }
  std::shared_ptr<cp_linop> h_;
  std::shared_ptr<Functor> fn_;
};

struct PcgResult {
  Matrix x;
  Index iterations = 0;
  double residual = 0.0;  // relative, recomputed from op at exit
  bool converged = false;
};
// pcg (linalg.hpp:76-77; linalg.cpp:143-192) on the device.
inline PcgResult pcg(const LinearOperator& op, const Matrix& rhs, const LinearOperator* preconditioner, double tol,
                     Index max_iter) {
  if (rhs.rows() != op.rows()) throw std::invalid_argument("pcg: rhs row count does not match the operator");
  PcgResult r;
  r.x.resize(rhs.rows(), rhs.cols());
  int64_t it = 0;
  double res = 0.0;
  int32_t conv = 0;
  const int rc = cp_pcg(detail::ctx(), op.handle(), rhs.data(), rhs.cols(),
                        preconditioner ? preconditioner->handle() : nullptr, tol, max_iter, r.x.data(), &it, &res,
                        &conv);
  if (preconditioner) preconditioner->rethrow(CP_OK);  // a functor preconditioner's own exception first
  op.rethrow(rc);
  r.iterations = it, r.residual = res, r.converged = conv != 0;
  return r;
}
inline PcgResult pcg(const LinearOperator& op, const Vector& rhs, const LinearOperator* preconditioner, double tol,
                     Index max_iter) {
  Matrix b(static_cast<Index>(rhs.size()), 1);
  std::memcpy(b.data(), rhs.data(), rhs.size() * sizeof(double));
  return pcg(op, b, preconditioner, tol, max_iter);
}
// power_iteration (linalg.hpp:82-83; linalg.cpp:194-242) on the device.
inline double power_iteration(const LinearOperator& op, double tol = 1e-9, Index max_iter = 10000) {
  double lam = 0.0;
  op.rethrow(cp_power_iteration(detail::ctx(), op.handle(), tol, max_iter, &lam));
  return lam;
}
// CholeskyFactor (linalg.hpp:17-33): (I + rho L)^{-1} on the device.
class CholeskyFactor {
 public:
  CholeskyFactor(const SparseMatrix& L, double rho) : size_(L.rows()), rho_(rho) {
    if (L.rows() != L.cols()) throw std::invalid_argument("cholesky: matrix must be square");
    cp_factor* f = nullptr;
    detail::check(cp_factor_create(detail::ctx(), L.rows(), L.colptr.data(), L.rowidx.data(), L.values.data(), rho, &f));
    f_.reset(f, cp_factor_destroy);
  }
  Index size() const { return size_; }
  double rho() const { return rho_; }
  Matrix solve(const Matrix& rhs) const {
    if (rhs.rows() != size_) throw std::invalid_argument("cholesky solve: rhs has wrong row count");
    Matrix out(rhs.rows(), rhs.cols());
    detail::check(cp_factor_solve(detail::ctx(), f_.get(), rhs.data(), rhs.cols(), out.data()));
    return out;
  }

 private:
  std::shared_ptr<cp_factor> f_;
  Index size_ = 0;
  double rho_ = 0.0;
};

// ---- solvers.hpp -------------------------------------------------------------
enum class Algorithm { ADMM, FastAMA, SSNAL };
inline const char* algorithm_name(Algorithm a) {
  switch (a) {
    case Algorithm::ADMM: return "admm";
    case Algorithm::FastAMA: return "ama";
    case Algorithm::SSNAL: return "ssnal";
  }
  return "?";
}
inline Algorithm algorithm_from_name(std::string_view name) {
  if (name == "admm") return Algorithm::ADMM;
  if (name == "ama" || name == "fast-ama" || name == "fastama") return Algorithm::FastAMA;
  if (name == "ssnal") return Algorithm::SSNAL;
  throw std::invalid_argument("unknown solver '" + std::string(name) + "' (expected ssnal, admm or ama)");
}

struct ProblemInstance {
  const DataMatrix* data = nullptr;
  const WeightedGraph* graph = nullptr;
  IncidenceOperator B;
  double gamma = 0.0;
  PenaltyNorm norm = PenaltyNorm::l2;
  std::shared_ptr<cp_data> dev;  // device copy of A

  ProblemInstance(const DataMatrix& data_, const WeightedGraph& graph_, double gamma_, PenaltyNorm norm_)
      : data(&data_), graph(&graph_), B(graph_), gamma(gamma_), norm(norm_) {
    if (data_.n() != graph_.nodes())
      throw std::invalid_argument("instance: graph has " + std::to_string(graph_.nodes()) + " nodes for " +
                                  std::to_string(data_.n()) + " samples");
    if (!(gamma >= 0.0) || !std::isfinite(gamma)) throw std::invalid_argument("instance: gamma must be finite and >= 0");
    dev = detail::upload(data_);
  }
  const Matrix& A() const { return data->values; }
  Index d() const { return data->d(); }
  Index n() const { return data->n(); }
  Index edge_count() const { return graph->edge_count(); }
  Vector penalty_radii() const {
    Vector r = graph->weights();
    for (double& x : r) x *= gamma;
    return r;
  }
};

struct TerminationRecord {
  double f_primal = 0.0, f_dual = 0.0, gap = 0.0;
  Index iterations = 0;
  bool converged = false;
  double wall_time = 0.0;
  Index newton = 0, cg = 0, armijo = 0;  // work counters (extension)
};

struct TraceRow {  // solvers.hpp:54-60
  Index iter = 0;
  double f_p = 0.0;
  double f_d = 0.0;
  double gap = 0.0;
  double elapsed_s = 0.0;
};

struct Solution {
  Matrix X;
  Matrix Z;
  TerminationRecord termination;
  std::vector<TraceRow> trace;  // filled when SolverConfig::collect_trace
};

struct SolverConfig {
  Algorithm algorithm = Algorithm::SSNAL;
  double epsilon = 1e-6;
  double kkt_factor = 10.0;
  Index max_iter = 0;
  std::optional<double> time_limit;
  double admm_rho = 1.0;
  double ama_step_safety = 0.99;
  double ssnal_sigma0 = 1.0;
  double armijo_mu = 1e-4;
  double backtrack_beta = 0.5;
  Index ssnal_newton_max = 50;
  Index pcg_max_iter = 500;
  bool collect_trace = false;

  Index resolved_max_iter() const { return max_iter > 0 ? max_iter : (algorithm == Algorithm::SSNAL ? 100 : 20000); }
  void validate() const {
    if (time_limit && !(*time_limit > 0.0)) throw std::invalid_argument("config: time_limit must be positive when set");
    cp_solver_config c = to_c();
    (void)c;
  }
  cp_solver_config to_c() const {
    cp_solver_config c;
    cp_solver_config_default(&c);
    c.algorithm = static_cast<int32_t>(algorithm);
    c.collect_trace = collect_trace ? 1 : 0;
    c.epsilon = epsilon;
    c.kkt_factor = kkt_factor;
    c.max_iter = max_iter;
    c.time_limit = time_limit ? *time_limit : 0.0;
    c.admm_rho = admm_rho;
    c.ama_step_safety = ama_step_safety;
    c.ssnal_sigma0 = ssnal_sigma0;
    c.armijo_mu = armijo_mu;
    c.backtrack_beta = backtrack_beta;
    c.ssnal_newton_max = ssnal_newton_max;
    c.pcg_max_iter = pcg_max_iter;
    return c;
  }
};

namespace detail {
inline TerminationRecord from_c(const cp_termination& t) {
  TerminationRecord r;
  r.f_primal = t.f_primal, r.f_dual = t.f_dual, r.gap = t.gap, r.iterations = t.iterations;
  r.converged = t.converged != 0, r.wall_time = t.wall_time;
  r.newton = t.newton, r.cg = t.cg, r.armijo = t.armijo;
  return r;
}
}  // namespace detail

// objectives (solvers.hpp:95-118)
inline double primal_objective(const ProblemInstance& inst, const Matrix& X) {
  if (X.rows() != inst.d() || X.cols() != inst.n()) throw std::invalid_argument("primal_objective: X has the wrong shape");
  double out = 0.0;
  detail::check(cp_primal_objective(detail::ctx(), inst.dev.get(), inst.graph->handle(), inst.gamma,
                                    penalty_q(inst.norm), X.data(), &out));
  return out;
}
inline double dual_objective(const ProblemInstance& inst, const Matrix& Z) {
  if (Z.rows() != inst.d() || Z.cols() != inst.edge_count())
    throw std::invalid_argument("dual_objective: Z has the wrong shape");
  double out = 0.0;
  detail::check(cp_dual_objective(detail::ctx(), inst.dev.get(), inst.graph->handle(), inst.gamma,
                                  penalty_q(inst.norm), Z.data(), &out));
  return out;
}
inline double duality_gap(double f_p, double f_d) { return std::abs(f_p - f_d) / (1.0 + std::abs(f_p) + std::abs(f_d)); }
inline Matrix recover_primal(const ProblemInstance& inst, const Matrix& Z) {
  Matrix T = inst.B.apply_transpose(Z);
  Matrix X(inst.d(), inst.n());
  for (Index k = 0; k < X.size(); ++k) X.data()[k] = inst.A().data()[k] - T.data()[k];
  return X;
}
inline double kkt_residual(const ProblemInstance& inst, const Matrix& X, const Matrix& Z) {
  if (X.rows() != inst.d() || X.cols() != inst.n()) throw std::invalid_argument("kkt_residual: X has the wrong shape");
  if (Z.rows() != inst.d() || Z.cols() != inst.edge_count())
    throw std::invalid_argument("kkt_residual: Z has the wrong shape");
  double out = 0.0;
  detail::check(cp_kkt_residual(detail::ctx(), inst.dev.get(), inst.graph->handle(), inst.gamma, penalty_q(inst.norm),
                                X.data(), Z.data(), &out));
  return out;
}
// AL subproblem pieces (solvers.hpp:143-156)
inline double ssnal_phi_value(const ProblemInstance& inst, const Matrix& Z, double sigma, const Matrix& X) {
  double out = 0.0;
  detail::check(cp_ssnal_phi_value(detail::ctx(), inst.dev.get(), inst.graph->handle(), inst.gamma,
                                   penalty_q(inst.norm), Z.data(), sigma, X.data(), &out));
  return out;
}
inline Matrix ssnal_phi_gradient(const ProblemInstance& inst, const Matrix& Z, double sigma, const Matrix& X) {
  Matrix out(inst.d(), inst.n());
  detail::check(cp_ssnal_phi_gradient(detail::ctx(), inst.dev.get(), inst.graph->handle(), inst.gamma,
                                      penalty_q(inst.norm), Z.data(), sigma, X.data(), out.data()));
  return out;
}
inline Matrix ssnal_hessian_apply(const ProblemInstance& inst, const Matrix& Z, double sigma, const Matrix& X,
                                  const Matrix& D) {
  Matrix out(inst.d(), inst.n());
  detail::check(cp_ssnal_hessian_apply(detail::ctx(), inst.dev.get(), inst.graph->handle(), inst.gamma,
                                       penalty_q(inst.norm), Z.data(), sigma, X.data(), D.data(), out.data()));
  return out;
}

// Per-path state: held by the device context (solvers.hpp:119-123).
struct SolveCache {};

// solve / solve_* (solvers.hpp:132-141)
inline Solution solve(const ProblemInstance& inst, const SolverConfig& config, const Solution* warm = nullptr,
                      SolveCache* = nullptr) {
  config.validate();
  cp_solver_config c = config.to_c();
  Solution sol;
  sol.X.resize(inst.d(), inst.n());
  sol.Z.resize(inst.d(), inst.edge_count());
  cp_termination t;
  detail::check(cp_solve(detail::ctx(), inst.dev.get(), inst.graph->handle(), inst.gamma, penalty_q(inst.norm), &c,
                         warm ? warm->X.data() : nullptr, warm ? warm->X.rows() : 0, warm ? warm->X.cols() : 0,
                         warm ? warm->Z.data() : nullptr, warm ? warm->Z.cols() : 0, sol.X.data(), sol.Z.data(),
                         &t));
  sol.termination = detail::from_c(t);
  if (config.collect_trace) {
    int64_t cnt = 0;
    detail::check(cp_last_trace(detail::ctx(), nullptr, 0, &cnt));
    std::vector<cp_trace_row> rows(static_cast<size_t>(cnt));
    detail::check(cp_last_trace(detail::ctx(), rows.data(), cnt, &cnt));
    for (const auto& r : rows) sol.trace.push_back(TraceRow{r.iter, r.f_p, r.f_d, r.gap, r.elapsed_s});
  }
  return sol;
}
inline Solution solve_ssnal(const ProblemInstance& inst, SolverConfig config, const Solution* warm = nullptr,
                            SolveCache* cache = nullptr) {
  config.algorithm = Algorithm::SSNAL;
  return solve(inst, config, warm, cache);
}
inline Solution solve_admm(const ProblemInstance& inst, SolverConfig config, const Solution* warm = nullptr,
                           SolveCache* cache = nullptr) {
  config.algorithm = Algorithm::ADMM;
  return solve(inst, config, warm, cache);
}
inline Solution solve_fast_ama(const ProblemInstance& inst, SolverConfig config, const Solution* warm = nullptr,
                               SolveCache* cache = nullptr) {
  config.algorithm = Algorithm::FastAMA;
  return solve(inst, config, warm, cache);
}

// ---- path.hpp ----------------------------------------------------------------
enum class Spacing { linear, geometric };
inline const char* spacing_name(Spacing s) { return s == Spacing::linear ? "linear" : "geometric"; }
inline Spacing spacing_from_name(std::string_view name) {
  if (name == "linear") return Spacing::linear;
  if (name == "geometric") return Spacing::geometric;
  throw std::invalid_argument("unknown spacing '" + std::string(name) + "' (expected linear or geometric)");
}

struct GammaSchedule {
  std::vector<double> values;
  double start = 0.0;
  double end = 0.0;
  Index count = 0;
  Spacing spacing = Spacing::geometric;
};
inline GammaSchedule make_schedule(double start, double end, Index count, Spacing spacing) {
  GammaSchedule s;
  s.values.assign(static_cast<size_t>(count > 0 ? count : 1), 0.0);
  detail::check(cp_make_schedule(start, end, count, spacing == Spacing::geometric ? 1 : 0, s.values.data()));
  s.values.resize(static_cast<size_t>(count));
  s.start = start, s.end = end, s.count = count, s.spacing = spacing;
  return s;
}

struct ClusterAssignment {
  std::vector<Index> labels;
  Index K = 0;
  Matrix centroids;
};
inline ClusterAssignment extract_clusters(const Matrix& X, const WeightedGraph& graph, double fuse_tol = 1e-3) {
  std::vector<int64_t> lab(static_cast<size_t>(X.cols()));
  int64_t K = 0;
  Matrix cent(X.rows(), X.cols());
  detail::check(cp_extract_clusters(detail::ctx(), graph.handle(), X.data(), X.rows(), X.cols(), fuse_tol, lab.data(),
                                    &K, cent.data()));
  ClusterAssignment out;
  out.labels.assign(lab.begin(), lab.end());
  out.K = K;
  out.centroids.resize(X.rows(), K);
  std::memcpy(out.centroids.data(), cent.data(), sizeof(double) * static_cast<size_t>(X.rows() * K));
  return out;
}
inline std::pair<Vector, Vector> two_point_closed_form(const Vector& a1, const Vector& a2, double w, double gamma) {
  if (a1.size() != a2.size()) throw std::invalid_argument("two_point_closed_form: dimension mismatch");
  if (!(w > 0.0)) throw std::invalid_argument("two_point_closed_form: weight must be positive");
  if (!(gamma >= 0.0)) throw std::invalid_argument("two_point_closed_form: gamma must be >= 0");
  double nc = 0.0;
  for (size_t k = 0; k < a1.size(); ++k) nc += (a1[k] - a2[k]) * (a1[k] - a2[k]);
  nc = std::sqrt(nc);
  if (nc == 0.0) return {a1, a2};
  const double s = std::min(2.0 * gamma * w / nc, 1.0);
  Vector x1 = a1, x2 = a2;
  for (size_t k = 0; k < a1.size(); ++k) {
    const double c = a1[k] - a2[k];
    x1[k] = a1[k] - 0.5 * s * c;
    x2[k] = a2[k] + 0.5 * s * c;
  }
  return {x1, x2};
}

struct PathOptions {
  bool warm_start = true;
  bool require_connected = false;
  double fuse_tol = 1e-3;
};

struct PathResult {
  GammaSchedule schedule;
  std::vector<Solution> solutions;
  std::vector<ClusterAssignment> assignments;
  std::vector<TerminationRecord> stats;
  SolverConfig solver;
  bool all_converged() const {
    for (const auto& s : stats)
      if (!s.converged) return false;
    return true;
  }
};

// run_path (path.hpp:71-73; path.cpp:110-142): the whole sweep on the GPU.
// X(gamma) and Z(gamma) land in one page-locked host slab shared by the
// returned matrices (streamed by the device while the next gamma is solved);
// centroids and trace rows arrive through the C-ABI path sink.
inline PathResult run_path(const DataMatrix& data, const WeightedGraph& graph, PenaltyNorm norm,
                           const GammaSchedule& schedule, const SolverConfig& config, const PathOptions& options = {}) {
  if (schedule.values.empty()) throw std::invalid_argument("run_path: empty schedule");
  if (data.n() != graph.nodes()) throw std::invalid_argument("run_path: graph size does not match the data");
  config.validate();
  auto dev = detail::upload(data);
  const Index T = static_cast<Index>(schedule.values.size());
  const Index d = data.d(), n = data.n(), E = graph.edge_count();
  const size_t mx = static_cast<size_t>(d * n), mz = static_cast<size_t>(d * E);
  void* raw = nullptr;
  detail::check(cp_host_alloc(static_cast<uint64_t>(T) * (mx + mz) * sizeof(double) + 8, &raw));
  std::shared_ptr<double> slab(static_cast<double*>(raw), [](double* p) { cp_host_free(p); });
  double* X = slab.get();
  double* Z = X + static_cast<size_t>(T) * mx;
  std::vector<int64_t> lab(static_cast<size_t>(T * n)), K(static_cast<size_t>(T));
  std::vector<cp_termination> terms(static_cast<size_t>(T));
  cp_solver_config c = config.to_c();
  cp_path_options o{options.warm_start ? 1 : 0, options.require_connected ? 1 : 0, options.fuse_tol};
  struct Sink {
    std::vector<Matrix> cent;
    std::vector<std::vector<TraceRow>> trace;
  } sk;
  sk.cent.resize(static_cast<size_t>(T));
  sk.trace.resize(static_cast<size_t>(T));
  cp_path_sink sink;
  sink.user = &sk;
  sink.centroids = [](void* u, int64_t t, int64_t k, int64_t dd, const double* cent) {
    Matrix m(dd, k);
    if (k) std::memcpy(m.data(), cent, sizeof(double) * static_cast<size_t>(dd * k));
    static_cast<Sink*>(u)->cent[static_cast<size_t>(t)] = std::move(m);
  };
  sink.trace = [](void* u, int64_t t, const cp_trace_row* rows, int64_t cnt) {
    auto& tr = static_cast<Sink*>(u)->trace[static_cast<size_t>(t)];
    for (int64_t k = 0; k < cnt; ++k)
      tr.push_back(TraceRow{rows[k].iter, rows[k].f_p, rows[k].f_d, rows[k].gap, rows[k].elapsed_s});
  };
  sink.skip_identity = 1;  // K = n: centroids = X (filled below from the returned X)
  detail::check(cp_run_path_ex(detail::ctx(), dev.get(), graph.handle(), penalty_q(norm), schedule.values.data(), T,
                               &c, &o, X, Z, lab.data(), K.data(), terms.data(), &sink));
  PathResult r;
  r.schedule = schedule;
  r.solver = config;
  for (Index t = 0; t < T; ++t) {
    Solution s;
    s.X = Matrix::adopt(d, n, slab, X + static_cast<size_t>(t) * mx);
    s.Z = Matrix::adopt(d, E, slab, Z + static_cast<size_t>(t) * mz);
    s.termination = detail::from_c(terms[static_cast<size_t>(t)]);
    s.trace = std::move(sk.trace[static_cast<size_t>(t)]);
    ClusterAssignment a;
    a.labels.assign(lab.begin() + t * n, lab.begin() + (t + 1) * n);
    a.K = K[static_cast<size_t>(t)];
    a.centroids = a.K == n && sk.cent[static_cast<size_t>(t)].size() == 0 && n > 0 ? s.X
                                                                                  : std::move(sk.cent[static_cast<size_t>(t)]);
    r.stats.push_back(s.termination);
    r.assignments.push_back(std::move(a));
    r.solutions.push_back(std::move(s));
  }
  return r;
}

// ---- bench.hpp: performance profiles over device solves (bench.cpp:23-116) -------
struct BenchTask {
  const DataMatrix* data = nullptr;
  const WeightedGraph* graph = nullptr;
  PenaltyNorm norm = PenaltyNorm::l2;
  GammaSchedule schedule;
};
struct MethodCurve {
  Algorithm method = Algorithm::SSNAL;
  std::vector<std::pair<double, Index>> points;  // (tau, problems solved within tau * T)
  Index solved_total = 0;
  double full_time = 0.0;
};
struct PerfProfile {
  double baseline_T = 0.0;
  Index problem_count = 0;
  std::vector<MethodCurve> curves;
};
struct BenchOptions {
  double epsilon = 1e-6;
  Index tau_max = 10;
  std::optional<double> cutoff_override;
  SolverConfig base_config;
  bool warm_start = true;
};
namespace detail {
struct SweepOutcome {
  std::vector<double> finish;
  double total_time = 0.0;
};
inline SweepOutcome sweep(const std::vector<BenchTask>& tasks, Algorithm method, const BenchOptions& options,
                          const double* budget) {
  SweepOutcome out;
  for (const BenchTask& task : tasks) {
    std::optional<Solution> prev;
    for (double gamma : task.schedule.values) {
      if (budget && out.total_time >= *budget) return out;
      SolverConfig config = options.base_config;
      config.algorithm = method;
      config.epsilon = options.epsilon;
      if (budget) {
        const double remaining = *budget - out.total_time;
        config.time_limit = config.time_limit ? std::min(*config.time_limit, remaining) : remaining;
      }
      ProblemInstance inst(*task.data, *task.graph, gamma, task.norm);
      const Solution* warm = (options.warm_start && prev) ? &*prev : nullptr;
      Solution sol = solve(inst, config, warm);
      out.total_time += sol.termination.wall_time;
      if (sol.termination.converged && (!budget || out.total_time <= *budget)) out.finish.push_back(out.total_time);
      prev = std::move(sol);
    }
  }
  return out;
}
}  // namespace detail
inline PerfProfile run_bench(const std::vector<BenchTask>& tasks, const std::vector<Algorithm>& methods,
                             const BenchOptions& options) {
  if (methods.empty()) throw std::invalid_argument("run_bench: no methods given");
  if (tasks.empty()) throw std::invalid_argument("run_bench: no tasks given");
  Index problems = 0;
  for (const BenchTask& t : tasks) {
    if (!t.data || !t.graph) throw std::invalid_argument("run_bench: task is missing data or graph");
    if (t.schedule.values.empty()) throw std::invalid_argument("run_bench: task has an empty schedule");
    problems += static_cast<Index>(t.schedule.values.size());
  }
  if (options.tau_max < 1) throw std::invalid_argument("run_bench: tau_max must be >= 1");
  options.base_config.validate();
  std::vector<detail::SweepOutcome> uncapped;
  for (Algorithm m : methods) uncapped.push_back(detail::sweep(tasks, m, options, nullptr));
  size_t best = 0;
  for (size_t i = 1; i < methods.size(); ++i) {
    const bool more = uncapped[i].finish.size() > uncapped[best].finish.size();
    const bool tie = uncapped[i].finish.size() == uncapped[best].finish.size() &&
                     uncapped[i].total_time < uncapped[best].total_time;
    if (more || tie) best = i;
  }
  if (uncapped[best].finish.empty()) throw std::runtime_error("run_bench: no baseline (no method solved any problem)");
  const double T = uncapped[best].total_time;
  const double cutoff = options.cutoff_override ? *options.cutoff_override : 10.0 * T;
  PerfProfile profile;
  profile.baseline_T = T;
  profile.problem_count = problems;
  for (size_t i = 0; i < methods.size(); ++i) {
    detail::SweepOutcome rerun;
    const detail::SweepOutcome* capped = &uncapped[i];
    if (uncapped[i].total_time > cutoff) {
      rerun = detail::sweep(tasks, methods[i], options, &cutoff);
      capped = &rerun;
    }
    MethodCurve curve;
    curve.method = methods[i];
    curve.full_time = uncapped[i].total_time;
    curve.solved_total = static_cast<Index>(capped->finish.size());
    for (Index tau = 1; tau <= options.tau_max; ++tau) {
      const double horizon = std::min(static_cast<double>(tau) * T, cutoff);
      Index count = 0;
      for (double t : capped->finish) count += t <= horizon ? 1 : 0;
      curve.points.emplace_back(static_cast<double>(tau), count);
    }
    profile.curves.push_back(std::move(curve));
  }
  return profile;
}
inline std::string format_double(double value);
inline std::string perf_profile_csv(const PerfProfile& profile) {
  std::string csv = "method,tau,solved\n";
  for (const MethodCurve& c : profile.curves)
    for (const auto& [tau, solved] : c.points) {
      csv += algorithm_name(c.method);
      csv += ',';
      csv += format_double(tau);
      csv += ',';
      csv += std::to_string(solved);
      csv += '\n';
    }
  return csv;
}

// ---- output formats (io.cpp:14-18, 120-140; path.cpp:144-177) ------------------
inline std::string format_double(double value) {
  char buf[64];
  auto res = std::to_chars(buf, buf + sizeof(buf), value);
  return std::string(buf, res.ptr);
}
inline void write_matrix_csv(const std::string& path, const Matrix& M) {
  std::ofstream out(path, std::ios::binary);
  if (!out) throw std::runtime_error("cannot open '" + path + "' for writing");
  for (Index r = 0; r < M.rows(); ++r) {
    for (Index c = 0; c < M.cols(); ++c) {
      if (c) out << ',';
      out << format_double(M(r, c));
    }
    out << '\n';
  }
  if (!out) throw std::runtime_error("write to '" + path + "' failed");
}
inline void export_graph_csv(const std::string& path, const WeightedGraph& graph) {
  std::ofstream out(path, std::ios::binary);
  if (!out) throw std::runtime_error("cannot open '" + path + "' for writing");
  out << "i,j,w\n";
  for (const Edge& e : graph.edges()) out << e.i << ',' << e.j << ',' << format_double(e.w) << '\n';
  if (!out) throw std::runtime_error("write to '" + path + "' failed");
}
// JSON with the reference's document shape and keys in nlohmann::json's order
// (std::map: sorted); numbers in std::to_chars shortest form.
inline std::string path_result_to_json(const PathResult& result, int indent = 2) {
  std::string o;
  auto nl = [&](int level) {
    if (indent >= 0) {
      o += '\n';
      o.append(static_cast<size_t>(indent * level), ' ');
    }
  };
  auto num = [&](double v) {
    if (!std::isfinite(v)) {
      o += "null";
      return;
    }
    std::string s = format_double(v);
    o += s;
  };
  auto key = [&](const char* k, int level, bool first) {
    if (!first) o += ',';
    nl(level);
    o += '"';
    o += k;
    o += indent >= 0 ? "\": " : "\":";
  };
  o += '{';
  key("per_gamma", 1, true);
  o += '[';
  for (size_t t = 0; t < result.stats.size(); ++t) {
    const TerminationRecord& rec = result.stats[t];
    const ClusterAssignment& asg = result.assignments[t];
    if (t) o += ',';
    nl(2);
    o += '{';
    key("K", 3, true);
    o += std::to_string(asg.K);
    key("converged", 3, false);
    o += rec.converged ? "true" : "false";
    key("f_d", 3, false);
    num(rec.f_dual);
    key("f_p", 3, false);
    num(rec.f_primal);
    key("gamma", 3, false);
    num(result.schedule.values[t]);
    key("gap", 3, false);
    num(rec.gap);
    key("iterations", 3, false);
    o += std::to_string(rec.iterations);
    key("labels", 3, false);
    o += '[';
    for (size_t i = 0; i < asg.labels.size(); ++i) {
      if (i) o += ',';
      nl(4);
      o += std::to_string(asg.labels[i]);
    }
    if (!asg.labels.empty()) nl(3);
    o += ']';
    key("wall_time_s", 3, false);
    num(rec.wall_time);
    nl(2);
    o += '}';
  }
  if (!result.stats.empty()) nl(1);
  o += ']';
  key("schedule", 1, false);
  o += '{';
  key("count", 2, true);
  o += std::to_string(result.schedule.count);
  key("end", 2, false);
  num(result.schedule.end);
  key("spacing", 2, false);
  o += '"';
  o += spacing_name(result.schedule.spacing);
  o += '"';
  key("start", 2, false);
  num(result.schedule.start);
  key("values", 2, false);
  o += '[';
  for (size_t i = 0; i < result.schedule.values.size(); ++i) {
    if (i) o += ',';
    nl(3);
    num(result.schedule.values[i]);
  }
  if (!result.schedule.values.empty()) nl(2);
  o += ']';
  nl(1);
  o += '}';
  key("solver", 1, false);
  o += '{';
  const SolverConfig& c = result.solver;
  key("admm_rho", 2, true);
  num(c.admm_rho);
  key("algorithm", 2, false);
  o += '"';
  o += algorithm_name(c.algorithm);
  o += '"';
  key("ama_step_safety", 2, false);
  num(c.ama_step_safety);
  key("epsilon", 2, false);
  num(c.epsilon);
  key("kkt_factor", 2, false);
  num(c.kkt_factor);
  key("max_iter", 2, false);
  o += std::to_string(c.resolved_max_iter());
  key("ssnal_sigma0", 2, false);
  num(c.ssnal_sigma0);
  if (c.time_limit) {
    key("time_limit", 2, false);
    num(*c.time_limit);
  }
  nl(1);
  o += '}';
  nl(0);
  o += '}';
  return o;
}

// generate_gaussian_mixture (io.hpp:41-44; io.cpp:142-165); centers as d-vectors.
struct SyntheticData {
  DataMatrix data;
  std::vector<Index> labels;
};
inline SyntheticData generate_gaussian_mixture(const std::vector<Vector>& centers, double spread, Index per_center,
                                               std::uint64_t seed) {
  if (centers.empty()) throw std::invalid_argument("mixture needs at least one center");
  const Index d = static_cast<Index>(centers.front().size()), m = static_cast<Index>(centers.size());
  for (const auto& c : centers)
    if (static_cast<Index>(c.size()) != d) throw std::invalid_argument("mixture centers differ in dimension");
  std::vector<double> C(static_cast<size_t>(d * m));
  for (Index k = 0; k < m; ++k) std::memcpy(C.data() + k * d, centers[static_cast<size_t>(k)].data(), sizeof(double) * static_cast<size_t>(d));
  Matrix A(d, m * (per_center > 0 ? per_center : 0));
  detail::check(cp_gaussian_mixture(C.data(), d, m, spread, per_center, seed, A.data()));
  SyntheticData s{make_data_matrix(std::move(A)), {}};
  for (Index k = 0; k < m; ++k)
    for (Index q = 0; q < per_center; ++q) s.labels.push_back(k);
  return s;
}

}  // namespace cluspath
