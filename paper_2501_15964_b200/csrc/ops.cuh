// Device operators of the solver path (objective.cpp, ssnal.cpp, ama.cpp,
// prox.cpp, linalg.cpp::pcg of the reference), each a fused HBM-streaming
// kernel over node rows or edge rows.  All pointers are device pointers; all
// reductions are fixed-order block partials (run-to-run deterministic).
#pragma once

#include <functional>

#include "graph.cuh"

namespace cpb {

enum { Q_LINF = 0, Q_L1 = 1, Q_L2 = 2 };  // Q_LINF: q = infinity (no reference counterpart)

// One penalty level on one (data, graph) pair: ProblemInstance (solvers.hpp:26-43).
struct Prob {
  Ctx* c = nullptr;
  Data* A = nullptr;
  const Graph* g = nullptr;
  double gamma = 0.0;
  int q = Q_L2;
  double* rad = nullptr;  // E: gamma * w_l (penalty_radii, objective.cpp:36)
  int64_t d() const { return A->d; }
  int64_t n() const { return A->n; }
  int64_t E() const { return g->E; }
};

// A set of edges for the edge passes: the contiguous range [e0, e0 + count),
// or list[0 .. count) when list is set (a partitioned solve's ghost edges).
struct EdgeSel {
  const int* list = nullptr;
  int64_t e0 = 0, count = 0;
  __host__ __device__ int64_t at(int64_t i) const { return list ? static_cast<int64_t>(list[i]) : e0 + i; }
};

void make_radii(Ctx& c, const Graph& g, double gamma, double* rad);
void make_thr(Ctx& c, int64_t E, const double* rad, double sigma, double* thr);

// ---- vector primitives (flat over count doubles) ---------------------------
double dot_dev(Ctx& c, const double* a, const double* b, int64_t count);
void axpy_dev(Ctx& c, double* out, const double* x, double a, const double* y, int64_t count);  // out = x + a*y
void neg_dev(Ctx& c, double* out, const double* x, int64_t count);
void copy_dev(Ctx& c, double* dst, const double* src, int64_t count);
double max_abs_dev(Ctx& c, const double* x, int64_t count);

// ---- prox / projection over edge columns (prox.cpp:73-93) ------------------
void prox_columns_dev(Ctx& c, int q, const double* V, const double* t, int64_t d, int64_t E, double* out);
void project_columns_dev(Ctx& c, int q, const double* Z, const double* r, int64_t d, int64_t E, double* out);
// Whether the last project_columns_dev moved any column (reads a device flag; syncs).
bool last_projection_changed(Ctx& c);
void prox_jacobian_apply_dev(Ctx& c, int q, const double* V, const double* t, const double* W, int64_t d, int64_t E,
                             double* out);
void prox_jacobian_diag_dev(Ctx& c, int q, const double* V, const double* t, int64_t d, int64_t E, double* out);

// ---- SSNAL pieces (ssnal.cpp:24-82) -----------------------------------------
// phi at X (or at X + alpha*D when D != nullptr, materialising Xt): writes V, nv.
// zz = ||Z||^2.  Returns phi (synchronous scalar read).
double eval_phi(const Prob& P, const double* X, const double* D, double alpha, double* Xt, const double* Z,
                double sigma, const double* thr, double zz, double* V, double* nv);
// Per-edge prox scale s (PV = s V for q=2), Jacobian (alpha, beta); returns #edges with beta != 0.
int64_t jac_params(const Prob& P, const double* nv, const double* thr, double* ps, double* jal, double* jbe);
// G = X - A + sigma B^T(V - PV) and the Jacobi diagonal; returns ||G||^2.
double grad_diag(const Prob& P, const double* X, const double* V, const double* ps, const double* jal,
                 const double* jbe, const double* thr, double sigma, double* G, double* diag, bool want_diag);
// Ap = p + sigma B^T((I - M) (p B)); pAp/pp partials into `part` (2 per block).
// mask / sgn: the edge_masks bits of q = 1 / inf (nullable: read V instead)
int hess_apply(const Prob& P, const double* p, const double* V, const double* jal, const double* jbe,
               const double* thr, double sigma, double* Ap, double* part, const void* cg_state = nullptr,
               const unsigned* mask = nullptr, const unsigned* sgn = nullptr);

// Block-Jacobi PCG on the SSNAL Newton system (linalg.cpp:143-192): solves
// H x = rhs from x0 = 0, stop on the worst relative feature-row residual.
struct PcgWork {
  double *x, *r, *p, *Ap, *diag;
};
struct PcgOut {
  int64_t iterations = 0;
  bool converged = false;
};
// A PCG operator: Ap = M p plus (pAp, pp) block partials in `part` (2 per
// block); returns the block count.  `cg_state` lets it no-op after the loop ends.
using PcgOp = std::function<int(const double* p, double* Ap, double* part, const void* cg_state)>;
// Generic device PCG (x0 = 0, or x0 = w.x when warm) on node-shaped d x n blocks.
// dist: node-partitioned over the context's communicator (comm.cuh) — each
// rank updates its own rows, the operator covers them (c.own_v0/own_v1), the
// block partials are all-reduced and p (then x) all-gathered; the work
// buffers must hold P * ceil(n / P) rows.
PcgOut pcg_dev(Ctx& c, int64_t n, int64_t d, const PcgOp& op, double op_bytes, const char* op_name,
               const double* rhs, PcgWork w, double tol, int64_t max_iter, bool warm, bool dist = false,
               const Graph* halo = nullptr, bool neg_rhs = false);  // neg_rhs: solve for b = -rhs  // dist: refresh p by halo exchange over this graph (else all-gather)
// the Newton system H D = -G: `G` is the gradient (negated inside the PCG's first pass)
PcgOut pcg_newton(const Prob& P, const double* V, const double* jal, const double* jbe, const double* thr,
                  double sigma, const double* G, PcgWork w, double tol, int64_t max_iter, int64_t n_active);

// ---- objectives / gap (objective.cpp:63-113) --------------------------------
struct GapOut {
  double fp = 0, fd = 0, gap = 0, kkt = 0;
};
GapOut eval_gap(const Prob& P, const double* X, const double* Z);
double primal_objective_dev(const Prob& P, const double* X);
double dual_objective_dev(const Prob& P, const double* Z);
double kkt_residual_dev(const Prob& P, const double* X, const double* Z);

// SSNAL multiplier step (ssnal.cpp:183-195) fused with the gap at the new Z.
struct MultOut {
  GapOut gap;
  double feas = 0;  // ||XB - PV|| / (1 + ||XB||)
  double zz = 0;    // ||Z||^2 at the new Z
};
// v_at_x: V = X B + Z / sigma at exactly this X (the edge kernel may then recompute V_l
// bitwise instead of reading it)
MultOut ssnal_multiplier(const Prob& P, const double* X, double* Z, const double* V, const double* ps,
                         const double* thr, double sigma, bool v_at_x = false);

// ---- fast AMA (ama.cpp:57-72) ---------------------------------------------
// Xh = A - Zhat B^T
void ama_primal(const Prob& P, const double* Zh, double* Xh);
// Znew = Pi(Zhat + step Xh B); Zhat = Znew + mom (Znew - Zprev); Zprev = Znew
void ama_dual_step(const Prob& P, const double* Xh, double* Zh, double* Zprev, double step, double mom,
                   const double* momp = nullptr);
void ama_momenta(const Prob& P, double* tm, int cnt);             // tm[0..cnt) = momenta, tm[cnt] = t
void ama_set_t(const Prob& P, double* tm, int cnt, double t);
// cnt AMA iterations + recover_primal into Xout + the gap partials as one cooperative kernel
// (small d, E).
// Returns the grid G (0 = not applicable: caller runs the per-kernel / graph path); *parts then
// holds the gap check's partial tables at (Xout, Zp) for gap_from_partials(P, *parts, G, G).
int ama_block_fused(const Prob& P, double* Xh, double* Zh, double* Zp, double* Xout, double step, double t0,
                    int cnt, double** parts);
GapOut gap_from_partials(const Prob& P, const double* dev_parts, int nbn, int nbe);

// The `active` flag of a PCG state (nullptr when none): operators no-op on it.
const int* cg_active_ptr(const void* cg_state);

}  // namespace cpb
