// Node-CSR gather kernels: every operator of the form
//     out_v = f( x_v, sum over incident edges l of v, ascending l, of +-g_l )
// (Bᵀ, the SSNAL gradient/diagonal/Hessian, the gap's Z Bᵀ, AMA's A - Z Bᵀ,
// ADMM's right-hand side and the Laplacian).  Accumulation runs in ascending
// edge id per (node, feature), exactly the order of the reference's scatter
// loop (graph.cpp:140-152), so sums are bitwise equal to it; there are no
// atomics.
//
// Geometry: d <= 32 -> sub-warp groups of gx = 2^ceil(log2 d) lanes, 256/gx
// nodes per block; d > 32 -> one node per block, gx = 32 * ceil(d / NF / 32)
// threads each owning NF features (f = tx + gx k) in registers.  Incident
// edges are consumed in batches of 8 with all 8 x NF row loads issued before
// use, so a hub node's latency chain is deg/8 memory round trips, not deg x d/32.
#pragma once

#include "graph.cuh"

namespace cpb {

struct NodeGeom {
  int gx, gy, nf, grid;
};
NodeGeom node_geom(Ctx& c, int64_t n, int64_t d);

// Bᵀ z (graph.cpp:140-152)
void gather_bt(Ctx& c, const Graph& g, const double* Z, int64_t d, double* out);
// Xh = A - Zh Bᵀ (ama.cpp:62-63)
void gather_a_minus_bt(Ctx& c, const Graph& g, const double* A, const double* Zh, int64_t d, double* Xh);
// R = A + (rho U - L) Bᵀ (admm.cpp:61)
void gather_admm_rhs(Ctx& c, const Graph& g, const double* A, const double* U, const double* L, double rho,
                     int64_t d, double* R);
// out = y + rho (L y); part[2b] = <y, out>, part[2b+1] = <y, y>  (I + rho L)
int gather_lap(Ctx& c, const Graph& g, const double* y, double rho, int64_t d, double* out, double* part,
               const int* active);
// gap node terms at (X, Z): part[4b + k] = ||X-A||^2, ||ZBᵀ||^2, <ZBᵀ, A>, ||X - A + ZBᵀ||^2
int gather_gap(Ctx& c, const Graph& g, const double* X, const double* A, const double* Z, int64_t d, double* part);
// SSNAL gradient and Jacobi diagonal (ssnal.cpp:41-44, :68-82); part[b] = ||G||^2
int gather_grad_diag(Ctx& c, const Graph& g, const double* X, const double* A, const double* V, const double* ps,
                     const double* jal, const double* jbe, const double* thr, int64_t d, double sigma, int q,
                     bool want_diag, double* G, double* diag, double* part);
// SSNAL Hessian (ssnal.cpp:56-64), two passes: per-edge bc_l = beta_l <v_l, p_i - p_j>,
// then the node gather; part[2b] = <p, Ap>, part[2b+1] = <p, p>.
// TMA-staged single-pass Hessian (hess_tma.cu): q = 2, even d in [256, 1024].
bool hess_tma_supported(int64_t d);
int hess_tma(Ctx& c, const Graph& g, const double* P, const double* V, const double* jal, const double* jbe,
             int64_t d, double sigma, double* Ap, double* part, const int* active);
// Edge ownership in a partitioned solve (c.own range): this rank's owned edges
// are the contiguous ids [e0, e1) (smaller endpoint owned); ghost edges enter an
// owned node from another rank's node (computed redundantly, never summed);
// row0/rows: every rank's owned range (to assemble full edge arrays).
struct EdgePart {
  uint64_t uid = 0;
  int64_t v0 = 0, v1 = -1;
  int nranks = 1;
  int64_t e0 = 0, e1 = 0, nghost = 0;
  DBuf<int> ghost;
  std::vector<int64_t> row0, rows;
};
const EdgePart& edge_part(Ctx& c, const Graph& g);

// Halo plan of a partitioned solve: for every other rank s, the owned nodes
// this rank sends to s (those adjacent to s's nodes) and the nodes of s it
// receives (s's nodes adjacent to this rank's), both in ascending id, so the
// two sides agree without negotiation (the graph is replicated).
struct HaloPlan {
  uint64_t uid = 0;
  int64_t v0 = 0, v1 = -1;
  int nranks = 1;
  std::vector<int64_t> send_off, recv_off;  // per rank, prefix offsets (size nranks + 1)
  DBuf<int> send_idx, recv_idx;
  int64_t nsend = 0, nrecv = 0;
};
const HaloPlan& halo_plan(Ctx& c, const Graph& g);
// p's halo rows <- the owning ranks' rows (p is a full-size node array).
void halo_exchange(Ctx& c, const Graph& g, double* p, int64_t d);

// mask / sgn (nullable): edge_masks bits for q = 1 / inf (then V is not read by the Hessian)
int hess_two_pass(Ctx& c, const Graph& g, const double* P, const double* V, const double* jal, const double* jbe,
                  const double* thr, int64_t d, double sigma, int q, double* bc, double* Ap, double* part,
                  const int* active, const unsigned* mask = nullptr, const unsigned* sgn = nullptr);
// Jacobian feature bits per edge from V: thr = t_l (q = 1) or theta_l (q = inf); 2 E ceil(d/32) words
void edge_masks(Ctx& c, const Graph& g, const double* V, const double* thr, int64_t d, int q, unsigned* mask,
                unsigned* sgn);

}  // namespace cpb
