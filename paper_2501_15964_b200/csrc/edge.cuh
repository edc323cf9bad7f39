// Register-resident edge-row kernels (edge.cu) for d <= 1024.
#pragma once

#include "graph.cuh"

namespace cpb {

bool edge_reg_supported(int64_t d);
int edge_grid(Ctx& c, int64_t E);
// eval_phi's edge pass; part[b] = envelope partial.  Returns the block count.
int phi_edge_reg(Ctx& c, const Graph& g, const double* X, const double* Z, const double* thr, const double* rad,
                 int64_t d, double sigma, int q, double* V, double* nv, double* part);
// SSNAL multiplier + gap edge terms; part[9 b + k] as k_mult.  Returns the block count.
int mult_reg(Ctx& c, const Graph& g, const double* X, double* Z, const double* V, const double* ps, const double* thr,
             const double* rad, int64_t d, double sigma, int q, double* part);

}  // namespace cpb
