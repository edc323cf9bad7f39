// Solver drivers (ssnal.cpp, ama.cpp, admm.cpp, objective.cpp:115-123) and the
// path engine (path.cpp).  Host C++ that sequences the device operators of
// ops.cuh; all iterates stay in HBM, only scalars cross to the host.
#pragma once

#include <map>

#include "ops.cuh"

namespace cpb {

// SolveCache (solvers.hpp:119-123): per-path state shared across gammas.
struct SolveCache {
  std::map<uint64_t, double> lambda_max;  // graph uid -> lambda_max(B B^T)
};

void validate_config(const cp_solver_config& c);  // objective.cpp:43-61
// TraceRow (solvers.hpp:54-60) after a gap evaluation, when collect_trace
inline void trace_gap(Ctx& c, const cp_solver_config& cfg, int64_t k, const GapOut& g, double elapsed) {
  if (cfg.collect_trace) c.trace.push_back(cp_trace_row{k, g.fp, g.fd, g.gap, elapsed});
}
int64_t resolved_max_iter(const cp_solver_config& c);

// Solve one instance.  X (d x n) and Z (d x E) are device buffers; when `warm`
// they hold the warm start (Z is re-projected onto the new radii), and on
// return they hold the solution (objective.cpp:115-123).
cp_termination solve_dev(Prob& P, const cp_solver_config& cfg, bool warm, double* X, double* Z, SolveCache& cache);

// extract_clusters (path.cpp:60-89): labels (device int n), returns K;
// centroids (device d x K, nullable).
int64_t extract_clusters_dev(Ctx& c, const Graph& g, const double* X, int64_t d, double fuse_tol, int* labels,
                             double* centroids);

// run_path (path.cpp:110-142).  Outputs are host buffers (nullable).
// sink (nullable): per-gamma centroids (host d x K) and trace rows.
void run_path_dev(Ctx& c, Data& A, const Graph& g, int q, const double* gammas, int64_t T,
                  const cp_solver_config& cfg, const cp_path_options& opt, double* X_out, double* Z_out,
                  int64_t* labels_out, int64_t* K_out, cp_termination* terms_out, const cp_path_sink* sink = nullptr);

}  // namespace cpb
