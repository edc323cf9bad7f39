/*
 * cluspath_b200.h — the C-ABI drop-in boundary of the B200-native
 * convex-clustering-path engine (libcluspath_b200.so, sm_100a).
 *
 * Every entry point below replaces one function of the reference C++ API
 * (the headers under /root/reference/proj/include/cluspath, namespace cluspath); the
 * replaced declaration is cited as header:line.  Plain pointers and sizes
 * only: no C++ or torch types cross this boundary.
 *
 * Layout.  A d x n matrix (Eigen::MatrixXd, column-major, types.hpp:12) is
 * passed as `const double*` of length d*n with each sample (node) contiguous;
 * a d x |E| edge matrix likewise with each edge contiguous.  Edges are
 * (i, j, w) with 0 <= i < j < n, kept sorted lexicographically
 * (graph.hpp:14-51).  Index = int64_t (types.hpp:11).
 *
 * Errors.  Every int-returning call returns CP_OK or an error code; the
 * message of the calling thread's last error is cp_last_error().  The code
 * tells the wrapper which exception the reference would throw:
 * CP_EINVAL -> std::invalid_argument, CP_ERUNTIME -> std::runtime_error.
 * Non-convergence is not an error (cp_termination.converged = 0,
 * solver_util.hpp:87-100).
 *
 * Ownership.  The caller owns every host buffer.  Device state (data, graph,
 * per-path solver state) is owned by the handles and lives until destroyed —
 * the per-path SolveCache of the reference (solvers.hpp:119-123) is held by
 * the cp_ctx.  One cp_ctx per host thread; calls are synchronous.
 */
#ifndef CLUSPATH_B200_H
#define CLUSPATH_B200_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define CP_OK 0
#define CP_EINVAL 1   /* std::invalid_argument */
#define CP_ERUNTIME 2 /* std::runtime_error    */
#define CP_ECUDA 3    /* CUDA failure (reported as runtime_error) */
#define CP_ENCCL 4    /* NCCL failure */

typedef struct cp_ctx cp_ctx;     /* one device, its streams, workspace and SolveCache */
typedef struct cp_data cp_data;   /* device-resident DataMatrix (types.hpp:16-22)     */
typedef struct cp_graph cp_graph; /* device-resident WeightedGraph (graph.hpp:23-51)   */

/* SolverConfig (solvers.hpp:72-93); cp_solver_config_default fills the reference defaults. */
typedef struct cp_solver_config {
  int32_t algorithm;      /* 0 ADMM, 1 FastAMA, 2 SSNAL (solvers.hpp:15) */
  int32_t collect_trace;  /* 1: record a cp_trace_row per gap evaluation (cp_last_trace, cp_path_sink) */
  double epsilon;         /* 1e-6 */
  double kkt_factor;      /* 10 */
  int64_t max_iter;       /* 0 -> 100 outer (SSNAL) or 20000 (ADMM, AMA) */
  double time_limit;      /* seconds; <= 0 means none */
  double admm_rho;        /* 1 */
  double ama_step_safety; /* 0.99 */
  double ssnal_sigma0;    /* 1 */
  double armijo_mu;       /* 1e-4 */
  double backtrack_beta;  /* 0.5 */
  int64_t ssnal_newton_max; /* 50 */
  int64_t pcg_max_iter;     /* 500 */
} cp_solver_config;

/* TerminationRecord (solvers.hpp:45-52) plus work counters. */
typedef struct cp_termination {
  double f_primal, f_dual, gap;
  int64_t iterations;
  int32_t converged, pad;
  double wall_time;
  int64_t newton, cg, armijo, hess_apply; /* counters (not in the reference record) */
} cp_termination;

/* TraceRow (solvers.hpp:54-60): one row per gap evaluation when collect_trace. */
typedef struct cp_trace_row {
  int64_t iter;
  double f_p, f_d, gap, elapsed_s;
} cp_trace_row;

/* PathOptions (path.hpp:51-55). */
typedef struct cp_path_options {
  int32_t warm_start;        /* 1 */
  int32_t require_connected; /* 0 */
  double fuse_tol;           /* 1e-3 */
} cp_path_options;

/* Per-kernel timing/bytes record for roofline accounting (no reference counterpart). */
typedef struct cp_kernel_stat {
  char name[40];
  int64_t launches;
  double ms;        /* summed CUDA-event time on the launching stream */
  double alg_bytes; /* summed algorithmic (compulsory) bytes */
} cp_kernel_stat;

/* ---- context ------------------------------------------------------------ */
int cp_ctx_create(int device, cp_ctx** out);
void cp_ctx_destroy(cp_ctx* ctx);
const char* cp_last_error(void);
int cp_ctx_synchronize(cp_ctx* ctx);
void cp_solver_config_default(cp_solver_config* cfg);
void cp_path_options_default(cp_path_options* opt);
/* Kernel statistics: enable CUDA-event timing of the hot kernels. */
int cp_stats_enable(cp_ctx* ctx, int on);
int cp_stats_reset(cp_ctx* ctx);
int cp_stats_get(cp_ctx* ctx, cp_kernel_stat* out, int max_entries, int* count);
/* Device/library identification: sm major/minor, SM count, kernel build arch. */
int cp_device_info(cp_ctx* ctx, int* sm_major, int* sm_minor, int* sm_count, int* built_arch);
/* How the last cp_knn_graph on this context ran: tensor_cores = 1 when the
 * tcgen05 3xTF32 candidate pass was used, segments = its column segments,
 * band_rows = rows settled by the second (threshold) tensor-core pass,
 * exact_rows = rows re-done by the exact FP64 tile kernel, worst_ratio =
 * max |d2~ - d2| / delta_i over the candidates re-checked (must be < 1). */
int cp_knn_info(cp_ctx* ctx, int* tensor_cores, int* segments, int64_t* band_rows, int64_t* exact_rows,
                double* worst_ratio);
/* Number of library kernel launches so far (process-wide). */
unsigned long long cp_launch_count(void);
/* CUDA-event timer on the context's stream; cp_timer_stop waits and returns ms. */
int cp_timer_start(cp_ctx* ctx);
int cp_timer_stop(cp_ctx* ctx, double* ms);
/* Evict L2 by writing a buffer larger than it (benchmark hygiene). */
int cp_flush_l2(cp_ctx* ctx);
/* Page-locked host buffers: run_path outputs placed in them are copied
   asynchronously, overlapped with the next gamma's solve. */
int cp_host_alloc(uint64_t bytes, void** out);
void cp_host_free(void* p);

/* ---- synthetic inputs (io.cpp:142-165; host code, libstdc++ <random>) -------- */
/* generate_gaussian_mixture(centers, spread, per_center, seed): centers d x m, out d x (m*per_center). */
int cp_gaussian_mixture(const double* centers, int64_t d, int64_t m, double spread, int64_t per_center, uint64_t seed,
                        double* out);
/* count draws of std::normal_distribution<double>(0,1) over std::mt19937_64(seed). */
int cp_normals(uint64_t seed, int64_t count, double* out);

/* ---- data (types.hpp:16-28; make_data_matrix graph.cpp:10-23) ------------ */
int cp_data_create(cp_ctx* ctx, const double* A, int64_t d, int64_t n, cp_data** out);
void cp_data_destroy(cp_data* data);

/* ---- graph (graph.hpp:23-92) --------------------------------------------- */
/* compute_knn_weights(data, k, phi) (graph.hpp:58; graph.cpp:75-114) */
int cp_knn_graph(cp_ctx* ctx, const cp_data* data, int64_t k, double phi, cp_graph** out);
/* Row-sharded kNN (graph.cpp:79-88 per row).  kd_dev and
 * kj_dev are DEVICE pointers to n x k arrays (double, int32): the k nearest
 * (d2, j) of every row in [r0, r1), ascending by (d2, j), are written at
 * their global row positions; other rows are untouched.  Bit-identical to the
 * rows cp_knn_graph computes, whatever the row range. */
int cp_knn_rows(cp_ctx* ctx, const cp_data* data, int64_t k, int64_t r0, int64_t r1, double* kd_dev,
                int32_t* kj_dev);
/* The graph from complete per-row lists (DEVICE pointers, n x k): union of
 * (min, max) pairs, sorted, unique, w = exp(-phi d2) (graph.cpp:89-111). */
int cp_graph_from_knn(cp_ctx* ctx, int64_t n, int64_t k, double phi, const double* kd_dev, const int32_t* kj_dev,
                      cp_graph** out);
/* Multi-GPU (one process per GPU): rank 0 creates a 128-byte
 * NCCL unique id, the caller distributes it (e.g. torch.distributed), and every
 * rank attaches a communicator to its context.  With a communicator, each SSNAL
 * Newton system's PCG is node-partitioned over the ranks (rows
 * [r ceil(n/P), (r+1) ceil(n/P))): Hessian applies and vector updates cover the
 * rank's rows, block partials are all-reduced and p / x all-gathered over
 * NVLink; the rest of the path is replicated.  nranks = 1 runs the same code
 * path on one GPU.  libnccl.so.2 is loaded at run time (CP_ENCCL if absent). */
int cp_nccl_unique_id(char out[128]);
int cp_ctx_set_comm(cp_ctx* ctx, int nranks, int rank, const char id[128]);
/* In-process group of nranks contexts driven by nranks host threads (the same
 * partitioned code path without NCCL, e.g. several ranks tested on one GPU:
 * collectives meet at host barriers, no kernel waits on another rank). */
typedef struct cp_local_group cp_local_group;
int cp_local_group_create(int nranks, cp_local_group** out);
void cp_local_group_destroy(cp_local_group* g);
int cp_ctx_set_local_comm(cp_ctx* ctx, cp_local_group* g, int rank);
/* Host-only: the query rows [r0, r1) of `rank` among `nranks` for the
 * row-sharded kNN: ceil(n / nranks) rows per rank, the last rank short. */
int cp_shard_rows(int64_t n, int nranks, int rank, int64_t* r0, int64_t* r1);
/* WeightedGraph(n, edges): sorts and validates (graph.hpp:29-31; graph.cpp:25-45) */
int cp_graph_from_edges(cp_ctx* ctx, int64_t n, const int64_t* i, const int64_t* j, const double* w, int64_t E,
                        cp_graph** out);
void cp_graph_destroy(cp_graph* g);
int64_t cp_graph_nodes(const cp_graph* g);      /* graph.hpp:33 */
int64_t cp_graph_edge_count(const cp_graph* g); /* graph.hpp:34 */
/* edges() in list order; d2 (nullable) receives the kNN squared distances
   (NaN for graphs built from an edge list). */
int cp_graph_export(cp_ctx* ctx, const cp_graph* g, int64_t* i, int64_t* j, double* w, double* d2);
int cp_graph_degrees(cp_ctx* ctx, const cp_graph* g, int64_t* degree); /* graph.hpp:43-44 */

/* IncidenceOperator::apply_into: X (d x n) -> X B (d x |E|) (graph.hpp:69-70; graph.cpp:122-132) */
int cp_incidence_apply(cp_ctx* ctx, const cp_graph* g, const double* X, int64_t d, int64_t n, double* out);
/* IncidenceOperator::apply_transpose_into: Z (d x |E|) -> Z B^T (d x n) (graph.hpp:74-75; graph.cpp:140-152) */
int cp_incidence_apply_t(cp_ctx* ctx, const cp_graph* g, const double* Z, int64_t d, int64_t E, double* out);
/* connected_components + component_count (graph.hpp:90-92; graph.cpp:169-202) */
/* IncidenceOperator::laplacian (graph.hpp:82; graph.cpp:154-167): B B^T
 * (weights do not enter) as compressed columns, n x n.  Call with colptr = NULL
 * to get *nnz, then with colptr (n + 1), rowidx (nnz) and values (nnz); rows are
 * ascending within each column (Eigen's compressed layout). */
int cp_graph_laplacian(cp_ctx* ctx, const cp_graph* g, int64_t* colptr, int64_t* rowidx, double* values,
                       int64_t* nnz);
int cp_connected_components(cp_ctx* ctx, const cp_graph* g, int64_t* labels, int64_t* K);
/* power_iteration(LinearOperator::sparse(B.laplacian())) (linalg.hpp:84-85; linalg.cpp:194-242) */
int cp_laplacian_lambda_max(cp_ctx* ctx, const cp_graph* g, double tol, int64_t max_iter, double* lambda);

/* ---- prox (prox.hpp:8-54) ------------------------------------------------- */
/* q in {1, 2}; prox_columns_into (prox.hpp:28-29; prox.cpp:73-80) */
int cp_prox_columns(cp_ctx* ctx, int q, const double* V, const double* thresholds, int64_t d, int64_t E,
                    double* out);
/* project_columns (prox.hpp:30-31; prox.cpp:82-93) */
int cp_project_columns(cp_ctx* ctx, int q, const double* Z, const double* radii, int64_t d, int64_t E, double* out);
/* ProxJacobian::diag for every column (prox.hpp:38-49; prox.cpp:106-132): out d x E */
/* ProxJacobian::apply (prox.hpp:38-47; prox.cpp:95-132) column-wise: out_l =
 * M_l W_l, M_l the structured Jacobian of prox_{t_l ||.||_q} at V_l. */
int cp_prox_jacobian_apply(cp_ctx* ctx, int q, const double* V, const double* thresholds, const double* W,
                           int64_t d, int64_t E, double* out);
int cp_prox_jacobian_diag(cp_ctx* ctx, int q, const double* V, const double* thresholds, int64_t d, int64_t E,
                          double* out);

/* ---- objectives (solvers.hpp:95-118, 143-156) ----------------------------- */
int cp_primal_objective(cp_ctx* ctx, const cp_data* A, const cp_graph* g, double gamma, int q, const double* X,
                        double* out);
int cp_dual_objective(cp_ctx* ctx, const cp_data* A, const cp_graph* g, double gamma, int q, const double* Z,
                      double* out);
int cp_kkt_residual(cp_ctx* ctx, const cp_data* A, const cp_graph* g, double gamma, int q, const double* X,
                    const double* Z, double* out);
int cp_ssnal_phi_value(cp_ctx* ctx, const cp_data* A, const cp_graph* g, double gamma, int q, const double* Z,
                       double sigma, const double* X, double* out);
int cp_ssnal_phi_gradient(cp_ctx* ctx, const cp_data* A, const cp_graph* g, double gamma, int q, const double* Z,
                          double sigma, const double* X, double* out);
int cp_ssnal_hessian_apply(cp_ctx* ctx, const cp_data* A, const cp_graph* g, double gamma, int q, const double* Z,
                           double sigma, const double* X, const double* D, double* out);

/* ---- solve (solvers.hpp:132-141) ----------------------------------------- */
/* solve / solve_ssnal / solve_admm / solve_fast_ama.  warmX/warmZ nullable (both or neither);
   their shapes are (wd x wn) and (wd x wE) and must match the instance. */
int cp_solve(cp_ctx* ctx, const cp_data* A, const cp_graph* g, double gamma, int q, const cp_solver_config* cfg,
             const double* warmX, int64_t warm_d, int64_t warm_n, const double* warmZ, int64_t warm_E, double* X,
             double* Z, cp_termination* term);

/* Solution::trace (solvers.hpp:54-66) of the most recent cp_solve on this
 * context (empty unless cfg->collect_trace).  Call with rows = NULL for *count. */
int cp_last_trace(cp_ctx* ctx, cp_trace_row* rows, int64_t max_rows, int64_t* count);

/* ---- linalg (linalg.hpp:17-87) --------------------------------------------- */
/* LinearOperator (linalg.hpp:38-65).  The operand is a rows x cols column-major
 * block; device-resident for the factory kinds.  A host callback
 * (LinearOperator(rows, fn, symmetric, positive_definite)) receives host
 * buffers and returns 0 on success; each apply is one device round trip. */
typedef struct cp_linop cp_linop;
typedef int (*cp_apply_fn)(void* user, const double* in, double* out, int64_t rows, int64_t cols);
int cp_linop_identity(cp_ctx* ctx, int64_t n, cp_linop** out);                             /* linalg.hpp:53 */
int cp_linop_dense(cp_ctx* ctx, const double* M, int64_t n, int positive_definite, cp_linop** out); /* :54 */
/* n x n compressed columns (Eigen::SparseMatrix<double> layout, int64 indices) (linalg.hpp:55-56) */
int cp_linop_sparse(cp_ctx* ctx, int64_t n, const int64_t* colptr, const int64_t* rowidx, const double* values,
                    int positive_definite, cp_linop** out);
/* jacobi(Vector diag) when cols = 1, jacobi(Matrix diag) otherwise (linalg.hpp:60-61) */
int cp_linop_jacobi(cp_ctx* ctx, const double* diag, int64_t rows, int64_t cols, cp_linop** out);
int cp_linop_callback(cp_ctx* ctx, int64_t rows, cp_apply_fn fn, void* user, int symmetric, int positive_definite,
                      cp_linop** out); /* linalg.hpp:45-46 */
int cp_linop_info(const cp_linop* op, int64_t* rows, int* symmetric, int* positive_definite);
void cp_linop_destroy(cp_linop* op);
int cp_linop_apply(cp_ctx* ctx, const cp_linop* op, const double* X, int64_t cols, double* out); /* :51 */
/* pcg(op, rhs, preconditioner, tol, max_iter) (linalg.hpp:76-77; linalg.cpp:143-192).
 * rhs / x: rows x cols host buffers; pre nullable (identity). */
int cp_pcg(cp_ctx* ctx, const cp_linop* op, const double* rhs, int64_t cols, const cp_linop* pre, double tol,
           int64_t max_iter, double* x, int64_t* iterations, double* residual, int32_t* converged);
/* power_iteration(op, tol, max_iter) (linalg.hpp:82-83; linalg.cpp:194-242) */
int cp_power_iteration(cp_ctx* ctx, const cp_linop* op, double tol, int64_t max_iter, double* lambda);
/* CholeskyFactor(L, rho) / solve(rhs) (linalg.hpp:17-33; linalg.cpp:32-54): M = I + rho L,
 * L n x n compressed columns; solve returns M^{-1} rhs (rows n, cols columns) to 1e-14
 * relative residual per column (device CG in place of the sparse factor). */
typedef struct cp_factor cp_factor;
int cp_factor_create(cp_ctx* ctx, int64_t n, const int64_t* colptr, const int64_t* rowidx, const double* values,
                     double rho, cp_factor** out);
int cp_factor_solve(cp_ctx* ctx, const cp_factor* f, const double* rhs, int64_t cols, double* out);
void cp_factor_destroy(cp_factor* f);
/* norm_value / dual_norm_value (prox.hpp:14-15; prox.cpp:25-31) of every column of a d x cols block */
int cp_norm_values(cp_ctx* ctx, int q, const double* V, int64_t d, int64_t cols, double* norm, double* dual);

/* ---- path (path.hpp:26-78) ------------------------------------------------ */
/* make_schedule(start, end, count, spacing) (path.hpp:26; path.cpp:21-58); spacing 0 linear, 1 geometric */
int cp_make_schedule(double start, double end, int64_t count, int geometric, double* out);
/* extract_clusters (path.hpp:41-42; path.cpp:60-89): labels n, K, centroids d x n (first K columns used) */
int cp_extract_clusters(cp_ctx* ctx, const cp_graph* g, const double* X, int64_t d, int64_t n, double fuse_tol,
                        int64_t* labels, int64_t* K, double* centroids);
/* run_path (path.hpp:71-73; path.cpp:110-142).  Outputs per gamma t (all nullable):
   X_out[t*d*n], Z_out[t*d*E], labels_out[t*n], K_out[t], terms_out[t]. */
int cp_run_path(cp_ctx* ctx, const cp_data* A, const cp_graph* g, int q, const double* gammas, int64_t T,
                const cp_solver_config* cfg, const cp_path_options* opt, double* X_out, double* Z_out,
                int64_t* labels_out, int64_t* K_out, cp_termination* terms_out);
/* Per-gamma callbacks of cp_run_path_ex (all nullable), called on the calling
 * thread in gamma order: the d x K centroids of ClusterAssignment (path.hpp:30-34,
 * filled by path.cpp:135; host memory valid during the call) and the solver's
 * trace rows (Solution::trace, when cfg->collect_trace). */
typedef struct cp_path_sink {
  void* user;
  void (*centroids)(void* user, int64_t t, int64_t K, int64_t d, const double* centroids);
  void (*trace)(void* user, int64_t t, const cp_trace_row* rows, int64_t count);
  /* 1: skip the centroids call when K = n (every node its own cluster, labels 0..n-1 and
     centroids = X bitwise); a caller that keeps X(gamma) reuses it instead of a d x n copy */
  int32_t skip_identity;
} cp_path_sink;
int cp_run_path_ex(cp_ctx* ctx, const cp_data* A, const cp_graph* g, int q, const double* gammas, int64_t T,
                   const cp_solver_config* cfg, const cp_path_options* opt, double* X_out, double* Z_out,
                   int64_t* labels_out, int64_t* K_out, cp_termination* terms_out, const cp_path_sink* sink);

#ifdef __cplusplus
}
#endif

#endif /* CLUSPATH_B200_H */
