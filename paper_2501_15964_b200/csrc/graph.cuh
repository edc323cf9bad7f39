// Device-resident data matrix and weighted graph (types.hpp:16-22,
// graph.hpp:23-51) plus the graph-level operations (kNN build, incidence
// operator, connected components, Laplacian spectral bound).
//
// HBM layout (SoA, 32-bit indices):
//   A        double[n][d]   one sample per row (Eigen d x n column-major bytes)
//   ei, ej   int32[E]       endpoints, i < j, lexicographic (i, j) order
//   w, d2    double[E]      weights; kNN squared distances (NaN if user edges)
//   off      int32[n+1]     node CSR over incident edges
//   adj_e    int32[2E]      incident edge ids, ascending per node (= ascending
//                            neighbour id: the order Bᵀ accumulates in, graph.cpp:140-152)
//   adj_o    int32[2E]      the other endpoint; sign = (other > node) ? +1 : -1
//   order    int32[n]       nodes by descending degree (work scheduling only)
#pragma once

#include <vector>

#include "common.cuh"

namespace cpb {

struct Data {
  int64_t d = 0, n = 0;
  DBuf<double> A;
  double normA = -1.0;  // ||A||_F, lazily computed
};

struct Graph {
  int64_t n = 0, E = 0, max_degree = 0;
  uint64_t uid = 0;
  DBuf<int> ei, ej, off, adj_e, adj_o, order;
  DBuf<double> w, d2;
};

// Builders.
std::unique_ptr<Graph> graph_from_edges(Ctx& c, int64_t n, const int64_t* i, const int64_t* j, const double* w,
                                        int64_t E);
std::unique_ptr<Graph> knn_graph(Ctx& c, const Data& A, int64_t k, double phi);
// Tensor-core kNN candidates + exact FP64 re-check (knn_tc.cu).  Fills kd/kj
// (n x k, ascending (d2, j)) for every row it can certify and lists the
// others in ovf; returns how many (they need the exact tile kernel).
bool knn_tc_enabled(Ctx& c, int64_t n, int64_t d, int64_t k);
int64_t knn_tc(Ctx& c, const Data& A, int64_t k, int64_t r0, int64_t r1, double* kd, int* kj, int* ovf);
// Row-sharded kNN: each rank fills rows [r0, r1) of the n x k
// lists, the lists are all-gathered, and every rank builds the same graph.
void knn_validate(const Data& A, int64_t k, double phi);
void knn_rows_dev(Ctx& c, const Data& A, int64_t k, int64_t r0, int64_t r1, double* kd, int* kj);
std::unique_ptr<Graph> graph_from_knn_dev(Ctx& c, int64_t n, int64_t k, double phi, const double* kd, const int* kj);
// Builds CSR/order for a graph whose ei/ej/w/d2 (sorted, validated) are set.
void finalize_graph(Ctx& c, Graph& g);
std::vector<int> bfs_sequence(Ctx& c, const Graph& g, std::vector<int>* off_out);
std::vector<int> lpt_lists(const std::vector<int64_t>& cost, int nw, int win);

// Incidence operator on device arrays (row layouts as above).
void incidence_apply_dev(Ctx& c, const Graph& g, const double* X, int64_t d, double* out);
void incidence_apply_t_dev(Ctx& c, const Graph& g, const double* Z, int64_t d, double* out);

// Connected components over the edges with flag[l] != 0 (all edges when flag
// is null).  labels: rank of each component's smallest node (graph.cpp:169-196).
int64_t components_dev(Ctx& c, const Graph& g, const unsigned char* flag, int* labels);

// IncidenceOperator::laplacian (graph.cpp:154-167) in CSC form (host outputs;
// colptr null: only the nonzero count is returned).
int64_t laplacian_csc(Ctx& c, const Graph& g, int64_t* colptr, int64_t* rowidx, double* values);

// power_iteration on L = B B^T (linalg.cpp:194-242).
double laplacian_lambda_max(Ctx& c, const Graph& g, double tol, int64_t max_iter);

// Data helpers.
double data_fro_norm(Ctx& c, Data& A);

}  // namespace cpb
