// linalg.hpp:17-87 on the device (see linalg.cu).
#pragma once

#include "ops.cuh"

namespace cpb {

// A LinearOperator (linalg.hpp:38-65): rows() = n; the operand is an n x cols
// column-major block.  Device-resident data for the factory kinds; a host
// callback for LinearOperator(rows, fn, ...).
struct LinOp {
  enum Kind { Identity, Dense, Sparse, Jacobi, Callback } kind = Identity;
  int64_t n = 0;
  bool symmetric = true, positive_definite = false;
  DBuf<double> vals;  // dense n x n (column-major) / sparse values / Jacobi diagonal
  int64_t jcols = 1;  // Jacobi: columns of the diagonal block (1: the Vector overload)
  DBuf<int> rowptr, col;
  int (*fn)(void*, const double*, double*, int64_t, int64_t) = nullptr;
  void* user = nullptr;
};

void linop_apply(Ctx& c, const LinOp& op, const double* X, int64_t cols, double* Y);
// Sparse operator from compressed columns (Eigen layout, int64 indices), holding
// scale * M + shift * I (shift = 0 for LinearOperator::sparse; 1 for I + rho L).
void linop_set_sparse(Ctx& c, LinOp& op, int64_t n, const int64_t* colptr, const int64_t* rowidx, const double* values,
                      double scale, double shift);

struct PcgResultDev {
  int64_t iterations = 0;
  double residual = 0.0;
  bool converged = false;
};
// pcg (linalg.cpp:143-192).  rhs, x: device n x cols.  per_column = 1 stops on
// the worst relative column residual (CholeskyFactor::solve) instead of rows.
PcgResultDev pcg_generic(Ctx& c, const LinOp& op, const double* rhs, int64_t cols, const LinOp* pre, double tol,
                         int64_t max_iter, double* x, int per_column = 0);
// power_iteration (linalg.cpp:194-242)
double power_generic(Ctx& c, const LinOp& op, double tol, int64_t max_iter);
// norm_value / dual_norm_value (prox.cpp:25-31) per column of a d x cols block
void norm_values_dev(Ctx& c, int q, const double* V, int64_t d, int64_t cols, double* nrm, double* dual);

}  // namespace cpb
