// l x l dense algebra of the preconditioner construction, on the device
// (dense_small.cu).  Host-vector wrappers upload, compute and download: the
// operands are l x l (l <= a few thousand), the work is l^3.
#pragma once

#include <vector>

#include "apc_internal.hpp"

namespace apc {

using Vec = std::vector<double>;

// upper Cholesky in place (column-major k x k; the lower part is zeroed):
// -1, or the first column with a non-positive pivot
int dpotrf_upper_dev(apc_ctx* ctx, i64 k, double* A);
// chol_upper (dense_factor.hpp:229-244) of a host Gram matrix; throws
// APC_NOT_POSITIVE(what, column) like the host routine
Vec dchol_upper(apc_ctx* ctx, i64 k, const Vec& g, const char* what);
// X (row-major k x ncols, device) <- T^{-1} X or T^{-T} X, T upper column-major
// (device); throws APC_SINGULAR on a zero diagonal
void dtrsm_rows_dev(apc_ctx* ctx, i64 k, const double* T, double* X, i64 ncols, bool transpose);
// tri_solve (dense_factor.hpp:406-424) on every column of a host k x ncols block
Vec dtri_solve_cols(apc_ctx* ctx, i64 k, const Vec& t, const Vec& x, i64 ncols, bool transpose);
// column-major C = A (m x k) B (k x n)
Vec dmatmul(apc_ctx* ctx, i64 m, i64 k, i64 n, const Vec& a, const Vec& b);

}  // namespace apc
