// Dense kernels of the per-rebuild preconditioner construction (blas.cu:
// hand-written DMMA GEMM / SYRK / blocked TRSM on tall-skinny blocks; never on
// the per-iteration path and never on the index-selecting path).
// Column-major throughout.
#pragma once

#include "apc_internal.hpp"

namespace apc {

// C = alpha op(A) op(B) + beta C
void dgemm(apc_ctx* ctx, bool ta, bool tb, i64 m, i64 n, i64 k, double alpha, const double* A, i64 lda,
           const double* B, i64 ldb, double beta, double* C, i64 ldc);
// C (n x n, upper triangle) = alpha A^T A + beta C, A is k x n
void dsyrk_t(apc_ctx* ctx, i64 n, i64 k, double alpha, const double* A, i64 lda, double beta, double* C, i64 ldc);
// B (m x n) <- B T^{-1}, T upper n x n
void dtrsm_right_upper(apc_ctx* ctx, i64 m, i64 n, const double* T, i64 ldt, double* B, i64 ldb);
void blas_destroy(apc_ctx* ctx);

}  // namespace apc
