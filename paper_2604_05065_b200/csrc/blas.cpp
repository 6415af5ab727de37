// cuBLAS wrappers (see blas.hpp).  One handle per context, bound to the
// library stream; deterministic (no atomics-based algorithms requested).
#include "blas.hpp"

#include <cublas_v2.h>

#include <string>

namespace apc {

namespace {
cublasHandle_t handle(apc_ctx* ctx) {
  if (!ctx->blas) {
    cublasHandle_t h;
    if (cublasCreate(&h) != CUBLAS_STATUS_SUCCESS) fail(APC_CUDA_ERROR, "cublasCreate failed");
    cublasSetStream(h, ctx->stream);
    cublasSetAtomicsMode(h, CUBLAS_ATOMICS_NOT_ALLOWED);
    ctx->blas = h;
  }
  return static_cast<cublasHandle_t>(ctx->blas);
}
void check(cublasStatus_t s, const char* what) {
  if (s != CUBLAS_STATUS_SUCCESS) fail(APC_CUDA_ERROR, std::string(what) + ": cuBLAS status " + std::to_string(s));
}
}  // namespace

void dgemm(apc_ctx* ctx, bool ta, bool tb, i64 m, i64 n, i64 k, double alpha, const double* A, i64 lda,
           const double* B, i64 ldb, double beta, double* C, i64 ldc) {
  if (m == 0 || n == 0) return;
  check(cublasDgemm(handle(ctx), ta ? CUBLAS_OP_T : CUBLAS_OP_N, tb ? CUBLAS_OP_T : CUBLAS_OP_N, (int)m, (int)n,
                    (int)k, &alpha, A, (int)lda, B, (int)ldb, &beta, C, (int)ldc),
        "cublasDgemm");
}

void dsyrk_t(apc_ctx* ctx, i64 n, i64 k, double alpha, const double* A, i64 lda, double beta, double* C, i64 ldc) {
  if (n == 0) return;
  check(cublasDsyrk(handle(ctx), CUBLAS_FILL_MODE_UPPER, CUBLAS_OP_T, (int)n, (int)k, &alpha, A, (int)lda, &beta,
                    C, (int)ldc),
        "cublasDsyrk");
}

void dtrsm_right_upper(apc_ctx* ctx, i64 m, i64 n, const double* T, i64 ldt, double* B, i64 ldb) {
  if (m == 0 || n == 0) return;
  const double one = 1.0;
  check(cublasDtrsm(handle(ctx), CUBLAS_SIDE_RIGHT, CUBLAS_FILL_MODE_UPPER, CUBLAS_OP_N, CUBLAS_DIAG_NON_UNIT,
                    (int)m, (int)n, &one, T, (int)ldt, B, (int)ldb),
        "cublasDtrsm");
}

void blas_destroy(apc_ctx* ctx) {
  if (ctx->blas) cublasDestroy(static_cast<cublasHandle_t>(ctx->blas));
  ctx->blas = nullptr;
}

}  // namespace apc
