// l x l dense algebra of the per-rebuild preconditioner construction on the
// device (dense_small.hpp): blocked upper Cholesky (chol_upper,
// dense_factor.hpp:229-244), triangular solves with many right-hand sides
// (tri_solve, dense_factor.hpp:406-424) and products through the DMMA GEMM of
// blas.cu.  Not on the index-selecting path: results are
// deterministic run to run, not bit-identical to the reference's loops.
#include <algorithm>

#include "blas.hpp"
#include "dense_small.hpp"

namespace apc {

namespace {

constexpr int kPotrfNB = 64;   // diagonal block (factored by one CTA in shared memory)
constexpr int kSmallT = 256;

// factor the nb x nb diagonal block A(k0:k0+nb, k0:k0+nb) in place (upper,
// column-major, ld), right-looking inside shared memory; *bad = first
// non-positive pivot's global index
__global__ void __launch_bounds__(kSmallT) potf2_kernel(double* A, long long ld, int k0, int nb, int* bad) {
  __shared__ double s[kPotrfNB * (kPotrfNB + 1)];
  __shared__ int fail;
  constexpr int L = kPotrfNB + 1;
  if (threadIdx.x == 0) fail = -1;
  for (int t = threadIdx.x; t < nb * nb; t += kSmallT) {
    const int i = t % nb, j = t / nb;
    s[j * L + i] = A[(k0 + j) * ld + k0 + i];
  }
  __syncthreads();
  for (int p = 0; p < nb; ++p) {
    if (threadIdx.x == 0) {
      const double d = s[p * L + p];
      if (!(d > 0.0) && fail < 0) fail = k0 + p;
      s[p * L + p] = d > 0.0 ? sqrt(d) : 1.0;
    }
    __syncthreads();
    const double dp = s[p * L + p];
    for (int j = p + 1 + threadIdx.x; j < nb; j += kSmallT) s[j * L + p] /= dp;  // row p of U
    __syncthreads();
    // trailing upper block: s(i, j) -= U(p, i) U(p, j), p < i <= j
    const int w = nb - p - 1;
    for (int t = threadIdx.x; t < w * w; t += kSmallT) {
      const int i = p + 1 + t % w, j = p + 1 + t / w;
      if (i <= j) s[j * L + i] -= s[i * L + p] * s[j * L + p];
    }
    __syncthreads();
  }
  for (int t = threadIdx.x; t < nb * nb; t += kSmallT) {
    const int i = t % nb, j = t / nb;
    A[(k0 + j) * ld + k0 + i] = i <= j ? s[j * L + i] : 0.0;
  }
  if (threadIdx.x == 0 && fail >= 0) atomicMin(bad, fail);
}

// B(k0:k0+nb, c) <- U^{-T} B(k0:k0+nb, c) for the columns c >= k0 + nb of the
// block row (U = the factored diagonal block): thread per column, forward
// substitution in column order
__global__ void __launch_bounds__(128) potrf_panel_kernel(double* A, long long ld, int k0, int nb, long long ncols) {
  __shared__ double u[kPotrfNB * kPotrfNB];
  for (int t = threadIdx.x; t < nb * nb; t += 128) u[t] = A[(k0 + t / nb) * ld + k0 + t % nb];
  __syncthreads();
  const long long c = k0 + nb + static_cast<long long>(blockIdx.x) * 128 + threadIdx.x;
  if (c >= k0 + nb + ncols) return;
  double x[kPotrfNB];
  double* col = A + c * ld + k0;
  for (int i = 0; i < nb; ++i) x[i] = col[i];
  for (int i = 0; i < nb; ++i) {
    double s = x[i];
    for (int j = 0; j < i; ++j) s -= u[i * nb + j] * x[j];
    x[i] = s / u[i * nb + i];
  }
  for (int i = 0; i < nb; ++i) col[i] = x[i];
}

// X (row-major k x ncols: X[i * ncols + c]) <- T^{-1} X or T^{-T} X for upper
// T (column-major k x k); thread per column, T read by broadcast
__global__ void __launch_bounds__(128) trsm_cols_kernel(const double* __restrict__ T, long long k, double* X,
                                                        long long ncols, int transpose, int* bad) {
  const long long c = static_cast<long long>(blockIdx.x) * 128 + threadIdx.x;
  if (c >= ncols) return;
  if (!transpose) {
    for (long long i = k - 1; i >= 0; --i) {
      double s = X[i * ncols + c];
      for (long long j = i + 1; j < k; ++j) s -= T[j * k + i] * X[j * ncols + c];
      const double d = T[i * k + i];
      if (d == 0.0) {
        atomicMin(bad, static_cast<int>(i));
        return;
      }
      X[i * ncols + c] = s / d;
    }
  } else {
    for (long long i = 0; i < k; ++i) {
      double s = X[i * ncols + c];
      for (long long j = 0; j < i; ++j) s -= T[i * k + j] * X[j * ncols + c];
      const double d = T[i * k + i];
      if (d == 0.0) {
        atomicMin(bad, static_cast<int>(i));
        return;
      }
      X[i * ncols + c] = s / d;
    }
  }
}

__global__ void zero_lower_kernel(double* A, long long k) {
  const long long q = static_cast<long long>(blockIdx.x) * blockDim.x + threadIdx.x;
  if (q < k * k && q % k > q / k) A[q] = 0.0;
}

__global__ void transpose_kernel(const double* __restrict__ a, long long m, long long n, double* __restrict__ t) {
  const long long q = static_cast<long long>(blockIdx.x) * blockDim.x + threadIdx.x;
  if (q < m * n) {
    const long long i = q % m, j = q / m;  // a(i, j), column-major m x n
    t[i * n + j] = a[q];
  }
}

int read_flag(apc_ctx* ctx, const int* d) {
  int h = 0;
  copy_sync(ctx->stream, &h, d, sizeof(int), cudaMemcpyDeviceToHost);
  return h;
}

DBuf<int> new_flag(apc_ctx* ctx) {
  DBuf<int> f(1);
  const int big = 0x7fffffff;
  APC_CUDA(cudaMemcpyAsync(f.p, &big, sizeof(int), cudaMemcpyHostToDevice, ctx->stream));
  return f;
}

void up(apc_ctx* ctx, DBuf<double>& d, const Vec& h) {
  d.alloc(std::max<i64>(1, static_cast<i64>(h.size())));
  if (!h.empty())
    APC_CUDA(cudaMemcpyAsync(d.p, h.data(), sizeof(double) * h.size(), cudaMemcpyHostToDevice, ctx->stream));
}

Vec down(apc_ctx* ctx, const double* d, i64 n) {
  Vec h(static_cast<size_t>(n));
  copy_sync(ctx->stream, h.data(), d, sizeof(double) * n, cudaMemcpyDeviceToHost);
  return h;
}

}  // namespace

int dpotrf_upper_dev(apc_ctx* ctx, i64 k, double* A) {
  cudaStream_t st = ctx->stream;
  DBuf<int> bad = new_flag(ctx);
  for (i64 k0 = 0; k0 < k; k0 += kPotrfNB) {
    const int nb = static_cast<int>(std::min<i64>(kPotrfNB, k - k0));
    potf2_kernel<<<1, kSmallT, 0, st>>>(A, k, static_cast<int>(k0), nb, bad.p);
    const i64 rest = k - k0 - nb;
    if (rest > 0) {
      potrf_panel_kernel<<<static_cast<unsigned>((rest + 127) / 128), 128, 0, st>>>(A, k, static_cast<int>(k0), nb,
                                                                                 rest);
      // trailing update A22 -= A12^T A12 (the full square; the lower part is ignored)
      const double* A12 = A + (k0 + nb) * k + k0;
      double* A22 = A + (k0 + nb) * k + k0 + nb;
      dgemm(ctx, true, false, rest, rest, nb, -1.0, A12, k, A12, k, 1.0, A22, k);
      ctx->launches += 2;
    } else {
      ctx->launches++;
    }
  }
  zero_lower_kernel<<<static_cast<unsigned>((k * k + 255) / 256), 256, 0, st>>>(A, k);
  ctx->launches++;
  APC_CUDA(cudaGetLastError());
  const int b = read_flag(ctx, bad.p);
  return b == 0x7fffffff ? -1 : b;
}

Vec dchol_upper(apc_ctx* ctx, i64 k, const Vec& g, const char* what) {
  DBuf<double> A;
  up(ctx, A, g);
  const int bad = dpotrf_upper_dev(ctx, k, A.p);
  if (bad >= 0) fail(APC_NOT_POSITIVE, what, bad);
  return down(ctx, A.p, k * k);
}

void dtrsm_rows_dev(apc_ctx* ctx, i64 k, const double* T, double* X, i64 ncols, bool transpose) {
  if (k == 0 || ncols == 0) return;
  DBuf<int> bad = new_flag(ctx);
  trsm_cols_kernel<<<static_cast<unsigned>((ncols + 127) / 128), 128, 0, ctx->stream>>>(T, k, X, ncols,
                                                                                       transpose ? 1 : 0, bad.p);
  ctx->launches++;
  APC_CUDA(cudaGetLastError());
  const int b = read_flag(ctx, bad.p);
  if (b != 0x7fffffff) fail(APC_SINGULAR, "tri_solve: zero diagonal", b);
}

Vec dtri_solve_cols(apc_ctx* ctx, i64 k, const Vec& t, const Vec& x, i64 ncols, bool transpose) {
  cudaStream_t st = ctx->stream;
  DBuf<double> dT, dX, dR(std::max<i64>(1, k * ncols));
  up(ctx, dT, t);
  up(ctx, dX, x);
  const unsigned g = static_cast<unsigned>((k * ncols + 255) / 256);
  transpose_kernel<<<std::max(1u, g), 256, 0, st>>>(dX.p, k, ncols, dR.p);  // column-major -> row-major
  dtrsm_rows_dev(ctx, k, dT.p, dR.p, ncols, transpose);
  transpose_kernel<<<std::max(1u, g), 256, 0, st>>>(dR.p, ncols, k, dX.p);  // back to column-major
  ctx->launches += 2;
  return down(ctx, dX.p, k * ncols);
}

Vec dmatmul(apc_ctx* ctx, i64 m, i64 k, i64 n, const Vec& a, const Vec& b) {
  DBuf<double> dA, dB, dC(std::max<i64>(1, m * n));
  up(ctx, dA, a);
  up(ctx, dB, b);
  dgemm(ctx, false, false, m, n, k, 1.0, dA.p, m, dB.p, k, 0.0, dC.p, m);
  return down(ctx, dC.p, m * n);
}

}  // namespace apc
