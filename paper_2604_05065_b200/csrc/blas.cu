// Dense kernels of the per-rebuild preconditioner construction (blas.hpp),
// hand-written for sm_100a instead of cuBLAS: FP64 GEMM on the tensor cores
// (mma.sync.m8n8k4.f64, DMMA) with either operand transposed, a split over K
// for the tall-skinny products (Q^T E with K = n rows, the Gram E^T E),
// reduced in a fixed order, and a blocked right upper-triangular solve (its
// off-diagonal updates are GEMMs, the 32 x 32 diagonal blocks a row-parallel
// substitution).  Never on the per-iteration path and never on the
// index-selecting path: results are deterministic run to run, not
// bit-identical to any particular BLAS.
//   QrAccumulator::append (preconditioner.hpp:435-476): P = Q^T E, E -= Q P,
//     G = E^T E, E <- E R^{-1}; the explicit basis V = Q_R V_M (:171-193);
//   the sparse-C Gram of CurState::c_gram (row blocks accumulated in order).
#include <algorithm>

#include "blas.hpp"

namespace apc {

namespace {

constexpr int kBM = 96, kBN = 64, kBK = 32;
constexpr int kSA = kBM + 4, kSB = kBK + 4;  // shared strides (doubles): conflict-free fragments
constexpr int kStage = kBK * kSA + kBN * kSB;

__device__ __forceinline__ void mma_f64(double (&d)[2], double a, double b) {
  asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0, %1}, {%2}, {%3}, {%0, %1};\n"
               : "+d"(d[0]), "+d"(d[1])
               : "d"(a), "d"(b));
}

__device__ __forceinline__ void cp8(double* smem, const double* g, bool ok) {
  const unsigned sa = static_cast<unsigned>(__cvta_generic_to_shared(smem));
  asm volatile("cp.async.ca.shared.global [%0], [%1], 8, %2;\n" ::"r"(sa), "l"(g), "r"(ok ? 8 : 0));
}

struct GemmArgs {
  const double* A;  // op(A)(i, k) = A[i * ai + k * ak]
  long long ai, ak;
  const double* B;  // op(B)(k, j) = B[k * bk + j * bj]
  long long bk, bj;
  double* C;        // col-major, ldc
  long long ldc;
  long long M, N, K, kchunk;  // kchunk: K range per split (grid.z)
  double alpha, beta;
  double* ws;       // split partials (M x N col-major per split), null without a split
};

// CTA: a 96 x 64 tile of C over the K range of split blockIdx.z; warp w owns
// columns [8w, 8w + 8) and all twelve 8-row tiles.  Operand staging follows
// the operand's contiguous dimension so the cp.async copies coalesce.
__global__ void __launch_bounds__(256, 2) gemm_dmma_kernel(GemmArgs g) {
  extern __shared__ double sm[];
  const int tid = threadIdx.x, lane = tid & 31, w = tid >> 5, gq = lane >> 2, t = lane & 3;
  const long long i0 = static_cast<long long>(blockIdx.x) * kBM, j0 = static_cast<long long>(blockIdx.y) * kBN;
  const long long kb = static_cast<long long>(blockIdx.z) * g.kchunk;
  const long long ke = kb + g.kchunk < g.K ? kb + g.kchunk : g.K;
  auto stage = [&](int buf, long long k0) {
    double* As = sm + buf * kStage;  // [k][i], stride kSA
    double* Bs = As + kBK * kSA;     // [j][k], stride kSB
    if (g.ai == 1) {
      for (int e = tid; e < kBK * kBM; e += 256) {
        const int kk = e / kBM, ii = e % kBM;
        const long long k = k0 + kk, i = i0 + ii;
        const bool ok = k < ke && i < g.M;
        cp8(As + kk * kSA + ii, ok ? g.A + i + k * g.ak : g.A, ok);
      }
    } else {
      for (int e = tid; e < kBK * kBM; e += 256) {
        const int ii = e / kBK, kk = e % kBK;
        const long long k = k0 + kk, i = i0 + ii;
        const bool ok = k < ke && i < g.M;
        cp8(As + kk * kSA + ii, ok ? g.A + i * g.ai + k * g.ak : g.A, ok);
      }
    }
    if (g.bk == 1) {
      for (int e = tid; e < kBN * kBK; e += 256) {
        const int jj = e / kBK, kk = e % kBK;
        const long long k = k0 + kk, j = j0 + jj;
        const bool ok = k < ke && j < g.N;
        cp8(Bs + jj * kSB + kk, ok ? g.B + k + j * g.bj : g.B, ok);
      }
    } else {
      for (int e = tid; e < kBN * kBK; e += 256) {
        const int kk = e / kBN, jj = e % kBN;
        const long long k = k0 + kk, j = j0 + jj;
        const bool ok = k < ke && j < g.N;
        cp8(Bs + jj * kSB + kk, ok ? g.B + k * g.bk + j * g.bj : g.B, ok);
      }
    }
    asm volatile("cp.async.commit_group;\n" ::);
  };
  double acc[kBM / 8][2];
#pragma unroll
  for (int q = 0; q < kBM / 8; ++q) acc[q][0] = acc[q][1] = 0.0;
  const long long nk = ke > kb ? (ke - kb + kBK - 1) / kBK : 0;
  if (nk > 0) stage(0, kb);
  for (long long c = 0; c < nk; ++c) {
    const int buf = static_cast<int>(c & 1);
    if (c + 1 < nk) {
      stage(buf ^ 1, kb + (c + 1) * kBK);
      asm volatile("cp.async.wait_group 1;\n" ::);
    } else {
      asm volatile("cp.async.wait_group 0;\n" ::);
    }
    __syncthreads();
    const double* As = sm + buf * kStage;
    const double* Bs = As + kBK * kSA;
#pragma unroll
    for (int kk = 0; kk < kBK; kk += 4) {
      const double b = Bs[(8 * w + gq) * kSB + kk + t];
#pragma unroll
      for (int q = 0; q < kBM / 8; ++q) mma_f64(acc[q], As[(kk + t) * kSA + 8 * q + gq], b);
    }
    __syncthreads();
  }
#pragma unroll
  for (int q = 0; q < kBM / 8; ++q) {
    const long long i = i0 + 8 * q + gq;
    if (i >= g.M) continue;
#pragma unroll
    for (int h = 0; h < 2; ++h) {
      const long long j = j0 + 8 * w + 2 * t + h;
      if (j >= g.N) continue;
      if (g.ws) {
        g.ws[static_cast<long long>(blockIdx.z) * g.M * g.N + j * g.M + i] = acc[q][h];
      } else {
        double* c = g.C + j * g.ldc + i;
        *c = g.beta == 0.0 ? g.alpha * acc[q][h] : g.alpha * acc[q][h] + g.beta * *c;
      }
    }
  }
}

// C = alpha * (sum of the split partials, split order) + beta * C
__global__ void gemm_reduce_kernel(const double* __restrict__ ws, int splits, long long M, long long N, double alpha,
                                   double beta, double* __restrict__ C, long long ldc) {
  const long long e = static_cast<long long>(blockIdx.x) * blockDim.x + threadIdx.x;
  if (e >= M * N) return;
  const long long i = e % M, j = e / M;
  double s = ws[e];
  for (int z = 1; z < splits; ++z) s += ws[z * M * N + e];
  double* c = C + j * ldc + i;
  *c = beta == 0.0 ? alpha * s : alpha * s + beta * *c;
}

// B(:, jb:jb+nb) <- B(:, jb:jb+nb) T(jb:jb+nb, jb:jb+nb)^{-1}, thread per row
constexpr int kTrsmNB = 32;
__global__ void __launch_bounds__(128)
trsm_diag_kernel(long long m, int nb, const double* __restrict__ T, long long ldt, double* __restrict__ B,
                 long long ldb) {
  __shared__ double Ts[kTrsmNB][kTrsmNB + 1];
  for (int e = threadIdx.x; e < nb * nb; e += blockDim.x) Ts[e % nb][e / nb] = T[(e / nb) * ldt + e % nb];
  __syncthreads();
  const long long r = static_cast<long long>(blockIdx.x) * blockDim.x + threadIdx.x;
  if (r >= m) return;
  double x[kTrsmNB];
#pragma unroll
  for (int j = 0; j < kTrsmNB; ++j) x[j] = j < nb ? B[j * ldb + r] : 0.0;
#pragma unroll
  for (int j = 0; j < kTrsmNB; ++j) {
    if (j >= nb) break;
    double s = x[j];
#pragma unroll
    for (int i = 0; i < kTrsmNB; ++i)
      if (i < j) s -= x[i] * Ts[i][j];
    x[j] = s / Ts[j][j];
  }
#pragma unroll
  for (int j = 0; j < kTrsmNB; ++j)
    if (j < nb) B[j * ldb + r] = x[j];
}

int num_sms(apc_ctx* ctx) { return ctx->num_sms > 0 ? ctx->num_sms : 148; }

void gemm(apc_ctx* ctx, long long M, long long N, long long K, double alpha, const double* A, long long ai,
          long long ak, const double* B, long long bk, long long bj, double beta, double* C, long long ldc) {
  if (M == 0 || N == 0) return;
  cudaStream_t st = ctx->stream;
  const int smem = 2 * kStage * static_cast<int>(sizeof(double));
  static bool attr = false;
  if (!attr) {
    APC_CUDA(cudaFuncSetAttribute(gemm_dmma_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, smem));
    attr = true;
  }
  const long long tiles = ((M + kBM - 1) / kBM) * ((N + kBN - 1) / kBN);
  // split K until the grid covers the SMs twice (tall-skinny products), chunks
  // a multiple of kBK; fixed split order in the reduction keeps runs identical
  long long splits = 1;
  const long long want = 2LL * num_sms(ctx);
  if (K > 4 * kBK && tiles < want) splits = std::min<long long>((want + tiles - 1) / tiles, (K + 4 * kBK - 1) / (4 * kBK));
  long long kchunk = (K + splits - 1) / splits;
  kchunk = (kchunk + kBK - 1) / kBK * kBK;
  splits = std::max<long long>(1, (K + kchunk - 1) / kchunk);
  GemmArgs g{A, ai, ak, B, bk, bj, C, ldc, M, N, K, std::max<long long>(kchunk, 1), alpha, beta, nullptr};
  DBuf<double> ws;
  if (splits > 1) {
    ws.alloc(splits * M * N);
    g.ws = ws.p;
  }
  dim3 grid(static_cast<unsigned>((M + kBM - 1) / kBM), static_cast<unsigned>((N + kBN - 1) / kBN),
            static_cast<unsigned>(splits));
  gemm_dmma_kernel<<<grid, 256, smem, st>>>(g);
  ctx->launches++;
  if (splits > 1) {
    gemm_reduce_kernel<<<static_cast<unsigned>((M * N + 255) / 256), 256, 0, st>>>(ws.p, static_cast<int>(splits), M,
                                                                                 N, alpha, beta, C, ldc);
    ctx->launches++;
    APC_CUDA(cudaStreamSynchronize(st));  // ws goes out of scope
  }
  APC_CUDA(cudaGetLastError());
}

}  // namespace

void dgemm(apc_ctx* ctx, bool ta, bool tb, i64 m, i64 n, i64 k, double alpha, const double* A, i64 lda,
           const double* B, i64 ldb, double beta, double* C, i64 ldc) {
  gemm(ctx, m, n, k, alpha, A, ta ? lda : 1, ta ? 1 : lda, B, tb ? ldb : 1, tb ? 1 : ldb, beta, C, ldc);
}

void dsyrk_t(apc_ctx* ctx, i64 n, i64 k, double alpha, const double* A, i64 lda, double beta, double* C, i64 ldc) {
  // the full square A^T A (callers read the upper triangle)
  gemm(ctx, n, n, k, alpha, A, lda, 1, A, 1, lda, beta, C, ldc);
}

void dtrsm_right_upper(apc_ctx* ctx, i64 m, i64 n, const double* T, i64 ldt, double* B, i64 ldb) {
  if (m == 0 || n == 0) return;
  for (i64 jb = 0; jb < n; jb += kTrsmNB) {
    const int nb = static_cast<int>(std::min<i64>(kTrsmNB, n - jb));
    if (jb > 0)  // B(:, jb:jb+nb) -= B(:, 0:jb) T(0:jb, jb:jb+nb)
      gemm(ctx, m, nb, jb, -1.0, B, 1, ldb, T + jb * ldt, 1, ldt, 1.0, B + jb * ldb, ldb);
    trsm_diag_kernel<<<static_cast<unsigned>((m + 127) / 128), 128, 0, ctx->stream>>>(m, nb, T + jb * ldt + jb, ldt,
                                                                                      B + jb * ldb, ldb);
    ctx->launches++;
  }
  APC_CUDA(cudaGetLastError());
}

void blas_destroy(apc_ctx*) {}

}  // namespace apc
