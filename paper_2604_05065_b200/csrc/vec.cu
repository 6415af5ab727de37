// Phase-boundary vector work on the device: warm-start right-hand side
// rhs = b_aug - A_mu x (solver.hpp:207-210), system relative residual
// ||A_mu x - b_aug|| / ||b|| (solver.hpp:147-153, 257-258) and x += dx
// (solver.hpp:238-240).  Residual norms use a fixed reduction tree and one
// scalar allreduce across row shards.
#include <algorithm>

#include "dev_common.cuh"
#include "lsqr.hpp"
#include "ops.cuh"
#include "vec.hpp"

namespace apc {

namespace {
constexpr int kT = 256;
inline unsigned nb(long long n) { return static_cast<unsigned>(std::max<long long>(1, (n + kT - 1) / kT)); }

// top rows (tail == 0): r_i = b_i - ax_i ; tail rows (tail == 1): r_j = 0 - mu x_j.
// Writes rhs (optional) and block partials of r^2.
__global__ void residual_kernel(const double* ax, const double* b, const double* x, long long len,
                                double mu, int tail, double* rhs, double* part) {
  __shared__ double sh[32];
  long long i = static_cast<long long>(blockIdx.x) * kT + threadIdx.x;
  double sq = 0.0;
  if (i < len) {
    const double r = tail ? 0.0 - mu * x[i] : b[i] - ax[i];
    if (rhs) rhs[i] = r;
    sq = r * r;
  }
  sq = block_sum<kT>(sq, sh);
  if (threadIdx.x == 0) part[blockIdx.x] = sq;
}

__global__ void sum_kernel(const double* part, long long n, double* out) {
  __shared__ double sh[32];
  double s = ordered_sum<kT>(part, n, sh);
  if (threadIdx.x == 0) *out = s;
}

__global__ void axpy_kernel(double* x, const double* d, long long n) {
  long long i = static_cast<long long>(blockIdx.x) * kT + threadIdx.x;
  if (i < n) x[i] += d[i];
}
}  // namespace

VecWork::VecWork(apc_mat& a, double mu_) : mu(mu_) {
  const long long len = a.mloc() + (mu > 0.0 ? a.n : 0);
  ax.alloc(std::max<long long>(1, len));
  part.alloc(nb(a.mloc()) + nb(a.n));
  scalar.alloc(1);
}

// r = [b; 0] - A_mu x  -> rhs (local rows + tail), returns ||r||^2 over all
// ranks (the replicated tail is counted on rank 0 only)
double residual(apc_mat& a, VecWork& w, const double* x, const double* b_local, double* rhs) {
  apc_ctx* ctx = a.ctx;
  cudaStream_t st = ctx->stream;
  op_fwd(a, w.mu, w.mu > 0.0, x, w.ax.p);
  const long long ntop = a.mloc() > 0 ? nb(a.mloc()) : 0;
  if (a.mloc() > 0) {
    residual_kernel<<<nb(a.mloc()), kT, 0, st>>>(w.ax.p, b_local, x, a.mloc(), w.mu, 0, rhs, w.part.p);
    ctx->launches++;
  }
  long long nparts = ntop;
  if (w.mu > 0.0) {
    residual_kernel<<<nb(a.n), kT, 0, st>>>(nullptr, nullptr, x, a.n, w.mu, 1,
                                             rhs ? rhs + a.mloc() : nullptr, w.part.p + ntop);
    ctx->launches++;
    if (ctx->rank == 0) nparts += nb(a.n);
  }
  sum_kernel<<<1, kT, 0, st>>>(w.part.p, nparts, w.scalar.p);
  ctx->launches++;
  comm_allreduce(ctx, w.scalar.p, 1);
  double h = 0.0;
  APC_CUDA(cudaMemcpyAsync(&h, w.scalar.p, sizeof(double), cudaMemcpyDeviceToHost, st));
  APC_CUDA(cudaStreamSynchronize(st));
  return h;
}

void axpy(apc_ctx* ctx, double* x, const double* d, long long n) {
  axpy_kernel<<<nb(n), kT, 0, ctx->stream>>>(x, d, n);
  ctx->launches++;
}

}  // namespace apc
