// One-sided (Hestenes) Jacobi SVD of the l x l preconditioner core M on the
// device: the same rotation formulas and stopping rule as small_svd
// (/root/reference/proj/include/aplicur/dense_factor.hpp:249-402; tol 1e-15,
// <= 60 sweeps), but in parallel round-robin order (l/2 disjoint column pairs
// per step, one CTA per pair), one CUDA graph per sweep.  Only sigma and V are
// needed by the preconditioner builders.  Not index-affecting.
// All sweeps run in ONE cooperative launch (jacobi_sweeps_kernel): CTAs take
// the round's pairs grid-stride, a grid barrier separates the rounds, and the
// rotation flag of each sweep (double-buffered) decides convergence on the
// device; the per-round launches (jacobi_round_kernel) remain as a fallback.
#include <cooperative_groups.h>

#include <algorithm>
#include <cmath>
#include <cstdlib>
#include <numeric>
#include <vector>

#include "dev_common.cuh"
#include "svd.hpp"

namespace apc {

namespace {

constexpr int kJT = 256;

__global__ void __launch_bounds__(kJT)
jacobi_round_kernel(double* __restrict__ W, double* __restrict__ V, long long p, long long n,
                    const int2* __restrict__ pairs, int* __restrict__ rotated) {
  __shared__ double sh[32];
  const int2 pr = pairs[blockIdx.x];
  if (pr.x < 0 || pr.y < 0) return;
  const long long j1 = pr.x < pr.y ? pr.x : pr.y, j2 = pr.x < pr.y ? pr.y : pr.x;
  double* c1 = W + j1 * p;
  double* c2 = W + j2 * p;
  double a = 0.0, b = 0.0, c = 0.0;
  for (long long i = threadIdx.x; i < p; i += kJT) {
    const double x = c1[i], y = c2[i];
    a += x * x;
    b += y * y;
    c += x * y;
  }
  a = block_sum<kJT>(a, sh);
  b = block_sum<kJT>(b, sh);
  c = block_sum<kJT>(c, sh);
  if (fabs(c) <= 1.0e-15 * sqrt(a * b) || c == 0.0) return;
  if (threadIdx.x == 0) *rotated = 1;
  const double zeta = (b - a) / (2.0 * c);
  const double tt = (zeta >= 0.0 ? 1.0 : -1.0) / (fabs(zeta) + sqrt(1.0 + zeta * zeta));
  const double cs = 1.0 / sqrt(1.0 + tt * tt);
  const double sn = cs * tt;
  for (long long i = threadIdx.x; i < p; i += kJT) {
    const double x = c1[i], y = c2[i];
    c1[i] = cs * x - sn * y;
    c2[i] = sn * x + cs * y;
  }
  double* v1 = V + j1 * n;
  double* v2 = V + j2 * n;
  for (long long i = threadIdx.x; i < n; i += kJT) {
    const double x = v1[i], y = v2[i];
    v1[i] = cs * x - sn * y;
    v2[i] = sn * x + cs * y;
  }
}

// one pair: the rotation of jacobi_round_kernel, block-wide
__device__ __forceinline__ bool jacobi_pair(double* __restrict__ W, double* __restrict__ V, long long p,
                                            long long n, int2 pr, double* sh) {
  if (pr.x < 0 || pr.y < 0) return false;
  const long long j1 = pr.x < pr.y ? pr.x : pr.y, j2 = pr.x < pr.y ? pr.y : pr.x;
  double* c1 = W + j1 * p;
  double* c2 = W + j2 * p;
  double a = 0.0, b = 0.0, c = 0.0;
  for (long long i = threadIdx.x; i < p; i += kJT) {
    const double x = __ldcg(c1 + i), y = __ldcg(c2 + i);
    a += x * x;
    b += y * y;
    c += x * y;
  }
  a = block_sum<kJT>(a, sh);
  b = block_sum<kJT>(b, sh);
  c = block_sum<kJT>(c, sh);
  if (fabs(c) <= 1.0e-15 * sqrt(a * b) || c == 0.0) return false;
  const double zeta = (b - a) / (2.0 * c);
  const double tt = (zeta >= 0.0 ? 1.0 : -1.0) / (fabs(zeta) + sqrt(1.0 + zeta * zeta));
  const double cs = 1.0 / sqrt(1.0 + tt * tt);
  const double sn = cs * tt;
  for (long long i = threadIdx.x; i < p; i += kJT) {
    const double x = __ldcg(c1 + i), y = __ldcg(c2 + i);
    c1[i] = cs * x - sn * y;
    c2[i] = sn * x + cs * y;
  }
  double* v1 = V + j1 * n;
  double* v2 = V + j2 * n;
  for (long long i = threadIdx.x; i < n; i += kJT) {
    const double x = __ldcg(v1 + i), y = __ldcg(v2 + i);
    v1[i] = cs * x - sn * y;
    v2[i] = sn * x + cs * y;
  }
  return true;
}

// every sweep of the tournament in one cooperative launch; flags[2] (one per
// sweep parity) are zero on entry; *sweeps_out = sweeps run, 0 rotations in
// the last one <=> converged
__global__ void __launch_bounds__(kJT)
jacobi_sweeps_kernel(double* __restrict__ W, double* __restrict__ V, long long p, long long n,
                     const int2* __restrict__ pairs, long long rounds, long long half, int max_sweeps,
                     int* __restrict__ flags, int* __restrict__ sweeps_out) {
  namespace cg = cooperative_groups;
  cg::grid_group grid = cg::this_grid();
  __shared__ double sh[32];
  for (int sw = 0; sw < max_sweeps; ++sw) {
    int* fl = flags + (sw & 1);
    bool any = false;
    for (long long r = 0; r < rounds; ++r) {
      for (long long q = blockIdx.x; q < half; q += gridDim.x) any |= jacobi_pair(W, V, p, n, pairs[r * half + q], sh);
      grid.sync();
    }
    if (any && threadIdx.x == 0) atomicOr(fl, 1);
    grid.sync();
    const int rot = atomicAdd(fl, 0);
    if (rot == 0) {
      if (blockIdx.x == 0 && threadIdx.x == 0) *sweeps_out = sw + 1;
      return;
    }
    // reset the other parity's flag for the next sweep (nobody reads it now)
    if (blockIdx.x == 0 && threadIdx.x == 0) flags[(sw + 1) & 1] = 0;
    grid.sync();
  }
  if (blockIdx.x == 0 && threadIdx.x == 0) *sweeps_out = -1;
}

__global__ void col_norms_kernel(const double* W, long long p, long long n, double* out) {
  __shared__ double sh[32];
  const long long j = blockIdx.x;
  double s = 0.0;
  for (long long i = threadIdx.x; i < p; i += kJT) s += W[j * p + i] * W[j * p + i];
  s = block_sum<kJT>(s, sh);
  if (threadIdx.x == 0) out[j] = sqrt(s);
}

__global__ void eye_kernel(double* V, long long n) {
  const long long e = static_cast<long long>(blockIdx.x) * blockDim.x + threadIdx.x;
  if (e < n * n) V[e] = (e / n == e % n) ? 1.0 : 0.0;
}

}  // namespace

void device_jacobi_svd(apc_ctx* ctx, i64 n, const Vec& M, Vec& sigma, Vec& V) {
  cudaStream_t st = ctx->stream;
  const i64 p = n;
  DBuf<double> dW(n * n), dV(n * n), dS(n);
  DBuf<int> flag(1);
  APC_CUDA(cudaMemcpyAsync(dW.p, M.data(), sizeof(double) * n * n, cudaMemcpyHostToDevice, st));
  eye_kernel<<<static_cast<unsigned>((n * n + 255) / 256), 256, 0, st>>>(dV.p, n);
  // circle-method tournament: n' - 1 rounds of n'/2 disjoint pairs (n' even)
  const i64 np = n + (n & 1), half = np / 2, rounds = np - 1;
  std::vector<int2> pairs(static_cast<size_t>(rounds * half));
  std::vector<int> ring(static_cast<size_t>(np));
  std::iota(ring.begin(), ring.end(), 0);
  for (i64 r = 0; r < rounds; ++r) {
    for (i64 k = 0; k < half; ++k) {
      int a = ring[k], b = ring[np - 1 - k];
      if (a >= n || b >= n) a = b = -1;  // bye
      pairs[r * half + k] = make_int2(a, b);
    }
    std::rotate(ring.begin() + 1, ring.end() - 1, ring.end());  // keep ring[0] fixed
  }
  DBuf<int2> dpairs(rounds * half);
  APC_CUDA(cudaMemcpyAsync(dpairs.p, pairs.data(), sizeof(int2) * pairs.size(), cudaMemcpyHostToDevice, st));
  static const bool per_round = std::getenv("APC_JACOBI_ROUNDS") != nullptr;
  if (!per_round && n > 1) {
    static int per_sm = -1;
    if (per_sm < 0)
      APC_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, jacobi_sweeps_kernel, kJT, 0));
    const long long grid = std::max<long long>(1, std::min<long long>(half, 1LL * per_sm * ctx->num_sms));
    DBuf<int> flags(3);
    APC_CUDA(cudaMemsetAsync(flags.p, 0, sizeof(int) * 3, st));
    long long pp = p, nn = n, rr = rounds, hh = half;
    int ms = 60;
    int* swo = flags.p + 2;
    void* args[] = {&dW.p, &dV.p, &pp, &nn, &dpairs.p, &rr, &hh, &ms, &flags.p, &swo};
    APC_CUDA(cudaLaunchCooperativeKernel(reinterpret_cast<const void*>(jacobi_sweeps_kernel), dim3(grid), dim3(kJT),
                                         args, 0, st));
    ctx->launches++;
    int sweeps = 0;
    copy_sync(st, &sweeps, swo, sizeof(int), cudaMemcpyDeviceToHost);
    if (sweeps < 0) fail(APC_NO_CONVERGENCE, "small_svd: Jacobi sweep cap reached");
  } else {
  // one sweep as a graph
  cudaGraph_t g = nullptr;
  cudaGraphExec_t ge = nullptr;
  APC_CUDA(cudaStreamBeginCapture(st, cudaStreamCaptureModeThreadLocal));
  for (i64 r = 0; r < rounds; ++r)
    jacobi_round_kernel<<<static_cast<unsigned>(half), kJT, 0, st>>>(dW.p, dV.p, p, n, dpairs.p + r * half, flag.p);
  APC_CUDA(cudaStreamEndCapture(st, &g));
  APC_CUDA(cudaGraphInstantiate(&ge, g, 0));
  bool converged = n <= 1;
  int h = 0;
  for (int sweep = 0; sweep < 60 && !converged; ++sweep) {
    APC_CUDA(cudaMemsetAsync(flag.p, 0, sizeof(int), st));
    APC_CUDA(cudaGraphLaunch(ge, st));
    ctx->launches += static_cast<std::uint64_t>(rounds);
    copy_sync(st, &h, flag.p, sizeof(int), cudaMemcpyDeviceToHost);
    converged = h == 0;
  }
  cudaGraphExecDestroy(ge);
  cudaGraphDestroy(g);
  if (!converged) fail(APC_NO_CONVERGENCE, "small_svd: Jacobi sweep cap reached");
  }
  col_norms_kernel<<<static_cast<unsigned>(n), kJT, 0, st>>>(dW.p, p, n, dS.p);
  ctx->launches++;
  Vec sig(static_cast<size_t>(n)), v(static_cast<size_t>(n * n));
  APC_CUDA(cudaMemcpyAsync(sig.data(), dS.p, sizeof(double) * n, cudaMemcpyDeviceToHost, st));
  copy_sync(st, v.data(), dV.p, sizeof(double) * n * n, cudaMemcpyDeviceToHost);
  std::vector<i64> ord(static_cast<size_t>(n));
  std::iota(ord.begin(), ord.end(), i64{0});
  std::stable_sort(ord.begin(), ord.end(), [&](i64 a, i64 b) { return sig[a] > sig[b]; });
  sigma.resize(static_cast<size_t>(n));
  V.resize(static_cast<size_t>(n * n));
  for (i64 jj = 0; jj < n; ++jj) {
    sigma[jj] = sig[ord[jj]];
    std::copy(v.begin() + ord[jj] * n, v.begin() + (ord[jj] + 1) * n, V.begin() + jj * n);
  }
}

}  // namespace apc
