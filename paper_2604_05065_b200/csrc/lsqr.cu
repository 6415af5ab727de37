// Device-resident LSQR phase: Golub-Kahan bidiagonalisation with the vector
// updates and norms fused into the operator kernels, scalars and stop rules on
// the GPU, and the whole iteration captured as a CUDA graph whose conditional
// WHILE node re-runs the body until the device stop flag is raised.
//
// Reference: lsqr_solve (/root/reference/proj/include/aplicur/lsqr.hpp:84-207),
// dynamic_stop_check (lsqr.hpp:65-72), right_preconditioned
// (operators.hpp:75-90), preconditioner applies (preconditioner.hpp:62-124,
// 279-339).
//
// Per iteration (plain / preconditioned):
//   [P^{-1} v -> z : project, core, expand]            (preconditioned only)
//   fwd   : u <- A z - alpha*u  (+ ||u_top||^2, fused in the SpMV/GEMV)
//   tail  : u_tail <- mu z - alpha*u_tail (+ ||u_tail||^2)       (mu > 0)
//   adj   : g <- A^T u (raw, local rows)         [+ NCCL allreduce(n+1)]
//   epi   : beta; g/beta; plain: v <- g - beta v, ||v||^2, alpha, rotation
//   [P^{-T} g : project, core, expand + v update + alpha, rotation]
//   upd   : v/alpha; y += t1 w; w = v + t2 w; ||y||; stop tests
// u and v are kept unnormalised between kernels and normalised on the fly
// (u/beta, v/alpha rounds exactly like the reference's in-place division).
#include <cuda_runtime.h>

#include <algorithm>
#include <chrono>
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <string>

#include <cooperative_groups.h>

#include "dev_common.cuh"
#include "lsqr.hpp"
#include "dense_pair.hpp"
#include "lsqr_persistent.hpp"
#include "ops.cuh"

namespace apc {

constexpr int kVecThreads = 256;

struct LsqrPtrs {
  LsqrState* st;
  TraceRow* trace;
  double* u;  // mloc (+ n tail)
  double* v;  // n
  double* w;
  double* y;
  double* z;  // P^{-1} v (or v itself when unpreconditioned)
  double* g;  // n + 1 (A^T u raw | ||u_top||^2)
  double* h;  // n (g / beta, input of P^{-T})
  double* fwd_part;
  double* tail_part;
  double* epi_part;
  double* upd_part;
  unsigned* ctr;  // [0] fwd, [1] tail, [2] epi, [3] upd
  long long mloc, n;
  double mu;
  int has_tail;
};

// ---------------------------------------------------------------------------
// scalar recurrences (single thread of the last block)
// ---------------------------------------------------------------------------
__device__ void finalize_alpha(LsqrState* st, TraceRow* trace, double alpha, double beta) {
  const double wall = (globaltimer_ns() - st->t0_ns) * 1e-6;
  if (st->iter < 0) {  // phase initialisation (lsqr.hpp:113-135)
    st->iter = 0;
    st->beta = beta;
    st->phibar = beta;
    st->phibar0 = beta;
    st->alpha = alpha;
    st->rhobar = alpha;
    st->opnorm2 = alpha * alpha;
    st->t1 = 0.0;
    st->t2 = 0.0;
    if (trace) trace[0] = TraceRow{beta, 0.0, 0.0, wall, 0, 0ull};
    if (alpha == 0.0) {
      st->done = 1;
      st->reason = kReasonGradientTol;
    }
    return;
  }
  // continue the bidiagonalisation (lsqr.hpp:139-164)
  st->alpha = alpha;
  st->beta = beta;
  st->opnorm2 += alpha * alpha + beta * beta;
  const double rho = hypot(st->rhobar, beta);
  const double c = st->rhobar / rho;
  const double s = beta / rho;
  const double theta = s * alpha;
  st->rhobar = -c * alpha;
  const double phi = c * st->phibar;
  const double phibar_prev = st->phibar;
  const double phibar = s * st->phibar;
  st->phibar = phibar;
  st->t1 = phi / rho;
  st->t2 = -theta / rho;
  st->cabs = fabs(c);
  const long long j = st->iter + 1;
  st->iter = j;
  if (!isfinite(phibar) || !isfinite(alpha) || !isfinite(beta)) {  // lsqr.hpp:173-174
    st->breakdown = 1;
    st->done = 1;
  }
  const double cvgrate = (phibar > 0.0 && phibar_prev > 0.0) ? log(phibar_prev / phibar)
                                                             : CUDART_INF;
  const double cvgdiff = phibar_prev - phibar;
  if (j == 1) st->cvgrate1 = cvgrate;
  st->t_cvgrate = cvgrate;
  st->t_cvgdiff = cvgdiff;
  if (trace && j < st->trace_cap)
    trace[j] = TraceRow{phibar, cvgrate, cvgdiff, wall, j, 1ull + 2ull * static_cast<unsigned long long>(j)};
}

// stop tests after the y/w update (lsqr.hpp:183-203)
__device__ void stop_tests(LsqrState* st, double ynorm) {
  const long long j = st->iter;
  if (j <= 0 || st->done) return;
  st->ynorm = ynorm;
  const double phibar = st->phibar;
  const double grad = phibar * st->alpha * st->cabs;
  const double sq = sqrt(st->opnorm2);
  const bool grad_small = grad <= st->eps * sq * phibar;
  const bool res_small = phibar <= st->eps * (sq * ynorm + st->phibar0);
  if (grad_small || res_small || phibar == 0.0) {
    st->done = 1;
    st->reason = kReasonGradientTol;
    return;
  }
  if (j >= 2 && st->nu > 0.0 && !isinf(st->nu)) {  // dynamic_stop_check (lsqr.hpp:65-72)
    const double rate = st->t_cvgrate, diff = st->t_cvgdiff;
    int dyn = kReasonNone;
    if (st->sigma_floor > 0.0 && diff < st->sigma_floor) dyn = kReasonDynamicDiff;
    else if (rate <= 0.0) dyn = kReasonDynamicRate;
    else if (st->cvgrate1 / rate > st->nu) dyn = kReasonDynamicRate;
    if (dyn != kReasonNone) {
      st->done = 1;
      st->reason = dyn;
      return;
    }
  }
  if (j >= st->cap) {
    st->done = 1;
    st->reason = kReasonIterationCap;
  }
}

// ---------------------------------------------------------------------------
// kernels
// ---------------------------------------------------------------------------
struct LsqrFwdEpi {  // u <- (A z) - alpha * u/beta ; ||u_top||^2 -> g[n]
  double* u;
  const LsqrState* st;
  double* part;
  unsigned* ctr;
  double* out_norm2;
  double alpha, beta;
  __device__ void begin() {
    alpha = st->alpha;
    beta = st->beta;
  }
  __device__ double load(long long r) { return u[r]; }
  __device__ double row(long long r, double av, double uo) {
    const double uh = beta > 0.0 ? uo / beta : uo;
    const double t = av - alpha * uh;
    u[r] = t;
    return t * t;
  }
  __device__ void tile_done(unsigned tile, unsigned ntiles, double sq) {
    __shared__ double sh[32];
    if (threadIdx.x == 0) part[tile] = sq;
    if (elect_last_block(ctr, ntiles)) {
      double s = ordered_sum<256>(part, ntiles, sh);
      if (threadIdx.x == 0) *out_norm2 = s;
    }
  }
};

// true-residual sample: ||b - A xs||^2 over the local rows -> *out_norm2
struct ResidSampleEpi {
  const double* b;
  double* part;
  unsigned* ctr;
  double* out_norm2;
  __device__ void begin() {}
  __device__ double load(long long r) { return b[r]; }
  __device__ double row(long long, double av, double bo) {
    const double t = av - bo;
    return t * t;
  }
  __device__ void tile_done(unsigned tile, unsigned ntiles, double sq) {
    __shared__ double sh[32];
    if (threadIdx.x == 0) part[tile] = sq;
    if (elect_last_block(ctr, ntiles)) {
      double s = ordered_sum<256>(part, ntiles, sh);
      if (threadIdx.x == 0) *out_norm2 = s;
    }
  }
};

// Explicit basis (dense B, n x l column-major): out = x + B s through the dense
// forward kernel (8 rows per thread, split over the l columns) instead of a
// thread-per-row chain over l.  mode 0: out_j = x_j + (B s)_j ; mode 1:
// v_j = (x_j + (B s)_j) - beta v_j, ||v||^2 -> alpha and the rotation (last block).
struct PcExpandEpi {
  LsqrPtrs P;
  const double* x;
  double* out;
  int mode;
  double beta;
  int fuse_tail;  // mode 0: also u_t <- mu z - alpha u_t/beta (lsqr_tail_kernel), ||u_t||^2
  double alpha;
  __device__ void begin() {
    if (mode == 1) beta = sqrt(P.g[P.n] + P.st->tail_norm2);
    if (mode == 0 && fuse_tail) {
      alpha = P.st->alpha;
      beta = P.st->beta;
    }
  }
  __device__ double load(long long j) { return mode == 1 ? P.v[j] : 0.0; }
  __device__ double row(long long j, double acc, double vj) {
    const double o = x[j] + acc;
    if (mode == 0) {
      out[j] = o;
      if (!fuse_tail) return 0.0;
      double* ut = P.u + P.mloc;
      const double uo = ut[j];
      const double uh = beta > 0.0 ? uo / beta : uo;
      const double t = P.mu * o - alpha * uh;
      ut[j] = t;
      return t * t;
    }
    const double t = o - beta * vj;
    P.v[j] = t;
    return t * t;
  }
  __device__ void tile_done(unsigned tile, unsigned ntiles, double sq) {
    __shared__ double sh[32];
    if (mode == 0) {
      if (!fuse_tail) return;
      if (threadIdx.x == 0) P.tail_part[tile] = sq;
      if (elect_last_block(P.ctr + 1, ntiles)) {
        const double s = ordered_sum<256>(P.tail_part, ntiles, sh);
        if (threadIdx.x == 0) P.st->tail_norm2 = s;
      }
      return;
    }
    if (threadIdx.x == 0) P.epi_part[tile] = sq;
    if (elect_last_block(P.ctr + 2, ntiles)) {
      const double s = ordered_sum<256>(P.epi_part, ntiles, sh);
      if (threadIdx.x == 0) finalize_alpha(P.st, P.trace, sqrt(s), beta);
    }
  }
};

// init: u <- rhs; ||rhs_top||^2 -> g[n] ; ||rhs_tail||^2 -> st->tail_norm2
__global__ void __launch_bounds__(kVecThreads)
lsqr_init_copy_kernel(LsqrPtrs P, const double* rhs, long long len, long long off, int tail) {
  __shared__ double sh[32];
  long long i = static_cast<long long>(blockIdx.x) * kVecThreads + threadIdx.x;
  double sq = 0.0;
  if (i < len) {
    double t = rhs[off + i];
    P.u[off + i] = t;
    sq = t * t;
  }
  sq = block_sum<kVecThreads>(sq, sh);
  double* part = tail ? P.tail_part : P.fwd_part;
  if (threadIdx.x == 0) part[blockIdx.x] = sq;
  if (elect_last_block(P.ctr + (tail ? 1 : 0), gridDim.x)) {
    double s = ordered_sum<kVecThreads>(part, gridDim.x, sh);
    if (threadIdx.x == 0) {
      if (tail) P.st->tail_norm2 = s;
      else P.g[P.n] = s;
    }
  }
}

// mu-tail rows of the augmented system: u_t <- mu z - alpha u_t/beta
__global__ void __launch_bounds__(kVecThreads) lsqr_tail_kernel(LsqrPtrs P) {
  __shared__ double sh[32];
  if (P.st->done) return;
  const double alpha = P.st->alpha, beta = P.st->beta;
  long long j = static_cast<long long>(blockIdx.x) * kVecThreads + threadIdx.x;
  double sq = 0.0;
  if (j < P.n) {
    double* ut = P.u + P.mloc;
    const double uo = ut[j];
    const double uh = beta > 0.0 ? uo / beta : uo;
    const double t = P.mu * P.z[j] - alpha * uh;
    ut[j] = t;
    sq = t * t;
  }
  sq = block_sum<kVecThreads>(sq, sh);
  if (threadIdx.x == 0) P.tail_part[blockIdx.x] = sq;
  if (elect_last_block(P.ctr + 1, gridDim.x)) {
    double s = ordered_sum<kVecThreads>(P.tail_part, gridDim.x, sh);
    if (threadIdx.x == 0) P.st->tail_norm2 = s;
  }
}

// beta from the (allreduced) ||u_top||^2 and the tail; g = A_mu^T u / beta.
// precond == 0: v <- g - beta v, ||v||^2 -> alpha -> rotation (last block).
// precond != 0: h <- g (input of P^{-T}).
__global__ void __launch_bounds__(kVecThreads) lsqr_epi_kernel(LsqrPtrs P, int precond) {
  __shared__ double sh[32];
  LsqrState* st = P.st;
  if (st->done) return;
  const double beta = sqrt(P.g[P.n] + st->tail_norm2);
  if (st->iter < 0 && beta == 0.0) {  // exact_zero_rhs (lsqr.hpp:113-118)
    if (blockIdx.x == 0 && threadIdx.x == 0) {
      P.trace[0] = TraceRow{0.0, 0.0, 0.0, (globaltimer_ns() - st->t0_ns) * 1e-6, 0, 0ull};
      st->phibar = 0.0;
      st->phibar0 = 0.0;
      st->done = 1;
      st->reason = kReasonExactZeroRhs;
    }
    return;
  }
  long long j = static_cast<long long>(blockIdx.x) * kVecThreads + threadIdx.x;
  double sq = 0.0;
  if (j < P.n) {
    double raw = P.g[j];  // split rows of A^T were summed by op_adj_raw
    if (P.has_tail) raw += P.mu * P.u[P.mloc + j];
    const double gj = beta > 0.0 ? raw / beta : raw;
    if (precond) {
      P.h[j] = gj;
    } else {
      const double t = gj - beta * P.v[j];
      P.v[j] = t;
      sq = t * t;
    }
  }
  if (precond) return;
  sq = block_sum<kVecThreads>(sq, sh);
  if (threadIdx.x == 0) P.epi_part[blockIdx.x] = sq;
  if (elect_last_block(P.ctr + 2, gridDim.x)) {
    double s = ordered_sum<kVecThreads>(P.epi_part, gridDim.x, sh);
    if (threadIdx.x == 0) finalize_alpha(st, P.trace, sqrt(s), beta);
  }
}

// v <- v/alpha ; y += t1 w ; w = v + t2 w ; ||y|| ; stop tests (lsqr.hpp:145-203)
__global__ void __launch_bounds__(kVecThreads)
lsqr_update_kernel(LsqrPtrs P, cudaGraphConditionalHandle cond, int use_cond) {
  __shared__ double sh[32];
  LsqrState* st = P.st;
  if (st->done) {
    if (use_cond && blockIdx.x == 0 && threadIdx.x == 0) cudaGraphSetConditional(cond, 0);
    return;
  }
  const double alpha = st->alpha, t1 = st->t1, t2 = st->t2;
  long long j = static_cast<long long>(blockIdx.x) * kVecThreads + threadIdx.x;
  double sq = 0.0;
  if (j < P.n) {
    const double vo = P.v[j];
    const double vh = alpha > 0.0 ? vo / alpha : vo;
    P.v[j] = vh;
    const double wo = P.w[j];
    const double yn = P.y[j] + t1 * wo;
    P.y[j] = yn;
    P.w[j] = vh + t2 * wo;
    sq = yn * yn;
  }
  sq = block_sum<kVecThreads>(sq, sh);
  if (threadIdx.x == 0) P.upd_part[blockIdx.x] = sq;
  if (elect_last_block(P.ctr + 3, gridDim.x)) {
    double s = ordered_sum<kVecThreads>(P.upd_part, gridDim.x, sh);
    if (threadIdx.x == 0) {
      stop_tests(st, sqrt(s));
      if (use_cond) cudaGraphSetConditional(cond, st->done ? 0u : 1u);
    }
  }
}

// ---------------------------------------------------------------------------
// true-residual sampling (the solver's observer, solver.hpp:222-236, 418-427)
// ---------------------------------------------------------------------------
// gate: sample iff this graph body completed iteration j >= 1 and j % stride == 0
__global__ void samp_gate_kernel(LsqrState* st, long long stride) {
  const long long j = st->iter;
  const bool take = j >= 1 && j != st->samp_last && !st->breakdown && j % stride == 0;
  st->samp_last = j;
  st->samp_skip = take ? 0 : 1;
}

// xs = d (+ x_base) ; tail: ||mu xs||^2 -> sc[1] (last block)
__global__ void __launch_bounds__(kVecThreads)
samp_combine_kernel(const LsqrState* st, const double* d, const double* x_base, double* xs, long long n,
                    double mu, double* part, unsigned* ctr, double* sc) {  // xs may alias d
  __shared__ double sh[32];
  if (st->samp_skip) return;
  const long long j = static_cast<long long>(blockIdx.x) * kVecThreads + threadIdx.x;
  double sq = 0.0;
  if (j < n) {
    const double v = x_base ? d[j] + x_base[j] : d[j];
    if (x_base) xs[j] = v;
    const double t = mu * v;
    sq = t * t;
  }
  if (mu <= 0.0) return;
  sq = block_sum<kVecThreads>(sq, sh);
  if (threadIdx.x == 0) part[blockIdx.x] = sq;
  if (elect_last_block(ctr, gridDim.x)) {
    const double s = ordered_sum<kVecThreads>(part, gridDim.x, sh);
    if (threadIdx.x == 0) sc[1] = s;
  }
}

__global__ void samp_zero_kernel(const LsqrState* st, double* sc) {
  if (!st->samp_skip) sc[0] = 0.0;
}

// sampled[j] = sqrt(top + tail) / bnorm (system_relres, solver.hpp:147-153)
__global__ void samp_final_kernel(const LsqrState* st, const double* sc, double bnorm, int tail,
                                  double* sampled, long long cap) {
  if (st->samp_skip) return;
  const long long j = st->iter;
  if (j < 0 || j >= cap) return;
  sampled[j] = bnorm > 0.0 ? sqrt(sc[0] + (tail ? sc[1] : 0.0)) / bnorm : 0.0;
}

// ---------------------------------------------------------------------------
// preconditioner kernels:  out = x + B (K (B^T x))  or  x + R^T (G (R x))
// ---------------------------------------------------------------------------
// Sparse and dense dot products of the preconditioner applies.  Each running
// sum adds its terms in index order (one chain per lane or thread); the loops
// are unrolled by hand so the loads of four terms are issued before the first
// add waits on them (the chains were latency bound: one index load and one
// dependent gather per term).  The add order, hence every bit, is the plain
// loops' own (APC_NO_GATHER_UNROLL builds the plain loops for A/B runs).
// lane-strided: sum over q = b0 + lane, b0 + lane + 32, ... < b1
__device__ __forceinline__ double gather_dot_lanes(const int* __restrict__ idx, const double* __restrict__ val,
                                                   const double* __restrict__ s, int b0, int b1, int lane) {
  double x = 0.0;
  int q = b0 + lane;
#ifndef APC_NO_GATHER_UNROLL
  for (; q + 96 < b1; q += 128) {
    const int i0 = idx[q], i1 = idx[q + 32], i2 = idx[q + 64], i3 = idx[q + 96];
    const double v0 = val[q], v1 = val[q + 32], v2 = val[q + 64], v3 = val[q + 96];
    const double s0 = s[i0], s1 = s[i1], s2 = s[i2], s3 = s[i3];
    x += v0 * s0;
    x += v1 * s1;
    x += v2 * s2;
    x += v3 * s3;
  }
#endif
  for (; q < b1; q += 32) x += val[q] * s[idx[q]];
  return x;
}
// one thread: sum over q = q0 .. q1-1 (acc carried in)
__device__ __forceinline__ double gather_dot_seq(const int* __restrict__ idx, const double* __restrict__ val,
                                                 const double* __restrict__ s, int q0, int q1, double acc) {
  int q = q0;
#ifndef APC_NO_GATHER_UNROLL
  for (; q + 3 < q1; q += 4) {
    const int i0 = idx[q], i1 = idx[q + 1], i2 = idx[q + 2], i3 = idx[q + 3];
    const double v0 = val[q], v1 = val[q + 1], v2 = val[q + 2], v3 = val[q + 3];
    const double s0 = s[i0], s1 = s[i1], s2 = s[i2], s3 = s[i3];
    acc += v0 * s0;
    acc += v1 * s1;
    acc += v2 * s2;
    acc += v3 * s3;
  }
#endif
  for (; q < q1; ++q) acc += val[q] * s[idx[q]];
  return acc;
}
// lane-strided dense row: sum over k = lane, lane + 32, ... < l of row[k] t[k]
__device__ __forceinline__ double row_dot_lanes(const double* __restrict__ row, const double* __restrict__ t,
                                                long long l, int lane) {
  double acc = 0.0;
  long long k = lane;
#ifndef APC_NO_GATHER_UNROLL
  for (; k + 96 < l; k += 128) {
    const double r0 = row[k], r1 = row[k + 32], r2 = row[k + 64], r3 = row[k + 96];
    const double t0 = t[k], t1 = t[k + 32], t2 = t[k + 64], t3 = t[k + 96];
    acc += r0 * t0;
    acc += r1 * t1;
    acc += r2 * t2;
    acc += r3 * t3;
  }
#endif
  for (; k < l; k += 32) acc += row[k] * t[k];
  return acc;
}

// s = K t with K stored row-major (KT[i * l + k] = K(i, k)): one warp per row,
// lanes stride k (coalesced), fixed shuffle tree
__global__ void pc_core_kernel(const double* __restrict__ KT, long long l,
                               const double* __restrict__ t, double* __restrict__ s,
                               const int* done) {
  if (done && *done) return;
  const long long i = (static_cast<long long>(blockIdx.x) * blockDim.x + threadIdx.x) >> 5;
  const int lane = threadIdx.x & 31;
  if (i >= l) return;
  double acc = row_dot_lanes(KT + i * l, t, l, lane);
  acc = warp_sum(acc);
  if (lane == 0) s[i] = acc;
}

// t = R x: one warp per (short) row of R, spread over many CTAs
__global__ void pc_rproj_kernel(const int* __restrict__ rptr, const int* __restrict__ ridx,
                                const double* __restrict__ rval, long long l, const double* __restrict__ x,
                                double* __restrict__ t, const int* done) {
  if (done && *done) return;
  const long long i = (static_cast<long long>(blockIdx.x) * blockDim.x + threadIdx.x) >> 5;
  const int lane = threadIdx.x & 31;
  if (i >= l) return;
  double acc = gather_dot_lanes(ridx, rval, x, rptr[i], rptr[i + 1], lane);
  acc = warp_sum(acc);
  if (lane == 0) t[i] = acc;
}

// implicit basis, one CTA: t = R x (warp per row of R), then s = K t
constexpr int kSmallThreads = 1024;
__global__ void __launch_bounds__(kSmallThreads)
pc_small_kernel(const int* __restrict__ rptr, const int* __restrict__ ridx, const double* __restrict__ rval,
                const double* __restrict__ KT, long long l, const double* __restrict__ x,
                double* __restrict__ t, double* __restrict__ s, const int* done) {
  extern __shared__ double tsh[];
  if (done && *done) return;
  const int w = threadIdx.x >> 5, lane = threadIdx.x & 31;
  constexpr int kW = kSmallThreads / 32;
  for (long long i = w; i < l; i += kW) {
    double acc = 0.0;
    for (int q = rptr[i] + lane; q < rptr[i + 1]; q += 32) acc += rval[q] * x[ridx[q]];
    acc = warp_sum(acc);
    if (lane == 0) tsh[i] = acc;
  }
  __syncthreads();
  for (long long i = w; i < l; i += kW) {
    const double* row = KT + i * l;
    double acc = 0.0;
    for (long long k = lane; k < l; k += 32) acc += row[k] * tsh[k];
    acc = warp_sum(acc);
    if (lane == 0) s[i] = acc;
  }
  if (t && threadIdx.x < l)
    for (long long i = threadIdx.x; i < l; i += kSmallThreads) t[i] = tsh[i];
}

// expand: o_j = x_j + (B s)_j (explicit) or x_j + (R^T s)_j (implicit), then
// mode 0: out[j] = o_j ; mode 1: v_j = o_j - beta v_j, ||v||^2 -> alpha (last block)
// mode 0 fusions (the iteration's z = P^{-1} v feeds them): xr[inv[j]] = z_j,
// the hot-relabelled copy of z for the forward (hot_permute_kernel); tail:
// u_t <- mu z - alpha u_t/beta with ||u_t||^2 (lsqr_tail_kernel)
struct ExpandFuse {
  double* xr;
  const int* inv;
  int tail;
};
__global__ void __launch_bounds__(kVecThreads)
pc_expand_kernel(LsqrPtrs P, int kind, const double* __restrict__ B, long long l,
                 const int* __restrict__ tptr, const int* __restrict__ tidx,
                 const double* __restrict__ tval, const double* __restrict__ s,
                 const double* __restrict__ x, double* __restrict__ out, int mode,
                 const int* done, ExpandFuse fz) {
  __shared__ double sh[32];
  // implicit basis: R^T rows longer than kExpandLong (the Zipf-head columns of
  // a sparse A appear in most selected rows) are summed by a whole warp
  // instead of one thread, so one column does not serialise the launch
  constexpr int kExpandLong = 32;
  __shared__ int defer[kVecThreads];
  __shared__ double dacc[kVecThreads];
  __shared__ int ndefer;
  if (done && *done) return;
  long long j = static_cast<long long>(blockIdx.x) * kVecThreads + threadIdx.x;
  const long long n = P.n;
  double beta = 0.0;
  if (mode == 1) beta = sqrt(P.g[n] + P.st->tail_norm2);
  double sq = 0.0;
  double acc = 0.0;
  bool deferred = false;
  if (kind != 1) {
    if (threadIdx.x == 0) ndefer = 0;
    __syncthreads();
    if (j < n) {
      const int q0 = tptr[j], q1 = tptr[j + 1];
      if (q1 - q0 > kExpandLong) {
        defer[atomicAdd(&ndefer, 1)] = threadIdx.x;
        deferred = true;
      } else {
        acc = gather_dot_seq(tidx, tval, s, q0, q1, acc);
      }
    }
    __syncthreads();
    const int lane = threadIdx.x & 31;
    for (int d = threadIdx.x >> 5; d < ndefer; d += kVecThreads / 32) {
      const long long jj = static_cast<long long>(blockIdx.x) * kVecThreads + defer[d];
      double a = gather_dot_lanes(tidx, tval, s, tptr[jj], tptr[jj + 1], lane);
      a = warp_sum(a);
      if (lane == 0) dacc[defer[d]] = a;
    }
    __syncthreads();
    if (deferred) acc = dacc[threadIdx.x];
  }
  if (j < n) {
    if (kind == 1) {
      for (long long t = 0; t < l; ++t) acc += B[t * n + j] * s[t];
    }
    const double o = x[j] + acc;
    if (mode == 0) {
      out[j] = o;
      if (fz.xr) fz.xr[fz.inv[j]] = o;
      if (fz.tail) {
        const double a0 = P.st->alpha, b0 = P.st->beta;
        double* ut = P.u + P.mloc;
        const double uo = ut[j];
        const double uh = b0 > 0.0 ? uo / b0 : uo;
        const double t = P.mu * o - a0 * uh;
        ut[j] = t;
        sq = t * t;
      }
    } else {
      const double t = o - beta * P.v[j];
      P.v[j] = t;
      sq = t * t;
    }
  }
  if (mode == 0) {
    if (!fz.tail) return;
    sq = block_sum<kVecThreads>(sq, sh);
    if (threadIdx.x == 0) P.tail_part[blockIdx.x] = sq;
    if (elect_last_block(P.ctr + 1, gridDim.x)) {
      const double ssum = ordered_sum<kVecThreads>(P.tail_part, gridDim.x, sh);
      if (threadIdx.x == 0) P.st->tail_norm2 = ssum;
    }
    return;
  }
  sq = block_sum<kVecThreads>(sq, sh);
  if (threadIdx.x == 0) P.epi_part[blockIdx.x] = sq;
  if (elect_last_block(P.ctr + 2, gridDim.x)) {
    double ssum = ordered_sum<kVecThreads>(P.epi_part, gridDim.x, sh);
    if (threadIdx.x == 0) finalize_alpha(P.st, P.trace, sqrt(ssum), beta);
  }
}

// ---------------------------------------------------------------------------
// The n-space part of one iteration in ONE cooperative launch (identity or
// implicit basis I + R^T G R).  After A^T u is complete it replaces
//   lsqr_epi -> pc_rproj -> pc_core -> pc_expand(mode 1) -> lsqr_update
//   -> [next iteration] pc_rproj -> pc_core -> pc_expand(mode 0, xr, mu-tail)
// (nine launches whose fixed costs dominated the ~100 us of n-space work per
// C5 iteration) by five grid barriers:
//   B  t = R h            h = (A^T u + mu u_t)/beta formed on the fly at R's columns
//   C  s = G_a t
//   D  v_raw = h + R^T s - beta v (own 256-column tiles; kept in h), ||v_raw||^2 per tile
//   E  alpha, rotation (every CTA, identical); v, y, w updates, ||y||^2 per tile;
//      t' = R v (v = v_raw/alpha at R's columns)
//   F  s' = G_f t'; stop tests (every CTA, identical); CTA 0 publishes the scalars
//   G  z = v + R^T s' for the NEXT iteration's forward (+ its hot-relabelled
//      copy, + the mu-tail rows u_t <- mu z - alpha u_t/beta, ||u_t||^2)
// Every per-element operation, every 256-column tile partial and every ordered
// sum over the tile partials is the unfused kernels' own, so the iterates are
// unchanged.  The scalar recurrence runs on a shared-memory copy of LsqrState in
// every CTA (all CTAs read the state before the first barrier; CTA 0 writes it
// back before the last one).
struct NspaceArgs {
  LsqrPtrs P;
  int kind;  // 0 identity, 2 implicit
  const int* rptr;
  const int* ridx;
  const double* rval;
  const int* tptr;
  const int* tidx;
  const double* tval;
  const double* Ga;  // P^{-T} middle operator (row-major l x l)
  const double* Gf;  // P^{-1}
  long long l;
  double* t;
  double* s;
  double* xr;  // hot-relabelled copy of z (nullptr: none)
  const int* inv;
  int fuse_tail;
  cudaGraphConditionalHandle cond;
  int use_cond;
  int noop;  // timing experiments only (APC_NSPACE_NOOP): skip the work
};
constexpr int kNsThreads = kVecThreads;  // 256-column tiles: the unfused kernels' blocks

// (R^T s)_j for column j = j0 + threadIdx.x: short R^T rows summed by the
// thread, rows longer than 32 entries (Zipf-head columns of a sparse A appear
// in most selected rows) by the whole warp -- pc_expand_kernel's split and sum
// orders, warp-synchronous (no block barrier)
__device__ __forceinline__ double ns_rts(const NspaceArgs& a, long long j0, long long n, const double* s) {
  constexpr int kExpandLong = 32;
  const long long j = j0 + threadIdx.x;
  const int lane = threadIdx.x & 31;
  int q0 = 0, q1 = 0;
  if (j < n) {
    q0 = a.tptr[j];
    q1 = a.tptr[j + 1];
  }
  const bool lng = q1 - q0 > kExpandLong;
  double acc = 0.0;
  if (!lng) acc = gather_dot_seq(a.tidx, a.tval, s, q0, q1, acc);
  unsigned m = __ballot_sync(0xffffffffu, lng);
  while (m) {
    const int L = __ffs(m) - 1;
    m &= m - 1;
    const int b0 = __shfl_sync(0xffffffffu, q0, L), b1 = __shfl_sync(0xffffffffu, q1, L);
    double x = gather_dot_lanes(a.tidx, a.tval, s, b0, b1, lane);
    x = warp_sum(x);
    if (lane == L) acc = x;
  }
  return acc;
}

// out = M x for row-major l x l M: warp per row over the grid (pc_core_kernel)
__device__ __forceinline__ void ns_core(const double* __restrict__ M, long long l, const double* t, double* out,
                                        long long gw, long long nw) {
  const int lane = threadIdx.x & 31;
  for (long long i = gw; i < l; i += nw) {
    double acc = row_dot_lanes(M + i * l, t, l, lane);
    acc = warp_sum(acc);
    if (lane == 0) out[i] = acc;
  }
}

// stage G for the tiles [tile0, ntiles) step tstep; the mu-tail norm by the last CTA
__device__ __forceinline__ void ns_stage_z(const NspaceArgs& a, double alpha, double beta, long long tile0,
                                           long long tstep, double* sh) {
  const LsqrPtrs& P = a.P;
  const long long n = P.n, ntiles = (n + kNsThreads - 1) / kNsThreads;
  const bool pre = a.kind == 2;
  for (long long tile = tile0; tile < ntiles; tile += tstep) {
    const long long j0 = tile * kNsThreads, j = j0 + threadIdx.x;
    const double acc = pre ? ns_rts(a, j0, n, a.s) : 0.0;
    double sq = 0.0;
    if (j < n) {
      const double vj = P.v[j];
      const double o = pre ? vj + acc : vj;
      if (pre) P.z[j] = o;
      if (a.xr) a.xr[a.inv[j]] = o;
      if (a.fuse_tail) {
        double* ut = P.u + P.mloc;
        const double uo = ut[j];
        const double uh = beta > 0.0 ? uo / beta : uo;
        const double t = P.mu * o - alpha * uh;
        ut[j] = t;
        sq = t * t;
      }
    }
    if (a.fuse_tail) {
      sq = block_sum<kNsThreads>(sq, sh);
      if (threadIdx.x == 0) P.tail_part[tile] = sq;
    }
  }
  if (a.fuse_tail && elect_last_block(P.ctr + 1, gridDim.x)) {
    const double ssum = ordered_sum<kNsThreads>(P.tail_part, ntiles, sh);
    if (threadIdx.x == 0) P.st->tail_norm2 = ssum;
  }
}

__global__ void __launch_bounds__(kNsThreads, 4) lsqr_nspace_kernel(NspaceArgs a) {
  namespace cg = cooperative_groups;
  cg::grid_group grid = cg::this_grid();
  __shared__ double sh[32];
  __shared__ LsqrState ls;
  const LsqrPtrs& P = a.P;
  if (threadIdx.x == 0) ls = *P.st;
  __syncthreads();
  if (a.noop) {  // count iterations only, stop at the cap
    if (blockIdx.x == 0 && threadIdx.x == 0) {
      const long long j = ++P.st->iter;
      if (j >= ls.cap) P.st->done = 1;
      if (a.use_cond) cudaGraphSetConditional(a.cond, j >= ls.cap ? 0u : 1u);
    }
    return;
  }
  if (ls.done) {
    if (a.use_cond && blockIdx.x == 0 && threadIdx.x == 0) cudaGraphSetConditional(a.cond, 0);
    return;
  }
  const long long n = P.n, l = a.l, ntiles = (n + kNsThreads - 1) / kNsThreads;
  const int lane = threadIdx.x & 31;
  const long long gw = static_cast<long long>(blockIdx.x) * (kNsThreads / 32) + (threadIdx.x >> 5);
  const long long nw = static_cast<long long>(gridDim.x) * (kNsThreads / 32);
  const bool pre = a.kind == 2;
  const double beta = sqrt(P.g[n] + ls.tail_norm2);
  auto hval = [&](long long c) {  // lsqr_epi_kernel's h_c
    double raw = P.g[c];
    if (P.has_tail) raw += P.mu * P.u[P.mloc + c];
    return beta > 0.0 ? raw / beta : raw;
  };
  if (pre) {  // B, C: s = G_a (R h)
    for (long long r = gw; r < l; r += nw) {
      double acc = 0.0;
      for (int q = a.rptr[r] + lane; q < a.rptr[r + 1]; q += 32) acc += a.rval[q] * hval(a.ridx[q]);
      acc = warp_sum(acc);
      if (lane == 0) a.t[r] = acc;
    }
    grid.sync();
    ns_core(a.Ga, l, a.t, a.s, gw, nw);
    grid.sync();
  }
  // D: v_raw (into h), ||v_raw||^2 per tile
  for (long long tile = blockIdx.x; tile < ntiles; tile += gridDim.x) {
    const long long j0 = tile * kNsThreads, j = j0 + threadIdx.x;
    const double acc = pre ? ns_rts(a, j0, n, a.s) : 0.0;
    double sq = 0.0;
    if (j < n) {
      const double h = hval(j);
      const double o = pre ? h + acc : h;
      const double t = o - beta * P.v[j];
      P.h[j] = t;
      sq = t * t;
    }
    sq = block_sum<kNsThreads>(sq, sh);
    if (threadIdx.x == 0) P.epi_part[tile] = sq;
  }
  grid.sync();
  // E: alpha and the rotation in every CTA; v, y, w; t' = R v
  {
    const double ssum = ordered_sum<kNsThreads>(P.epi_part, ntiles, sh);
    if (threadIdx.x == 0) finalize_alpha(&ls, blockIdx.x == 0 ? P.trace : nullptr, sqrt(ssum), beta);
    __syncthreads();
  }
  const double alpha = ls.alpha, t1 = ls.t1, t2 = ls.t2;
  for (long long tile = blockIdx.x; tile < ntiles; tile += gridDim.x) {
    const long long j = tile * kNsThreads + threadIdx.x;
    double sq = 0.0;
    if (j < n) {
      const double vo = P.h[j];
      const double vh = alpha > 0.0 ? vo / alpha : vo;
      P.v[j] = vh;
      const double wo = P.w[j];
      const double yn = P.y[j] + t1 * wo;
      P.y[j] = yn;
      P.w[j] = vh + t2 * wo;
      sq = yn * yn;
    }
    sq = block_sum<kNsThreads>(sq, sh);
    if (threadIdx.x == 0) P.upd_part[tile] = sq;
  }
  if (pre) {
    for (long long r = gw; r < l; r += nw) {
      double acc = 0.0;
      for (int q = a.rptr[r] + lane; q < a.rptr[r + 1]; q += 32) {
        const double vo = P.h[a.ridx[q]];
        acc += a.rval[q] * (alpha > 0.0 ? vo / alpha : vo);
      }
      acc = warp_sum(acc);
      if (lane == 0) a.t[r] = acc;
    }
  }
  grid.sync();
  // F: s' = G_f t'; stop tests; CTA 0 publishes the scalars
  if (pre) ns_core(a.Gf, l, a.t, a.s, gw, nw);
  {
    const double ysum = ordered_sum<kNsThreads>(P.upd_part, ntiles, sh);
    if (threadIdx.x == 0) stop_tests(&ls, sqrt(ysum));
    __syncthreads();
  }
  if (blockIdx.x == 0 && threadIdx.x == 0) {
    *P.st = ls;
    if (a.use_cond) cudaGraphSetConditional(a.cond, ls.done ? 0u : 1u);
  }
  if (ls.done) return;  // identical in every CTA: nobody waits at the barrier below
  grid.sync();
  // G: the next iteration's z
  ns_stage_z(a, ls.alpha, ls.beta, blockIdx.x, gridDim.x, sh);
}

// stage G alone (before the first loop iteration): one CTA per tile
__global__ void __launch_bounds__(kNsThreads) lsqr_nspace_z_kernel(NspaceArgs a) {
  __shared__ double sh[32];
  const LsqrState* st = a.P.st;
  if (st->done) return;
  ns_stage_z(a, st->alpha, st->beta, blockIdx.x, gridDim.x, sh);
}

namespace {
__global__ void zero_kernel(double* p, long long n) {
  long long i = static_cast<long long>(blockIdx.x) * blockDim.x + threadIdx.x;
  if (i < n) p[i] = 0.0;
}
__global__ void stamp_t0_kernel(LsqrState* st) { st->t0_ns = globaltimer_ns(); }
inline unsigned nb(long long n, int t = kVecThreads) {
  return static_cast<unsigned>(std::max<long long>(1, (n + t - 1) / t));
}
}  // namespace

// ---------------------------------------------------------------------------
// workspace
// ---------------------------------------------------------------------------
struct LsqrWork {
  apc_ctx* ctx = nullptr;
  long long mloc = 0, n = 0, ulen = 0;
  double mu = 0.0;
  DBuf<double> u, v, w, z, g, h, t, s, fwd_part, tail_part, epi_part, upd_part, pc_part, pers_part, pcf_part;
  DBuf<unsigned> ctr, pc_ctr, pcf_ctr;
  DBuf<LsqrState> st;
  DBuf<TraceRow> trace;
  DBuf<double> xs, samp_part, samp_tpart, samp_sc, sampled, samp_xr;  // true-residual sampling
  LsqrState* hst = nullptr;  // pinned
  cudaEvent_t ev[2] = {nullptr, nullptr};
  cudaEvent_t tev[2] = {nullptr, nullptr};  // timing of the iteration loop
};

LsqrWork* lsqr_work_create(apc_mat& a, double mu) {
  auto* w = new LsqrWork();
  w->ctx = a.ctx;
  w->mloc = a.mloc();
  w->n = a.n;
  w->mu = mu;
  w->ulen = a.mloc() + (mu > 0.0 ? a.n : 0);
  const long long n = a.n;
  w->u.alloc(std::max<long long>(1, w->ulen));
  w->v.alloc(std::max<long long>(1, n));
  w->w.alloc(std::max<long long>(1, n));
  w->z.alloc(std::max<long long>(1, n));
  w->g.alloc(n + 1);
  w->h.alloc(std::max<long long>(1, n));
  const long long ntiles = std::max<long long>(fwd_num_tiles(a), nb(w->mloc));
  w->fwd_part.alloc(std::max<long long>(1, ntiles));
  w->tail_part.alloc(nb(n));
  w->epi_part.alloc(nb(n));
  w->upd_part.alloc(nb(n));
  w->ctr.alloc(8);
  APC_CUDA(cudaMemsetAsync(w->ctr.p, 0, w->ctr.bytes(), a.ctx->stream));
  w->st.alloc(1);
  w->hst = static_cast<LsqrState*>(ctx_pinned(a.ctx, 2, sizeof(LsqrState) * 2));
  APC_CUDA(cudaEventCreateWithFlags(&w->ev[0], cudaEventDisableTiming));
  APC_CUDA(cudaEventCreateWithFlags(&w->ev[1], cudaEventDisableTiming));
  APC_CUDA(cudaEventCreate(&w->tev[0]));
  APC_CUDA(cudaEventCreate(&w->tev[1]));
  // operator scratch sized up front (no allocation during graph capture)
  if (!a.sparse) {
    DenseFwdPlan fp = dense_fwd_plan(a);
    DenseAdjPlan ap = dense_adj_plan(a);
    ctx_scratch(a.ctx, std::max(fp.nsplit * a.mloc(), ap.msplit * a.n));
    ctx_counters(a.ctx, std::max(fp.ntiles, ap.ngroups));
  }
  return w;
}

void lsqr_work_destroy(LsqrWork* w) {
  if (!w) return;
  for (auto& e : w->ev)
    if (e) cudaEventDestroy(e);
  for (auto& e : w->tev)
    if (e) cudaEventDestroy(e);
  delete w;
}

// ---------------------------------------------------------------------------
// preconditioner application pieces (enqueue on the ctx stream)
// ---------------------------------------------------------------------------
namespace {

// s = K (B^T x)  (explicit)  or  s = G (R x)  (implicit, one fused CTA)
void pc_project_core(LsqrWork* w, PrecondDev& p, const double* x, bool transpose, const int* done) {
  apc_ctx* ctx = w->ctx;
  const double* KT = transpose ? p.Ka.p : p.Kf.p;
  if (p.kind == 1) {
    DenseAdjPlan pl = dense_adj_plan(p.n, p.l, ctx->num_sms);
    launch_dense_adj(ctx, p.B.p, p.n, p.l, x, w->t.p, done, pl.msplit > 1 ? w->pc_part.p : nullptr,
                     pl.msplit > 1 ? w->pc_ctr.p : nullptr);
    pc_core_kernel<<<nb(p.l * 32), kVecThreads, 0, ctx->stream>>>(KT, p.l, w->t.p, w->s.p, done);
    ctx->launches++;
  } else {
    // two wide launches beat one latency-bound CTA (pc_small_kernel) by ~3x
    pc_rproj_kernel<<<nb(p.l * 32, 128), 128, 0, ctx->stream>>>(p.R.ptr.p, p.R.idx.p, p.R.val.p, p.l, x,
                                                                w->t.p, done);
    pc_core_kernel<<<nb(p.l * 32, 128), 128, 0, ctx->stream>>>(KT, p.l, w->t.p, w->s.p, done);
    ctx->launches += 2;
  }
}

// returns true when the fusions asked for were applied (xr only on the
// implicit-basis kernel; the mu-tail on both)
bool pc_expand(LsqrWork* w, const LsqrPtrs& P, PrecondDev& p, const double* x, double* out,
               int mode, const int* done, ExpandFuse fz = ExpandFuse{nullptr, nullptr, 0}) {
  if (p.kind == 1 && !std::getenv("APC_PC_EXPAND_ROWS")) {
    if (fz.xr) return false;
    const DenseFwdPlan pl = dense_fwd_plan(p.n, p.l, w->ctx->num_sms);
    dim3 grid(static_cast<unsigned>(pl.ntiles), static_cast<unsigned>(pl.nsplit));
    const PcExpandEpi epi{P, x, out, mode, 0.0, fz.tail, 0.0};
    dense_fwd_kernel<PcExpandEpi><<<grid, kDenseFwdThreads, 0, w->ctx->stream>>>(
        p.B.p, p.n, p.n, p.l, w->s.p, pl.cols_per_split, pl.nsplit > 1 ? w->pcf_part.p : nullptr,
        pl.nsplit > 1 ? w->pcf_ctr.p : nullptr, done, epi);
    w->ctx->launches++;
    if (pl.nsplit > 1) {
      dense_split_epi_kernel<PcExpandEpi><<<static_cast<unsigned>((p.n + 255) / 256), 256, 0, w->ctx->stream>>>(
          w->pcf_part.p, static_cast<int>(pl.nsplit), p.n, done, epi);
      w->ctx->launches++;
    }
    return true;
  }
  pc_expand_kernel<<<nb(w->n), kVecThreads, 0, w->ctx->stream>>>(
      P, p.kind, p.B.p, p.l, p.RT.ptr.p, p.RT.idx.p, p.RT.val.p, w->s.p, x, out, mode, done, fz);
  w->ctx->launches++;
  return true;
}

void ensure_pc_buffers(LsqrWork* w, PrecondDev& p) {
  w->t.ensure(std::max<long long>(1, p.l));
  w->s.ensure(std::max<long long>(1, p.l));
  if (p.kind == 1) {
    DenseAdjPlan pl = dense_adj_plan(p.n, p.l, w->ctx->num_sms);
    w->pc_part.ensure(std::max<long long>(1, pl.msplit * p.l));
    if (w->pc_ctr.n < pl.ngroups) {
      w->pc_ctr.alloc(pl.ngroups);
      APC_CUDA(cudaMemsetAsync(w->pc_ctr.p, 0, w->pc_ctr.bytes(), w->ctx->stream));
    }
    const DenseFwdPlan fp = dense_fwd_plan(p.n, p.l, w->ctx->num_sms);
    w->pcf_part.ensure(std::max<long long>(1, fp.nsplit * p.n));
    if (w->pcf_ctr.n < fp.ntiles) {
      w->pcf_ctr.alloc(fp.ntiles);
      APC_CUDA(cudaMemsetAsync(w->pcf_ctr.p, 0, w->pcf_ctr.bytes(), w->ctx->stream));
    }
  }
}

// the fused n-space path (lsqr_nspace_kernel): identity or implicit basis;
// APC_NSPACE=0 keeps the unfused kernels
bool nspace_enabled(const LsqrWork* w, const PrecondDev* p) {
  static const bool env = std::getenv("APC_NSPACE") && std::atoi(std::getenv("APC_NSPACE")) != 0;
  return env && w->n > 0 && (!p || p->kind == 0 || p->kind == 2);
}

NspaceArgs nspace_args(LsqrWork* w, apc_mat& a, PrecondDev* p, const LsqrPtrs& P, cudaGraphConditionalHandle cond,
                       int use_cond) {
  NspaceArgs na{};
  na.P = P;
  na.kind = p && p->kind == 2 ? 2 : 0;
  if (na.kind == 2) {
    na.rptr = p->R.ptr.p;
    na.ridx = p->R.idx.p;
    na.rval = p->R.val.p;
    na.tptr = p->RT.ptr.p;
    na.tidx = p->RT.idx.p;
    na.tval = p->RT.val.p;
    na.Ga = p->Ka.p;
    na.Gf = p->Kf.p;
    na.l = p->l;
  }
  na.t = w->t.p;
  na.s = w->s.p;
  const bool xr = w->mloc > 0 && fwd_takes_permuted(a);
  na.xr = xr ? a.hot.xr.p : nullptr;
  na.inv = xr ? a.hot.inv.p : nullptr;
  na.fuse_tail = P.has_tail;
  na.cond = cond;
  na.use_cond = use_cond;
  na.noop = std::getenv("APC_NSPACE_NOOP") ? 1 : 0;
  return na;
}

int nspace_grid(apc_ctx* ctx, long long n) {
  static int per_sm = -1;
  if (per_sm < 0) {
    int occ = 0;
    APC_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, lsqr_nspace_kernel, kNsThreads, 0));
    const char* e = std::getenv("APC_NSPACE_CTAS_PER_SM");
    per_sm = std::max(1, std::min(occ, e ? std::atoi(e) : 4));
  }
  const long long ntiles = (n + kNsThreads - 1) / kNsThreads;
  return static_cast<int>(std::max<long long>(1, std::min<long long>(ntiles, static_cast<long long>(per_sm) * ctx->num_sms)));
}

// the z of the first loop iteration (stage G of lsqr_nspace_kernel)
void enqueue_nspace_z(LsqrWork* w, apc_mat& a, PrecondDev* p, const LsqrPtrs& P) {
  apc_ctx* ctx = w->ctx;
  if (p && p->kind == 2) pc_project_core(w, *p, P.v, false, &P.st->done);
  NspaceArgs na = nspace_args(w, a, p, P, cudaGraphConditionalHandle{}, 0);
  lsqr_nspace_z_kernel<<<nb(w->n), kNsThreads, 0, ctx->stream>>>(na);
  ctx->launches++;
}

// one iteration on the fused n-space path: fwd, adj, [allreduce], n-space
void enqueue_iteration_nspace(LsqrWork* w, apc_mat& a, PrecondDev* p, const LsqrPtrs& P,
                              cudaGraphConditionalHandle cond, int use_cond) {
  apc_ctx* ctx = w->ctx;
  cudaStream_t st = ctx->stream;
  const int* done = &P.st->done;
  NspaceArgs na = nspace_args(w, a, p, P, cond, use_cond);
  const double* z = na.kind == 2 ? P.z : P.v;
  LsqrFwdEpi epi{P.u, P.st, P.fwd_part, P.ctr + 0, P.g + P.n, 0.0, 0.0};
  if (w->mloc > 0) {
    launch_fwd(a, z, done, epi, st, na.xr != nullptr);
  } else {
    lsqr_init_copy_kernel<<<1, kVecThreads, 0, st>>>(P, P.u, 0, 0, 0);
    ctx->launches++;
  }
  op_adj_raw(a, P.u, P.g, done);
  comm_allreduce(ctx, P.g, w->n + 1);
  void* args[] = {&na};
  APC_CUDA(cudaLaunchCooperativeKernel(reinterpret_cast<const void*>(lsqr_nspace_kernel),
                                       dim3(nspace_grid(ctx, w->n)), dim3(kNsThreads), args, 0, st));
  ctx->launches++;
}

// one LSQR iteration (all kernels no-op once st->done is raised)
void enqueue_iteration(LsqrWork* w, apc_mat& a, PrecondDev* p, const LsqrPtrs& P,
                       cudaGraphConditionalHandle cond, int use_cond) {
  if (nspace_enabled(w, p)) {
    enqueue_iteration_nspace(w, a, p, P, cond, use_cond);
    return;
  }
  apc_ctx* ctx = w->ctx;
  cudaStream_t st = ctx->stream;
  const int* done = &P.st->done;
  const bool pre = p && p->kind != 0;
  const double* z = P.v;
  // kernel fusions of the preconditioned single-rank iteration (APC_FUSE=0 turns them off)
  static const bool fuse_env = !std::getenv("APC_FUSE") || std::atoi(std::getenv("APC_FUSE")) != 0;
  bool tail_fused = false, x_permuted = false;
  if (pre) {  // z = P^{-1} v (+ its hot-relabelled copy, + the mu-tail rows of u)
    pc_project_core(w, *p, P.v, false, done);
    const bool want_xr = fuse_env && w->mloc > 0 && fwd_takes_permuted(a);
    const bool want_tail = fuse_env && P.has_tail;
    ExpandFuse fz{want_xr ? a.hot.xr.p : nullptr, want_xr ? a.hot.inv.p : nullptr, want_tail ? 1 : 0};
    if (pc_expand(w, P, *p, P.v, P.z, 0, done, fz)) {
      x_permuted = want_xr;
      tail_fused = want_tail;
    } else {
      pc_expand(w, P, *p, P.v, P.z, 0, done, ExpandFuse{nullptr, nullptr, want_tail ? 1 : 0});
      tail_fused = want_tail;
    }
    z = P.z;
  }
  LsqrFwdEpi epi{P.u, P.st, P.fwd_part, P.ctr + 0, P.g + P.n, 0.0, 0.0};
  // dense A of 64 MB or more: u, ||u||^2 and A^T u in one kernel that reads A once
  const bool pair_fused = w->mloc > 0 && !a.sparse && dense_pair_ready(a);
  if (pair_fused) {
    launch_dense_pair(a, z, P.u, P.st, P.g, done);
  } else if (w->mloc > 0) {
    launch_fwd(a, z, done, epi, st, x_permuted);
  } else {
    // empty shard: publish ||u_top||^2 = 0 through the init-copy path
    lsqr_init_copy_kernel<<<1, kVecThreads, 0, st>>>(P, P.u, 0, 0, 0);
    ctx->launches++;
  }
  if (P.has_tail && !tail_fused) {
    LsqrPtrs Pz = P;
    Pz.z = const_cast<double*>(z);
    lsqr_tail_kernel<<<nb(w->n), kVecThreads, 0, st>>>(Pz);
    ctx->launches++;
  }
  // A^T u with the epilogue h = (A^T u + mu u_t)/beta where the columns are
  // finalised (one rank: no allreduce between them): the tail scatter and the
  // head combine apply it and the separate lsqr_epi_kernel pass over n goes
  // away (same operations per column: same bits).  Opt-in (APC_FUSE_EPI=1):
  // on C5 the random u_t gather and the division in the scatter cost what the
  // coalesced pass did (791 vs 787 us per iteration, profiles/r2e_dense_pair.md)
  const bool epi_env = std::getenv("APC_FUSE_EPI") && std::atoi(std::getenv("APC_FUSE_EPI")) != 0;  // per enqueue: the tests toggle it
  const bool epi_fused =
      fuse_env && epi_env && pre && ctx->nranks == 1 && w->mloc > 0 &&
      op_adj_epi(a, P.u, P.h, done,
                 AdjEpi{P.has_tail ? P.u + P.mloc : nullptr, P.mu, P.g + P.n, P.has_tail ? &P.st->tail_norm2 : nullptr});
  if (!epi_fused) {
    if (!pair_fused) op_adj_raw(a, P.u, P.g, done);
    comm_allreduce(ctx, P.g, w->n + 1);
    lsqr_epi_kernel<<<nb(w->n), kVecThreads, 0, st>>>(P, pre ? 1 : 0);
    ctx->launches++;
  }
  if (pre) {  // v = P^{-T} h - beta v ; alpha ; rotation
    pc_project_core(w, *p, P.h, true, done);
    pc_expand(w, P, *p, P.h, nullptr, 1, done);
  }
  lsqr_update_kernel<<<nb(w->n), kVecThreads, 0, st>>>(P, cond, use_cond);
  ctx->launches++;
}

// the observer's sample after iteration j (no-ops unless the gate opens)
void enqueue_sample(LsqrWork* w, apc_mat& a, PrecondDev* p, const LsqrPtrs& P, const SampleCfg& sc,
                    long long cap) {
  apc_ctx* ctx = w->ctx;
  cudaStream_t st = ctx->stream;
  const long long n = w->n;
  samp_gate_kernel<<<1, 1, 0, st>>>(P.st, sc.stride);
  ctx->launches++;
  const int* skip = &P.st->samp_skip;
  const double* xs = P.y;
  if (p && p->kind != 0) {  // P^{-1} y
    pc_project_core(w, *p, P.y, false, skip);
    pc_expand(w, P, *p, P.y, w->xs.p, 0, skip);
    xs = w->xs.p;
  }
  if (sc.x_base || P.has_tail) {  // + x ; ||mu xs||^2
    double* out = sc.x_base ? w->xs.p : const_cast<double*>(xs);
    samp_combine_kernel<<<nb(n), kVecThreads, 0, st>>>(P.st, xs, sc.x_base, out, n, P.has_tail ? P.mu : 0.0,
                                                       w->samp_tpart.p, P.ctr + 5, w->samp_sc.p);
    ctx->launches++;
    xs = out;
  }
  if (w->mloc > 0) {
    double* xr_buf = fwd_takes_permuted(a) ? w->samp_xr.p : nullptr;  // sized in lsqr_phase
    launch_fwd(a, xs, skip, ResidSampleEpi{sc.b_local, w->samp_part.p, P.ctr + 4, w->samp_sc.p}, st, false, xr_buf);
  } else {
    samp_zero_kernel<<<1, 1, 0, st>>>(P.st, w->samp_sc.p);
    ctx->launches++;
  }
  comm_allreduce(ctx, w->samp_sc.p, 1);
  samp_final_kernel<<<1, 1, 0, st>>>(P.st, w->samp_sc.p, sc.bnorm, P.has_tail, w->sampled.p, cap);
  ctx->launches++;
}

}  // namespace

void precond_apply(apc_ctx* ctx, PrecondDev& p, bool transpose, const double* x, double* out) {
  if (p.kind == 0) {
    APC_CUDA(cudaMemcpyAsync(out, x, sizeof(double) * p.n, cudaMemcpyDeviceToDevice, ctx->stream));
    return;
  }
  LsqrWork tmp;
  tmp.ctx = ctx;
  tmp.n = p.n;
  ensure_pc_buffers(&tmp, p);
  LsqrPtrs P{};
  P.n = p.n;
  pc_project_core(&tmp, p, x, transpose, nullptr);
  pc_expand(&tmp, P, p, x, out, 0, nullptr);
  APC_CUDA(cudaStreamSynchronize(ctx->stream));
  APC_CUDA(cudaGetLastError());
}

// ---------------------------------------------------------------------------
// one phase
// ---------------------------------------------------------------------------
void lsqr_phase(LsqrWork* w, apc_mat& a, double mu, const PrecondDev* pc, const double* rhs_d,
                const StopCfg& stop, int phase, double* y_d, PhaseOut& out, const SampleCfg* samp) {
  (void)phase;
  apc_ctx* ctx = w->ctx;
  cudaStream_t st = ctx->stream;
  PrecondDev* p = const_cast<PrecondDev*>(pc);
  const long long n = w->n;
  require(mu == w->mu, APC_INVALID_ARGUMENT, "lsqr_phase: workspace built for another mu");
  if (p && p->kind != 0) ensure_pc_buffers(w, *p);
  // the panel copy of a large dense A is built here, outside any graph capture
  if (!a.sparse && w->mloc > 0) dense_pair_ready(a);
  const long long cap = stop.max_iters > 0 ? stop.max_iters : 4 * n;
  w->trace.ensure(cap + 1);
  const bool sampling = samp && samp->stride > 0;
  if (sampling) {
    w->xs.ensure(std::max<long long>(1, n));
    w->samp_part.ensure(w->fwd_part.n);
    w->samp_tpart.ensure(nb(n));
    w->samp_sc.ensure(2);
    w->sampled.ensure(cap + 1);
    if (fwd_takes_permuted(a)) w->samp_xr.ensure(std::max<long long>(1, n));
    APC_CUDA(cudaMemsetAsync(w->sampled.p, 0xFF, sizeof(double) * (cap + 1), st));  // NaN
  }

  LsqrState h{};
  h.eps = stop.eps_lsqr;
  h.nu = stop.nu_lsqr;
  h.sigma_floor = stop.sigma_floor;
  h.iter = -1;  // initialisation pending
  h.cap = cap;
  h.trace_cap = cap + 1;
  h.reason = kReasonNone;
  std::memcpy(&w->hst[0], &h, sizeof(h));
  APC_CUDA(cudaMemcpyAsync(w->st.p, &w->hst[0], sizeof(LsqrState), cudaMemcpyHostToDevice, st));

  LsqrPtrs P{};
  P.st = w->st.p;
  P.trace = w->trace.p;
  P.u = w->u.p;
  P.v = w->v.p;
  P.w = w->w.p;
  P.y = y_d;
  P.z = w->z.p;
  P.g = w->g.p;
  P.h = w->h.p;
  P.fwd_part = w->fwd_part.p;
  P.tail_part = w->tail_part.p;
  P.epi_part = w->epi_part.p;
  P.upd_part = w->upd_part.p;
  P.ctr = w->ctr.p;
  P.mloc = w->mloc;
  P.n = n;
  P.mu = mu;
  P.has_tail = mu > 0.0 ? 1 : 0;

  auto t_start = std::chrono::steady_clock::now();
  // ---- initialisation: u = rhs, beta, v = P^{-T} A^T u / beta, alpha, w = v
  stamp_t0_kernel<<<1, 1, 0, st>>>(w->st.p);
  zero_kernel<<<nb(n), kVecThreads, 0, st>>>(w->v.p, n);
  zero_kernel<<<nb(n), kVecThreads, 0, st>>>(w->w.p, n);
  zero_kernel<<<nb(n), kVecThreads, 0, st>>>(y_d, n);
  ctx->launches += 4;
  lsqr_init_copy_kernel<<<nb(w->mloc), kVecThreads, 0, st>>>(P, rhs_d, w->mloc, 0, 0);
  ctx->launches++;
  if (P.has_tail) {
    lsqr_init_copy_kernel<<<nb(n), kVecThreads, 0, st>>>(P, rhs_d, n, w->mloc, 1);
    ctx->launches++;
  }
  const int* done = &w->st.p->done;
  const bool pre = p && p->kind != 0;
  op_adj_raw(a, P.u, P.g, done);
  comm_allreduce(ctx, P.g, n + 1);
  lsqr_epi_kernel<<<nb(n), kVecThreads, 0, st>>>(P, pre ? 1 : 0);
  ctx->launches++;
  if (pre) {
    pc_project_core(w, *p, P.h, true, done);
    pc_expand(w, P, *p, P.h, nullptr, 1, done);
  }
  lsqr_update_kernel<<<nb(n), kVecThreads, 0, st>>>(P, cudaGraphConditionalHandle{}, 0);
  ctx->launches++;
  APC_CUDA(cudaGetLastError());

  // ---- iterations: graph with a conditional WHILE node (single rank), or
  // batches of captured iterations polled from the host (multi-rank: the
  // NCCL call stays outside conditional bodies)
  // APC_LSQR_MODE: "while" (default, 1 rank) | "batch" (graph of 8 iterations,
  // host-polled; used for multi-rank) | "eager" (no graph; for kernel profiling)
  const char* mode_env = std::getenv("APC_LSQR_MODE");
  const std::string mode = mode_env ? mode_env : "";
  const bool eager = mode == "eager" || !comm_graph_safe(ctx);
  const bool persistent =
      !sampling && (mode.empty() || mode == "persistent") && persistent_eligible(a, p, ctx);
  const bool use_while = !persistent && ctx->nranks == 1 && mode != "batch" && !eager;
  if (!persistent && nspace_enabled(w, p)) enqueue_nspace_z(w, a, p, P);
  cudaGraph_t graph = nullptr;
  cudaGraphExec_t exec = nullptr;
  const std::uint64_t launches_before_capture = ctx->launches;
  std::uint64_t per_iter = 0;
  APC_CUDA(cudaEventRecord(w->tev[0], st));
  if (persistent) {
    // one cooperative launch runs every iteration (L2-resident sparse systems)
    if (p && p->kind == 2) {
      w->s.ensure(std::max<long long>(1, p->l));
      w->t.ensure(std::max<long long>(1, p->l));
    }
    w->pers_part.ensure(4LL * persistent_max_grid(ctx));
    const char* bps = std::getenv("APC_PERSISTENT_BLOCKS_PER_SM");
    const bool prof = std::getenv("APC_PERSISTENT_PROF") != nullptr;
    DBuf<unsigned long long> d_prof(prof ? 64 * 16 + 16LL * persistent_max_grid(ctx) : 0);
    if (prof) APC_CUDA(cudaMemsetAsync(d_prof.p, 0, d_prof.bytes(), st));
    PersistentBuffers pb{w->u.p, w->v.p, w->g.p, w->w.p, y_d, w->z.p, w->h.p, w->s.p, w->t.p, w->pers_part.p,
                         w->st.p, w->trace.p, bps ? std::atoi(bps) : 0, prof ? d_prof.p : nullptr};
    lsqr_persistent_run(a, mu, p, pb);
    per_iter = 0;
    if (prof) {
      std::vector<unsigned long long> h(static_cast<size_t>(d_prof.n));
      copy_sync(st, h.data(), d_prof.p, sizeof(unsigned long long) * h.size(), cudaMemcpyDeviceToHost);
      // 16 stamps per iteration (lsqr_persistent.cu STAMP(k)); interval k runs
      // from stamp k to the next recorded one
      static const char* names[16] = {"S12proj", "S12z", "B1", "zcopy", "-", "S3loop", "S3red", "B2",
                                      "beta+stop", "S4loop", "B3", "S56proj", "S56v", "B4", "S7", "-"};
      double acc[16] = {0};
      int cnt = 0;
      for (int it = 2; it < 63; ++it) {
        if (h[(it + 1) * 16] == 0) break;
        for (int k = 0; k < 16; ++k) {
          const unsigned long long a0 = h[it * 16 + k];
          if (!a0) continue;
          unsigned long long a1 = 0;
          for (int q = k + 1; q < 16 && !a1; ++q) a1 = h[it * 16 + q];
          if (!a1) a1 = h[(it + 1) * 16];
          acc[k] += (a1 - a0) * 1e-3;
        }
        ++cnt;
      }
      if (cnt) {
        std::fprintf(stderr, "persistent stage us/iter (%d its):", cnt);
        double tot = 0.0;
        for (int k = 0; k < 16; ++k)
          if (acc[k] > 0.0) {
            std::fprintf(stderr, " %s %.2f", names[k], acc[k] / cnt);
            tot += acc[k] / cnt;
          }
        std::fprintf(stderr, " | total %.2f\n", tot);
        // per-CTA interval sums (iterations 2..63): min / median / max over CTAs
        std::fprintf(stderr, "per-CTA us/iter min/med/max:");
        for (int k = 1; k < 16; ++k) {
          std::vector<double> v;
          for (int b = 0; b < persistent_max_grid(ctx); ++b) {
            const unsigned long long x = h[64 * 16 + b * 16 + k];
            if (x) v.push_back(x * 1e-3 / 62.0);
          }
          if (v.empty()) continue;
          std::sort(v.begin(), v.end());
          std::fprintf(stderr, " [%s %.1f/%.1f/%.1f]", names[k - 1], v.front(), v[v.size() / 2], v.back());
        }
        std::fprintf(stderr, "\n");
      }
    }
  } else if (use_while) {
    APC_CUDA(cudaGraphCreate(&graph, 0));
    cudaGraphConditionalHandle cond;
    APC_CUDA(cudaGraphConditionalHandleCreate(&cond, graph, 1, cudaGraphCondAssignDefault));
    cudaGraphNodeParams cp{};
    cp.type = cudaGraphNodeTypeConditional;
    cp.conditional.handle = cond;
    cp.conditional.type = cudaGraphCondTypeWhile;
    cp.conditional.size = 1;
    cudaGraphNode_t node;
    APC_CUDA(cudaGraphAddNode(&node, graph, nullptr, 0, &cp));
    cudaGraph_t body = cp.conditional.phGraph_out[0];
    APC_CUDA(cudaStreamBeginCaptureToGraph(st, body, nullptr, nullptr, 0,
                                           cudaStreamCaptureModeThreadLocal));
    // APC_WHILE_UNROLL iterations per pass of the body (kernels after the stop
    // exit on `done`): fewer body relaunches per iteration
    static const int unroll = std::max(1, std::getenv("APC_WHILE_UNROLL") ? std::atoi(std::getenv("APC_WHILE_UNROLL")) : 1);
    for (int k = 0; k < unroll; ++k) {
      enqueue_iteration(w, a, p, P, cond, 1);
      if (sampling) enqueue_sample(w, a, p, P, *samp, cap + 1);
    }
    per_iter = (ctx->launches - launches_before_capture) / unroll;
    APC_CUDA(cudaStreamEndCapture(st, &body));
    APC_CUDA(cudaGraphInstantiate(&exec, graph, 0));
    // skip the loop entirely if initialisation already stopped
    APC_CUDA(cudaMemcpyAsync(&w->hst[1], w->st.p, sizeof(LsqrState), cudaMemcpyDeviceToHost, st));
    APC_CUDA(cudaStreamSynchronize(st));
    if (!w->hst[1].done) APC_CUDA(cudaGraphLaunch(exec, st));
  } else if (eager) {
    for (;;) {
      for (int k = 0; k < 8; ++k) {
        enqueue_iteration(w, a, p, P, cudaGraphConditionalHandle{}, 0);
        if (sampling) enqueue_sample(w, a, p, P, *samp, cap + 1);
      }
      APC_CUDA(cudaMemcpyAsync(&w->hst[1], w->st.p, sizeof(LsqrState), cudaMemcpyDeviceToHost, st));
      APC_CUDA(cudaStreamSynchronize(st));
      if (w->hst[1].done) break;
    }
    per_iter = 0;  // eager launches were counted as issued
  } else {
    constexpr int kBatch = 8;
    APC_CUDA(cudaStreamBeginCapture(st, cudaStreamCaptureModeThreadLocal));
    for (int k = 0; k < kBatch; ++k) {
      enqueue_iteration(w, a, p, P, cudaGraphConditionalHandle{}, 0);
      if (sampling) enqueue_sample(w, a, p, P, *samp, cap + 1);
    }
    per_iter = (ctx->launches - launches_before_capture) / kBatch;
    APC_CUDA(cudaStreamEndCapture(st, &graph));
    APC_CUDA(cudaGraphInstantiate(&exec, graph, 0));
    for (long long launch = 0;; ++launch) {
      const int slot = static_cast<int>(launch & 1);
      APC_CUDA(cudaGraphLaunch(exec, st));
      APC_CUDA(cudaMemcpyAsync(&w->hst[slot], w->st.p, sizeof(LsqrState), cudaMemcpyDeviceToHost, st));
      APC_CUDA(cudaEventRecord(w->ev[slot], st));
      if (launch >= 1) {
        APC_CUDA(cudaEventSynchronize(w->ev[slot ^ 1]));
        if (w->hst[slot ^ 1].done) break;
      }
    }
  }
  APC_CUDA(cudaEventRecord(w->tev[1], st));
  APC_CUDA(cudaMemcpyAsync(&w->hst[0], w->st.p, sizeof(LsqrState), cudaMemcpyDeviceToHost, st));
  APC_CUDA(cudaStreamSynchronize(st));
  APC_CUDA(cudaGetLastError());
  {
    float ms = 0.f;
    APC_CUDA(cudaEventElapsedTime(&ms, w->tev[0], w->tev[1]));
    out.device_ms = ms;
  }
  if (exec) cudaGraphExecDestroy(exec);
  if (graph) cudaGraphDestroy(graph);
  out.ms = std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now() - t_start).count();

  const LsqrState& f = w->hst[0];
  out.breakdown = f.breakdown != 0;
  out.iters = f.iter < 0 ? 0 : f.iter;
  // count executed (graph-replayed) kernels, not captured ones
  if (!eager && !persistent)
    ctx->launches = launches_before_capture + per_iter * static_cast<std::uint64_t>(out.iters);
  out.reason = f.reason;
  const long long nrows = out.iters + 1;
  out.rows.resize(static_cast<size_t>(nrows));
  static_assert(sizeof(TraceRowH) == sizeof(TraceRow), "trace row layout");
  copy_sync(st, out.rows.data(), w->trace.p, sizeof(TraceRow) * nrows, cudaMemcpyDeviceToHost);
  if (sampling) {
    out.sampled.resize(static_cast<size_t>(nrows));
    copy_sync(st, out.sampled.data(), w->sampled.p, sizeof(double) * nrows, cudaMemcpyDeviceToHost);
  } else {
    out.sampled.clear();
  }
  if (out.breakdown) fail(APC_NUMERICAL_BREAKDOWN, "lsqr_solve: non-finite recurrence");
}

}  // namespace apc
