// Device-side helpers shared by the sm_100a kernels.  All .cu files of the
// library are compiled with -fmad=false: no FMA contraction, so every
// product/sum rounds exactly like the reference's SSE2 build
// (/root/reference/proj/CMakeLists.txt:3-11, no -march).
#pragma once

#include <cuda_runtime.h>
#include <math_constants.h>

#include <cstdint>

namespace apc {

constexpr int kWarp = 32;

__device__ __forceinline__ double warp_sum(double v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  return v;
}

// Deterministic block sum (fixed tree; every thread gets the result).
template <int NT>
__device__ __forceinline__ double block_sum(double v, double* sh) {
  v = warp_sum(v);
  const int w = threadIdx.x >> 5, l = threadIdx.x & 31;
  __syncthreads();
  if (l == 0) sh[w] = v;
  __syncthreads();
  double r = 0.0;
  if (w == 0) {
    r = (l < NT / 32) ? sh[l] : 0.0;
    r = warp_sum(r);
    if (l == 0) sh[0] = r;
  }
  __syncthreads();
  r = sh[0];
  __syncthreads();
  return r;
}

// "Last block done" election: every block publishes its partial, then the
// block that increments the counter last sees all partials and reduces them
// in index order -- a deterministic grid reduction without a second launch.
// Returns true in exactly one block; that block resets the counter.
__device__ __forceinline__ bool elect_last_block(unsigned int* counter, unsigned int nblocks) {
  __shared__ bool last;
  __threadfence();
  __syncthreads();
  if (threadIdx.x == 0) {
    unsigned int prev = atomicAdd(counter, 1u);
    last = (prev == nblocks - 1);
    if (last) *counter = 0u;
  }
  __syncthreads();
  if (last) __threadfence();
  return last;
}

// Sum partials[0..n) in a fixed order with one block (deterministic).
template <int NT>
__device__ __forceinline__ double ordered_sum(const volatile double* partials, long long n,
                                              double* sh) {
  // each thread sums a contiguous stripe, then the stripes are tree-summed in
  // thread order: fixed association for fixed (n, NT)
  long long per = (n + NT - 1) / NT;
  long long b = per * threadIdx.x, e = b + per < n ? b + per : n;
  // the stripe's loads are issued 8 at a time before the (in-order) adds: a
  // volatile load per add made the last block's sum a chain of L2 round trips
  // (~5 us at the LSQR kernels' 1563 tiles).  L2 loads (__ldcg): the partials
  // come from other SMs, ordered by elect_last_block's fences.
  const double* p = const_cast<const double*>(partials);
  double s = 0.0;
  for (long long i = b; i < e; i += 8) {
    double t[8];
#pragma unroll
    for (int k = 0; k < 8; ++k) t[k] = i + k < e ? __ldcg(p + i + k) : 0.0;
#pragma unroll
    for (int k = 0; k < 8; ++k)
      if (i + k < e) s += t[k];
  }
  return block_sum<NT>(s, sh);
}

__device__ __forceinline__ unsigned long long globaltimer_ns() {
  unsigned long long t;
  asm volatile("mov.u64 %0, %globaltimer;" : "=l"(t));
  return t;
}

// ---------------------------------------------------------------------------
// LSQR device state (one per phase) -- the scalars of lsqr_solve
// (/root/reference/proj/include/aplicur/lsqr.hpp:84-207) kept on the GPU so
// the iteration never round-trips to the host.
// ---------------------------------------------------------------------------
struct LsqrState {
  double alpha, beta;          // current Golub-Kahan scalars
  double rhobar, phibar, phibar0;
  double opnorm2;              // running ||op||_F^2 estimate (lsqr.hpp:134,154)
  double cvgrate1;
  double t1, t2, cabs;         // rotation outputs consumed by the y/w update
  double tail_norm2;           // ||u_tail||^2 (mu rows; replicated on all ranks)
  double ynorm;
  double t_cvgrate, t_cvgdiff; // cvgrate / cvgdiff of the latest iteration
  double eps, nu, sigma_floor; // StopConfig (lsqr.hpp:54-59)
  long long iter;              // completed iterations j
  long long cap;
  long long trace_cap;
  int done;                    // 1: stop (no further kernel does work)
  int reason;                  // StopReason (lsqr.hpp:17-24)
  int breakdown;               // 1: non-finite recurrence (numerical_breakdown)
  int samp_skip;               // 1: this iteration takes no true-residual sample
  unsigned long long t0_ns;
  long long samp_last;         // iteration of the last sampling gate
};

struct TraceRow {  // LsqrTraceRow (lsqr.hpp:38-47)
  double phibar, cvgrate, cvgdiff, wall_ms;
  long long iter;
  unsigned long long matvecs;
};

enum StopReasonDev {  // lsqr.hpp:17-24
  kReasonNone = 0,
  kReasonGradientTol = 1,
  kReasonDynamicRate = 2,
  kReasonDynamicDiff = 3,
  kReasonIterationCap = 4,
  kReasonExactZeroRhs = 5,
};

}  // namespace apc
