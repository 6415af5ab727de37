// Persistent cooperative LSQR phase for L2-resident sparse systems (the
// BASELINE C2 shape): ONE kernel launch runs every iteration of a phase, with
// grid-wide barriers between the dependent stages instead of ~11 kernel
// launches per iteration.  Each CTA carries its own copy of the scalar
// recurrence (alpha, beta, rhobar, phibar, ... of lsqr.hpp:132-203): every CTA
// reduces the same block partials in the same fixed order, so all copies stay
// bit-identical and no scalar ever round-trips through a broadcast.
//
// Stages per iteration (implicit preconditioner P^{-1} = I + R^T G R, R the
// l selected rows of A):
//   S12 t = R v, d_q = RT_q * (Gf t)_i, z = v + sum d      (per CTA)  | B1
//       stop tests of the previous iteration (its ||y|| partials are
//       complete only now; nothing persistent was written since)
//   S3  z -> shared memory ; u <- A z - alpha u/beta_old (SELL-32, thread
//       per row) ; u_tail <- mu z - alpha u_t/beta_old ; ||u||^2 partials| B2
//   S4  beta ; h = (A^T u + mu u_t)/beta  (warp per row of A^T)         | B3
//   S56 t = R h ; v_raw = h + R^T Ga t - beta v ; ||v_raw||^2  (per CTA)| B4
//   S7  alpha, rotation ; v = v_raw/alpha ; y += t1 w ; w = v + t2 w ;
//       ||y||^2 partials  (no barrier: the next S12 reads v_raw/alpha,
//       bit-identical to v, and every other read of v is the owner's own)
// "Per CTA" stages: each CTA owns a contiguous column range, recomputes the
// (short) l-vector t itself and only the (G t)_i its columns need, which
// saves the two grid barriers a grid-wide projection would cost.  Large R
// falls back to the grid-wide projection (two extra barriers per use).
// Unpreconditioned phases skip S12/S56; S4 then writes v_raw directly.
#include <cooperative_groups.h>
#include <cub/cub.cuh>

#include <algorithm>
#include <cstdlib>
#include <map>
#include <mutex>
#include <tuple>
#include <vector>

#include "dev_common.cuh"
#include "lsqr.hpp"
#include "lsqr_persistent.hpp"

namespace cg = cooperative_groups;

namespace apc {

#define STAMP(k)                                                                                 \
  if (P.prof && threadIdx.x == 0 && j < 64) {                                                      \
    const unsigned long long now_ = globaltimer_ns();                                              \
    if (blockIdx.x == 0) P.prof[j * 16 + (k)] = now_;                                              \
    if (j >= 2) P.prof[64 * 16 + blockIdx.x * 16 + (k)] += now_ - prev_stamp;                      \
    prev_stamp = now_;                                                                             \
  }

namespace {

// threads per CTA (template PT): one fat CTA per SM keeps grid barriers cheap;
// 1024 threads cap registers at 64, 512 allow 128 (no spills, fewer warps)
#ifndef APC_SELL_U
#define APC_SELL_U 8
#endif
constexpr int kSellU = APC_SELL_U;  // SELL entries per predicated load block
constexpr long long kSmemBudget = 200 * 1024;  // dynamic shared memory (z / projection scratch)

struct PArgs {
  // A: CSR rows (mloc) and CSR of A^T (n rows, no split rows)
  const int *aptr, *aidx;
  const double* aval;
  const int *tptr, *tidx;
  const double* tval;
  // SELL-32 copy of A (null: thread-per-row CSR walk)
  const int *soff, *sidx;
  const double* sval;
  long long nchunks;
  long long mloc, n;
  double mu;
  int has_tail;
  int zsmem;  // 1: every CTA stages z in shared memory for the forward gathers
  // preconditioner (implicit) or identity
  int pre;
  int fused;          // 1: per-CTA projection (small R), 0: grid-wide
  long long cchunk;   // columns owned per CTA
  const int *rptr, *ridx;
  const double* rval;
  const int *rtptr, *rtidx;
  const double* rtval;
  const double *Gf, *Ga;  // row-major l x l
  long long l;
  int rnnz;        // nnz(R) (fused: products staged per CTA)
  long long qmax;  // max R^T entries over the CTAs' column ranges (fused)
  int regs;  // 1: phase-constant projection operands held in registers (small R, l <= 256)
  // vectors
  double *u, *v, *vr, *w, *y, *z, *h, *s, *t;
  double* part;  // 4 slots x kPartStride
  unsigned long long* prof;  // optional stage timestamps (first 64 iterations)
  LsqrState* st;
  TraceRow* trace;
};

// Cache policy of the A^T u loads (A/B knobs): u gathers are random with no
// L1 reuse; the CSR(A^T) streams are read once per iteration.
#ifndef APC_GATHER_CG
#define APC_GATHER_CG 1
#endif
#ifndef APC_STREAM_CS
#define APC_STREAM_CS 0
#endif
__device__ __forceinline__ double ld_gather(const double* p) {
  if constexpr (APC_GATHER_CG) return __ldcg(p);
  else return *p;
}
template <class T>
__device__ __forceinline__ T ld_stream(const T* p) {
  if constexpr (APC_STREAM_CS) return __ldcs(p);
  else return __ldg(p);
}

// sum_{k < len} val[s k] * (x[idx[s k]] / xdiv), added strictly in k order; U
// entries per block are loaded under predicates so one block costs one memory
// round trip (a plain loop would pay one per entry)
template <int U, bool kDiv>
__device__ __forceinline__ double seq_dot(const int* idx, const double* val, int s, int len, const double* x,
                                          double xdiv = 1.0) {
  double acc = 0.0;
  for (int k0 = 0; k0 < len; k0 += U) {
    int i[U];
    double a[U], xv[U];
#pragma unroll
    for (int u = 0; u < U; ++u) {
      const bool ok = k0 + u < len;
      i[u] = ok ? __ldg(idx + s * (k0 + u)) : 0;
      a[u] = ok ? __ldg(val + s * (k0 + u)) : 0.0;
    }
#pragma unroll
    for (int u = 0; u < U; ++u) xv[u] = (k0 + u < len) ? x[i[u]] : 0.0;
#pragma unroll
    for (int u = 0; u < U; ++u)
      if (k0 + u < len) acc += a[u] * (kDiv ? xv[u] / xdiv : xv[u]);
  }
  return acc;
}

// Grid sums of per-CTA partials (layout part[slot * kPartStride + cta]): warp
// 0 of every CTA sums each requested slot in the same fixed order (lane
// stripes, then butterfly) and shares the results through shared memory --
// one reader per SM keeps the few hot partial lines from being hammered.
constexpr int kPartStride = 2048;
template <int NS>
__device__ __forceinline__ void grid_sums(const double* part, const int (&slots)[NS], int nblocks, double* out_sh,
                                          double (&out)[NS]) {
  if (threadIdx.x < 32) {
    double v[NS];
#pragma unroll
    for (int k = 0; k < NS; ++k) v[k] = 0.0;
    for (int b0 = 0; b0 < nblocks; b0 += 256) {  // all loads of a block in flight at once
      double x[NS][8];
#pragma unroll
      for (int u = 0; u < 8; ++u) {
        const int b = b0 + threadIdx.x + 32 * u;
#pragma unroll
        for (int k = 0; k < NS; ++k) x[k][u] = b < nblocks ? part[slots[k] * kPartStride + b] : 0.0;
      }
#pragma unroll
      for (int u = 0; u < 8; ++u)
#pragma unroll
        for (int k = 0; k < NS; ++k)
          if (b0 + threadIdx.x + 32 * u < nblocks) v[k] += x[k][u];
    }
#pragma unroll
    for (int k = 0; k < NS; ++k) {
      const double t = warp_sum(v[k]);
      if (threadIdx.x == 0) out_sh[k] = t;
    }
  }
  __syncthreads();
#pragma unroll
  for (int k = 0; k < NS; ++k) out[k] = out_sh[k];
}

// CTA partial sums of up to two values -> part[blockIdx.x * 4 + slot] (fixed
// order: lanes by butterfly, warps in index order).  One block barrier; the
// caller's next grid barrier orders the reuse of `red`.
template <int PT>
__device__ __forceinline__ void cta_partial(double a, double b, double* red, double* part, int slot_a,
                                            int slot_b) {
  a = warp_sum(a);
  b = warp_sum(b);
  const int w = threadIdx.x >> 5;
  if ((threadIdx.x & 31) == 0) {
    red[w] = a;
    red[32 + w] = b;
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    double sa = 0.0, sb = 0.0;
    for (int k = 0; k < PT / 32; ++k) {
      sa += red[k];
      sb += red[32 + k];
    }
    part[slot_a * kPartStride + blockIdx.x] = sa;
    if (slot_b >= 0) part[slot_b * kPartStride + blockIdx.x] = sb;
  }
}

// t = M (x / xdiv), s = K t for the l x n sparse M (R) and row-major K, spread
// over the whole grid (one warp per row in each half, a barrier between them).
__device__ void grid_project(cg::grid_group& grid, const int* mptr, const int* midx, const double* mval,
                             const double* KT, long long l, const double* x, double xdiv, double* t,
                             double* s_out, long long gwarp, long long nwarps, int lane) {
  for (long long i = gwarp; i < l; i += nwarps) {
    double acc = 0.0;
    for (int q = mptr[i] + lane; q < mptr[i + 1]; q += 32) acc += mval[q] * (x[midx[q]] / xdiv);
    acc = warp_sum(acc);
    if (lane == 0) t[i] = acc;
  }
  grid.sync();
  for (long long i = gwarp; i < l; i += nwarps) {
    const double* row = KT + i * l;
    double acc = 0.0;
    for (long long k = lane; k < l; k += 32) acc += row[k] * t[k];
    acc = warp_sum(acc);
    if (lane == 0) s_out[i] = acc;
  }
}

// Per-CTA projection for the columns [c0, c1) this CTA owns:
//   psh[q] = R_val[q] * (x[R_idx[q]] / xdiv)   every entry of R (entry-parallel)
//   tsh[i] = sum_q psh[q] over row i, in order  (= (R x)_i)
//   dsh[q - RT_ptr[c0]] = RT_val[q] * (K tsh)_{RT_idx[q]}   for q of the range
// The K rows are fetched before t exists, so the stage costs about two memory
// round trips (R entries -> x gathers) instead of one per dependent load.
template <int PT>
__device__ void cta_project(const PArgs& P, const double* x, double xdiv, const double* K, double* tsh,
                            double* dsh, double* psh, long long c0, long long c1, int warp, int lane) {
  const int nr = P.rnnz;
  for (int q0 = threadIdx.x; q0 < nr; q0 += 4 * PT) {
    int i[4];
    double a[4], xv[4];
#pragma unroll
    for (int u = 0; u < 4; ++u) {
      const int q = q0 + u * PT;
      i[u] = q < nr ? __ldg(P.ridx + q) : 0;
      a[u] = q < nr ? __ldg(P.rval + q) : 0.0;
    }
#pragma unroll
    for (int u = 0; u < 4; ++u) xv[u] = q0 + u * PT < nr ? x[i[u]] : 0.0;
#pragma unroll
    for (int u = 0; u < 4; ++u)
      if (q0 + u * PT < nr) psh[q0 + u * PT] = a[u] * (xv[u] / xdiv);
  }
  const int qb0 = __ldg(P.rtptr + c0), qb1 = __ldg(P.rtptr + c1);
  const int qa = qb0 + warp;
  const bool small = P.l <= 256;
  double g[8];
#pragma unroll
  for (int u = 0; u < 8; ++u) g[u] = 0.0;
  if (small && qa < qb1) {
    const double* row = K + static_cast<long long>(__ldg(P.rtidx + qa)) * P.l;
#pragma unroll
    for (int u = 0; u < 8; ++u)
      if (lane + 32 * u < P.l) g[u] = __ldg(row + lane + 32 * u);
  }
  __syncthreads();
  for (long long i = threadIdx.x; i < P.l; i += PT) {
    const int b = __ldg(P.rptr + i), e = __ldg(P.rptr + i + 1);
    double acc = 0.0;
    for (int q = b; q < e; ++q) acc += psh[q];
    tsh[i] = acc;
  }
  __syncthreads();
  for (int q = qa; q < qb1; q += PT / 32) {
    double acc = 0.0;
    if (small && q == qa) {
#pragma unroll
      for (int u = 0; u < 8; ++u)
        if (lane + 32 * u < P.l) acc += g[u] * tsh[lane + 32 * u];
    } else {
      const double* row = K + static_cast<long long>(__ldg(P.rtidx + q)) * P.l;
      for (long long k = lane; k < P.l; k += 32) acc += __ldg(row + k) * tsh[k];
    }
    acc = warp_sum(acc);
    if (lane == 0) dsh[q - qb0] = __ldg(P.rtval + q) * acc;
  }
  __syncthreads();
}

// The phase-constant operands of the per-CTA projection held in registers
// (small R, l <= 256): R entries (4 per thread), the thread's row bounds of R,
// this warp's first R^T entry and its rows of Gf / Ga.
struct ProjRegs {
  int ri[4];
  double rv[4];
  int rb, re;
  int qb0, qb1, qa;
  long long gi;  // K row of this warp's first R^T entry (-1: none)
};

template <int PT>
__device__ __forceinline__ void proj_regs_load(const PArgs& P, ProjRegs& R, long long c0, long long c1, int warp) {
#pragma unroll
  for (int u = 0; u < 4; ++u) {
    const int q = threadIdx.x + u * PT;
    R.ri[u] = q < P.rnnz ? __ldg(P.ridx + q) : 0;
    R.rv[u] = q < P.rnnz ? __ldg(P.rval + q) : 0.0;
  }
  R.rb = threadIdx.x < P.l ? __ldg(P.rptr + threadIdx.x) : 0;
  R.re = threadIdx.x < P.l ? __ldg(P.rptr + threadIdx.x + 1) : 0;
  R.qb0 = __ldg(P.rtptr + c0);
  R.qb1 = __ldg(P.rtptr + c1);
  R.qa = R.qb0 + warp;
  R.gi = R.qa < R.qb1 ? static_cast<long long>(__ldg(P.rtidx + R.qa)) * P.l : -1;
}

// cta_project with the operands of ProjRegs: one memory round trip (the x
// gathers) plus three block barriers.  Same arithmetic and order as cta_project.
template <int PT, bool kFwd>
__device__ __forceinline__ void cta_project_reg(const PArgs& P, const ProjRegs& R, const double* x, double xdiv,
                                                double* tsh, double* dsh, double* psh, int lane) {
  const int nr = P.rnnz;
  double xv[4];
#pragma unroll
  for (int u = 0; u < 4; ++u) xv[u] = threadIdx.x + u * PT < nr ? x[R.ri[u]] : 0.0;
#pragma unroll
  for (int u = 0; u < 4; ++u)
    if (threadIdx.x + u * PT < nr) psh[threadIdx.x + u * PT] = R.rv[u] * (xv[u] / xdiv);
  for (int q = threadIdx.x + 4 * PT; q < nr; q += PT)  // beyond the register-held entries
    psh[q] = __ldg(P.rval + q) * (x[__ldg(P.ridx + q)] / xdiv);
  const double* K = kFwd ? P.Gf : P.Ga;
  double g[8];  // this warp's first K row, fetched before t exists
#pragma unroll
  for (int u = 0; u < 8; ++u) g[u] = (R.gi >= 0 && lane + 32 * u < P.l) ? __ldg(K + R.gi + lane + 32 * u) : 0.0;
  __syncthreads();
  if (threadIdx.x < P.l) {
    double acc = 0.0;
    for (int q = R.rb; q < R.re; ++q) acc += psh[q];
    tsh[threadIdx.x] = acc;
  }
  __syncthreads();
  for (int q = R.qa; q < R.qb1; q += PT / 32) {
    double acc = 0.0;
    if (q == R.qa) {
#pragma unroll
      for (int u = 0; u < 8; ++u)
        if (lane + 32 * u < P.l) acc += g[u] * tsh[lane + 32 * u];
    } else {
      const double* row = K + static_cast<long long>(__ldg(P.rtidx + q)) * P.l;
      for (long long k = lane; k < P.l; k += 32) acc += __ldg(row + k) * tsh[k];
    }
    acc = warp_sum(acc);
    if (lane == 0) dsh[q - R.qb0] = __ldg(P.rtval + q) * acc;
  }
  __syncthreads();
}

__device__ __forceinline__ unsigned smem_u32(const void* p) {
  return static_cast<unsigned>(__cvta_generic_to_shared(p));
}

template <int PT, bool kRegs>
__global__ void __launch_bounds__(PT, 1) lsqr_persistent_kernel(PArgs P) {
  extern __shared__ double dyn[];  // z copy (S3) / t, d, products (S12, S56): disjoint in time
  __shared__ double red[64];
  __shared__ double gsh[4];
  cg::grid_group grid = cg::this_grid();
  const long long gtid = static_cast<long long>(blockIdx.x) * PT + threadIdx.x;
  const long long gsize = static_cast<long long>(gridDim.x) * PT;
  const long long gwarp = gtid >> 5, nwarps = gsize >> 5;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int nb = gridDim.x;
  // owned columns of the n-length stages
  const long long cb = static_cast<long long>(blockIdx.x) * P.cchunk;
  const long long c0 = cb < P.n ? cb : P.n;
  const long long c1 = c0 + P.cchunk < P.n ? c0 + P.cchunk : P.n;
  LsqrState* st = P.st;
  // replicated scalar recurrence (initialised by the phase-init kernels)
  double alpha = st->alpha, beta = st->beta, rhobar = st->rhobar, phibar = st->phibar;
  const double phibar0 = st->phibar0;
  double opnorm2 = st->opnorm2, cvgrate1 = st->cvgrate1;
  const double eps = st->eps, nu = st->nu, floor_ = st->sigma_floor;
  const long long cap = st->cap, tcap = st->trace_cap;
  long long j = st->iter;
  const unsigned long long t0 = st->t0_ns;
  if (st->done) return;
  // quantities of the last completed iteration, tested after the next B2
  bool pending = false, nonfinite = false;
  double cc = 0.0, cvgrate = 0.0, cvgdiff = 0.0;
  // v of the next S12 = vsrc / vdiv (first iteration: the initialised v)
  const double* vsrc = P.v;
  double vdiv = 1.0;
  double* tsh = dyn;
  double* dsh = dyn + P.l;
  double* psh = dsh + P.qmax;
  unsigned long long prev_stamp = 0;
  ProjRegs R;
  constexpr bool regs = kRegs;
  if (regs && P.fused) proj_regs_load<PT>(P, R, c0, c1, warp);
  // z staging by one bulk (TMA) copy per iteration, completion on an mbarrier
  __shared__ __align__(8) unsigned long long zbar;
  unsigned zphase = 0;
  const bool ztma = P.zsmem && ((P.n * 8) % 16 == 0);
  if (ztma && threadIdx.x == 0) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(smem_u32(&zbar)) : "memory");
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncthreads();

  for (;;) {
    // ---- S12: z = v + R^T Gf R v
    STAMP(0);
    if (P.pre) {
      if (P.fused) {
        if (regs) cta_project_reg<PT, true>(P, R, vsrc, vdiv, tsh, dsh, psh, lane);
        else cta_project<PT>(P, vsrc, vdiv, P.Gf, tsh, dsh, psh, c0, c1, warp, lane);
        STAMP(1);
        const int qb0 = __ldg(P.rtptr + c0);
        for (long long c = c0 + threadIdx.x; c < c1; c += PT) {
          double acc = 0.0;
          for (int q = __ldg(P.rtptr + c); q < __ldg(P.rtptr + c + 1); ++q) acc += dsh[q - qb0];
          P.z[c] = P.v[c] + acc;
        }
      } else {
        grid_project(grid, P.rptr, P.ridx, P.rval, P.Gf, P.l, vsrc, vdiv, P.t, P.s, gwarp, nwarps, lane);
        grid.sync();
        for (long long c = c0 + threadIdx.x; c < c1; c += PT) {
          double acc = 0.0;
          for (int q = P.rtptr[c]; q < P.rtptr[c + 1]; ++q) acc += P.rtval[q] * P.s[P.rtidx[q]];
          P.z[c] = P.v[c] + acc;
        }
      }
    }
    STAMP(2);
    grid.sync();  // B1
    STAMP(3);
    // ---- S3: u <- A z - alpha u/beta ; tail rows
    const double* zg = P.pre ? P.z : P.v;
    const double* zs = zg;
    if (ztma) {
      // B1 ordered every generic access to dyn and the z stores of all CTAs
      // before this point; the proxy fence hands them to the async proxy
      if (threadIdx.x == 0) {
        const unsigned bytes = static_cast<unsigned>(P.n * 8);
        asm volatile("fence.proxy.async;" ::: "memory");
        asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(&zbar)), "r"(bytes)
                     : "memory");
        for (unsigned off = 0; off < bytes; off += 32768) {
          const unsigned len = bytes - off < 32768 ? bytes - off : 32768;
          asm volatile(
              "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
                  smem_u32(reinterpret_cast<char*>(dyn) + off)),
              "l"(reinterpret_cast<const char*>(zg) + off), "r"(len), "r"(smem_u32(&zbar))
              : "memory");
        }
      }
      asm volatile(
          "{\n .reg .pred p;\n ZWAIT_%=:\n mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n @!p bra ZWAIT_%=;\n}" ::"r"(
              smem_u32(&zbar)),
          "r"(zphase)
          : "memory");
      zphase ^= 1u;
      zs = dyn;
    } else if (P.zsmem) {
      const long long h2 = P.n >> 1;
      const double2* src = reinterpret_cast<const double2*>(zg);
      double2* dst = reinterpret_cast<double2*>(dyn);
#pragma unroll 4
      for (long long i = threadIdx.x; i < h2; i += PT) dst[i] = src[i];
      if ((P.n & 1) && threadIdx.x == 0) dyn[P.n - 1] = zg[P.n - 1];
      __syncthreads();
      zs = dyn;
    }
    STAMP(5);
    {
      double sq = 0.0, sqt = 0.0;
      const double rb = beta;
      if (P.sidx) {
        // SELL-32: warp = 32 consecutive rows, lane = row; idx/val coalesced
        for (long long ch = gwarp; ch < P.nchunks; ch += nwarps) {
          const long long r = ch * 32 + lane;
          const bool ok = r < P.mloc;
          const int len = ok ? __ldg(P.aptr + r + 1) - __ldg(P.aptr + r) : 0;
          const double uo = ok ? P.u[r] : 0.0;
          const long long off = __ldg(P.soff + ch) + lane;
          const double acc = seq_dot<kSellU, false>(P.sidx + off, P.sval + off, 32, len, zs);
          if (ok) {
            const double uh = rb > 0.0 ? uo / rb : uo;
            const double t = acc - alpha * uh;
            P.u[r] = t;
            sq += t * t;
          }
        }
      } else {
        // thread per row (rows are short)
        for (long long r = gtid; r < P.mloc; r += gsize) {
          const int b = __ldg(P.aptr + r), e = __ldg(P.aptr + r + 1);
          const double uo = P.u[r];
          const double acc = seq_dot<8, false>(P.aidx + b, P.aval + b, 1, e - b, zs);
          const double uh = rb > 0.0 ? uo / rb : uo;
          const double t = acc - alpha * uh;
          P.u[r] = t;
          sq += t * t;
        }
      }
      if (P.has_tail) {
        double* ut = P.u + P.mloc;
        for (long long c = gtid; c < P.n; c += gsize) {
          const double uo = ut[c];
          const double uh = rb > 0.0 ? uo / rb : uo;
          const double t = P.mu * zs[c] - alpha * uh;
          ut[c] = t;
          sqt += t * t;
        }
      }
      STAMP(6);
      cta_partial<PT>(sq, sqt, red, P.part, 0, 1);
    }
    STAMP(7);
    grid.sync();  // B2
    STAMP(8);
    // beta of this iteration and ||y|| of the previous one in one pass
    double sums[3];
    grid_sums<3>(P.part, {0, 1, 3}, nb, gsh, sums);
    const double s3 = pending ? sums[2] : 0.0;
    const double bnew = sqrt(sums[0] + sums[1]);
    if (pending) {
      // ---- stop tests of iteration j (lsqr.hpp:183-203), identical in every
      // CTA; the S12/S3 work done since only touched z and u (scratch)
      const double ynorm = sqrt(s3);
      int reason = kReasonNone;
      bool stop = false;
      if (nonfinite) {
        stop = true;
      } else {
        const double grad = phibar * alpha * fabs(cc);
        const double sqn = sqrt(opnorm2);
        if (grad <= eps * sqn * phibar || phibar <= eps * (sqn * ynorm + phibar0) || phibar == 0.0) {
          stop = true;
          reason = kReasonGradientTol;
        } else if (j >= 2 && nu > 0.0 && !isinf(nu)) {
          if (floor_ > 0.0 && cvgdiff < floor_) reason = kReasonDynamicDiff;
          else if (cvgrate <= 0.0) reason = kReasonDynamicRate;
          else if (cvgrate1 / cvgrate > nu) reason = kReasonDynamicRate;
          stop = reason != kReasonNone;
        }
        if (!stop && j >= cap) {
          stop = true;
          reason = kReasonIterationCap;
        }
      }
      if (blockIdx.x == 0 && threadIdx.x == 0) {
        if (j < tcap)
          P.trace[j] = TraceRow{phibar, cvgrate, cvgdiff, (globaltimer_ns() - t0) * 1e-6, j,
                                1ull + 2ull * static_cast<unsigned long long>(j)};
        if (stop) {
          st->alpha = alpha;
          st->beta = beta;
          st->rhobar = rhobar;
          st->phibar = phibar;
          st->opnorm2 = opnorm2;
          st->cvgrate1 = cvgrate1;
          st->ynorm = ynorm;
          st->iter = j;
          st->done = 1;
          st->reason = reason;
          st->breakdown = nonfinite ? 1 : 0;
        }
      }
      if (stop) return;
    }
    STAMP(9);
    // ---- S4: h = (A^T u + mu u_t) / beta  [plain: v_raw = h - beta v, ||v_raw||^2]
    {
      double sq = 0.0;
      auto finish = [&](long long c, double acc) {
        if (P.has_tail) acc += P.mu * P.u[P.mloc + c];
        const double gj = bnew > 0.0 ? acc / bnew : acc;
        if (P.pre) {
          P.h[c] = gj;
        } else {
          const double t = gj - bnew * P.v[c];
          P.vr[c] = t;
          sq += t * t;
        }
      };
      // two rows of A^T per warp pass, 4 predicated entries per lane and row:
      // up to 8 independent gathers in flight per lane
      for (long long c = gwarp; c < P.n; c += 2 * nwarps) {
        const long long c2 = c + nwarps;
        const bool has2 = c2 < P.n;
        const int b1 = __ldg(P.tptr + c), n1 = __ldg(P.tptr + c + 1) - b1;
        const int b2 = has2 ? __ldg(P.tptr + c2) : 0, n2 = has2 ? __ldg(P.tptr + c2 + 1) - b2 : 0;
        const int nmax = max(n1, n2);
        double acc1 = 0.0, acc2 = 0.0;
        for (int k0 = lane; k0 < nmax; k0 += 128) {
          int i1[4], i2[4];
          double v1[4], v2[4], g1[4], g2[4];
#pragma unroll
          for (int u = 0; u < 4; ++u) {
            const int q = k0 + 32 * u;
            i1[u] = q < n1 ? ld_stream(P.tidx + b1 + q) : 0;
            v1[u] = q < n1 ? ld_stream(P.tval + b1 + q) : 0.0;
            i2[u] = q < n2 ? ld_stream(P.tidx + b2 + q) : 0;
            v2[u] = q < n2 ? ld_stream(P.tval + b2 + q) : 0.0;
          }
#pragma unroll
          for (int u = 0; u < 4; ++u) {
            const int q = k0 + 32 * u;
            g1[u] = q < n1 ? ld_gather(P.u + i1[u]) : 0.0;
            g2[u] = q < n2 ? ld_gather(P.u + i2[u]) : 0.0;
          }
#pragma unroll
          for (int u = 0; u < 4; ++u) {
            const int q = k0 + 32 * u;
            if (q < n1) acc1 += v1[u] * g1[u];
            if (q < n2) acc2 += v2[u] * g2[u];
          }
        }
        acc1 = warp_sum(acc1);
        acc2 = warp_sum(acc2);
        if (lane == 0) {
          finish(c, acc1);
          if (has2) finish(c2, acc2);
        }
      }
      if (!P.pre) cta_partial<PT>(sq, 0.0, red, P.part, 2, -1);
    }
    STAMP(10);
    grid.sync();  // B3
    STAMP(11);
    if (P.pre) {
      // ---- S56: v_raw = h + R^T Ga R h - beta v ; ||v_raw||^2
      double sq = 0.0;
      if (P.fused) {
        if (regs) cta_project_reg<PT, false>(P, R, P.h, 1.0, tsh, dsh, psh, lane);
        else cta_project<PT>(P, P.h, 1.0, P.Ga, tsh, dsh, psh, c0, c1, warp, lane);
        STAMP(12);
        const int qb0 = __ldg(P.rtptr + c0);
        for (long long c = c0 + threadIdx.x; c < c1; c += PT) {
          double acc = 0.0;
          for (int q = __ldg(P.rtptr + c); q < __ldg(P.rtptr + c + 1); ++q) acc += dsh[q - qb0];
          const double t = (P.h[c] + acc) - bnew * P.v[c];
          P.vr[c] = t;
          sq += t * t;
        }
      } else {
        grid_project(grid, P.rptr, P.ridx, P.rval, P.Ga, P.l, P.h, 1.0, P.t, P.s, gwarp, nwarps, lane);
        grid.sync();
        for (long long c = c0 + threadIdx.x; c < c1; c += PT) {
          double acc = 0.0;
          for (int q = P.rtptr[c]; q < P.rtptr[c + 1]; ++q) acc += P.rtval[q] * P.s[P.rtidx[q]];
          const double t = (P.h[c] + acc) - bnew * P.v[c];
          P.vr[c] = t;
          sq += t * t;
        }
      }
      cta_partial<PT>(sq, 0.0, red, P.part, 2, -1);
      STAMP(13);
      grid.sync();  // B4
    }
    STAMP(14);
    // ---- S7: alpha ; rotation (lsqr.hpp:145-171) ; owner-column updates ; ||y||^2
    // (the owner's first column is fetched before the alpha reduction)
    const long long cf = c0 + threadIdx.x;
    double vo = 0.0, wo = 0.0, yo = 0.0;
    if (cf < c1) {
      vo = P.vr[cf];
      wo = P.w[cf];
      yo = P.y[cf];
    }
    double sa[1];
    grid_sums<1>(P.part, {2}, nb, gsh + 3, sa);
    const double anew = sqrt(sa[0]);
    beta = bnew;
    alpha = anew;
    opnorm2 += alpha * alpha + beta * beta;
    const double rho = hypot(rhobar, beta);
    cc = rhobar / rho;
    const double s = beta / rho;
    const double theta = s * alpha;
    rhobar = -cc * alpha;
    const double phi = cc * phibar;
    const double phibar_prev = phibar;
    phibar = s * phibar;
    const double t1 = phi / rho, t2 = -theta / rho;
    ++j;
    nonfinite = !isfinite(phibar) || !isfinite(alpha) || !isfinite(beta);
    cvgrate = (phibar > 0.0 && phibar_prev > 0.0) ? log(phibar_prev / phibar) : CUDART_INF;
    cvgdiff = phibar_prev - phibar;
    if (j == 1) cvgrate1 = cvgrate;
    vdiv = alpha > 0.0 ? alpha : 1.0;
    vsrc = P.vr;
    {
      double sq = 0.0;
      for (long long c = cf; c < c1; c += PT) {
        if (c != cf) {
          vo = P.vr[c];
          wo = P.w[c];
          yo = P.y[c];
        }
        const double vh = vo / vdiv;
        P.v[c] = vh;
        const double yn = yo + t1 * wo;
        P.y[c] = yn;
        P.w[c] = vh + t2 * wo;
        sq += yn * yn;
      }
      cta_partial<PT>(sq, 0.0, red, P.part, 3, -1);
    }
    pending = true;
    if (P.prof && blockIdx.x == 0 && threadIdx.x == 0 && j - 1 < 64) P.prof[(j - 1) * 16 + 15] = globaltimer_ns();
  }
}

// ---- SELL-32 build from the CSR (once per matrix)
__global__ void sell_width_kernel(const int* __restrict__ ptr, long long rows, long long chunks,
                                  int* __restrict__ width) {
  const long long ch = static_cast<long long>(blockIdx.x) * blockDim.x + threadIdx.x;
  if (ch > chunks) return;
  if (ch == chunks) {
    width[ch] = 0;
    return;
  }
  int w = 0;
  const long long rend = ch * 32 + 32 < rows ? ch * 32 + 32 : rows;
  for (long long r = ch * 32; r < rend; ++r) w = max(w, ptr[r + 1] - ptr[r]);
  width[ch] = 32 * w;
}

__global__ void sell_fill_kernel(const int* __restrict__ ptr, const int* __restrict__ idx,
                                 const double* __restrict__ val, long long rows, const int* __restrict__ off,
                                 int* __restrict__ sidx, double* __restrict__ sval) {
  const long long r = static_cast<long long>(blockIdx.x) * blockDim.x + threadIdx.x;
  if (r >= rows) return;
  const long long base = off[r >> 5] + (r & 31);
  const int b = ptr[r], e = ptr[r + 1];
  for (int q = b; q < e; ++q) {
    sidx[base + 32LL * (q - b)] = idx[q];
    sval[base + 32LL * (q - b)] = val[q];
  }
}

void build_sell(apc_mat& a) {
  apc_ctx* ctx = a.ctx;
  cudaStream_t st = ctx->stream;
  Sell& s = a.sell;
  const long long rows = a.a.rows;
  s.rows = rows;
  s.chunks = (rows + 31) / 32;
  s.off.alloc(s.chunks + 1);
  DBuf<int> width(s.chunks + 1);
  sell_width_kernel<<<static_cast<unsigned>((s.chunks + 1 + 255) / 256), 256, 0, st>>>(a.a.ptr.p, rows, s.chunks,
                                                                                         width.p);
  size_t tmp = 0;
  cub::DeviceScan::ExclusiveSum(nullptr, tmp, width.p, s.off.p, static_cast<int>(s.chunks + 1), st);
  DBuf<unsigned char> tbuf(static_cast<long long>(std::max<size_t>(tmp, 1)));
  APC_CUDA(cub::DeviceScan::ExclusiveSum(tbuf.p, tmp, width.p, s.off.p, static_cast<int>(s.chunks + 1), st));
  int slots = 0;
  copy_sync(st, &slots, s.off.p + s.chunks, sizeof(int), cudaMemcpyDeviceToHost);
  s.slots = slots;
  s.idx.alloc(std::max(1, slots));
  s.val.alloc(std::max(1, slots));
  APC_CUDA(cudaMemsetAsync(s.idx.p, 0, s.idx.bytes(), st));
  APC_CUDA(cudaMemsetAsync(s.val.p, 0, s.val.bytes(), st));
  if (rows > 0)
    sell_fill_kernel<<<static_cast<unsigned>((rows + 255) / 256), 256, 0, st>>>(a.a.ptr.p, a.a.idx.p, a.a.val.p,
                                                                               rows, s.off.p, s.idx.p, s.val.p);
  APC_CUDA(cudaGetLastError());
  ctx->launches += rows > 0 ? 3 : 2;
  APC_CUDA(cudaStreamSynchronize(st));
}

// occupancy of a kernel variant at a dynamic shared-memory size, with the
// opt-in attribute set; cached (the driver calls take locks that a concurrent
// NVML poller also takes, and would otherwise run at every LSQR phase)
int occupancy(void* kfn, int threads, size_t smem) {
  static std::mutex mu;
  static std::map<std::tuple<int, void*, int, size_t>, int> cache;
  std::lock_guard<std::mutex> lk(mu);
  int dev = 0;
  APC_CUDA(cudaGetDevice(&dev));
  const auto key = std::make_tuple(dev, kfn, threads, smem);
  auto it = cache.find(key);
  if (it != cache.end()) return it->second;
  if (smem > 48 * 1024)
    APC_CUDA(cudaFuncSetAttribute(kfn, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(smem)));
  int per_sm = 0;
  APC_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kfn, threads, smem));
  cache[key] = per_sm;
  return per_sm;
}

}  // namespace

bool persistent_eligible(const apc_mat& a, const PrecondDev* p, const apc_ctx* ctx) {
  if (ctx->nranks != 1 || !a.sparse) return false;
  if (a.at.n_parts != 0) return false;  // a row of A^T longer than one work unit
  if (p && p->kind == 1) return false;  // explicit dense basis: graph path
  if (p && p->kind == 2 && p->l > 6000) return false;
  return true;
}

void lsqr_persistent_run(apc_mat& a, double mu, const PrecondDev* p, const PersistentBuffers& b) {
  apc_ctx* ctx = a.ctx;
  PArgs P{};
  P.aptr = a.a.ptr.p;
  P.aidx = a.a.idx.p;
  P.aval = a.a.val.p;
  P.tptr = a.at.ptr.p;
  P.tidx = a.at.idx.p;
  P.tval = a.at.val.p;
  P.mloc = a.mloc();
  P.n = a.n;
  P.mu = mu;
  P.has_tail = mu > 0.0 ? 1 : 0;
  P.pre = (p && p->kind == 2) ? 1 : 0;
  // the SELL copy pays for itself when the CSR is L2-resident (the gathers,
  // not HBM, bound the forward product); APC_PERSISTENT_SELL=0 disables it
  const char* sell_env = std::getenv("APC_PERSISTENT_SELL");
  const bool want_sell = (sell_env ? std::atoi(sell_env) != 0 : true) && a.a.nnz * 12 <= (96LL << 20) &&
                         a.a.nnz * 3 / 2 + 32 * 64 < (1LL << 31);
  if (want_sell) {
    if (a.sell.rows != a.a.rows || !a.sell.off.p) build_sell(a);
    P.soff = a.sell.off.p;
    P.sidx = a.sell.idx.p;
    P.sval = a.sell.val.p;
    P.nchunks = a.sell.chunks;
  }
  const char* pte = std::getenv("APC_PERSISTENT_PT");
  const int pt = (pte && std::atoi(pte) == 1024) ? 1024 : 512;
  void* kfn = pt == 512 ? reinterpret_cast<void*>(lsqr_persistent_kernel<512, false>)
                        : reinterpret_cast<void*>(lsqr_persistent_kernel<1024, false>);
  int per_sm = 0;
  per_sm = occupancy(kfn, pt, 0);
  const int blocks_per_sm = std::max(1, std::min(per_sm, b.blocks_per_sm > 0 ? b.blocks_per_sm : 3));
  const int grid = ctx->num_sms * blocks_per_sm;
  P.cchunk = std::max<long long>(1, (a.n + grid - 1) / grid);
  long long smem_doubles = 1;
  if (P.pre) {
    P.rptr = p->R.ptr.p;
    P.ridx = p->R.idx.p;
    P.rval = p->R.val.p;
    P.rtptr = p->RT.ptr.p;
    P.rtidx = p->RT.idx.p;
    P.rtval = p->RT.val.p;
    P.Gf = p->Kf.p;
    P.Ga = p->Ka.p;
    P.l = p->l;
    // per-CTA projection when R is small: every CTA re-walks nnz(R) and reads
    // one K row per R^T entry of its columns
    const char* fe = std::getenv("APC_PERSISTENT_FUSED");
    const bool want_fused = (fe ? std::atoi(fe) != 0 : true) && p->R.nnz <= 32768 && p->R.nnz * p->l <= (8LL << 20);
    if (want_fused) {
      std::vector<int> hp(static_cast<size_t>(a.n + 1));
      copy_sync(ctx->stream, hp.data(), p->RT.ptr.p, sizeof(int) * hp.size(), cudaMemcpyDeviceToHost);
      long long qmax = 0;
      for (long long c0 = 0; c0 < a.n; c0 += P.cchunk)
        qmax = std::max<long long>(qmax, hp[std::min<long long>(a.n, c0 + P.cchunk)] - hp[c0]);
      if ((P.l + qmax + p->R.nnz) * 8 <= kSmemBudget) {
        P.fused = 1;
        P.rnnz = static_cast<int>(p->R.nnz);
        P.qmax = qmax;
        smem_doubles = std::max(smem_doubles, P.l + qmax + p->R.nnz);
      }
    }
  }
  const char* ze = std::getenv("APC_PERSISTENT_ZSMEM");
  if ((ze ? std::atoi(ze) != 0 : true) && P.n * 8 <= kSmemBudget) {
    P.zsmem = 1;
    smem_doubles = std::max(smem_doubles, P.n);
  }
  P.u = b.u;
  P.v = b.v;
  P.vr = b.vr;
  P.w = b.w;
  P.y = b.y;
  P.z = b.z;
  P.h = b.h;
  P.s = b.s;
  P.t = b.t;
  P.prof = b.prof;
  P.st = b.st;
  P.trace = b.trace;
  const char* re = std::getenv("APC_PERSISTENT_REGS");
  P.regs = ((re ? std::atoi(re) != 0 : false) && P.fused && P.rnnz <= 4 * pt && P.l <= pt && P.l <= 256) ? 1 : 0;
  if (P.regs)
    kfn = pt == 512 ? reinterpret_cast<void*>(lsqr_persistent_kernel<512, true>)
                    : reinterpret_cast<void*>(lsqr_persistent_kernel<1024, true>);
  const size_t smem = sizeof(double) * static_cast<size_t>(smem_doubles);
  per_sm = occupancy(kfn, pt, smem);
  require(per_sm >= blocks_per_sm, APC_CUDA_ERROR, "persistent LSQR: grid does not fit co-resident");
  P.part = b.part;
  require(grid <= kPartStride, APC_CUDA_ERROR, "persistent LSQR: grid larger than the partial stride");
  void* args[] = {&P};
  APC_CUDA(cudaLaunchCooperativeKernel(kfn, dim3(grid), dim3(pt), args, smem, ctx->stream));
  ctx->launches++;
}

int persistent_max_grid(apc_ctx* ctx) { return std::max(ctx->num_sms * 8, kPartStride); }

}  // namespace apc
