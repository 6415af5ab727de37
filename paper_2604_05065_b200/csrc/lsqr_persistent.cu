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
#include <vector>

#include "dev_common.cuh"
#include "lsqr.hpp"
#include "lsqr_persistent.hpp"

namespace cg = cooperative_groups;

namespace apc {

#define STAMP(k) \
  if (P.prof && blockIdx.x == 0 && threadIdx.x == 0 && j < 64) P.prof[j * 8 + (k)] = globaltimer_ns()

namespace {

constexpr int kPT = 1024;  // threads per CTA: one fat CTA per SM keeps grid barriers cheap
constexpr int kNW = kPT / 32;
constexpr long long kSmemBudget = 200 * 1024;  // dynamic shared memory the kernel may use

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
  // vectors
  double *u, *v, *vr, *w, *y, *z, *h, *s, *t;
  double* part;  // gridDim.x x 4
  unsigned long long* prof;  // optional stage timestamps (first 64 iterations)
  LsqrState* st;
  TraceRow* trace;
};

__device__ __forceinline__ double grid_sum(const double* part, int slot, int nblocks, double* sh) {
  // every CTA sums the same per-CTA partials in the same order
  double v = 0.0;
  for (int b = threadIdx.x; b < nblocks; b += kPT) v += part[b * 4 + slot];
  return block_sum<kPT>(v, sh);
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
//   tsh = R (x / xdiv)                 (all l rows, thread per row, in order)
//   dsh[q - RT_ptr[c0]] = RT_val[q] * (K tsh)_{RT_idx[q]}   for q of the range
__device__ void cta_project(const PArgs& P, const double* x, double xdiv, const double* K, double* tsh,
                            double* dsh, long long c0, long long c1, int warp, int lane) {
  for (long long i = threadIdx.x; i < P.l; i += kPT) {
    const int b = __ldg(P.rptr + i), e = __ldg(P.rptr + i + 1);
    double acc = 0.0;
    for (int q = b; q < e; ++q) acc += __ldg(P.rval + q) * (x[__ldg(P.ridx + q)] / xdiv);
    tsh[i] = acc;
  }
  __syncthreads();
  const int qb0 = __ldg(P.rtptr + c0), qb1 = __ldg(P.rtptr + c1);
  for (int q = qb0 + warp; q < qb1; q += kNW) {
    const double* row = K + static_cast<long long>(__ldg(P.rtidx + q)) * P.l;
    double acc = 0.0;
    for (long long k = lane; k < P.l; k += 32) acc += __ldg(row + k) * tsh[k];
    acc = warp_sum(acc);
    if (lane == 0) dsh[q - qb0] = __ldg(P.rtval + q) * acc;
  }
  __syncthreads();
}

__global__ void __launch_bounds__(kPT, 1) lsqr_persistent_kernel(PArgs P) {
  extern __shared__ double dyn[];  // z copy (S3) / t + d (S12, S56): disjoint in time
  __shared__ double red[32];
  cg::grid_group grid = cg::this_grid();
  const long long gtid = static_cast<long long>(blockIdx.x) * kPT + threadIdx.x;
  const long long gsize = static_cast<long long>(gridDim.x) * kPT;
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
  // quantities of the last completed iteration, tested after the next B1
  bool pending = false, nonfinite = false;
  double cc = 0.0, cvgrate = 0.0, cvgdiff = 0.0;
  // v of the next S12 = vsrc / vdiv (first iteration: the initialised v)
  const double* vsrc = P.v;
  double vdiv = 1.0;
  double* tsh = dyn;
  double* dsh = dyn + P.l;

  for (;;) {
    // ---- S12: z = v + R^T Gf R v
    STAMP(0);
    if (P.pre) {
      if (P.fused) {
        cta_project(P, vsrc, vdiv, P.Gf, tsh, dsh, c0, c1, warp, lane);
        const int qb0 = __ldg(P.rtptr + c0);
        for (long long c = c0 + threadIdx.x; c < c1; c += kPT) {
          double acc = 0.0;
          for (int q = __ldg(P.rtptr + c); q < __ldg(P.rtptr + c + 1); ++q) acc += dsh[q - qb0];
          P.z[c] = P.v[c] + acc;
        }
      } else {
        grid_project(grid, P.rptr, P.ridx, P.rval, P.Gf, P.l, vsrc, vdiv, P.t, P.s, gwarp, nwarps, lane);
        grid.sync();
        for (long long c = c0 + threadIdx.x; c < c1; c += kPT) {
          double acc = 0.0;
          for (int q = P.rtptr[c]; q < P.rtptr[c + 1]; ++q) acc += P.rtval[q] * P.s[P.rtidx[q]];
          P.z[c] = P.v[c] + acc;
        }
      }
    }
    grid.sync();  // B1
    STAMP(1);
    if (pending) {
      // ---- stop tests of iteration j (lsqr.hpp:183-203), identical in every CTA
      const double ynorm = sqrt(grid_sum(P.part, 3, nb, red));
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
    // ---- S3: u <- A z - alpha u/beta ; tail rows
    const double* zg = P.pre ? P.z : P.v;
    const double* zs = zg;
    if (P.zsmem) {
      const long long h2 = P.n >> 1;
      const double2* src = reinterpret_cast<const double2*>(zg);
      double2* dst = reinterpret_cast<double2*>(dyn);
      for (long long i = threadIdx.x; i < h2; i += kPT) dst[i] = src[i];
      if ((P.n & 1) && threadIdx.x == 0) dyn[P.n - 1] = zg[P.n - 1];
      __syncthreads();
      zs = dyn;
    }
    STAMP(2);
    {
      double sq = 0.0, sqt = 0.0;
      const double rb = beta;
      if (P.sidx) {
        // SELL-32: warp = 32 consecutive rows, lane = row; idx/val coalesced
        for (long long ch = gwarp; ch < P.nchunks; ch += nwarps) {
          const long long r = ch * 32 + lane;
          const bool ok = r < P.mloc;
          const int len = ok ? __ldg(P.aptr + r + 1) - __ldg(P.aptr + r) : 0;
          const long long off = __ldg(P.soff + ch) + lane;
          const int* ip = P.sidx + off;
          const double* vp = P.sval + off;
          double acc = 0.0;
          int k = 0;
          for (; k + 4 <= len; k += 4) {
            const int i0 = __ldg(ip + 32 * k), i1 = __ldg(ip + 32 * (k + 1));
            const int i2 = __ldg(ip + 32 * (k + 2)), i3 = __ldg(ip + 32 * (k + 3));
            const double a0 = __ldg(vp + 32 * k), a1 = __ldg(vp + 32 * (k + 1));
            const double a2 = __ldg(vp + 32 * (k + 2)), a3 = __ldg(vp + 32 * (k + 3));
            const double z0 = zs[i0], z1 = zs[i1], z2 = zs[i2], z3 = zs[i3];
            acc += a0 * z0;
            acc += a1 * z1;
            acc += a2 * z2;
            acc += a3 * z3;
          }
          for (; k < len; ++k) acc += __ldg(vp + 32 * k) * zs[__ldg(ip + 32 * k)];
          if (ok) {
            const double uo = P.u[r];
            const double uh = rb > 0.0 ? uo / rb : uo;
            const double t = acc - alpha * uh;
            P.u[r] = t;
            sq += t * t;
          }
        }
      } else {
        // thread per row (rows are short): 4-wide unrolling keeps gathers in flight
        for (long long r = gtid; r < P.mloc; r += gsize) {
          const int b = __ldg(P.aptr + r), e = __ldg(P.aptr + r + 1);
          double acc = 0.0;
          int q = b;
          for (; q + 4 <= e; q += 4) {
            const int i0 = __ldg(P.aidx + q), i1 = __ldg(P.aidx + q + 1);
            const int i2 = __ldg(P.aidx + q + 2), i3 = __ldg(P.aidx + q + 3);
            const double a0 = __ldg(P.aval + q), a1 = __ldg(P.aval + q + 1);
            const double a2 = __ldg(P.aval + q + 2), a3 = __ldg(P.aval + q + 3);
            const double z0 = zs[i0], z1 = zs[i1], z2 = zs[i2], z3 = zs[i3];
            acc += a0 * z0;
            acc += a1 * z1;
            acc += a2 * z2;
            acc += a3 * z3;
          }
          for (; q < e; ++q) acc += __ldg(P.aval + q) * zs[__ldg(P.aidx + q)];
          const double uo = P.u[r];
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
      sq = block_sum<kPT>(sq, red);
      sqt = block_sum<kPT>(sqt, red);
      if (threadIdx.x == 0) {
        P.part[blockIdx.x * 4 + 0] = sq;
        P.part[blockIdx.x * 4 + 1] = sqt;
      }
    }
    grid.sync();  // B2
    STAMP(3);
    // ---- S4: beta ; h = (A^T u + mu u_t) / beta  [plain: v_raw = h - beta v, ||v_raw||^2]
    const double bnew = sqrt(grid_sum(P.part, 0, nb, red) + grid_sum(P.part, 1, nb, red));
    {
      double sq = 0.0;
      for (long long c = gwarp; c < P.n; c += nwarps) {
        double a0 = 0.0, a1 = 0.0, a2 = 0.0, a3 = 0.0;
        const int e = __ldg(P.tptr + c + 1);
        int q = __ldg(P.tptr + c) + lane;
        for (; q + 96 < e; q += 128) {
          const int i0 = __ldg(P.tidx + q), i1 = __ldg(P.tidx + q + 32);
          const int i2 = __ldg(P.tidx + q + 64), i3 = __ldg(P.tidx + q + 96);
          const double v0 = __ldg(P.tval + q), v1 = __ldg(P.tval + q + 32);
          const double v2 = __ldg(P.tval + q + 64), v3 = __ldg(P.tval + q + 96);
          a0 += v0 * P.u[i0];
          a1 += v1 * P.u[i1];
          a2 += v2 * P.u[i2];
          a3 += v3 * P.u[i3];
        }
        for (; q < e; q += 32) a0 += __ldg(P.tval + q) * P.u[__ldg(P.tidx + q)];
        double acc = warp_sum((a0 + a1) + (a2 + a3));
        if (lane == 0) {
          if (P.has_tail) acc += P.mu * P.u[P.mloc + c];
          const double gj = bnew > 0.0 ? acc / bnew : acc;
          if (P.pre) {
            P.h[c] = gj;
          } else {
            const double t = gj - bnew * P.v[c];
            P.vr[c] = t;
            sq += t * t;
          }
        }
      }
      if (!P.pre) {
        sq = block_sum<kPT>(sq, red);
        if (threadIdx.x == 0) P.part[blockIdx.x * 4 + 2] = sq;
      }
    }
    grid.sync();  // B3
    STAMP(4);
    if (P.pre) {
      // ---- S56: v_raw = h + R^T Ga R h - beta v ; ||v_raw||^2
      double sq = 0.0;
      if (P.fused) {
        cta_project(P, P.h, 1.0, P.Ga, tsh, dsh, c0, c1, warp, lane);
        const int qb0 = __ldg(P.rtptr + c0);
        for (long long c = c0 + threadIdx.x; c < c1; c += kPT) {
          double acc = 0.0;
          for (int q = __ldg(P.rtptr + c); q < __ldg(P.rtptr + c + 1); ++q) acc += dsh[q - qb0];
          const double t = (P.h[c] + acc) - bnew * P.v[c];
          P.vr[c] = t;
          sq += t * t;
        }
      } else {
        grid_project(grid, P.rptr, P.ridx, P.rval, P.Ga, P.l, P.h, 1.0, P.t, P.s, gwarp, nwarps, lane);
        grid.sync();
        for (long long c = c0 + threadIdx.x; c < c1; c += kPT) {
          double acc = 0.0;
          for (int q = P.rtptr[c]; q < P.rtptr[c + 1]; ++q) acc += P.rtval[q] * P.s[P.rtidx[q]];
          const double t = (P.h[c] + acc) - bnew * P.v[c];
          P.vr[c] = t;
          sq += t * t;
        }
      }
      sq = block_sum<kPT>(sq, red);
      if (threadIdx.x == 0) P.part[blockIdx.x * 4 + 2] = sq;
      grid.sync();  // B4
    }
    STAMP(5);
    // ---- S7: alpha ; rotation (lsqr.hpp:145-171) ; owner-column updates ; ||y||^2
    const double anew = sqrt(grid_sum(P.part, 2, nb, red));
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
      for (long long c = c0 + threadIdx.x; c < c1; c += kPT) {
        const double vh = P.vr[c] / vdiv;
        P.v[c] = vh;
        const double wo = P.w[c];
        const double yn = P.y[c] + t1 * wo;
        P.y[c] = yn;
        P.w[c] = vh + t2 * wo;
        sq += yn * yn;
      }
      sq = block_sum<kPT>(sq, red);
      if (threadIdx.x == 0) P.part[blockIdx.x * 4 + 3] = sq;
    }
    pending = true;
    if (P.prof && blockIdx.x == 0 && threadIdx.x == 0 && j - 1 < 64) P.prof[(j - 1) * 8 + 6] = globaltimer_ns();
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
  int per_sm = 0;
  APC_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, lsqr_persistent_kernel, kPT, 0));
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
      if ((P.l + qmax) * 8 <= kSmemBudget) {
        P.fused = 1;
        smem_doubles = std::max(smem_doubles, P.l + qmax);
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
  void* kfn = reinterpret_cast<void*>(lsqr_persistent_kernel);
  const size_t smem = sizeof(double) * static_cast<size_t>(smem_doubles);
  APC_CUDA(cudaFuncSetAttribute(kfn, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(smem)));
  APC_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kfn, kPT, smem));
  require(per_sm >= blocks_per_sm, APC_CUDA_ERROR, "persistent LSQR: grid does not fit co-resident");
  P.part = b.part;
  void* args[] = {&P};
  APC_CUDA(cudaLaunchCooperativeKernel(kfn, dim3(grid), dim3(kPT), args, smem, ctx->stream));
  ctx->launches++;
}

int persistent_max_grid(apc_ctx* ctx) { return ctx->num_sms * 8; }

}  // namespace apc
