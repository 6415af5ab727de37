// Persistent cooperative LSQR phase for L2-resident sparse systems (the
// BASELINE C2 shape): ONE kernel launch runs every iteration of a phase, with
// grid-wide barriers between the dependent stages instead of ~11 kernel
// launches per iteration.  Each CTA carries its own copy of the scalar
// recurrence (alpha, beta, rhobar, phibar, ... of lsqr.hpp:132-203): every CTA
// reduces the same block partials in the same fixed order, so all copies stay
// bit-identical and no scalar ever round-trips through a broadcast.
//
// Stages per iteration (implicit preconditioner P^{-1} = I + R^T G R):
//   S1  CTA 0: t = R v, s = Gf t                                   | sync
//   S2  z = v + R^T s                                              | sync
//   S3  u <- A z - alpha u/beta_old ; u_tail <- mu z - alpha u_t/beta_old ;
//       ||u||^2 block partials                                     | sync
//   S4  beta ; h = (A^T u + mu u_t)/beta  (warp per row of A^T)    | sync
//   S5  CTA 0: t = R h, s = Ga t                                   | sync
//   S6  v = h + R^T s - beta v ; ||v||^2 partials                  | sync
//   S7  alpha, rotation ; v /= alpha ; y += t1 w ; w = v + t2 w ;
//       ||y||^2 partials                                           | sync
//   S8  ||y|| ; stop tests (lsqr.hpp:183-203) ; trace row
// Unpreconditioned phases skip S1, S2, S5 and fuse S6 into S4.
#include <cooperative_groups.h>

#include <algorithm>
#include <cstdlib>

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

struct PArgs {
  // A: CSR rows (mloc) and CSR of A^T (n rows, no split rows)
  const int *aptr, *aidx;
  const double* aval;
  const int *tptr, *tidx;
  const double* tval;
  long long mloc, n;
  double mu;
  int has_tail;
  int group;  // lanes per row of the forward SpMV (4/8/16/32)
  int zsmem;  // 1: z staged per CTA in shared memory (n small)
  // preconditioner (implicit) or identity
  int pre;
  const int *rptr, *ridx;
  const double* rval;
  const int *rtptr, *rtidx;
  const double* rtval;
  const double *Gf, *Ga;  // row-major l x l
  long long l;
  // vectors
  double *u, *v, *w, *y, *z, *h, *s, *t;
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

// s = K (M x) for the l x n sparse M (R) and row-major K, spread over the
// whole grid (one warp per row in each half, a barrier between them): the
// rows are short, so the stage is latency-bound and wants many warps.
__device__ void grid_project(cg::grid_group& grid, const int* mptr, const int* midx, const double* mval,
                             const double* KT, long long l, const double* x, double* t, double* s_out,
                             long long gwarp, long long nwarps, int lane) {
  for (long long i = gwarp; i < l; i += nwarps) {
    double acc = 0.0;
    for (int q = mptr[i] + lane; q < mptr[i + 1]; q += 32) acc += mval[q] * x[midx[q]];
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

template <int G>
__global__ void __launch_bounds__(kPT, 1) lsqr_persistent_kernel(PArgs P) {
  extern __shared__ double tsh[];  // l doubles (preconditioner)
  __shared__ double red[32];
  cg::grid_group grid = cg::this_grid();
  const long long gtid = static_cast<long long>(blockIdx.x) * kPT + threadIdx.x;
  const long long gsize = static_cast<long long>(gridDim.x) * kPT;
  const long long gwarp = gtid >> 5, nwarps = gsize >> 5;
  const int lane = threadIdx.x & 31;
  const int nb = gridDim.x;
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
  // small n: every CTA builds its own copy of z in shared memory (the forward
  // SpMV then gathers from smem instead of L2, and the z stage needs no grid
  // barrier); otherwise z goes through global memory
  const double* zsrc = P.zsmem ? tsh : (P.pre ? P.z : P.v);

  for (;;) {
    // ---- S1/S2: z = v + R^T Gf R v
    STAMP(0);
    if (P.pre) {
      grid_project(grid, P.rptr, P.ridx, P.rval, P.Gf, P.l, P.v, P.t, P.s, gwarp, nwarps, lane);
      grid.sync();
      STAMP(1);
    }
    if (P.zsmem) {
      for (long long c = threadIdx.x; c < P.n; c += kPT) {
        double acc = 0.0;
        if (P.pre)
          for (int q = P.rtptr[c]; q < P.rtptr[c + 1]; ++q) acc += P.rtval[q] * P.s[P.rtidx[q]];
        tsh[c] = P.pre ? P.v[c] + acc : P.v[c];
      }
      __syncthreads();
      STAMP(2);
    } else if (P.pre) {
      for (long long c = gtid; c < P.n; c += gsize) {
        double acc = 0.0;
        for (int q = P.rtptr[c]; q < P.rtptr[c + 1]; ++q) acc += P.rtval[q] * P.s[P.rtidx[q]];
        P.z[c] = P.v[c] + acc;
      }
      grid.sync();
      STAMP(2);
    }
    // ---- S3: u <- A z - alpha u/beta ; tail rows
    {
      double sq = 0.0, sqt = 0.0;
      // thread per row (rows are short): every load of a row is independent of
      // the add chain, so 4-wide unrolling keeps several gathers in flight
      for (long long r = gtid; r < P.mloc; r += gsize) {
        const int b = P.aptr[r], e = P.aptr[r + 1];
        double acc = 0.0;
        int q = b;
        for (; q + 4 <= e; q += 4) {
          const int c0 = P.aidx[q], c1 = P.aidx[q + 1], c2 = P.aidx[q + 2], c3 = P.aidx[q + 3];
          const double v0 = P.aval[q], v1 = P.aval[q + 1], v2 = P.aval[q + 2], v3 = P.aval[q + 3];
          const double z0 = zsrc[c0], z1 = zsrc[c1], z2 = zsrc[c2], z3 = zsrc[c3];
          acc += v0 * z0;
          acc += v1 * z1;
          acc += v2 * z2;
          acc += v3 * z3;
        }
        for (; q < e; ++q) acc += P.aval[q] * zsrc[P.aidx[q]];
        {
          const double uo = P.u[r];
          const double uh = beta > 0.0 ? uo / beta : uo;
          const double t = acc - alpha * uh;
          P.u[r] = t;
          sq += t * t;
        }
      }
      if (P.has_tail) {
        double* ut = P.u + P.mloc;
        for (long long c = gtid; c < P.n; c += gsize) {
          const double uo = ut[c];
          const double uh = beta > 0.0 ? uo / beta : uo;
          const double t = P.mu * zsrc[c] - alpha * uh;
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
    grid.sync();
    STAMP(3);
    // ---- S4: beta ; h = (A^T u + mu u_t) / beta  [plain: v = h - beta v, ||v||^2]
    const double bnew = sqrt(grid_sum(P.part, 0, nb, red) + grid_sum(P.part, 1, nb, red));
    {
      double sq = 0.0;
      for (long long c = gwarp; c < P.n; c += nwarps) {
        double acc = 0.0, acc2 = 0.0;
        const int e = P.tptr[c + 1];
        int q = P.tptr[c] + lane;
        for (; q + 32 < e; q += 64) {
          const int i0 = P.tidx[q], i1 = P.tidx[q + 32];
          const double v0 = P.tval[q], v1 = P.tval[q + 32];
          acc += v0 * P.u[i0];
          acc2 += v1 * P.u[i1];
        }
        if (q < e) acc += P.tval[q] * P.u[P.tidx[q]];
        acc = warp_sum(acc + acc2);
        if (lane == 0) {
          if (P.has_tail) acc += P.mu * P.u[P.mloc + c];
          const double gj = bnew > 0.0 ? acc / bnew : acc;
          if (P.pre) {
            P.h[c] = gj;
          } else {
            const double t = gj - bnew * P.v[c];
            P.v[c] = t;
            sq += t * t;
          }
        }
      }
      if (!P.pre) {
        sq = block_sum<kPT>(sq, red);
        if (threadIdx.x == 0) P.part[blockIdx.x * 4 + 2] = sq;
      }
    }
    grid.sync();
    STAMP(4);
    if (P.pre) {
      // ---- S5/S6: v = h + R^T Ga R h - beta v ; ||v||^2
      grid_project(grid, P.rptr, P.ridx, P.rval, P.Ga, P.l, P.h, P.t, P.s, gwarp, nwarps, lane);
      grid.sync();
      STAMP(5);
      double sq = 0.0;
      for (long long c = gtid; c < P.n; c += gsize) {
        double acc = 0.0;
        for (int q = P.rtptr[c]; q < P.rtptr[c + 1]; ++q) acc += P.rtval[q] * P.s[P.rtidx[q]];
        const double t = (P.h[c] + acc) - bnew * P.v[c];
        P.v[c] = t;
        sq += t * t;
      }
      sq = block_sum<kPT>(sq, red);
      if (threadIdx.x == 0) P.part[blockIdx.x * 4 + 2] = sq;
      grid.sync();
      STAMP(6);
    }
    // ---- S7: alpha ; rotation (lsqr.hpp:145-171) ; vector updates ; ||y||^2
    const double anew = sqrt(grid_sum(P.part, 2, nb, red));
    beta = bnew;
    alpha = anew;
    opnorm2 += alpha * alpha + beta * beta;
    const double rho = hypot(rhobar, beta);
    const double c = rhobar / rho;
    const double s = beta / rho;
    const double theta = s * alpha;
    rhobar = -c * alpha;
    const double phi = c * phibar;
    const double phibar_prev = phibar;
    phibar = s * phibar;
    const double t1 = phi / rho, t2 = -theta / rho;
    ++j;
    const bool nonfinite = !isfinite(phibar) || !isfinite(alpha) || !isfinite(beta);
    const double cvgrate = (phibar > 0.0 && phibar_prev > 0.0) ? log(phibar_prev / phibar) : CUDART_INF;
    const double cvgdiff = phibar_prev - phibar;
    if (j == 1) cvgrate1 = cvgrate;
    {
      double sq = 0.0;
      for (long long cc = gtid; cc < P.n; cc += gsize) {
        const double vo = P.v[cc];
        const double vh = alpha > 0.0 ? vo / alpha : vo;
        P.v[cc] = vh;
        const double wo = P.w[cc];
        const double yn = P.y[cc] + t1 * wo;
        P.y[cc] = yn;
        P.w[cc] = vh + t2 * wo;
        sq += yn * yn;
      }
      sq = block_sum<kPT>(sq, red);
      if (threadIdx.x == 0) P.part[blockIdx.x * 4 + 3] = sq;
    }
    grid.sync();
    if (P.prof && blockIdx.x == 0 && threadIdx.x == 0 && j - 1 < 64) P.prof[(j - 1) * 8 + 7] = globaltimer_ns();
    // ---- S8: stop tests (identical decision in every CTA)
    const double ynorm = sqrt(grid_sum(P.part, 3, nb, red));
    int reason = kReasonNone;
    bool stop = false;
    if (nonfinite) {
      stop = true;
    } else {
      const double grad = phibar * alpha * fabs(c);
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
  }
  P.u = b.u;
  P.v = b.v;
  P.w = b.w;
  P.y = b.y;
  P.z = b.z;
  P.h = b.h;
  P.s = b.s;
  P.t = b.t;
  P.prof = b.prof;
  P.st = b.st;
  P.trace = b.trace;
  const int G = csr_group_size_p(a.a.avg_row_nnz);
  void* kfn = nullptr;
  switch (G) {
    case 4: kfn = reinterpret_cast<void*>(lsqr_persistent_kernel<4>); break;
    case 8: kfn = reinterpret_cast<void*>(lsqr_persistent_kernel<8>); break;
    case 16: kfn = reinterpret_cast<void*>(lsqr_persistent_kernel<16>); break;
    default: kfn = reinterpret_cast<void*>(lsqr_persistent_kernel<32>); break;
  }
  P.group = G;
  // measured on C2: the per-CTA z build costs more (latency-bound RT walk) than
  // the L2 gathers it saves, so shared-memory z is opt-in only
  P.zsmem = (P.n * 8 <= 200 * 1024 && std::getenv("APC_PERSISTENT_ZSMEM")) ? 1 : 0;
  const size_t smem = sizeof(double) * static_cast<size_t>(std::max<long long>(1, P.zsmem ? P.n : 1));
  if (smem > 48 * 1024) APC_CUDA(cudaFuncSetAttribute(kfn, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
  int per_sm = 0;
  APC_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kfn, kPT, smem));
  // fewer CTAs make each grid barrier cheaper; the L2-resident stages need
  // only a couple of CTAs per SM to saturate
  const int blocks_per_sm = std::max(1, std::min(per_sm, b.blocks_per_sm > 0 ? b.blocks_per_sm : 3));
  const int grid = ctx->num_sms * blocks_per_sm;
  double* part = b.part;
  P.part = part;
  void* args[] = {&P};
  APC_CUDA(cudaLaunchCooperativeKernel(kfn, dim3(grid), dim3(kPT), args, smem, ctx->stream));
  ctx->launches++;
}

int persistent_max_grid(apc_ctx* ctx) { return ctx->num_sms * 8; }

}  // namespace apc
