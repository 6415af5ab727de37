// Fused dense operator pair of one LSQR iteration on sm_100a:
//
//     u <- A z - alpha * u/beta      (Matrix::matvec, matrix.hpp:151-171, with
//                                     the u update of lsqr.hpp:139-145)
//     ||u||^2                        (-> beta)
//     g  = A^T u                     (Matrix::matvec_transpose, matrix.hpp:186-195)
//
// dense_fwd_kernel + dense_adj_kernel stream A from HBM twice per iteration
// (16 m n bytes, at 99% of the HBM roof: nothing left to gain there).  This
// kernel reads A ONCE: a row panel of A stays in shared memory between the two
// products.
//
//   * A^T u needs whole entries of u, i.e. complete rows of A z, so a panel of
//     rb rows must be held on chip across all n columns.  One SM cannot (n x 8
//     bytes per row); a GROUP of g CTAs can: CTA j of the group keeps the
//     rb x W slice of its W = n/g columns, the g partial row sums meet through
//     L2 (rb doubles per CTA and panel, g <= 37: a few % of the tile bytes).
//   * The panel copy of A (DensePanels, apc_internal.hpp) makes that slice one
//     contiguous run, so a tile is a single bulk (TMA) copy completing on an
//     mbarrier, however small rb is (rb = 4 at n = 50000).
//   * Warp-specialised, every role loops over the group's panels on its own and
//     meets the others only through mbarriers, so the exchange latency of one
//     panel hides behind the tiles of the next ones (S stages of ~40 KB):
//       producer (1 thread)  empty[s] -> bulk copy -> full[s]
//       P1 (8 warps)         full[s]  -> partial rows of A z (own columns) -> p1[s]
//       X  (7 warps, one panel each in turn; with the producer and the 16
//          compute warps that is 24 warps: 25 would round to 28 in the
//          register file and cap the kernel at 72 registers with spills)
//                            p1[s] -> publish the CTA's rb partials as flagged
//                            words (two 8-byte words {32 data bits | (launch
//                            epoch, panel) tag}: a matching tag proves the data,
//                            no fence / counter / flag poll), gather the group's
//                            g partials the same way and add them in CTA order
//                            (every CTA gets the same bits) -> u of the panel in
//                            shared memory -> ub[s]; the panel's designated CTA
//                            folds -alpha*u_old/beta into its partial, stores u
//                            and adds ||u||^2
//       P2 (8 warps)         ub[s] -> column sums of the tile times u, kept in
//                            registers over ALL panels -> empty[s]
//     At the end the groups' column sums and the CTAs' norm partials are added
//     in a fixed order (reruns are bit-identical).
//   * All CTAs must be co-resident (they wait on each other): cooperative
//     launch, one CTA per SM.
#include "dense_pair.hpp"
#include "dev_common.cuh"

#include <algorithm>
#include <cstdlib>

namespace apc {

namespace {

constexpr int kDpRoleThreads = 256;  // P1 and P2: 8 warps each
#ifndef APC_DP_NX
#define APC_DP_NX 7
#endif
#ifndef APC_DP_EVICT
#define APC_DP_EVICT 1
#endif
#ifndef APC_DP_BATCH
#define APC_DP_BATCH 5
#endif
constexpr int kDpNX = APC_DP_NX;     // exchange warps
constexpr int kDpBatch = APC_DP_BATCH;         // partials polled together by one lane
constexpr int kDpThreads = 32 + kDpNX * 32 + 2 * kDpRoleThreads;
constexpr int kDpKmax = 22;          // tile elements per P1/P2 thread
constexpr int kDpTileMax = kDpKmax * kDpRoleThreads;  // 5632 doubles = 44 KB
constexpr int kDpMaxStages = 12;
constexpr size_t kDpSmemMax = 227 * 1024;

struct DpArgs {
  const double* ap;
  long long mloc, n, npanels;
  int rb, W, g, gact, ng, stages, nslot;  // gact: CTAs of a group that own columns
  const double* z;
  double* u;
  const LsqrState* st;
  double* part;
  double* gpart;
  double* nrmp;
  unsigned* cnt;
  double* gout;
  const int* done;
  int debug;  // APC_DP_DEBUG (experiments only; results are wrong when set)
};

__device__ __forceinline__ unsigned dp_smem(const void* p) {
  return static_cast<unsigned>(__cvta_generic_to_shared(p));
}
__device__ __forceinline__ void dp_bar_init(unsigned long long* b, unsigned count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(dp_smem(b)), "r"(count) : "memory");
}
__device__ __forceinline__ void dp_bar_arrive(unsigned long long* b) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(dp_smem(b)) : "memory");
}
__device__ __forceinline__ void dp_bar_expect(unsigned long long* b, unsigned bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(dp_smem(b)), "r"(bytes) : "memory");
}
__device__ __forceinline__ void dp_bar_wait(unsigned long long* b, unsigned parity) {
  asm volatile(
      "{\n .reg .pred p;\n DPWAIT_%=:\n mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n @!p bra DPWAIT_%=;\n}" ::"r"(
          dp_smem(b)),
      "r"(parity)
      : "memory");
}
// A is streamed once per launch and is far larger than L2: its lines are
// marked evict-first so the explicit basis B, K and the n-space vectors of the
// LSQR iteration (~100 MB) stay L2-resident from one iteration to the next
__device__ __forceinline__ unsigned long long dp_evict_first_policy() {
  unsigned long long pol;
  asm volatile("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(pol));
  return pol;
}
__device__ __forceinline__ void dp_bulk(void* dst, const void* src, unsigned bytes, unsigned long long* bar,
                                        unsigned long long pol) {
#if APC_DP_EVICT
  asm volatile(
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes.L2::cache_hint [%0], [%1], %2, [%3], %4;" ::"r"(
          dp_smem(dst)),
      "l"(src), "r"(bytes), "r"(dp_smem(bar)), "l"(pol)
      : "memory");
#else
  (void)pol;
  asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
                   dp_smem(dst)),
               "l"(src), "r"(bytes), "r"(dp_smem(bar))
               : "memory");
#endif
}
__device__ __forceinline__ void dp_st_ll(ulonglong2* p, unsigned long long w0, unsigned long long w1) {
  asm volatile("st.volatile.global.v2.u64 [%0], {%1, %2};" ::"l"(p), "l"(w0), "l"(w1) : "memory");
}
__device__ __forceinline__ void dp_ld_ll(const ulonglong2* p, unsigned long long& w0, unsigned long long& w1) {
  asm volatile("ld.volatile.global.v2.u64 {%0, %1}, [%2];" : "=l"(w0), "=l"(w1) : "l"(p) : "memory");
}
__device__ __forceinline__ unsigned dp_ld_acquire(const unsigned* p) {
  unsigned v;
  asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}

__global__ void __launch_bounds__(kDpThreads, 1) dense_pair_kernel(DpArgs a) {
  extern __shared__ __align__(128) unsigned char dp_raw[];
  if (a.done && *a.done) return;
  const int S = a.stages, rb = a.rb;
  const int q = blockIdx.x / a.g, jg = blockIdx.x % a.g;   // group, CTA within the group
  const long long c0 = static_cast<long long>(jg) * a.W;   // first column of the slice
  const bool active = jg < a.gact;
  const int Wj = active ? static_cast<int>(a.n - c0 < a.W ? a.n - c0 : a.W) : 0;
  const int elems = Wj * rb;                                // doubles per tile
  const int tile_stride = a.W * rb;                         // doubles between stages (16-byte multiple)
  // the group's panels: p = q + ng * i
  const int ni = static_cast<int>(active && a.npanels > q ? (a.npanels - q + a.ng - 1) / a.ng : 0);  // < 2^21 (dp_plan)

  double* tiles = reinterpret_cast<double*>(dp_raw);
  double* sred = tiles + static_cast<size_t>(S) * tile_stride;  // S x 8 warps x 32
  double* us = sred + static_cast<size_t>(S) * 8 * 32;          // S x 32
  unsigned long long* bars = reinterpret_cast<unsigned long long*>(us + static_cast<size_t>(S) * 32);
  unsigned long long* full = bars;
  unsigned long long* empty = bars + S;
  unsigned long long* p1b = bars + 2 * S;
  unsigned long long* ub = bars + 3 * S;
  double* nrm_s = reinterpret_cast<double*>(bars + 4 * S);  // kDpNX
  __shared__ int last_flag;

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  if (threadIdx.x == 0) {
    for (int s = 0; s < S; ++s) {
      dp_bar_init(full + s, 1);
      dp_bar_init(empty + s, kDpRoleThreads);
      dp_bar_init(p1b + s, 8);
      dp_bar_init(ub + s, 1);
    }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncthreads();

  if (warp == 0) {
    // ---------------- producer ----------------
    if (lane == 0) {
      const unsigned bytes = static_cast<unsigned>(elems) * 8u;
      const unsigned long long pol = dp_evict_first_policy();
      // stage / round parity by counting: no 64-bit divisions in the per-panel loops
      int s = 0;
      unsigned ph = 0;
      for (int i = 0; i < ni; ++i, s = s + 1 == S ? 0 : s + 1, ph ^= s == 0 ? 1u : 0u) {
        dp_bar_wait(empty + s, ph ^ 1u);
        const long long p = q + static_cast<long long>(a.ng) * i;
        const double* src = a.ap + (p * a.n + c0) * rb;
        double* dst = tiles + static_cast<size_t>(s) * tile_stride;
        if (a.debug & 8) {
          dp_bar_arrive(full + s);
          continue;
        }
        dp_bar_expect(full + s, bytes);
        for (unsigned off = 0; off < bytes; off += 16384u) {
          const unsigned len = bytes - off < 16384u ? bytes - off : 16384u;
          dp_bulk(reinterpret_cast<unsigned char*>(dst) + off, reinterpret_cast<const unsigned char*>(src) + off, len,
                  full + s, pol);
        }
      }
    }
  } else if (warp <= kDpNX) {
    // ---------------- exchange ----------------
    const int xw = warp - 1;
    double alpha = 0.0, beta = 0.0;
    if (a.st) {
      alpha = a.st->alpha;
      beta = a.st->beta;
    }
    const int r = lane % rb, qq = lane / rb, nq = 32 / rb;
    const unsigned epoch = a.cnt[2];  // launches so far (bumped by the last CTA of each launch)
    double nrm = 0.0;
    // at most S exchange warps take part: a warp's first panel must belong to
    // round 0 of its stage (a parity wait on a fresh mbarrier for round 1
    // passes at once), and its later ones then follow completed rounds
    const int nxw = S < kDpNX ? S : kDpNX;
    for (int i = xw < nxw ? xw : ni; i < ni; i += nxw) {
      const int s = i % S;
      const unsigned ph = static_cast<unsigned>((i / S) & 1);
      const long long p = q + static_cast<long long>(a.ng) * i;
      const bool mine = i % a.gact == jg;  // this CTA finalises the panel's u
      const long long row = p * rb + lane;
      double uo = 0.0;
      if (mine && a.st && lane < rb && row < a.mloc) uo = a.u[row];
      // flag-in-word exchange (no fence, no counter): every partial travels as
      // two 8-byte words {32 data bits | 32-bit flag}; a word is written and
      // read whole, so a word whose flag is this launch's (epoch, panel) tag
      // carries this panel's bits.  The slot held (epoch, i - nslot) or an
      // (epoch - 1, .) tag before.
      ulonglong2* slot = reinterpret_cast<ulonglong2*>(a.part) +
                         ((static_cast<long long>(q) * a.nslot + i % a.nslot) * a.g) * rb;
      const unsigned long long flag =
          static_cast<unsigned long long>(((epoch & 0x7FFu) << 21) | (static_cast<unsigned>(i + 1) & 0x1FFFFFu)) << 32;
      dp_bar_wait(p1b + s, ph);
      if (lane < rb) {
        const double* sr = sred + (static_cast<size_t>(s) * 8) * 32 + lane;
        double pv = 0.0;
#pragma unroll
        for (int w = 0; w < 8; ++w) pv += sr[w * 32];
        if (mine && a.st) pv -= alpha * (beta > 0.0 ? uo / beta : uo);
        const unsigned long long bits = static_cast<unsigned long long>(__double_as_longlong(pv));
        dp_st_ll(slot + static_cast<long long>(jg) * rb + lane, (bits & 0xFFFFFFFFull) | flag, (bits >> 32) | flag);
      }
      // the g partials of row r, CTA order; nq lanes share a row
      double sum = 0.0;
      for (int j0 = (a.debug & 1) ? a.gact : qq; j0 < a.gact; j0 += kDpBatch * nq) {
        unsigned long long lo[kDpBatch], hi[kDpBatch];
        bool ok;
        do {
#pragma unroll
          for (int k = 0; k < kDpBatch; ++k) {
            const int jj = j0 + k * nq;
            if (jj < a.gact) dp_ld_ll(slot + static_cast<long long>(jj) * rb + r, lo[k], hi[k]);
            else lo[k] = hi[k] = flag;
          }
          ok = true;
#pragma unroll
          for (int k = 0; k < kDpBatch; ++k)
            ok = ok && (lo[k] & 0xFFFFFFFF00000000ull) == flag && (hi[k] & 0xFFFFFFFF00000000ull) == flag;
        } while (!ok);
#pragma unroll
        for (int k = 0; k < kDpBatch; ++k) {
          const int jj = j0 + k * nq;
          if (jj < a.gact)
            sum += __longlong_as_double(static_cast<long long>((lo[k] & 0xFFFFFFFFull) | (hi[k] << 32)));
        }
      }
      for (int o = rb; o < 32; o <<= 1) sum += __shfl_xor_sync(0xffffffffu, sum, o);
      if (lane < rb) us[s * 32 + lane] = sum;
      __syncwarp();
      if (lane == 0) dp_bar_arrive(ub + s);
      if (mine && lane < rb && row < a.mloc) {
        a.u[row] = sum;
        nrm += sum * sum;
      }
    }
    nrm = warp_sum(nrm);
    if (lane == 0) nrm_s[xw] = nrm;
  } else if (warp <= kDpNX + 8) {
    // ---------------- P1: partial rows of A z ----------------
    const int t = threadIdx.x - 32 * (1 + kDpNX);
    const int w1 = t >> 5;
    double zr[kDpKmax];
#pragma unroll
    for (int k = 0; k < kDpKmax; ++k) {
      const int e = t + k * kDpRoleThreads;
      zr[k] = e < elems ? __ldg(a.z + c0 + e / rb) : 0.0;
    }
    for (long long i = 0; i < ni; ++i) {
      const int s = static_cast<int>(i % S);
      const unsigned ph = static_cast<unsigned>((i / S) & 1);
      dp_bar_wait(full + s, ph);
      const double* tile = tiles + static_cast<size_t>(s) * tile_stride + t;
      double acc = 0.0;
#pragma unroll
      for (int k = 0; k < kDpKmax; ++k)
        if (t + k * kDpRoleThreads < elems) acc += tile[k * kDpRoleThreads] * zr[k];
      for (int o = 16; o >= rb; o >>= 1) acc += __shfl_xor_sync(0xffffffffu, acc, o);
      if (lane < rb) sred[(static_cast<size_t>(s) * 8 + w1) * 32 + lane] = acc;
      __syncwarp();
      if (lane == 0) dp_bar_arrive(p1b + s);
    }
  } else {
    // ---------------- P2: column sums of the tile times u ----------------
    const int t = threadIdx.x - 32 * (1 + kDpNX) - kDpRoleThreads;
    const int r = t % rb;
    double acc[kDpKmax];
#pragma unroll
    for (int k = 0; k < kDpKmax; ++k) acc[k] = 0.0;
    for (long long i = 0; i < ni; ++i) {
      const int s = static_cast<int>(i % S);
      const unsigned ph = static_cast<unsigned>((i / S) & 1);
      dp_bar_wait(full + s, ph);  // the async-proxy writes of the tile
      dp_bar_wait(ub + s, ph);
      const double uv = us[s * 32 + r];
      const double* tile = tiles + static_cast<size_t>(s) * tile_stride + t;
#pragma unroll
      for (int k = 0; k < kDpKmax; ++k)
        if (t + k * kDpRoleThreads < elems) acc[k] += tile[k * kDpRoleThreads] * uv;
      dp_bar_arrive(empty + s);
    }
    double* gp = a.gpart + static_cast<long long>(q) * a.n + c0;
#pragma unroll
    for (int k = 0; k < kDpKmax; ++k) {
      double v = acc[k];
      for (int o = rb >> 1; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
      const int e = t + k * kDpRoleThreads;
      if (r == 0 && e < elems) __stcg(gp + e / rb, v);
    }
  }

  // ---------------- finish: the groups' column sums and the norm ----------------
  const unsigned G = gridDim.x;
  unsigned* fin = a.cnt;
  __syncthreads();
  if (threadIdx.x == 0) {
    double sn = 0.0;
    for (int k = 0; k < kDpNX; ++k) sn += nrm_s[k];
    __stcg(a.nrmp + blockIdx.x, sn);
    __threadfence();
    atomicAdd(fin, 1u);
    while (dp_ld_acquire(fin) < G) {
    }
  }
  __syncthreads();
  const long long cs = (a.n + G - 1) / G;
  const long long cb = static_cast<long long>(blockIdx.x) * cs;
  for (long long c = cb + threadIdx.x; c < cb + cs && c < a.n; c += kDpThreads) {
    double v = 0.0;
    for (int k = 0; k < a.ng; ++k) v += __ldcg(a.gpart + static_cast<long long>(k) * a.n + c);
    a.gout[c] = v;
  }
  if (blockIdx.x == 0 && warp == 0) {
    double v = 0.0;
    for (unsigned k = lane; k < G; k += 32) v += __ldcg(a.nrmp + k);
    v = warp_sum(v);
    if (lane == 0) a.gout[a.n] = v;
  }
  // the last CTA through re-arms the counters for the next launch
  __syncthreads();
  if (threadIdx.x == 0) last_flag = atomicAdd(fin + 1, 1u) == G - 1 ? 1 : 0;
  __syncthreads();
  if (last_flag && threadIdx.x == 0) {
    a.cnt[0] = 0u;
    a.cnt[1] = 0u;
    a.cnt[2] = a.cnt[2] + 1u;
  }
}

// ap[(p n + c) rb + r] = A(p rb + r, c)
__global__ void __launch_bounds__(256)
dense_panel_pack_kernel(const double* __restrict__ A, long long ld, long long mloc, long long n, int rb,
                        long long total, double* __restrict__ ap) {
  const long long stride = static_cast<long long>(gridDim.x) * blockDim.x;
  for (long long e = static_cast<long long>(blockIdx.x) * blockDim.x + threadIdx.x; e < total; e += stride) {
    const long long r = e % rb, pc = e / rb;
    const long long c = pc % n, p = pc / n;
    const long long row = p * rb + r;
    ap[e] = row < mloc ? __ldcs(A + c * ld + row) : 0.0;
  }
}

__global__ void __launch_bounds__(1024) pair_norm2_kernel(const double* __restrict__ y, long long m, double* out) {
  __shared__ double sh[32];
  double s = 0.0;
  for (long long i = threadIdx.x; i < m; i += 1024) s += y[i] * y[i];
  s = block_sum<1024>(s, sh);
  if (threadIdx.x == 0) *out = s;
}

int dp_env() {  // read per matrix (the tests force the path on small shapes)
  const char* e = std::getenv("APC_DENSE_PAIR");
  return e ? std::atoi(e) : -1;
}
int dp_env_int(const char* name, int dflt) {
  const char* e = std::getenv(name);
  return e ? std::atoi(e) : dflt;
}

size_t dp_smem_bytes(int stages, int tile_stride) {
  return static_cast<size_t>(stages) * (static_cast<size_t>(tile_stride) * 8 + 8 * 32 * 8 + 32 * 8 + 4 * 8) +
         kDpNX * 8 + 128;
}

bool dp_plan(apc_mat& a, DensePanels& d) {
  const int G = a.ctx->num_sms;
  const i64 mloc = a.mloc(), n = a.n;
  int ng = dp_env_int("APC_DP_GROUPS", G % 4 == 0 ? 4 : (G % 2 == 0 ? 2 : 1));
  if (ng < 1 || G % ng != 0) return false;
  const int g = G / ng;
  const int W = static_cast<int>((n + g - 1) / g);
  const int gact = static_cast<int>((n + W - 1) / W);  // CTAs of a group that own columns (the others idle)
  int rb = 32;
  while (rb >= 2 && static_cast<i64>(rb) * W > kDpTileMax) rb >>= 1;
  const int rb_env = dp_env_int("APC_DP_RB", 0);
  if (rb_env >= 2 && rb_env <= rb && (rb_env & (rb_env - 1)) == 0) rb = rb_env;
  if (rb < 2) return false;
  const int tile_stride = W * rb;
  int S = kDpMaxStages;
  while (S >= 3 && dp_smem_bytes(S, tile_stride) > kDpSmemMax) --S;
  const int s_env = dp_env_int("APC_DP_STAGES", 0);
  if (s_env >= 3 && s_env <= S) S = s_env;
  if (S < 3) return false;
  d.mloc = mloc;
  d.n = n;
  d.rb = rb;
  d.W = W;
  d.g = g;
  d.gact = gact;
  d.ng = ng;
  d.stages = S;
  d.nslot = 2 * S + 2;
  d.npanels = (mloc + rb - 1) / rb;
  if (d.npanels / ng + 2 >= (i64{1} << 21)) return false;  // the panel tag of the exchange has 21 bits
  d.smem = dp_smem_bytes(S, tile_stride);
  return true;
}

}  // namespace

bool dense_pair_ready(apc_mat& a) {
  DensePanels& d = a.panels;
  if (d.state != 0) return d.state > 0;
  d.state = -1;
  const int env = dp_env();
  if (env == 0 || a.sparse || a.mloc() <= 0 || a.n <= 0) return false;
  const double bytes = 8.0 * static_cast<double>(a.mloc()) * static_cast<double>(a.n);
  // measured down to 60 MB (L2-resident) the single pass still wins (3000 x 2500: 1.34x,
  // 10007 x 4001: 1.65x, profiles/r2e_dense_pair.md); below that the launch is
  // latency-bound either way and the panel copy is not worth its bytes
  if (env < 0 && bytes < 64e6) return false;
  if (!dp_plan(a, d)) return false;
  // narrow matrices: a panel costs ~0.8 us of pipeline latency whatever its
  // size, so tiles under 16 KB (n < ~2500) lose to the two streaming passes
  // (20000 x 1000: 0.126 ms against 0.083 ms)
  if (env < 0 && static_cast<i64>(d.rb) * d.W * 8 < 16384) return false;
  size_t free_b = 0, total_b = 0;
  APC_CUDA(cudaMemGetInfo(&free_b, &total_b));
  const size_t need = static_cast<size_t>(d.npanels) * d.n * d.rb * 8;
  if (env < 0 && free_b < need + (size_t{4} << 30)) {
    pool_trim();
    APC_CUDA(cudaMemGetInfo(&free_b, &total_b));
    if (free_b < need + (size_t{4} << 30)) return false;
  }
  APC_CUDA(cudaFuncSetAttribute(dense_pair_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                static_cast<int>(d.smem)));
  int per_sm = 0;
  APC_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, dense_pair_kernel, kDpThreads, d.smem));
  if (per_sm < 1) return false;
  cudaStream_t st = a.ctx->stream;
  const i64 total = d.npanels * d.n * d.rb;
  d.ap.alloc(total);
  d.part.alloc(2 * static_cast<i64>(d.ng) * d.nslot * d.g * d.rb);  // two 8-byte words per partial
  APC_CUDA(cudaMemsetAsync(d.part.p, 0, d.part.bytes(), st));
  d.gpart.alloc(static_cast<i64>(d.ng) * d.n);
  d.nrmp.alloc(static_cast<i64>(d.ng) * d.g);
  d.cnt.alloc(4);  // finish counters (zero between launches) and the launch epoch
  APC_CUDA(cudaMemsetAsync(d.cnt.p, 0, d.cnt.bytes(), st));
  dense_panel_pack_kernel<<<a.ctx->num_sms * 16, 256, 0, st>>>(a.dense.p, a.mloc(), a.mloc(), a.n, d.rb, total,
                                                               d.ap.p);
  a.ctx->launches++;
  APC_CUDA(cudaGetLastError());
  d.state = 1;
  return true;
}

void pair_norm2(apc_ctx* ctx, const double* y, long long m, double* out) {
  pair_norm2_kernel<<<1, 1024, 0, ctx->stream>>>(y, m, out);
  ctx->launches++;
}

void launch_dense_pair(apc_mat& a, const double* z, double* u, const LsqrState* st, double* g, const int* done) {
  DensePanels& d = a.panels;
  DpArgs args{d.ap.p, d.mloc, d.n, d.npanels, d.rb, d.W, d.g, d.gact, d.ng, d.stages, d.nslot,
              z, u, st, d.part.p, d.gpart.p, d.nrmp.p, d.cnt.p, g, done, dp_env_int("APC_DP_DEBUG", 0)};
  void* kargs[] = {&args};
  APC_CUDA(cudaLaunchCooperativeKernel(reinterpret_cast<const void*>(dense_pair_kernel), dim3(d.ng * d.g),
                                       dim3(kDpThreads), kargs, d.smem, a.ctx->stream));
  a.ctx->launches++;
}

}  // namespace apc
