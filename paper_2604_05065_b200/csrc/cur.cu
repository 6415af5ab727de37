// Exact-order CUR kernels + the DeviceCur state machine (see cur.hpp).
//
// "Exact order" means: every output element is produced by the same sequence
// of IEEE operations as the reference's scalar loops (products and sums
// rounded separately, -fmad=false, sums in the reference's index order).  The
// parallelism comes from independent output elements, never from reordering a
// sum.  This is what makes I, J and rho_history bit-identical to the CPU.
#include <cooperative_groups.h>
#include <cub/device/device_radix_sort.cuh>
#include <cub/device/device_scan.cuh>

#include <algorithm>
#include <memory>
#include <chrono>
#include <climits>
#include <cmath>
#include <cstring>
#include <functional>
#include <numeric>

#include "blas.hpp"
#include "cur.hpp"
#include "lsqr.hpp"
#include "rng_dev.hpp"
#include "dev_common.cuh"
#include "ops.cuh"

namespace apc {

namespace {

constexpr int kT = 256;
inline unsigned nb(long long n, int t = kT) {
  return static_cast<unsigned>(std::max<long long>(1, (n + t - 1) / t));
}

// A(i, j) of a CSR matrix (columns sorted within rows): binary search
__device__ __forceinline__ double csr_at(const int* ptr, const int* idx, const double* val, long long i,
                                         long long j) {
  int lo = ptr[i], hi = ptr[i + 1];
  while (lo < hi) {
    int mid = (lo + hi) >> 1;
    if (idx[mid] < j) lo = mid + 1;
    else hi = mid;
  }
  return (lo < ptr[i + 1] && idx[lo] == j) ? val[lo] : 0.0;
}

// ---------------------------------------------------------------------------
// sketch Y = S * A (sparse sign), sketch.hpp:77-162.  One warp per column of
// A; Y(:, j) lives in shared memory; rows k in ascending order, each adding
// +-scale*A(k, j) to its xi rows (distinct within k, so lanes never collide).
// ---------------------------------------------------------------------------
constexpr int kSketchWarps = 8;

// Stage the S columns of a 32-row chunk (rows k0..k0+cnt-1 of A) in the warp's
// shared slice: one coalesced load round instead of a dependent load per row.
__device__ __forceinline__ void stage_s(const int* __restrict__ srow, const signed char* __restrict__ ssgn,
                                        long long k0, int cnt, int xi, int lane, int* rs, signed char* sg) {
  const int tot = cnt * xi;
  const long long base = k0 * xi;
  for (int e = lane; e < tot; e += 32) {
    rs[e] = srow[base + e];
    sg[e] = ssgn[base + e];
  }
  __syncwarp();
}

// same for a gathered list of rows (CSC column chunk): entry q is row kq
__device__ __forceinline__ void stage_s_rows(const int* __restrict__ srow, const signed char* __restrict__ ssgn,
                                             long long kq, bool valid, int xi, int lane, int* rs, signed char* sg) {
  if (valid)
    for (int t = 0; t < xi; ++t) {
      rs[lane * xi + t] = srow[kq * xi + t];
      sg[lane * xi + t] = ssgn[kq * xi + t];
    }
  __syncwarp();
}

struct SketchSmem {  // per-warp slices of the dynamic shared memory
  double* y;
  int* rs;
  signed char* sg;
};

__device__ __forceinline__ SketchSmem sketch_smem(double* base, int s, int xi, int w) {
  SketchSmem m;
  m.y = base + static_cast<long long>(w) * s;
  int* ri = reinterpret_cast<int*>(base + static_cast<long long>(kSketchWarps) * s);
  m.rs = ri + w * 32 * xi;
  signed char* sb = reinterpret_cast<signed char*>(ri + kSketchWarps * 32 * xi);
  m.sg = sb + w * 32 * xi;
  return m;
}

__global__ void __launch_bounds__(kSketchWarps * 32)
sketch_ss_dense_kernel(const double* __restrict__ A, long long m, long long n, int s, int xi,
                       const int* __restrict__ srow, const signed char* __restrict__ ssgn,
                       double scale, double mu_scale, int aug, int carry, double* __restrict__ Y) {
  extern __shared__ double ysh[];
  const int w = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const long long j = static_cast<long long>(blockIdx.x) * kSketchWarps + w;
  if (j >= n) return;
  SketchSmem sm = sketch_smem(ysh, s, xi, w);
  double* yc = sm.y;
  // carry: the running sums continue from the previous row block's (sharded setup)
  for (int i = lane; i < s; i += 32) yc[i] = carry ? Y[j * s + i] : 0.0;
  __syncwarp();
  const double* col = A + j * m;
  for (long long k0 = 0; k0 < m; k0 += 32) {
    const long long k = k0 + lane;
    const double v = k < m ? col[k] : 0.0;
    const int cnt = static_cast<int>(m - k0 < 32 ? m - k0 : 32);
    stage_s(srow, ssgn, k0, cnt, xi, lane, sm.rs, sm.sg);
    for (int kk = 0; kk < cnt; ++kk) {
      const double vk = __shfl_sync(0xffffffffu, v, kk);
      if (vk != 0.0) {
        const double sv = scale * vk;
        if (lane < xi) yc[sm.rs[kk * xi + lane]] += sv * static_cast<double>(sm.sg[kk * xi + lane]);
      }
      __syncwarp();
    }
  }
  if (aug && lane < xi) {  // mu tail: column m + j of S (sketch.hpp:152-160)
    const long long e = (m + j) * xi + lane;
    yc[srow[e]] += mu_scale * static_cast<double>(ssgn[e]);
  }
  __syncwarp();
  for (int i = lane; i < s; i += 32) Y[j * s + i] = yc[i];
}

// Dense A, inverted over S: every sketch row r keeps its own list of the A
// rows k that feed it (ascending k, packed k << 1 | sign > 0), so Y(r, j) is
// one thread's running sum, added in exactly the reference's k order
// (sketch.hpp:77-111: rows ascending, zero entries skipped).  A CTA takes
// kInvCols columns; their rows are staged kInvRows at a time in shared memory
// (coalesced, each A element read once), and each thread walks its list
// through the chunk for all kInvCols columns at once.  A is streamed once:
// HBM-bound instead of one dependent shared-memory update per row of A.
#ifndef APC_INV_COLS
#define APC_INV_COLS 4
#endif
constexpr int kInvCols = APC_INV_COLS;  // columns of A per CTA
constexpr int kInvRows = 256;
__device__ __forceinline__ unsigned inv_smem_u32(const void* p) {
  return static_cast<unsigned>(__cvta_generic_to_shared(p));
}
__device__ __forceinline__ void inv_bulk(void* dst, const void* src, unsigned bytes, unsigned long long* bar) {
  asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
                   inv_smem_u32(dst)),
               "l"(src), "r"(bytes), "r"(inv_smem_u32(bar))
               : "memory");
}
// chunk [c0, c0 + rows) of the CTA's columns and the chunk's S entries -> one
// buffer (bulk copies completing on bar; plain loads when a copy would be
// misaligned)
__device__ __forceinline__ void inv_stage(const double* __restrict__ A, long long m, long long j0, int nc,
                                          long long c0, int rows, const short* __restrict__ ent, int xi,
                                          double* abuf, short* ebuf, unsigned long long* bar, bool tma) {
  const unsigned abytes = static_cast<unsigned>(rows) * 8u;
  const unsigned ebytes = static_cast<unsigned>(rows) * static_cast<unsigned>(xi) * 2u;
  const short* esrc = ent + c0 * xi;
  if (tma) {
    if (threadIdx.x == 0) {
      // the block barrier ordered the generic reads of this buffer; hand it to the async proxy
      asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
      asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(inv_smem_u32(bar)),
                   "r"(abytes * static_cast<unsigned>(nc) + ebytes)
                   : "memory");
      for (int c = 0; c < nc; ++c) inv_bulk(abuf + c * kInvRows, A + (j0 + c) * m + c0, abytes, bar);
      inv_bulk(ebuf, esrc, ebytes, bar);
    }
  } else {
    for (int c = 0; c < nc; ++c) {
      const double* col = A + (j0 + c) * m + c0;
      for (int i = threadIdx.x; i < rows; i += blockDim.x) abuf[c * kInvRows + i] = __ldcs(col + i);
    }
    for (int i = threadIdx.x; i < rows * xi; i += blockDim.x) ebuf[i] = esrc[i];
  }
}
__device__ __forceinline__ void inv_wait(unsigned long long* bar, unsigned phase) {
  asm volatile(
      "{\n .reg .pred p;\n IWAIT_%=:\n mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n @!p bra IWAIT_%=;\n}" ::"r"(
          inv_smem_u32(bar)),
      "r"(phase)
      : "memory");
}

// Dense A, inverted over S: Y(r, j) is one thread's running sum over the A rows
// k that feed sketch row r, added in exactly the reference's k order
// (sketch.hpp:77-111: rows ascending, zero entries skipped).  The S entries are
// stored chunk-major: for each chunk of kInvRows rows of A, by target row r,
// k ascending within r, packed (k - chunk start) << 1 | sign > 0 in 16 bits,
// with cptr[chunk * (s + 1) + r] the offset of r's run inside the chunk.  A
// CTA takes kInvCols columns; every chunk (those columns' rows and the chunk's
// S entries) is staged by TMA bulk copies, double-buffered, and each thread
// walks its run in shared memory for all kInvCols columns at once.  A is read
// from HBM exactly once.
__global__ void __launch_bounds__(1024)
sketch_ss_dense_inv_kernel(const double* __restrict__ A, long long m, long long n, int s, int xi,
                           const int* __restrict__ cptr, const short* __restrict__ ent,
                           const int* __restrict__ srow, const signed char* __restrict__ ssgn, double scale,
                           double mu_scale, int aug, int carry, double* __restrict__ Y) {
  // [2 x (kInvCols x kInvRows doubles)] [2 x (kInvRows x xi shorts)] [s x kInvCols doubles: mu tail]
  extern __shared__ __align__(16) double dyn_inv[];
  __shared__ __align__(8) unsigned long long bars[2];
  double* abuf = dyn_inv;
  short* ebuf = reinterpret_cast<short*>(dyn_inv + 2 * kInvCols * kInvRows);
  const int estride = (kInvRows * xi + 7) & ~7;  // shorts per entry buffer (16-byte multiple)
  double* ysh = reinterpret_cast<double*>(ebuf + 2 * estride);
  const long long j0 = static_cast<long long>(blockIdx.x) * kInvCols;
  const int nc = static_cast<int>(n - j0 < kInvCols ? n - j0 : kInvCols);
  const int r = threadIdx.x;
  const bool own = r < s;
  double acc[kInvCols];
#pragma unroll
  for (int c = 0; c < kInvCols; ++c) acc[c] = (carry && own && c < nc) ? Y[(j0 + c) * s + r] : 0.0;
  // bulk copies need 16-byte aligned columns and copy sizes
  const bool tma = (m % 2 == 0) && (xi % 8 == 0) && ((reinterpret_cast<unsigned long long>(A) & 15ull) == 0) &&
                   ((reinterpret_cast<unsigned long long>(ent) & 15ull) == 0);
  if (threadIdx.x == 0) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(inv_smem_u32(&bars[0])) : "memory");
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(inv_smem_u32(&bars[1])) : "memory");
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncthreads();
  const long long nchunks = (m + kInvRows - 1) / kInvRows;
  auto rows_of = [&](long long ch) { return static_cast<int>(m - ch * kInvRows < kInvRows ? m - ch * kInvRows : kInvRows); };
  if (nchunks > 0) inv_stage(A, m, j0, nc, 0, rows_of(0), ent, xi, abuf, ebuf, &bars[0], tma);
  int rb = own ? __ldg(cptr + r) : 0, re = own ? __ldg(cptr + r + 1) : 0;
  for (long long ch = 0; ch < nchunks; ++ch) {
    const int b = static_cast<int>(ch & 1);
    if (ch + 1 < nchunks)  // the other buffer was released by the barrier at the end of ch - 1
      inv_stage(A, m, j0, nc, (ch + 1) * kInvRows, rows_of(ch + 1), ent, xi, abuf + (1 - b) * kInvCols * kInvRows,
                ebuf + (1 - b) * estride, &bars[1 - b], tma);
    // this thread's run in the next chunk (prefetched while this one is walked)
    int nrb = 0, nre = 0;
    if (own && ch + 1 < nchunks) {
      nrb = __ldg(cptr + (ch + 1) * (s + 1) + r);
      nre = __ldg(cptr + (ch + 1) * (s + 1) + r + 1);
    }
    if (tma) inv_wait(&bars[b], static_cast<unsigned>((ch >> 1) & 1));
    else __syncthreads();
    // sv = scale * A(k, j) once per element (the reference computes it once per
    // row k and adds sv * (+-1) to each of its xi targets).  A zero A(k, j) is
    // skipped by the reference; a nonzero one whose sv underflows to +-0 would
    // add +-0, which cannot change a sum that starts at +0 -- so testing sv
    // instead of A(k, j) keeps every bit.
    double* asw = abuf + b * kInvCols * kInvRows;
    for (int i = threadIdx.x; i < nc * kInvRows; i += blockDim.x) asw[i] = scale * asw[i];
    __syncthreads();
    const double* as = asw;
    const short* es = ebuf + b * estride;
    for (int i = rb; i < re; ++i) {
      const int e = es[i];
      const int kk = e >> 1;
      const bool pos = (e & 1) != 0;
#pragma unroll
      for (int c = 0; c < kInvCols; ++c) {
        const double sv = as[c * kInvRows + kk];
        if (c < nc && sv != 0.0) acc[c] += pos ? sv : -sv;  // sv * (+-1.0), exact
      }
    }
    rb = nrb;
    re = nre;
    __syncthreads();  // every thread is done with buffer b before it is refilled
  }
  if (aug) {  // mu tail: column m + j of S (sketch.hpp:152-160), added last
#pragma unroll
    for (int c = 0; c < kInvCols; ++c)
      if (own && c < nc) ysh[c * s + r] = acc[c];
    __syncthreads();
    if (threadIdx.x < xi)
      for (int c = 0; c < nc; ++c) {
        const long long e = (m + j0 + c) * xi + threadIdx.x;
        ysh[c * s + srow[e]] += mu_scale * static_cast<double>(ssgn[e]);
      }
    __syncthreads();
    for (int c = 0; c < nc; ++c)
      if (own) Y[(j0 + c) * s + r] = ysh[c * s + r];
  } else {
#pragma unroll
    for (int c = 0; c < kInvCols; ++c)
      if (own && c < nc) Y[(j0 + c) * s + r] = acc[c];
  }
}

// chunk-major inverted index of S over its first m columns: entry e = k * xi + q
// keyed by (chunk of k) * s + target row, sorted stably (k ascending within a
// key); every chunk holds exactly rows * xi entries, so chunk c starts at
// c * kInvRows * xi
__global__ void sketch_inv_keys_kernel(const int* __restrict__ srow, long long cnt, int xi, int s,
                                       int* __restrict__ keys, int* __restrict__ vals) {
  const long long e = static_cast<long long>(blockIdx.x) * blockDim.x + threadIdx.x;
  if (e >= cnt) return;
  const long long k = e / xi;
  keys[e] = static_cast<int>((k / kInvRows) * s + srow[e]);
  vals[e] = static_cast<int>(e);
}
__global__ void sketch_inv_pack_kernel(const int* __restrict__ vals, long long cnt, int xi,
                                       const signed char* __restrict__ ssgn, short* __restrict__ ent) {
  const long long i = static_cast<long long>(blockIdx.x) * blockDim.x + threadIdx.x;
  if (i >= cnt) return;
  const int e = vals[i];
  const int k = e / xi;
  ent[i] = static_cast<short>(((k % kInvRows) << 1) | (ssgn[e] > 0 ? 1 : 0));
}
// cptr[ch * (s + 1) + r] = offset of (ch, r)'s run inside chunk ch
__global__ void sketch_inv_ptr_kernel(const int* __restrict__ skeys, long long cnt, long long nchunks, int s, int xi,
                                      int* __restrict__ cptr) {
  const long long t = static_cast<long long>(blockIdx.x) * blockDim.x + threadIdx.x;
  if (t >= nchunks * (s + 1)) return;
  const long long ch = t / (s + 1), r = t % (s + 1);
  const long long key = ch * s + r;  // r == s: the next chunk's first key
  long long lo = 0, hi = cnt;  // first entry with key >= key
  while (lo < hi) {
    const long long mid = (lo + hi) >> 1;
    if (skeys[mid] < key) lo = mid + 1;
    else hi = mid;
  }
  cptr[t] = static_cast<int>(lo - ch * kInvRows * xi);
}

// CSC input: the device CSR(A^T) rows are the reference CSC columns
__global__ void __launch_bounds__(kSketchWarps * 32)
sketch_ss_csc_kernel(const int* __restrict__ cptr, const int* __restrict__ ridx,
                     const double* __restrict__ cval, long long m, long long n, int s, int xi,
                     const int* __restrict__ srow, const signed char* __restrict__ ssgn,
                     double scale, double mu_scale, int aug, int heavy, int carry, double* __restrict__ Y) {
  extern __shared__ double ysh[];
  const int w = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const long long j = static_cast<long long>(blockIdx.x) * kSketchWarps + w;
  if (j >= n) return;
  SketchSmem sm = sketch_smem(ysh, s, xi, w);
  double* yc = sm.y;
  const int b = cptr[j], e = cptr[j + 1];
  if (e - b > heavy) return;  // long columns: the inverted-index kernels below
  for (int i = lane; i < s; i += 32) yc[i] = carry ? Y[j * s + i] : 0.0;
  __syncwarp();
  for (int p0 = b; p0 < e; p0 += 32) {
    const int p = p0 + lane;
    const double v = p < e ? cval[p] : 0.0;
    const int k = p < e ? ridx[p] : 0;
    const int cnt = e - p0 < 32 ? e - p0 : 32;
    stage_s_rows(srow, ssgn, k, p < e, xi, lane, sm.rs, sm.sg);
    for (int q = 0; q < cnt; ++q) {
      const double vk = __shfl_sync(0xffffffffu, v, q);
      const double sv = scale * vk;
      if (lane < xi) yc[sm.rs[q * xi + lane]] += sv * static_cast<double>(sm.sg[q * xi + lane]);
      __syncwarp();
    }
  }
  if (aug && lane < xi) {
    const long long ee = (m + j) * xi + lane;
    yc[srow[ee]] += mu_scale * static_cast<double>(ssgn[ee]);
  }
  __syncwarp();
  for (int i = lane; i < s; i += 32) Y[j * s + i] = yc[i];
}

// Inverted-index sketch for long columns.  The reference's chain for output
// (i, j) is: for the stored rows k of column j in ascending order, whenever
// row i is one of S(:, k)'s xi rows, add (scale * A(k, j)) * sign.  Emitting
// one (key = slot(j) * s + i, value = entry * xi + t) pair per (entry, t) and
// stable-sorting by key gathers each chain contiguously, still in ascending
// entry order; one thread per (j, i) then walks its chain.  The critical path
// is the chain length (~ nnz(j) * xi / s), not nnz(j).
__global__ void heavy_pairs_kernel(const int* __restrict__ cptr, const int* __restrict__ ridx,
                                   const int* __restrict__ bcols, const long long* __restrict__ boff, int nb,
                                   long long total, int s, int xi, const int* __restrict__ srow,
                                   unsigned* __restrict__ keys, unsigned* __restrict__ vals) {
  const long long q = static_cast<long long>(blockIdx.x) * blockDim.x + threadIdx.x;  // batch entry
  if (q >= total) return;
  int lo = 0, hi = nb;  // slot: last b with boff[b] <= q
  while (hi - lo > 1) {
    const int mid = (lo + hi) >> 1;
    if (boff[mid] <= q) lo = mid;
    else hi = mid;
  }
  const long long p = cptr[bcols[lo]] + (q - boff[lo]);
  const long long k = ridx[p];
  for (int t = 0; t < xi; ++t) {
    keys[q * xi + t] = static_cast<unsigned>(lo) * static_cast<unsigned>(s) + static_cast<unsigned>(srow[k * xi + t]);
    vals[q * xi + t] = static_cast<unsigned>(p * xi + t);
  }
}

__global__ void heavy_walk_kernel(const unsigned* __restrict__ keys, const unsigned* __restrict__ vals,
                                  long long npairs, const int* __restrict__ bcols, int nb, int s, int xi,
                                  const int* __restrict__ ridx, const double* __restrict__ cval,
                                  const signed char* __restrict__ ssgn, const int* __restrict__ srow,
                                  double scale, double mu_scale, int aug, long long m, int carry,
                                  double* __restrict__ Y) {
  const long long key = static_cast<long long>(blockIdx.x) * blockDim.x + threadIdx.x;
  if (key >= static_cast<long long>(nb) * s) return;
  // segment [lower_bound(key), lower_bound(key + 1)) of the sorted keys
  auto lower = [&](unsigned kk) {
    long long lo = 0, hi = npairs;
    while (lo < hi) {
      const long long mid = (lo + hi) >> 1;
      if (keys[mid] < kk) lo = mid + 1;
      else hi = mid;
    }
    return lo;
  };
  const long long b = lower(static_cast<unsigned>(key)), e = lower(static_cast<unsigned>(key + 1));
  const int i = static_cast<int>(key % s);
  const long long j = bcols[key / s];
  double acc = carry ? Y[j * s + i] : 0.0;
  long long q = b;
  for (; q + 4 <= e; q += 4) {  // loads ahead of the (ordered) add chain
    double sv[4], sg[4];
#pragma unroll
    for (int u = 0; u < 4; ++u) {
      const unsigned ev = vals[q + u];
      const long long p = ev / xi;
      sv[u] = scale * cval[p];
      sg[u] = static_cast<double>(ssgn[static_cast<long long>(ridx[p]) * xi + ev % xi]);
    }
#pragma unroll
    for (int u = 0; u < 4; ++u) acc += sv[u] * sg[u];
  }
  for (; q < e; ++q) {
    const unsigned ev = vals[q];
    const long long p = ev / xi;
    acc += (scale * cval[p]) * static_cast<double>(ssgn[static_cast<long long>(ridx[p]) * xi + ev % xi]);
  }
  if (aug) {
    for (int t = 0; t < xi; ++t)
      if (srow[(m + j) * xi + t] == i) acc += mu_scale * static_cast<double>(ssgn[(m + j) * xi + t]);
  }
  Y[j * s + i] = acc;
}

// ---------------------------------------------------------------------------
// Gaussian sketch Y = S A via matmul (sketch.hpp:189-192 -> matrix.hpp:351-361):
// Y(i, j) = sum_k A(k, j) * S(i, k), k ascending.  Register-tiled FP64 GEMM
// whose k loop runs in order with separate DMUL/DADD: the exact chain of the
// reference, at GEMM data reuse.
// ---------------------------------------------------------------------------
// Tile GI (sketch rows: 32/64/96/112, chosen per s to limit padding, e.g.
// 112 for C3's s = 111, 96 for s = 275) x 64 (columns of A), k in chunks of 16,
// double-buffered shared memory with a register prefetch of the next chunk;
// each thread owns a (GI/16) x 4 block strided by 16 so shared reads are
// conflict-free or broadcast.
constexpr int kGK = 16;

template <int kGI, int kGJ>
__global__ void __launch_bounds__(256)
sketch_gauss_dense_kernel(const double* __restrict__ S, int s, const double* __restrict__ A, long long m,
                          long long n, int carry, double* __restrict__ Y) {
  constexpr int kGA = kGI / 16, kGC = kGJ / 16;
  __shared__ double Ss[2][kGK][kGI];
  __shared__ double As[2][kGK][kGJ];
  const int tid = threadIdx.x, tx = tid & 15, ty = tid >> 4;
  const long long i0 = static_cast<long long>(blockIdx.y) * kGI;
  const long long j0 = static_cast<long long>(blockIdx.x) * kGJ;
  constexpr int kSL = kGK * kGI / 256, kAL = kGK * kGJ / 256;  // loads per thread per chunk
  double rs[kSL], ra[kAL];
  auto fetch = [&](long long k0) {
#pragma unroll
    for (int r = 0; r < kSL; ++r) {
      const int e = tid + 256 * r, kk = e / kGI, ii = e % kGI;
      const long long k = k0 + kk;
      rs[r] = (k < m && i0 + ii < s) ? S[k * s + i0 + ii] : 0.0;
    }
#pragma unroll
    for (int r = 0; r < kAL; ++r) {
      const int e = tid + 256 * r, jj = e / kGK, kk = e % kGK;
      const long long k = k0 + kk;
      ra[r] = (k < m && j0 + jj < n) ? A[(j0 + jj) * m + k] : 0.0;
    }
  };
  auto stash = [&](int buf) {
#pragma unroll
    for (int r = 0; r < kSL; ++r) {
      const int e = tid + 256 * r;
      Ss[buf][e / kGI][e % kGI] = rs[r];
    }
#pragma unroll
    for (int r = 0; r < kAL; ++r) {
      const int e = tid + 256 * r;
      As[buf][e % kGK][e / kGK] = ra[r];
    }
  };
  double acc[kGA][kGC];
#pragma unroll
  for (int a = 0; a < kGA; ++a)
#pragma unroll
    for (int c = 0; c < kGC; ++c) {
      const long long i = i0 + ty + 16 * a, j = j0 + tx + 16 * c;
      acc[a][c] = (carry && i < s && j < n) ? Y[j * s + i] : 0.0;  // sharded setup: continue the k chain
    }
  fetch(0);
  stash(0);
  __syncthreads();
  int buf = 0;
  for (long long k0 = 0; k0 < m; k0 += kGK) {
    const bool more = k0 + kGK < m;
    if (more) fetch(k0 + kGK);  // global loads in flight during the chunk's arithmetic
#pragma unroll 4
    for (int kk = 0; kk < kGK; ++kk) {
      double sa[kGA], ab[kGC];
#pragma unroll
      for (int a = 0; a < kGA; ++a) sa[a] = Ss[buf][kk][ty + 16 * a];
#pragma unroll
      for (int c = 0; c < kGC; ++c) ab[c] = As[buf][kk][tx + 16 * c];
#pragma unroll
      for (int a = 0; a < kGA; ++a)
#pragma unroll
        for (int c = 0; c < kGC; ++c) acc[a][c] = __dadd_rn(acc[a][c], __dmul_rn(ab[c], sa[a]));
    }
    if (more) {
      stash(buf ^ 1);
      __syncthreads();
      buf ^= 1;
    }
  }
#pragma unroll
  for (int a = 0; a < kGA; ++a)
#pragma unroll
    for (int c = 0; c < kGC; ++c) {
      const long long i = i0 + ty + 16 * a, j = j0 + tx + 16 * c;
      if (i < s && j < n) Y[j * s + i] = acc[a][c];
    }
}

template <int GI>
void launch_gauss_exact_gi(cudaStream_t st, int gj, dim3 grid, const double* S, int s, const double* A, long long m,
                           long long n, int carry, double* Y) {
  switch (gj) {
    case 16: sketch_gauss_dense_kernel<GI, 16><<<grid, 256, 0, st>>>(S, s, A, m, n, carry, Y); break;
    case 32: sketch_gauss_dense_kernel<GI, 32><<<grid, 256, 0, st>>>(S, s, A, m, n, carry, Y); break;
    default: sketch_gauss_dense_kernel<GI, 64><<<grid, 256, 0, st>>>(S, s, A, m, n, carry, Y); break;
  }
}

void launch_sketch_gauss_exact(cudaStream_t st, int num_sms, const double* S, int s, const double* A, long long m,
                               long long n, double* Y, int carry = 0) {
  int best = 96;
  long long pad = (s + 95) / 96 * 96;
  for (int gi : {112, 64, 32}) {  // fewest padded rows; ties keep the larger tile
    const long long p = (s + gi - 1) / gi * static_cast<long long>(gi);
    if (p < pad) {
      pad = p;
      best = gi;
    }
  }
  // column tile: the widest that still gives >= 4 CTAs per SM (the k chains
  // cannot be split, so a narrow output -- C3: s = 111, n = 1e4 -- needs
  // narrow tiles to fill the GPU: 157 CTAs of 64 columns left half of it idle)
  const long long rt = (s + best - 1) / best;
  int gj = 64;
  while (gj > 16 && ((n + gj - 1) / gj) * rt < 4LL * num_sms) gj /= 2;
  dim3 grid(static_cast<unsigned>((n + gj - 1) / gj), static_cast<unsigned>(rt));
  switch (best) {
    case 112: launch_gauss_exact_gi<112>(st, gj, grid, S, s, A, m, n, carry, Y); break;
    case 64: launch_gauss_exact_gi<64>(st, gj, grid, S, s, A, m, n, carry, Y); break;
    case 32: launch_gauss_exact_gi<32>(st, gj, grid, S, s, A, m, n, carry, Y); break;
    default: launch_gauss_exact_gi<96>(st, gj, grid, S, s, A, m, n, carry, Y); break;
  }
}

// ---------------------------------------------------------------------------
// Opt-in fast Gaussian sketch (sketch_kind 2): Y = S A on the FP64 tensor cores
// (DMMA, mma.sync.m8n8k4.f64).  The MMA accumulates with fused multiply-adds in
// hardware order, so Y is not bit-identical to matmul (matrix.hpp:351-361);
// the CUR indices built from it are checked against the exact path's in
// tests/test_gpu_dmma.py.  CTA tile: 96 sketch rows x 64 columns of A, k in
// chunks of 32 staged by cp.async (double-buffered); warp w owns columns
// [8w, 8w + 8) of the tile and all 12 m8 row tiles (24 fp64 accumulators).
// Shared layouts keep the fragment loads conflict-free: S chunk [k][row]
// (stride 100 = 4 mod 16 doubles), A chunk [col][k] (stride 36).
// ---------------------------------------------------------------------------
// sketch-row tile DI: 112 rows cover s <= 112 in one tile (C3's s = 111 ran
// as 96 + a 15-live-row tile: 42% of its MMAs on padding), 96 otherwise
constexpr int kDJ = 64, kDK = 32, kDAL = kDK + 4;
template <int DI>
struct DmmaTile {
  static constexpr int SL = DI + 4;                  // S chunk stride (doubles): 4 mod 16 keeps fragments conflict-free
  static constexpr int Stage = kDK * SL + kDJ * kDAL;  // doubles per stage
};

__device__ __forceinline__ void dmma_m8n8k4(double (&d)[2], double a, double b) {
  asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0, %1}, {%2}, {%3}, {%0, %1};\n"
               : "+d"(d[0]), "+d"(d[1])
               : "d"(a), "d"(b));
}

__device__ __forceinline__ void cp_async8(double* smem, const double* gmem, bool ok) {
  const unsigned sa = static_cast<unsigned>(__cvta_generic_to_shared(smem));
  const int bytes = ok ? 8 : 0;  // 0: zero-fill
  asm volatile("cp.async.ca.shared.global [%0], [%1], 8, %2;\n" ::"r"(sa), "l"(gmem), "r"(bytes));
}

template <int kDI>
__global__ void __launch_bounds__(256, 2)
sketch_gauss_dmma_kernel(const double* __restrict__ S, int s, const double* __restrict__ A, long long m,
                         long long n, double* __restrict__ Y) {
  constexpr int kDSL = DmmaTile<kDI>::SL, kDStage = DmmaTile<kDI>::Stage;
  extern __shared__ double dsm[];
  const int tid = threadIdx.x, lane = tid & 31, w = tid >> 5;
  const int g = lane >> 2, t = lane & 3;
  const long long i0 = static_cast<long long>(blockIdx.y) * kDI;
  const long long j0 = static_cast<long long>(blockIdx.x) * kDJ;
  // split over k (grid.z): this CTA's chunk range; partial Y per split
  const long long nkall = (m + kDK - 1) / kDK;
  const long long kper = (nkall + gridDim.z - 1) / gridDim.z;
  const long long kc0 = blockIdx.z * kper, kc1 = kc0 + kper < nkall ? kc0 + kper : nkall;
  Y += static_cast<long long>(blockIdx.z) * s * n;
  auto stage = [&](int buf, long long k0) {
    double* Ss = dsm + buf * kDStage;
    double* As = Ss + kDK * kDSL;
    // S chunk: kDK columns of S (rows i0..i0+kDI), 8-byte copies, zero-filled past s / m
    for (int e = tid; e < kDK * kDI; e += 256) {
      const int kk = e / kDI, ii = e % kDI;
      const long long k = k0 + kk, i = i0 + ii;
      const bool ok = k < m && i < s;
      cp_async8(Ss + kk * kDSL + ii, ok ? S + k * s + i : S, ok);
    }
    // A chunk: kDJ columns of A, kDK consecutive rows each
    for (int e = tid; e < kDJ * kDK; e += 256) {
      const int jj = e / kDK, kk = e % kDK;
      const long long k = k0 + kk, j = j0 + jj;
      const bool ok = k < m && j < n;
      cp_async8(As + jj * kDAL + kk, ok ? A + j * m + k : A, ok);
    }
    asm volatile("cp.async.commit_group;\n" ::);
  };
  double acc[kDI / 8][2];
#pragma unroll
  for (int q = 0; q < kDI / 8; ++q) acc[q][0] = acc[q][1] = 0.0;
  const long long nk = kc1 > kc0 ? kc1 - kc0 : 0;
  if (nk > 0) stage(0, kc0 * kDK);
  for (long long c = 0; c < nk; ++c) {
    const int buf = static_cast<int>(c & 1);
    if (c + 1 < nk) {
      stage(buf ^ 1, (kc0 + c + 1) * kDK);
      asm volatile("cp.async.wait_group 1;\n" ::);
    } else {
      asm volatile("cp.async.wait_group 0;\n" ::);
    }
    __syncthreads();
    const double* Ss = dsm + buf * kDStage;
    const double* As = Ss + kDK * kDSL;
#pragma unroll
    for (int kk = 0; kk < kDK; kk += 4) {
      const double b = As[(8 * w + g) * kDAL + kk + t];  // B fragment: A(k0 + kk + t, j0 + 8w + g)
#pragma unroll
      for (int q = 0; q < kDI / 8; ++q) {
        const double a = Ss[(kk + t) * kDSL + 8 * q + g];  // A fragment: S(i0 + 8q + g, k0 + kk + t)
        dmma_m8n8k4(acc[q], a, b);
      }
    }
    __syncthreads();
  }
#pragma unroll
  for (int q = 0; q < kDI / 8; ++q) {
    const long long i = i0 + 8 * q + g;
    const long long j = j0 + 8 * w + 2 * t;
    if (i < s) {
      if (j < n) Y[j * s + i] = acc[q][0];
      if (j + 1 < n) Y[(j + 1) * s + i] = acc[q][1];
    }
  }
}

// Y = sum of the k-split partials, split order
__global__ void dmma_split_sum_kernel(const double* __restrict__ part, int splits, long long cnt,
                                      double* __restrict__ Y) {
  const long long q = static_cast<long long>(blockIdx.x) * blockDim.x + threadIdx.x;
  if (q >= cnt) return;
  double v = part[q];
  for (int z = 1; z < splits; ++z) v += part[z * cnt + q];
  Y[q] = v;
}

template <int DI>
void launch_sketch_gauss_dmma_t(apc_ctx* ctx, const double* S, int s, const double* A, long long m, long long n,
                                double* Y) {
  cudaStream_t st = ctx->stream;
  static bool attr = false;
  const int smem = 2 * DmmaTile<DI>::Stage * static_cast<int>(sizeof(double));
  if (!attr) {
    APC_CUDA(cudaFuncSetAttribute(sketch_gauss_dmma_kernel<DI>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem));
    attr = true;
  }
  // k splits until the grid fills the co-resident slots (2 CTAs per SM)
  const long long tiles = ((n + kDJ - 1) / kDJ) * ((s + DI - 1) / DI);
  const long long slots = 2LL * ctx->num_sms;
  const long long nkall = (m + kDK - 1) / kDK;
  const int splits = static_cast<int>(std::max<long long>(1, std::min<long long>((slots + tiles - 1) / std::max<long long>(1, tiles),
                                                                                   nkall / 8)));
  dim3 grid(static_cast<unsigned>((n + kDJ - 1) / kDJ), static_cast<unsigned>((s + DI - 1) / DI),
            static_cast<unsigned>(splits));
  if (splits == 1) {
    sketch_gauss_dmma_kernel<DI><<<grid, 256, smem, st>>>(S, s, A, m, n, Y);
    return;
  }
  DBuf<double> part(static_cast<long long>(splits) * s * n);
  sketch_gauss_dmma_kernel<DI><<<grid, 256, smem, st>>>(S, s, A, m, n, part.p);
  const long long cnt = static_cast<long long>(s) * n;
  dmma_split_sum_kernel<<<static_cast<unsigned>((cnt + 255) / 256), 256, 0, st>>>(part.p, splits, cnt, Y);
  APC_CUDA(cudaStreamSynchronize(st));  // part goes out of scope
}

void launch_sketch_gauss_dmma(apc_ctx* ctx, const double* S, int s, const double* A, long long m, long long n,
                              double* Y) {
  if (s <= 112) launch_sketch_gauss_dmma_t<112>(ctx, S, s, A, m, n, Y);
  else launch_sketch_gauss_dmma_t<96>(ctx, S, s, A, m, n, Y);
}

// sparse A with a Gaussian S: per (i, j) chain over the stored rows of column j
__global__ void sketch_gauss_csc_kernel(const double* __restrict__ S, int s, const int* __restrict__ cptr,
                                        const int* __restrict__ ridx, const double* __restrict__ cval,
                                        long long n, int carry, double* __restrict__ Y) {
  const int lane = threadIdx.x & 31;
  const long long j = (static_cast<long long>(blockIdx.x) * blockDim.x + threadIdx.x) >> 5;
  if (j >= n) return;
  for (int i = lane; i < s; i += 32) {
    double acc = carry ? Y[j * s + i] : 0.0;
    for (int p = cptr[j]; p < cptr[j + 1]; ++p) acc += cval[p] * S[static_cast<long long>(ridx[p]) * s + i];
    Y[j * s + i] = acc;
  }
}

// ---------------------------------------------------------------------------
// LUPP pivot order (dense_factor.hpp:119-157), right-looking and exact:
// one launch per step k applies step k-1's elimination to every unpivoted row
// (w(r,c) -= (w(r,k-1)/pval) * w(prow,c), skipped when pval or the factor is
// 0), then elects step k's pivot = max |w(r,k)|, ties to the lowest row index.
// ---------------------------------------------------------------------------
struct LuppPivot {
  double pval;
  long long prow;
};

__device__ __forceinline__ bool better(double m1, long long i1, double m2, long long i2) {
  return m1 > m2 || (m1 == m2 && i1 < i2);
}

__global__ void __launch_bounds__(kT)
lupp_step_kernel(double* __restrict__ W, long long ld, long long rows, long long cols, int k,
                 char* __restrict__ piv, long long* __restrict__ order, double* __restrict__ mags,
                 LuppPivot* __restrict__ pv, double* __restrict__ pmag, long long* __restrict__ pidx,
                 unsigned* __restrict__ ctr) {
  __shared__ double sm[kT / 32];
  __shared__ long long si[kT / 32];
  const long long r = static_cast<long long>(blockIdx.x) * kT + threadIdx.x;
  double best = -1.0;
  long long bidx = LLONG_MAX;
  if (r < rows && !piv[r]) {
    if (k > 0) {
      const double pval = pv->pval;
      const long long prow = pv->prow;
      if (pval != 0.0) {
        const double f = W[(k - 1) * ld + r] / pval;
        if (f != 0.0)
          for (long long c = k; c < cols; ++c) W[c * ld + r] -= f * W[c * ld + prow];
      }
    }
    best = fabs(W[static_cast<long long>(k) * ld + r]);
    bidx = r;
  }
  for (int o = 16; o > 0; o >>= 1) {
    const double om = __shfl_xor_sync(0xffffffffu, best, o);
    const long long oi = __shfl_xor_sync(0xffffffffu, bidx, o);
    if (better(om, oi, best, bidx)) {
      best = om;
      bidx = oi;
    }
  }
  const int w = threadIdx.x >> 5, lane = threadIdx.x & 31;
  if (lane == 0) {
    sm[w] = best;
    si[w] = bidx;
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    for (int q = 1; q < kT / 32; ++q)
      if (better(sm[q], si[q], best, bidx)) {
        best = sm[q];
        bidx = si[q];
      }
    pmag[blockIdx.x] = best;
    pidx[blockIdx.x] = bidx;
  }
  if (!elect_last_block(ctr, gridDim.x)) return;
  // final election over block partials (a total order: any tree gives the same winner)
  best = -1.0;
  bidx = LLONG_MAX;
  for (long long q = threadIdx.x; q < gridDim.x; q += kT) {
    const double om = ((volatile double*)pmag)[q];
    const long long oi = ((volatile long long*)pidx)[q];
    if (better(om, oi, best, bidx)) {
      best = om;
      bidx = oi;
    }
  }
  for (int o = 16; o > 0; o >>= 1) {
    const double om = __shfl_xor_sync(0xffffffffu, best, o);
    const long long oi = __shfl_xor_sync(0xffffffffu, bidx, o);
    if (better(om, oi, best, bidx)) {
      best = om;
      bidx = oi;
    }
  }
  __syncthreads();
  if (lane == 0) {
    sm[w] = best;
    si[w] = bidx;
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    for (int q = 1; q < kT / 32; ++q)
      if (better(sm[q], si[q], best, bidx)) {
        best = sm[q];
        bidx = si[q];
      }
    order[k] = bidx;
    mags[k] = best;
    piv[bidx] = 1;
    pv->prow = bidx;
    pv->pval = ((volatile double*)W)[static_cast<long long>(k) * ld + bidx];
  }
}

// ---------------------------------------------------------------------------
// The same pivot order from ONE cooperative launch, blocked (dense_factor.hpp:
// 119-157).  Every element w(r, c) still receives the updates of steps
// 0, 1, ... in step order with the reference's skips (pval == 0, factor == 0)
// and separately rounded products and differences, so the elimination and the
// elections are bit-identical to the right-looking loop; only WHEN an update
// is applied changes.  Steps come in panels of kLuppPanel columns:
//   panel step k: unpivoted rows apply step k-1 to the panel columns [k, kend)
//     and store its multiplier in w(r, k-1); local max |w(r, k)| (ties: lowest
//     row); one grid barrier; every CTA reduces the per-CTA candidates in the
//     same order, so all agree on the pivot without a second barrier;
//   U rows: the panel's pivot rows get the panel's earlier steps on the
//     trailing columns (thread per column, pivot order); grid barrier;
//   trailing update: every other unpivoted row applies the panel's steps to
//     the trailing columns, multipliers in registers, U rows in shared memory.
// Traffic per element and panel instead of per step: ~kLuppPanel x fewer
// passes over the rows x columns matrix (C5's E^col is 8e6 x 250).
// ---------------------------------------------------------------------------
constexpr int kLuppPanel = 16;
constexpr int kLuppThreads = 256;
constexpr int kLuppUCols = 256;  // trailing columns staged in shared memory per pass

struct LuppCoopArgs {
  double* W;
  long long ld, rows, cols;
  int steps;
  char* piv;
  long long* order;
  double* mags;
  double* cmag;      // 2 x grid candidates (double-buffered by step parity)
  long long* cidx;
  long long* prows;  // steps
};

__device__ __forceinline__ void block_best(double& best, long long& bidx, double* sm, long long* si) {
  const int lane = threadIdx.x & 31, wp = threadIdx.x >> 5;
  for (int o = 16; o > 0; o >>= 1) {
    const double om = __shfl_xor_sync(0xffffffffu, best, o);
    const long long oi = __shfl_xor_sync(0xffffffffu, bidx, o);
    if (better(om, oi, best, bidx)) {
      best = om;
      bidx = oi;
    }
  }
  __syncthreads();
  if (lane == 0) {
    sm[wp] = best;
    si[wp] = bidx;
  }
  __syncthreads();
  best = sm[0];
  bidx = si[0];
  for (int q = 1; q < kLuppThreads / 32; ++q)
    if (better(sm[q], si[q], best, bidx)) {
      best = sm[q];
      bidx = si[q];
    }
}

__global__ void __launch_bounds__(kLuppThreads)
lupp_coop_kernel(LuppCoopArgs P) {
  namespace cg = cooperative_groups;
  cg::grid_group grid = cg::this_grid();
  __shared__ double sm[kLuppThreads / 32];
  __shared__ long long si[kLuppThreads / 32];
  __shared__ double U[kLuppPanel * kLuppUCols];
  __shared__ long long spr[kLuppPanel];
  double* W = P.W;
  const long long ld = P.ld, rows = P.rows, cols = P.cols;
  const long long T = static_cast<long long>(gridDim.x) * kLuppThreads;
  const long long t0 = static_cast<long long>(blockIdx.x) * kLuppThreads + threadIdx.x;
  const int G = gridDim.x;
  for (int c0 = 0; c0 < P.steps; c0 += kLuppPanel) {
    const int kend = min(P.steps, c0 + kLuppPanel);
    double pv = 0.0;   // pivot value / row of the previous step (this CTA's copy)
    long long pr = 0;
    for (int k = c0; k < kend; ++k) {
      double best = -1.0;
      long long bidx = LLONG_MAX;
      for (long long r = t0; r < rows; r += T) {
        if (P.piv[r]) continue;
        if (k > c0) {
          double f = 0.0;
          if (pv != 0.0) {
            f = W[(k - 1) * ld + r] / pv;
            if (f != 0.0)
              for (long long c = k; c < kend; ++c) W[c * ld + r] -= f * __ldcg(W + c * ld + pr);
          }
          W[(k - 1) * ld + r] = f;  // the multiplier (0: the reference skipped this row)
        }
        const double mag = fabs(W[static_cast<long long>(k) * ld + r]);
        if (better(mag, r, best, bidx)) {
          best = mag;
          bidx = r;
        }
      }
      block_best(best, bidx, sm, si);
      const int buf = (k & 1) * G;
      if (threadIdx.x == 0) {
        P.cmag[buf + blockIdx.x] = best;
        P.cidx[buf + blockIdx.x] = bidx;
      }
      grid.sync();
      // every CTA elects the same pivot from the same candidates (a total order)
      best = -1.0;
      bidx = LLONG_MAX;
      for (int q = threadIdx.x; q < G; q += kLuppThreads) {
        const double om = __ldcg(P.cmag + buf + q);
        const long long oi = __ldcg(P.cidx + buf + q);
        if (better(om, oi, best, bidx)) {
          best = om;
          bidx = oi;
        }
      }
      block_best(best, bidx, sm, si);
      if (bidx >= t0 && (bidx - t0) % T == 0) P.piv[bidx] = 1;  // the owning thread marks it
      pv = __ldcg(W + static_cast<long long>(k) * ld + bidx);   // written before the barrier by its owner
      pr = bidx;
      if (blockIdx.x == 0 && threadIdx.x == 0) {
        P.order[k] = bidx;
        P.mags[k] = best;
        P.prows[k] = bidx;
      }
      if (threadIdx.x == 0) spr[k - c0] = bidx;
    }
    // multipliers of the panel's last step for the remaining unpivoted rows
    for (long long r = t0; r < rows; r += T) {
      if (P.piv[r]) continue;
      const double f = pv != 0.0 ? W[static_cast<long long>(kend - 1) * ld + r] / pv : 0.0;
      W[static_cast<long long>(kend - 1) * ld + r] = f;
    }
    if (kend >= cols) {
      grid.sync();
      continue;
    }
    __syncthreads();
    // U rows: pivot row i of the panel gets steps c0..i-1 on the trailing columns
    for (long long c = kend + t0; c < cols; c += T) {
      for (int i = 1; i < kend - c0; ++i) {
        const long long ri = spr[i];
        double v = __ldcg(W + c * ld + ri);
        for (int j = 0; j < i; ++j) {
          const double f = __ldcg(W + static_cast<long long>(c0 + j) * ld + ri);
          if (f != 0.0) v -= f * (j == 0 ? __ldcg(W + c * ld + spr[j]) : W[c * ld + spr[j]]);
        }
        W[c * ld + ri] = v;
      }
    }
    grid.sync();
    // trailing update of every other unpivoted row, kLuppUCols columns at a time
    const int np = kend - c0;
    for (long long cb = kend; cb < cols; cb += kLuppUCols) {
      const int nc = static_cast<int>(cols - cb < kLuppUCols ? cols - cb : kLuppUCols);
      __syncthreads();
      for (int e = threadIdx.x; e < np * nc; e += kLuppThreads) {
        const int j = e / nc, cc = e % nc;
        U[j * kLuppUCols + cc] = __ldcg(W + (cb + cc) * ld + spr[j]);
      }
      __syncthreads();
      for (long long r = t0; r < rows; r += T) {
        if (P.piv[r]) continue;
        double f[kLuppPanel];
#pragma unroll
        for (int j = 0; j < kLuppPanel; ++j) f[j] = j < np ? W[static_cast<long long>(c0 + j) * ld + r] : 0.0;
        for (int cc = 0; cc < nc; ++cc) {
          double v = W[(cb + cc) * ld + r];
#pragma unroll
          for (int j = 0; j < kLuppPanel; ++j)
            if (f[j] != 0.0) v -= f[j] * U[j * kLuppUCols + cc];
          W[(cb + cc) * ld + r] = v;
        }
      }
    }
    grid.sync();
  }
}

// ---------------------------------------------------------------------------
// Row-sharded LUPP: the row pivots of the sharded setup, where every rank
// holds its block of the rows of E^col (dense_factor.hpp:119-157).  Step k:
//   lupp_dist_local_kernel: the local unpivoted rows apply step k-1 (the
//     pivot row's values from the replicated `pr`), then the local best
//     |w(r, k)| is elected (ties: the lowest GLOBAL row); the last CTA writes
//     the candidate [mag, global row, that row's w(0..cols-1)];
//   comm_allgather of the candidates (bit-exact);
//   lupp_dist_elect_kernel: every rank elects the same winner from the same
//     gathered candidates (a total order), records it, marks it pivoted on
//     its owner and copies its row into `pr` for step k+1.
// The per-row elimination (separately rounded quotient, products and
// differences; skips on a zero pivot or factor) and the election are
// lupp_step_kernel's, so the order and magnitudes equal one rank's.
// ---------------------------------------------------------------------------
__global__ void __launch_bounds__(kT)
lupp_dist_local_kernel(double* __restrict__ W, long long ld, long long rows, long long cols, int k, long long row0,
                       char* __restrict__ piv, const double* __restrict__ pr, double* __restrict__ pmag,
                       long long* __restrict__ pidx, unsigned* __restrict__ ctr, double* __restrict__ cand) {
  __shared__ double sm[kT / 32];
  __shared__ long long si[kT / 32];
  const long long r = static_cast<long long>(blockIdx.x) * kT + threadIdx.x;
  double best = -1.0;
  long long bidx = LLONG_MAX;
  if (r < rows && !piv[r]) {
    if (k > 0) {
      const double pval = pr[k - 1];
      if (pval != 0.0) {
        const double f = W[(k - 1) * ld + r] / pval;
        if (f != 0.0)
          for (long long c = k; c < cols; ++c) W[c * ld + r] -= f * pr[c];
      }
    }
    best = fabs(W[static_cast<long long>(k) * ld + r]);
    bidx = row0 + r;
  }
  for (int o = 16; o > 0; o >>= 1) {
    const double om = __shfl_xor_sync(0xffffffffu, best, o);
    const long long oi = __shfl_xor_sync(0xffffffffu, bidx, o);
    if (better(om, oi, best, bidx)) {
      best = om;
      bidx = oi;
    }
  }
  const int w = threadIdx.x >> 5, lane = threadIdx.x & 31;
  if (lane == 0) {
    sm[w] = best;
    si[w] = bidx;
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    for (int q = 1; q < kT / 32; ++q)
      if (better(sm[q], si[q], best, bidx)) {
        best = sm[q];
        bidx = si[q];
      }
    pmag[blockIdx.x] = best;
    pidx[blockIdx.x] = bidx;
  }
  if (!elect_last_block(ctr, gridDim.x)) return;
  __shared__ double wbest;
  __shared__ long long widx;
  if (threadIdx.x == 0) {
    best = -1.0;
    bidx = LLONG_MAX;
    for (unsigned q = 0; q < gridDim.x; ++q) {
      const double om = ((volatile double*)pmag)[q];
      const long long oi = ((volatile long long*)pidx)[q];
      if (better(om, oi, best, bidx)) {
        best = om;
        bidx = oi;
      }
    }
    wbest = best;
    widx = bidx;
    cand[0] = best;  // -1: no unpivoted row on this rank
    cand[1] = best < 0.0 ? -1.0 : static_cast<double>(bidx);
  }
  __syncthreads();
  if (wbest >= 0.0)
    for (long long c = threadIdx.x; c < cols; c += kT) cand[2 + c] = __ldcg(W + c * ld + (widx - row0));
}

__global__ void lupp_dist_elect_kernel(const double* __restrict__ gath, int nranks, long long stride, int k,
                                       long long cols, long long row0, long long rows, char* __restrict__ piv,
                                       double* __restrict__ pr, long long* __restrict__ order,
                                       double* __restrict__ mags) {
  __shared__ int win;
  if (threadIdx.x == 0) {
    double best = -1.0;
    long long bidx = LLONG_MAX;
    int wp = 0;
    for (int p = 0; p < nranks; ++p) {
      const double mg = gath[p * stride];
      if (mg < 0.0) continue;
      const long long i = static_cast<long long>(gath[p * stride + 1]);
      if (better(mg, i, best, bidx)) {
        best = mg;
        bidx = i;
        wp = p;
      }
    }
    order[k] = bidx;
    mags[k] = best;
    if (bidx >= row0 && bidx < row0 + rows) piv[bidx - row0] = 1;
    win = wp;
  }
  __syncthreads();
  for (long long c = threadIdx.x; c < cols; c += blockDim.x) pr[c] = gath[win * stride + 2 + c];
}

// W (n x s column-major) = E^T with rows in J zeroed (cur.hpp:254-261)
__global__ void transpose_zero_kernel(const double* __restrict__ E, long long s, long long n,
                                      const int* __restrict__ colsel, double* __restrict__ W) {
  const long long idx = static_cast<long long>(blockIdx.x) * blockDim.x + threadIdx.x;
  if (idx >= s * n) return;
  const long long c = idx / n, r = idx % n;
  W[idx] = colsel[r] ? 0.0 : E[r * s + c];
}

// ---------------------------------------------------------------------------
// refresh: H = U R (core solve per column, cur.hpp:119-144,175-181) and
// E^row = Y - Y(:,J) H (cur.hpp:306-312)
// ---------------------------------------------------------------------------
// ---------------------------------------------------------------------------
// CoreFactor::build on the device (cur.hpp:59-114): the l x l intersection
// block A(I, J) factored by Householder QR (dense_factor.hpp:40-72) or LU with
// partial pivoting, in the reference's exact operation order: every norm and
// dot is one thread's left-to-right chain, every update a separately rounded
// product and difference.  One cooperative launch: CTA c owns kCoreCols
// consecutive columns (one thread each) in shared memory (stride l + 1:
// conflict-free); step j's reflector (or pivot and multipliers) is formed by
// the owner of column j right after its own update of step j - 1, published
// in a double-buffered global vector, and one grid barrier later every owner
// of a later column applies it.  Outputs: the factor col-major (a / lu) and
// transposed (row-major, for the warp solve), the reflectors col-major, the
// LU permutation, and the singularity verdict (dmin <= 1e-14 dmax, or a zero
// LU pivot) in flag[0].
// ---------------------------------------------------------------------------
constexpr int kCoreCols = 16;

struct CoreBuildArgs {
  const double* blk;  // l x l col-major
  long long l;
  int kind;           // 0 QR, 1 LU
  double* fa;         // l x l col-major factor (R / LU)
  double* fat;        // l x l row-major factor
  double* hh;         // l x l col-major reflectors (QR)
  long long* perm;    // l (LU)
  double* vbuf;       // 2 x l
  double* sbuf;       // 2 x 4 step scalars (skip / pivot row / pivot value)
  int* flag;          // [0] singular
};

__global__ void __launch_bounds__(kCoreCols)
core_build_kernel(CoreBuildArgs P) {
  namespace cg = cooperative_groups;
  cg::grid_group grid = cg::this_grid();
  extern __shared__ double csm[];
  const long long l = P.l, ls = l + 1;
  double* col = csm;                       // kCoreCols x ls
  double* v = csm + kCoreCols * ls;        // l: the step's reflector / multipliers
  const long long jj = static_cast<long long>(blockIdx.x) * kCoreCols + threadIdx.x;  // my column
  const bool own = jj < l;
  double* c = col + threadIdx.x * ls;
  if (own)
    for (long long i = 0; i < l; ++i) c[i] = P.blk[jj * l + i];
  long long perm_k = 0;
  double dmax = 0.0, dmin = CUDART_INF;
  bool singular = false;
  for (long long j = 0; j < l; ++j) {
    double* vb = P.vbuf + (j & 1) * l;
    double* sb = P.sbuf + (j & 1) * 4;
    if (own && jj == j) {
      if (P.kind == 0) {  // reflector of step j (dense_factor.hpp:49-63)
        double norm2 = 0.0;
        for (long long i = j; i < l; ++i) norm2 += c[i] * c[i];
        const double norm = sqrt(norm2);
        int skip = norm == 0.0;
        if (!skip) {
          const double alpha = (c[j] >= 0.0) ? -norm : norm;
          for (long long i = j; i < l; ++i) vb[i] = c[i];
          vb[j] -= alpha;
          double vn2 = 0.0;
          for (long long i = j; i < l; ++i) vn2 += vb[i] * vb[i];
          const double vn = sqrt(vn2);
          if (vn == 0.0) {
            skip = 1;
            for (long long i = j; i < l; ++i) P.hh[j * l + i] = vb[i];
          } else {
            for (long long i = j; i < l; ++i) {
              vb[i] /= vn;
              P.hh[j * l + i] = vb[i];
            }
            c[j] = alpha;
            for (long long i = j + 1; i < l; ++i) c[i] = 0.0;
          }
        }
        sb[0] = skip;
      } else {  // pivot of step k = j: first max |.| (cur.hpp:76-87)
        long long best = j;
        double bm = -1.0;
        for (long long i = j; i < l; ++i) {
          const double mg = fabs(c[i]);
          if (mg > bm) {
            bm = mg;
            best = i;
          }
        }
        if (best != j) {
          const double t = c[j];
          c[j] = c[best];
          c[best] = t;
        }
        const double piv = c[j];
        sb[1] = static_cast<double>(best);
        sb[2] = piv;
        if (piv != 0.0)
          for (long long i = j + 1; i < l; ++i) {
            const double fac = c[i] / piv;
            c[i] = fac;
            vb[i] = fac;
          }
      }
    }
    grid.sync();
    if (P.kind == 0) {
      if (__ldcg(sb) != 0.0) continue;  // zero column below the diagonal: nothing to reflect
      for (long long i = j + threadIdx.x; i < l; i += kCoreCols) v[i] = __ldcg(vb + i);
      __syncthreads();
      if (own && jj > j) {  // dense_factor.hpp:64-70
        double dot = 0.0;
        for (long long i = j; i < l; ++i) dot += v[i] * c[i];
        dot *= 2.0;
        for (long long i = j; i < l; ++i) c[i] -= dot * v[i];
      }
      __syncthreads();
    } else {
      const long long best = static_cast<long long>(__ldcg(sb + 1));
      const double piv = __ldcg(sb + 2);
      if (threadIdx.x == 0 && blockIdx.x == 0) {
        dmax = fmax(dmax, fabs(piv));
        dmin = fmin(dmin, fabs(piv));
        if (piv == 0.0) singular = true;
        // perm swap (cur.hpp:83-85), kept in P.perm by one thread
        if (j == 0)
          for (long long i = 0; i < l; ++i) P.perm[i] = i;
        if (best != j) {
          const long long t = P.perm[j];
          P.perm[j] = P.perm[best];
          P.perm[best] = t;
        }
        (void)perm_k;
      }
      if (piv == 0.0) break;  // the reference fails here (singular)
      for (long long i = j + 1 + threadIdx.x; i < l; i += kCoreCols) v[i] = __ldcg(vb + i);
      __syncthreads();
      if (own && jj != j) {
        if (best != j) {  // whole-row swap, every column
          const double t = c[j];
          c[j] = c[best];
          c[best] = t;
        }
        if (jj > j) {
          const double ck = c[j];
          for (long long i = j + 1; i < l; ++i) c[i] -= v[i] * ck;
        }
      }
      __syncthreads();
    }
  }
  if (own) {
    for (long long i = 0; i < l; ++i) {
      P.fa[jj * l + i] = c[i];
      P.fat[i * l + jj] = c[i];
    }
  }
  if (P.kind == 1) {
    if (blockIdx.x == 0 && threadIdx.x == 0) P.flag[0] = (singular || !(dmin > 1e-14 * dmax)) ? 1 : 0;
    return;
  }
  grid.sync();
  if (blockIdx.x == 0 && threadIdx.x == 0) {  // dmin / dmax of |R(j, j)| (cur.hpp:67-74)
    double mn = CUDART_INF, mx = 0.0;
    for (long long j = 0; j < l; ++j) {
      const double d = fabs(__ldcg(P.fa + j * l + j));
      mn = fmin(mn, d);
      mx = fmax(mx, d);
    }
    P.flag[0] = !(mn > 1e-14 * mx) ? 1 : 0;
  }
}

// row-major (l x b) -> col-major (l x b)
__global__ void rm_to_cm_kernel(const double* __restrict__ X, long long l, long long b, double* __restrict__ Y) {
  const long long e = static_cast<long long>(blockIdx.x) * blockDim.x + threadIdx.x;
  if (e >= l * b) return;
  const long long i = e / b, t = e % b;
  Y[t * l + i] = X[e];
}
// gather R(:, J+) row-major (l x b) from R row-major (l x n)
__global__ void gather_rcols_rm_kernel(const double* __restrict__ R, long long n, long long l,
                                       const long long* __restrict__ jp, long long b, double* __restrict__ out) {
  const long long e = static_cast<long long>(blockIdx.x) * blockDim.x + threadIdx.x;
  if (e >= l * b) return;
  const long long i = e / b, t = e % b;
  out[e] = R[i * n + jp[t]];
}

__global__ void core_solve_cols_kernel(const double* __restrict__ R, double* __restrict__ H, long long l,
                                       long long n, int kind, const double* __restrict__ hh,
                                       const double* __restrict__ fa, const long long* __restrict__ perm) {
  const long long j = static_cast<long long>(blockIdx.x) * blockDim.x + threadIdx.x;
  if (j >= n) return;
  double* y = H + j;  // y[i] at H[i * n + j]
  if (kind == 0) {
    for (long long i = 0; i < l; ++i) y[i * n] = R[i * n + j];
    for (long long t = 0; t < l; ++t) {  // y <- Q^T y (dense_factor.hpp:75-83)
      const double* v = hh + t * l;
      double d = 0.0;
      for (long long i = t; i < l; ++i) d += v[i] * y[i * n];
      d *= 2.0;
      for (long long i = t; i < l; ++i) y[i * n] -= d * v[i];
    }
    for (long long i = l - 1; i >= 0; --i) {  // back substitution
      double sacc = y[i * n];
      for (long long q = i + 1; q < l; ++q) sacc -= fa[q * l + i] * y[q * n];
      y[i * n] = sacc / fa[i * l + i];
    }
  } else {
    for (long long i = 0; i < l; ++i) y[i * n] = R[perm[i] * n + j];
    for (long long i = 1; i < l; ++i)
      for (long long q = 0; q < i; ++q) y[i * n] -= fa[q * l + i] * y[q * n];
    for (long long i = l - 1; i >= 0; --i) {
      for (long long q = i + 1; q < l; ++q) y[i * n] -= fa[q * l + i] * y[q * n];
      y[i * n] /= fa[i * l + i];
    }
  }
}

// Same product, warp per column: y = R(:, j) lives in registers, lane k
// holding rows [k KP, (k + 1) KP).  Every reduction keeps the reference's
// sequential order by walking the lanes in order (a running value handed on
// with one shuffle per lane, each lane adding its rows in order); the
// elementwise updates (y -= d v) are lane-parallel.  The chains are bound by
// FP64 latency (~9-18 cycles per step) instead of one memory round trip per
// step as in the thread-per-column kernel above.  fat: the factor transposed
// (row-major), so a lane's run of one row is contiguous.
template <int KP>
__global__ void __launch_bounds__(128)
core_solve_warp_kernel(const double* __restrict__ R, double* __restrict__ H, int l, long long n, int kind,
                       const double* __restrict__ hh, const double* __restrict__ fat,
                       const long long* __restrict__ perm) {
  const long long j = (static_cast<long long>(blockIdx.x) * blockDim.x + threadIdx.x) >> 5;
  const int lane = threadIdx.x & 31;
  if (j >= n) return;
  const int base = lane * KP;
  double y[KP];
#pragma unroll
  for (int e = 0; e < KP; ++e) {
    const int i = base + e;
    y[e] = i < l ? R[(kind == 0 ? static_cast<long long>(i) : perm[i]) * n + j] : 0.0;
  }
  const int lastlane = (l - 1) / KP;
  if (kind == 0) {
    for (int t = 0; t < l; ++t) {  // y <- Q^T y (dense_factor.hpp:75-83)
      const double* v = hh + static_cast<long long>(t) * l;
      double vr[KP];
#pragma unroll
      for (int e = 0; e < KP; ++e) {
        const int i = base + e;
        vr[e] = (i >= t && i < l) ? __ldg(v + i) : 0.0;
      }
      // d = sum_{i >= t} v_i y_i in index order: lanes t/KP .. lastlane in turn
      double d = 0.0;
      for (int k = t / KP; k <= lastlane; ++k) {
        if (lane == k) {
#pragma unroll
          for (int e = 0; e < KP; ++e) {
            const int i = base + e;
            if (i >= t && i < l) d += vr[e] * y[e];
          }
        }
        d = __shfl_sync(0xffffffffu, d, k);
      }
      d *= 2.0;
#pragma unroll
      for (int e = 0; e < KP; ++e) {
        const int i = base + e;
        if (i >= t && i < l) y[e] -= d * vr[e];
      }
    }
    for (int i = l - 1; i >= 0; --i) {  // back substitution, q = i+1 .. l-1 ascending
      const int li = i / KP, ei = i % KP;
      const double* row = fat + static_cast<long long>(i) * l;  // row i of the factor
      double fr[KP];
#pragma unroll
      for (int e = 0; e < KP; ++e) {
        const int q = base + e;
        fr[e] = (q > i && q < l) ? __ldg(row + q) : 0.0;
      }
      double sacc = 0.0;
#pragma unroll
      for (int e = 0; e < KP; ++e)
        if (e == ei) sacc = y[e];
      sacc = __shfl_sync(0xffffffffu, sacc, li);
      for (int k = li; k <= lastlane; ++k) {
        if (lane == k) {
#pragma unroll
          for (int e = 0; e < KP; ++e) {
            const int q = base + e;
            if (q > i && q < l) sacc -= fr[e] * y[e];
          }
        }
        sacc = __shfl_sync(0xffffffffu, sacc, k);
      }
      if (lane == li) {
        const double dv = __ldg(row + i);
#pragma unroll
        for (int e = 0; e < KP; ++e)
          if (e == ei) y[e] = sacc / dv;
      }
    }
  } else {
    for (int i = 1; i < l; ++i) {  // forward: y_i -= L(i, q) y_q, q = 0 .. i-1 ascending
      const int li = i / KP, ei = i % KP;
      const double* row = fat + static_cast<long long>(i) * l;
      double fr[KP];
#pragma unroll
      for (int e = 0; e < KP; ++e) {
        const int q = base + e;
        fr[e] = q < i ? __ldg(row + q) : 0.0;
      }
      double r = 0.0;
#pragma unroll
      for (int e = 0; e < KP; ++e)
        if (e == ei) r = y[e];
      r = __shfl_sync(0xffffffffu, r, li);
      for (int k = 0; k <= li; ++k) {
        if (lane == k) {
#pragma unroll
          for (int e = 0; e < KP; ++e) {
            const int q = base + e;
            if (q < i) r -= fr[e] * y[e];
          }
        }
        r = __shfl_sync(0xffffffffu, r, k);
      }
      if (lane == li) {
#pragma unroll
        for (int e = 0; e < KP; ++e)
          if (e == ei) y[e] = r;
      }
    }
    for (int i = l - 1; i >= 0; --i) {  // back: y_i -= U(i, q) y_q, q ascending; y_i /= U(i, i)
      const int li = i / KP, ei = i % KP;
      const double* row = fat + static_cast<long long>(i) * l;
      double fr[KP];
#pragma unroll
      for (int e = 0; e < KP; ++e) {
        const int q = base + e;
        fr[e] = (q > i && q < l) ? __ldg(row + q) : 0.0;
      }
      double r = 0.0;
#pragma unroll
      for (int e = 0; e < KP; ++e)
        if (e == ei) r = y[e];
      r = __shfl_sync(0xffffffffu, r, li);
      for (int k = li; k <= lastlane; ++k) {
        if (lane == k) {
#pragma unroll
          for (int e = 0; e < KP; ++e) {
            const int q = base + e;
            if (q > i && q < l) r -= fr[e] * y[e];
          }
        }
        r = __shfl_sync(0xffffffffu, r, k);
      }
      if (lane == li) {
        const double dv = __ldg(row + i);
#pragma unroll
        for (int e = 0; e < KP; ++e)
          if (e == ei) y[e] = r / dv;
      }
    }
  }
#pragma unroll
  for (int e = 0; e < KP; ++e) {
    const int i = base + e;
    if (i < l) H[static_cast<long long>(i) * n + j] = y[e];
  }
}

// lanes over sketch rows i, one warp per column j: E(i,j) = Y(i,j) - sum_t H(t,j) SC(i,t)
__global__ void eres_kernel(const double* __restrict__ Y, const double* __restrict__ SC,
                            const double* __restrict__ H, long long s, long long n, long long l,
                            double* __restrict__ E) {
  const long long j = (static_cast<long long>(blockIdx.x) * blockDim.x + threadIdx.x) >> 5;
  const int lane = threadIdx.x & 31;
  if (j >= n) return;
  for (long long i0 = 0; i0 < s; i0 += 32) {
    const long long i = i0 + lane;
    double acc = 0.0;
    for (long long t = 0; t < l; ++t) {
      const double h = H[t * n + j];
      if (h == 0.0) continue;
      if (i < s) acc += h * SC[t * s + i];
    }
    if (i < s) E[j * s + i] = Y[j * s + i] - acc;
  }
}

// SparseSignEmbedding columns (sketch.hpp:31-49) from the raw draws of the
// embedding stream: column c consumes draws [2 x c, 2 x c + 2 x) -- x for
// Floyd's below(t + 1) picks, x for the signs -- exactly as the sequential
// construction does whenever below() accepts every draw; a rejected draw
// (probability < s / 2^64 per draw) raises *bad and the host redoes the
// embedding sequentially.
__global__ void ss_columns_kernel(const std::uint64_t* __restrict__ raw, long long ncols, int s, int x,
                                  int* __restrict__ rows, signed char* __restrict__ sg, int* __restrict__ bad) {
  const long long c = static_cast<long long>(blockIdx.x) * blockDim.x + threadIdx.x;
  if (c >= ncols) return;
  const std::uint64_t* d = raw + c * 2 * x;
  int pick[64];
  int cnt = 0;
  for (int t = s - x; t < s; ++t) {
    const std::uint64_t nn = static_cast<std::uint64_t>(t) + 1;
    const std::uint64_t v = d[cnt];
    if (!(v < ~0ULL - (~0ULL % nn))) atomicExch(bad, 1);
    const int r = static_cast<int>(v % nn);
    bool dup = false;
    for (int q = 0; q < cnt; ++q) dup = dup || pick[q] == r;
    pick[cnt++] = dup ? t : r;
  }
  for (int q = 1; q < cnt; ++q) {  // insertion sort (distinct values)
    const int key = pick[q];
    int p = q - 1;
    while (p >= 0 && pick[p] > key) {
      pick[p + 1] = pick[p];
      --p;
    }
    pick[p + 1] = key;
  }
  for (int q = 0; q < x; ++q) {
    rows[c * x + q] = pick[q];
    sg[c * x + q] = static_cast<signed char>((d[x + q] & 1ULL) ? 1 : -1);
  }
}

// rho probes: out(i, p) = (E w_p)_i with the dense matvec chain (j ascending,
// zero entries of w skipped), sketch.hpp:219-221 -> matrix.hpp:156-162.
// Each output is one sequential chain of n DMUL+DADD (the reference order).
// The FP64 pipe, not memory, bounds such chains (measured: ~18 cycles per
// step for one warp on an SM, ~35-70 with 18 warps sharing it), so the
// chains are spread one warp per SM: CTA = (probe p, 32 consecutive rows i),
// and the E rows / probe entries of the next kProbeStages-1 column chunks are
// in flight as cp.async copies into shared memory while the current chunk runs.
constexpr int kProbeJ = 32;       // columns per stage
constexpr int kProbeStages = 4;   // cp.async pipeline depth
__device__ __forceinline__ void cp_async8(void* smem, const void* gmem) {
  asm volatile("cp.async.ca.shared.global [%0], [%1], 8;" ::"r"(static_cast<unsigned>(__cvta_generic_to_shared(smem))),
               "l"(gmem)
               : "memory");
}
__global__ void __launch_bounds__(32)
probe_kernel(const double* __restrict__ E, long long s, long long n, const double* __restrict__ W,
             double* __restrict__ out) {
  __shared__ double et[kProbeStages][kProbeJ][32];
  __shared__ double wt[kProbeStages][kProbeJ];
  const int lane = threadIdx.x;
  const long long p = blockIdx.y;
  const long long i = static_cast<long long>(blockIdx.x) * 32 + lane;
  const bool act = i < s;
  const double* w = W + p * n;
  const long long nchunk = (n + kProbeJ - 1) / kProbeJ;
  auto issue = [&](long long c) {
    const int st = static_cast<int>(c % kProbeStages);
    const long long j0 = c * kProbeJ;
    for (int jj = 0; jj < kProbeJ; ++jj)
      if (act && j0 + jj < n) cp_async8(&et[st][jj][lane], E + (j0 + jj) * s + i);
    if (j0 + lane < n) cp_async8(&wt[st][lane], w + j0 + lane);
  };
  for (int c = 0; c < kProbeStages - 1; ++c) {
    if (c < nchunk) issue(c);
    asm volatile("cp.async.commit_group;" ::: "memory");
  }
  double acc = 0.0;
  for (long long c = 0; c < nchunk; ++c) {
    if (c + kProbeStages - 1 < nchunk) issue(c + kProbeStages - 1);
    asm volatile("cp.async.commit_group;" ::: "memory");
    asm volatile("cp.async.wait_group %0;" ::"n"(kProbeStages - 1) : "memory");
    __syncwarp();
    const int st = static_cast<int>(c % kProbeStages);
    const int jn = static_cast<int>(n - c * kProbeJ < kProbeJ ? n - c * kProbeJ : kProbeJ);
    if (act)
      for (int jj = 0; jj < jn; ++jj) {
        const double wv = wt[st][jj];
        if (wv != 0.0) acc += wv * et[st][jj][lane];
      }
    __syncwarp();
  }
  if (act) out[p * s + i] = acc;
}

// ---------------------------------------------------------------------------
// gathers
// ---------------------------------------------------------------------------
// A(I, J) of the target; rows i >= m of the augmented stack are amu * e_{i-m}
// (AugmentedOperator::extract_block, matrix.hpp:460-473)
__global__ void gather_block_kernel(const double* A, long long m, const int* ptr, const int* idx,
                                    const double* val, int sparse, const long long* I, const long long* J,
                                    long long li, long long lj, double amu, double* out) {
  const long long e = static_cast<long long>(blockIdx.x) * blockDim.x + threadIdx.x;
  if (e >= li * lj) return;
  const long long jj = e / li, ii = e % li;
  const long long i = I[ii];
  if (i >= m) out[e] = (i - m == J[jj]) ? amu : 0.0;
  else out[e] = sparse ? csr_at(ptr, idx, val, i, J[jj]) : A[J[jj] * m + i];
}

// rows I[q] of the target -> R row-major (q in [0, cnt)), dense source
__global__ void gather_rows_dense_kernel(const double* A, long long m, long long n, const long long* I,
                                         long long cnt, double amu, double* R) {
  const long long e = static_cast<long long>(blockIdx.x) * blockDim.x + threadIdx.x;
  if (e >= cnt * n) return;
  const long long q = e / n, c = e % n;
  const long long i = I[q];
  R[e] = i < m ? A[c * m + i] : (c == i - m ? amu : 0.0);
}

__global__ void scatter_rows_csr_kernel(const int* ptr, const int* idx, const double* val, long long m,
                                        long long n, const long long* I, long long cnt, double amu, double* R) {
  const long long q = blockIdx.x;
  if (q >= cnt) return;
  const long long i = I[q];
  if (i >= m) {  // augmented identity row
    if (threadIdx.x == 0) R[q * n + (i - m)] = amu;
    return;
  }
  for (int p = ptr[i] + threadIdx.x; p < ptr[i + 1]; p += blockDim.x) R[q * n + idx[p]] = val[p];
}

// E^col rows m..m+n-1 of the augmented target: A-part is amu at row m + J+[jj];
// C's row m + j holds amu in the column t with J[t] == j (a one-term chain)
__global__ void ecol_tail_kernel(long long m, long long n, long long ld, const int* __restrict__ colpos,
                                 long long l, const long long* __restrict__ Jp, long long b,
                                 const double* __restrict__ urj, const int* __restrict__ rowsel, double amu,
                                 double* __restrict__ out) {
  const long long j = static_cast<long long>(blockIdx.x) * blockDim.x + threadIdx.x;
  if (j >= n) return;
  const bool zero = rowsel[m + j] != 0;
  const int t = colpos[j];
  for (long long jj = 0; jj < b; ++jj) {
    double v = 0.0;
    if (!zero) {
      const double aval = (Jp[jj] == j) ? amu : 0.0;
      if (l > 0) {
        double acc = 0.0;
        if (t >= 0) {
          const double x = urj[jj * l + t];
          if (x != 0.0) acc += x * amu;
        }
        v = aval - acc;
      } else {
        v = aval;
      }
    }
    out[jj * ld + m + j] = v;
  }
}

// SC = Y(:, J) (s x l column-major)
__global__ void gather_sc_kernel(const double* Y, long long s, const long long* J, long long l, double* SC) {
  const long long e = static_cast<long long>(blockIdx.x) * blockDim.x + threadIdx.x;
  if (e >= s * l) return;
  const long long t = e / s, i = e % s;
  SC[e] = Y[J[t] * s + i];
}

// R(q[t], :) = packed row t (the sharded setup's R rows from their owner)
__global__ void place_rows_kernel(const double* __restrict__ pk, const long long* __restrict__ q, long long cnt,
                                  long long n, double* __restrict__ R) {
  const long long e = static_cast<long long>(blockIdx.x) * blockDim.x + threadIdx.x;
  if (e >= cnt * n) return;
  const long long t = e / n, c = e % n;
  R[q[t] * n + c] = pk[e];
}

// R(:, J+) from the row-major R (l x b, column-major)
__global__ void gather_rcols_kernel(const double* R, long long n, long long l, const long long* Jp, long long b,
                                    double* out) {
  const long long e = static_cast<long long>(blockIdx.x) * blockDim.x + threadIdx.x;
  if (e >= l * b) return;
  const long long jj = e / l, i = e % l;
  out[e] = R[i * n + Jp[jj]];
}

// ---------------------------------------------------------------------------
// E^col = A(:, J+) - C (U R(:, J+)), rows I zeroed (cur.hpp:268-283)
// ---------------------------------------------------------------------------
constexpr int kEcolTile = 8;

__global__ void ecol_dense_kernel(const double* __restrict__ A, long long m, long long ld,
                                  const long long* __restrict__ J, long long l, const long long* __restrict__ Jp,
                                  long long b, const double* __restrict__ urj, const int* __restrict__ rowsel,
                                  double* __restrict__ out) {
  const long long i = static_cast<long long>(blockIdx.x) * blockDim.x + threadIdx.x;
  const long long jj0 = static_cast<long long>(blockIdx.y) * kEcolTile;
  if (i >= m) return;
  double acc[kEcolTile];
#pragma unroll
  for (int q = 0; q < kEcolTile; ++q) acc[q] = 0.0;
  for (long long t = 0; t < l; ++t) {
    const double c = A[J[t] * m + i];
#pragma unroll
    for (int q = 0; q < kEcolTile; ++q) {
      if (jj0 + q < b) {
        const double x = urj[(jj0 + q) * l + t];
        if (x != 0.0) acc[q] += x * c;
      }
    }
  }
  const bool zero = rowsel[i] != 0;
#pragma unroll
  for (int q = 0; q < kEcolTile; ++q) {
    const long long jj = jj0 + q;
    if (jj < b) out[jj * ld + i] = zero ? 0.0 : (l > 0 ? A[Jp[jj] * m + i] - acc[q] : A[Jp[jj] * m + i]);
  }
}

// sparse A: per row i, C(i, :) entries (t ascending) from crow lists
__global__ void ecol_sparse_kernel(const int* __restrict__ ptr, const int* __restrict__ idx,
                                   const double* __restrict__ val, long long m, long long ld,
                                   const int* __restrict__ cptr,
                                   const int* __restrict__ ct, const double* __restrict__ cv, long long l,
                                   const long long* __restrict__ Jp, long long b, const double* __restrict__ urj,
                                   const int* __restrict__ rowsel, double* __restrict__ out) {
  const long long i = static_cast<long long>(blockIdx.x) * blockDim.x + threadIdx.x;
  if (i >= m) return;
  const bool zero = rowsel[i] != 0;
  for (long long jj = 0; jj < b; ++jj) {
    double v = 0.0;
    if (!zero) {
      const double aval = csr_at(ptr, idx, val, i, Jp[jj]);
      double acc = 0.0;
      if (l > 0)
        for (int e = cptr[i]; e < cptr[i + 1]; ++e) {
          const double x = urj[jj * l + ct[e]];
          if (x != 0.0) acc += x * cv[e];
        }
      v = l > 0 ? aval - acc : aval;
    }
    out[jj * ld + i] = v;
  }
}

// C row lists: entries of CSR(A) row i whose column is in J, as (t = position in J, value), t ascending
__global__ void crow_count_kernel(const int* ptr, const int* idx, long long m, const int* colpos, int* cnt) {
  const long long i = static_cast<long long>(blockIdx.x) * blockDim.x + threadIdx.x;
  if (i >= m) return;
  int c = 0;
  for (int p = ptr[i]; p < ptr[i + 1]; ++p) c += colpos[idx[p]] >= 0;
  cnt[i] = c;
}

__global__ void crow_fill_kernel(const int* ptr, const int* idx, const double* val, long long m, const int* colpos,
                                 const int* cptr, int* ct, double* cv) {
  const long long i = static_cast<long long>(blockIdx.x) * blockDim.x + threadIdx.x;
  if (i >= m) return;
  int q = cptr[i];
  const int q0 = q;
  for (int p = ptr[i]; p < ptr[i + 1]; ++p) {
    const int t = colpos[idx[p]];
    if (t < 0) continue;
    // insertion by t (rows hold few entries)
    int at = q;
    while (at > q0 && ct[at - 1] > t) {
      ct[at] = ct[at - 1];
      cv[at] = cv[at - 1];
      --at;
    }
    ct[at] = t;
    cv[at] = val[p];
    ++q;
  }
}

// Exact-order Gram of a dense column block: G(i, j) = sum_r C(r, i) C(r, j) with
// r ascending and separate mul/add, i.e. chol_gram's loop (dense_factor.hpp:
// 199-209) element by element; 64 x 64 output tiles (upper-triangle tiles only).
__global__ void __launch_bounds__(256)
gram_exact_kernel(const double* __restrict__ C, long long m, long long l, double* __restrict__ G) {
  constexpr int T = 64, K = 16;
  __shared__ double Ci[K][T + 1];
  __shared__ double Cj[K][T + 1];
  const long long i0 = static_cast<long long>(blockIdx.y) * T, j0 = static_cast<long long>(blockIdx.x) * T;
  if (i0 > j0 + T - 1) return;  // strictly-lower tile
  const int tx = threadIdx.x & 15, ty = threadIdx.x >> 4;
  double acc[4][4];
#pragma unroll
  for (int a = 0; a < 4; ++a)
#pragma unroll
    for (int c = 0; c < 4; ++c) acc[a][c] = 0.0;
  for (long long k0 = 0; k0 < m; k0 += K) {
    for (int e = threadIdx.x; e < K * T; e += 256) {
      const int cc = e / K, kk = e % K;
      const long long r = k0 + kk;
      Ci[kk][cc] = (r < m && i0 + cc < l) ? C[(i0 + cc) * m + r] : 0.0;
      Cj[kk][cc] = (r < m && j0 + cc < l) ? C[(j0 + cc) * m + r] : 0.0;
    }
    __syncthreads();
    for (int kk = 0; kk < K; ++kk) {
      double a4[4], b4[4];
#pragma unroll
      for (int a = 0; a < 4; ++a) a4[a] = Ci[kk][ty + 16 * a];
#pragma unroll
      for (int c = 0; c < 4; ++c) b4[c] = Cj[kk][tx + 16 * c];
#pragma unroll
      for (int a = 0; a < 4; ++a)
#pragma unroll
        for (int c = 0; c < 4; ++c) acc[a][c] = __dadd_rn(acc[a][c], __dmul_rn(a4[a], b4[c]));
    }
    __syncthreads();
  }
#pragma unroll
  for (int a = 0; a < 4; ++a)
#pragma unroll
    for (int c = 0; c < 4; ++c) {
      const long long i = i0 + ty + 16 * a, j = j0 + tx + 16 * c;
      if (i <= j && j < l) G[j * l + i] = acc[a][c];
    }
}

// C = A(:, J) dense (m x l column-major) from a dense A
__global__ void gather_cols_kernel(const double* A, long long m, const long long* J, long long l, double* C) {
  const long long e = static_cast<long long>(blockIdx.x) * blockDim.x + threadIdx.x;
  if (e >= m * l) return;
  const long long t = e / m, i = e % m;
  C[e] = A[J[t] * m + i];
}

// rows [r0, r0 + rb) of C = A(:, J) densified from CSR(A) (rb x l, zero-filled by caller)
__global__ void densify_rows_kernel(const int* ptr, const int* idx, const double* val, long long r0, long long rb,
                                    const int* colpos, double* D) {
  const long long q = static_cast<long long>(blockIdx.x) * blockDim.x + threadIdx.x;
  if (q >= rb) return;
  const long long i = r0 + q;
  for (int p = ptr[i]; p < ptr[i + 1]; ++p) {
    const int t = colpos[idx[p]];
    if (t >= 0) D[static_cast<long long>(t) * rb + q] = val[p];
  }
}

__global__ void set_flags_kernel(int* flags, const long long* ids, long long cnt, int value) {
  const long long e = static_cast<long long>(blockIdx.x) * blockDim.x + threadIdx.x;
  if (e < cnt) flags[ids[e]] = value;
}

__global__ void set_colpos_kernel(int* colpos, const long long* J, long long l) {
  const long long t = static_cast<long long>(blockIdx.x) * blockDim.x + threadIdx.x;
  if (t < l) colpos[J[t]] = static_cast<int>(t);
}

template <class T>
void upload(apc_ctx* ctx, DBuf<T>& d, const T* h, i64 n) {
  d.ensure(std::max<i64>(1, n));
  if (n > 0) APC_CUDA(cudaMemcpyAsync(d.p, h, sizeof(T) * n, cudaMemcpyHostToDevice, ctx->stream));
}

template <class T>
std::vector<T> download(apc_ctx* ctx, const T* d, i64 n) {
  std::vector<T> h(static_cast<size_t>(std::max<i64>(0, n)));
  if (n > 0) APC_CUDA(cudaMemcpyAsync(h.data(), d, sizeof(T) * n, cudaMemcpyDeviceToHost, ctx->stream));
  APC_CUDA(cudaStreamSynchronize(ctx->stream));
  return h;
}

}  // namespace

// ---------------------------------------------------------------------------
// device LUPP driver
// ---------------------------------------------------------------------------
LuppOut device_lupp(apc_ctx* ctx, double* w, i64 rows, i64 cols, i64 max_pivots) {
  LuppOut out;
  i64 steps = std::min(rows, cols);
  if (max_pivots >= 0) steps = std::min(steps, max_pivots);
  if (steps <= 0) return out;
  cudaStream_t st = ctx->stream;
  const unsigned nbk = nb(rows);
  DBuf<char> piv(rows);
  DBuf<long long> order(steps), pidx(nbk);
  DBuf<double> mags(steps), pmag(nbk);
  DBuf<LuppPivot> pv(1);
  DBuf<unsigned> ctr(1);
  APC_CUDA(cudaMemsetAsync(piv.p, 0, rows, st));
  APC_CUDA(cudaMemsetAsync(ctr.p, 0, sizeof(unsigned), st));
  static const bool coop = !std::getenv("APC_LUPP_STEPS");
  if (coop) {
    // one cooperative launch: as many co-resident CTAs as the rows need
    static int per_sm = -1;
    if (per_sm < 0)
      APC_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, lupp_coop_kernel, kLuppThreads, 0));
    const long long want = (rows + kLuppThreads - 1) / kLuppThreads;
    const int grid = static_cast<int>(std::max<long long>(1, std::min<long long>(want, 1LL * per_sm * ctx->num_sms)));
    DBuf<double> cmag(2 * grid);
    DBuf<long long> cidx(2 * grid), prows(steps);
    LuppCoopArgs args{w, rows, rows, cols, static_cast<int>(steps), piv.p, order.p, mags.p, cmag.p, cidx.p, prows.p};
    void* kargs[] = {&args};
    APC_CUDA(cudaLaunchCooperativeKernel(reinterpret_cast<const void*>(lupp_coop_kernel), dim3(grid),
                                         dim3(kLuppThreads), kargs, 0, st));
    ctx->launches++;
  } else {
    for (i64 k = 0; k < steps; ++k) {
      lupp_step_kernel<<<nbk, kT, 0, st>>>(w, rows, rows, cols, static_cast<int>(k), piv.p, order.p, mags.p,
                                           pv.p, pmag.p, pidx.p, ctr.p);
    }
    ctx->launches += static_cast<std::uint64_t>(steps);
  }
  APC_CUDA(cudaGetLastError());
  auto o = download(ctx, order.p, steps);
  out.order.assign(o.begin(), o.end());
  out.mags = download(ctx, mags.p, steps);
  return out;
}

// Pivot order of LUPP over a row-sharded column-major matrix: this rank's
// rows [row0, row0 + rows) of a rows_global x cols matrix (w destroyed).  Every
// rank returns the same order (global rows) and magnitudes, equal to
// device_lupp over the whole matrix.  One step = two launches and one allgather.
LuppOut device_lupp_dist(apc_ctx* ctx, double* w, i64 rows, i64 row0, i64 rows_global, i64 cols, i64 max_pivots) {
  LuppOut out;
  i64 steps = std::min(rows_global, cols);
  if (max_pivots >= 0) steps = std::min(steps, max_pivots);
  if (steps <= 0) return out;
  cudaStream_t st = ctx->stream;
  const unsigned nbk = std::max(1u, nb(rows));
  const i64 stride = cols + 2;
  DBuf<char> piv(std::max<i64>(1, rows));
  DBuf<long long> order(steps), pidx(nbk);
  DBuf<double> mags(steps), pmag(nbk), pr(cols), cand(stride), gath(stride * ctx->nranks);
  DBuf<unsigned> ctr(1);
  APC_CUDA(cudaMemsetAsync(piv.p, 0, piv.bytes(), st));
  APC_CUDA(cudaMemsetAsync(ctr.p, 0, sizeof(unsigned), st));
  for (i64 k = 0; k < steps; ++k) {
    lupp_dist_local_kernel<<<nbk, kT, 0, st>>>(w, std::max<i64>(1, rows), rows, cols, static_cast<int>(k), row0,
                                               piv.p, pr.p, pmag.p, pidx.p, ctr.p, cand.p);
    comm_allgather(ctx, cand.p, stride, gath.p);
    lupp_dist_elect_kernel<<<1, 128, 0, st>>>(gath.p, ctx->nranks, stride, static_cast<int>(k), cols, row0, rows,
                                              piv.p, pr.p, order.p, mags.p);
  }
  ctx->launches += 2 * static_cast<std::uint64_t>(steps);
  APC_CUDA(cudaGetLastError());
  auto o = download(ctx, order.p, steps);
  out.order.assign(o.begin(), o.end());
  out.mags = download(ctx, mags.p, steps);
  return out;
}

// ---------------------------------------------------------------------------
// DeviceCur
// ---------------------------------------------------------------------------
DeviceCur::DeviceCur(apc_mat& a, i64 block, std::uint64_t seed, i64 xi, i64 probes, int core_kind,
                     int sketch_kind, i64 max_rank, double aug_mu, bool distributed)
    : a_(a), ctx_(a.ctx), m_(a.m), n_(a.n), block_size_(block), probes_(probes), max_rank_(max_rank),
      mt_(a.m + (aug_mu > 0.0 ? a.n : 0)), amu_(aug_mu > 0.0 ? aug_mu : 0.0), core_kind_(core_kind),
      rho_(std::numeric_limits<double>::infinity()), probe_rng_(seed, Stream::probes) {
  require(!(amu_ > 0.0 && sketch_kind != 0), APC_NOT_APPLICABLE,
          "CurState: the reference has no Gaussian sketch of the augmented stack");
  require(block >= 1, APC_INVALID_ARGUMENT, "CurState: block size must be >= 1");
  require(block <= n_, APC_INVALID_ARGUMENT, "CurState: block size exceeds column count");
  require(sketch_kind >= 0 && sketch_kind <= 2, APC_INVALID_ARGUMENT, "CurState: sketch kind must be 0, 1 or 2");
  dist_ = distributed && ctx_->nranks > 1;
  row0_ = dist_ ? a.r0 : 0;
  mloc_ = dist_ ? a.mloc() : m_;
  if (!dist_) {
    require(a.r0 == 0 && a.r1 == a.m, APC_NOT_APPLICABLE, "CurState: needs the full matrix on this rank");
  } else {
    require(amu_ == 0.0, APC_NOT_APPLICABLE,
            "CurState: the sharded setup has no augmented target [A; mu I] (pass the whole matrix on rank 0)");
    // every rank's row block: contiguous, in rank order, covering [0, m)
    const int P = ctx_->nranks;
    DBuf<double> mine(2), all(2 * P);
    const double mr[2] = {static_cast<double>(a.r0), static_cast<double>(a.r1)};
    APC_CUDA(cudaMemcpyAsync(mine.p, mr, sizeof(mr), cudaMemcpyHostToDevice, ctx_->stream));
    comm_allgather(ctx_, mine.p, 2, all.p);
    std::vector<double> h = download(ctx_, all.p, 2 * P);
    bounds_.resize(static_cast<size_t>(P + 1));
    for (int p = 0; p < P; ++p) {
      require(h[2 * p] == (p == 0 ? 0.0 : h[2 * p - 1]) && h[2 * p] <= h[2 * p + 1], APC_INVALID_ARGUMENT,
              "CurState: the sharded setup needs contiguous row blocks in rank order");
      bounds_[p] = static_cast<i64>(h[2 * p]);
    }
    require(h[2 * P - 1] == static_cast<double>(m_), APC_INVALID_ARGUMENT,
            "CurState: the row blocks of the sharded setup must cover every row");
    bounds_[P] = m_;
  }
  s_ = static_cast<i64>(std::ceil(1.1 * static_cast<double>(block)));
  const std::uint64_t emb_seed = splitmix(seed ^ 0x5ce7c3a1b2d4f688ULL);
  cudaStream_t st = ctx_->stream;
  Y_.alloc(std::max<i64>(1, s_ * n_));
  E_.alloc(std::max<i64>(1, s_ * n_));
  // Y = S A over this rank's rows.  Sharded: ONE running sum per entry of Y in
  // row order, carried from rank to rank -- rank p continues the sums rank p-1
  // broadcast, the last rank's Y reaches everyone -- so every chain is the
  // reference's and Y is bit-identical to one rank's.
  auto run_carried = [&](const std::function<void(int)>& f) {
    if (!dist_) {
      f(0);
      return;
    }
    APC_CUDA(cudaMemsetAsync(Y_.p, 0, Y_.bytes(), st));
    for (int p = 0; p < ctx_->nranks; ++p) {
      if (p == ctx_->rank) f(p > 0 ? 1 : 0);
      comm_bcast(ctx_, Y_.p, s_ * n_, p);
    }
  };
  cudaEvent_t ev0, ev1;
  APC_CUDA(cudaEventCreate(&ev0));
  APC_CUDA(cudaEventCreate(&ev1));
  const auto th0 = std::chrono::steady_clock::now();
  if (sketch_kind == 0) {
    // SparseSignEmbedding ctor (sketch.hpp:20-50), host RNG, bit-identical
    const i64 x = std::min(xi, s_);
    std::vector<int> rows(static_cast<size_t>(mt_ * x));
    std::vector<signed char> sg(static_cast<size_t>(mt_ * x));
    // Every column consumes exactly 2*xi draws (xi for Floyd's below(t+1),
    // xi for the signs) unless below() rejects a draw (probability < s/2^64):
    // draw the raw stream sequentially, build the columns in parallel, and
    // fall back to the sequential construction if any draw would be rejected.
    auto build_column = [&](i64 c, auto&& next_draw) {
      i64 pickbuf[64];
      std::vector<i64> big;
      i64* pick = pickbuf;
      if (x > 64) {
        big.resize(static_cast<size_t>(x));
        pick = big.data();
      }
      size_t cnt = 0;
      for (i64 t = s_ - x; t < s_; ++t) {
        const i64 r = static_cast<i64>(next_draw(static_cast<std::uint64_t>(t) + 1));
        bool dup = false;
        for (size_t q = 0; q < cnt; ++q)
          if (pick[q] == r) {
            dup = true;
            break;
          }
        pick[cnt++] = dup ? t : r;
      }
      std::sort(pick, pick + cnt);
      for (size_t q = 0; q < cnt; ++q) rows[c * x + q] = static_cast<int>(pick[q]);
      return cnt;
    };
    HostRng rng(emb_seed);
    bool ok = x <= 64;
    // device path: the raw stream and the columns are produced on the GPU
    DBuf<int> d_rows;
    DBuf<signed char> d_sg;
    bool on_device = false;
    if (ok && mt64_device_ok() && !std::getenv("APC_HOST_EMBEDDING")) {
      DBuf<std::uint64_t> raw(mt_ * 2 * x);
      DBuf<int> bad(1);
      APC_CUDA(cudaMemsetAsync(bad.p, 0, sizeof(int), st));
      mt64_stream_device(ctx_, splitmix(emb_seed), mt_ * 2 * x, raw.p);
      d_rows.alloc(mt_ * x);
      d_sg.alloc(mt_ * x);
      ss_columns_kernel<<<nb(mt_), kT, 0, st>>>(raw.p, mt_, static_cast<int>(s_), static_cast<int>(x), d_rows.p,
                                               d_sg.p, bad.p);
      ctx_->launches++;
      int hb = 0;
      copy_sync(st, &hb, bad.p, sizeof(int), cudaMemcpyDeviceToHost);
      on_device = hb == 0;
      ok = on_device;  // a rejected draw: redo sequentially below
    }
    if (ok && !on_device) {
      std::vector<std::uint64_t> raw(static_cast<size_t>(mt_ * 2 * x));
      for (auto& d : raw) d = rng.bits();
      std::vector<char> bad(static_cast<size_t>(std::max<i64>(1, mt_)), 0);
      host_parallel_for(mt_, [&](i64 b, i64 e) {
        for (i64 c = b; c < e; ++c) {
          const std::uint64_t* d = raw.data() + c * 2 * x;
          i64 k = 0;
          build_column(c, [&](std::uint64_t nn) {
            const std::uint64_t v = d[k++];
            if (!HostRng::below_accepts(v, nn)) bad[c] = 1;
            return v % nn;
          });
          for (i64 q = 0; q < x; ++q) sg[c * x + q] = static_cast<signed char>((d[x + q] & 1ULL) ? 1 : -1);
        }
      }, 16 * x);
      for (char f : bad) ok = ok && !f;
    }
    if (!ok) {  // sequential reference construction (sketch.hpp:31-49)
      HostRng seq(emb_seed);
      for (i64 c = 0; c < mt_; ++c) {
        const size_t cnt = build_column(c, [&](std::uint64_t nn) { return seq.below(nn); });
        for (size_t q = 0; q < cnt; ++q) sg[c * x + q] = static_cast<signed char>(seq.sign() > 0 ? 1 : -1);
      }
    }
    const double scale = 1.0 / std::sqrt(static_cast<double>(x));
    embed_ms_ = std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now() - th0).count();
    if (!on_device) {
      upload(ctx_, d_rows, rows.data(), mt_ * x);
      upload(ctx_, d_sg, sg.data(), mt_ * x);
    }
    APC_CUDA(cudaEventRecord(ev0, st));
    const double mu_scale = amu_ * scale;  // mu * scale_ * ss[q] (sketch.hpp:158)
    const int aug = amu_ > 0.0 ? 1 : 0;
    const size_t smem = sizeof(double) * kSketchWarps * s_ + (sizeof(int) + 1) * kSketchWarps * 32 * x;
    if (smem > 48 * 1024) {
      APC_CUDA(cudaFuncSetAttribute(sketch_ss_dense_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
      APC_CUDA(cudaFuncSetAttribute(sketch_ss_csc_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
    }
    const i64 ml = mloc_;  // this rank's rows (all of A unless distributed)
    const int* srow = d_rows.p + row0_ * x;  // S columns of those rows
    const signed char* ssg = d_sg.p + row0_ * x;
    auto sketch_rows = [&](int carry) {
      if (ml == 0) return;
      const unsigned g = nb(n_, kSketchWarps);
      const char* inv_env = std::getenv("APC_SKETCH_INV");
      const bool inv = !a.sparse && (inv_env ? std::atoi(inv_env) != 0 : true) && s_ <= 1024 && ml * x < (1LL << 30) &&
                       ((ml + kInvRows - 1) / kInvRows) * s_ < (1LL << 30);
      if (inv) {
        // chunk-major inverted index of S (rows of A feeding each sketch row, k ascending)
        const long long cnt = ml * x;
        const long long nchunks = (ml + kInvRows - 1) / kInvRows;
        DBuf<int> keys(cnt), vals(cnt), skeys(cnt), svals(cnt), cptr(nchunks * (s_ + 1));
        DBuf<short> ent(cnt + 8);
        sketch_inv_keys_kernel<<<nb(cnt, 256), 256, 0, st>>>(srow, cnt, static_cast<int>(x), static_cast<int>(s_),
                                                             keys.p, vals.p);
        int end_bit = 1;
        while ((1LL << end_bit) < nchunks * s_ + 1 && end_bit < 31) ++end_bit;
        size_t tb = 0;
        cub::DeviceRadixSort::SortPairs(nullptr, tb, keys.p, skeys.p, vals.p, svals.p, static_cast<int>(cnt), 0, end_bit,
                                        st);
        DBuf<char> tmp(static_cast<long long>(std::max<size_t>(tb, 1)));
        APC_CUDA(cub::DeviceRadixSort::SortPairs(tmp.p, tb, keys.p, skeys.p, vals.p, svals.p, static_cast<int>(cnt), 0,
                                                 end_bit, st));
        sketch_inv_pack_kernel<<<nb(cnt, 256), 256, 0, st>>>(svals.p, cnt, static_cast<int>(x), ssg, ent.p);
        sketch_inv_ptr_kernel<<<nb(nchunks * (s_ + 1), 256), 256, 0, st>>>(skeys.p, cnt, nchunks, static_cast<int>(s_),
                                                                          static_cast<int>(x), cptr.p);
        const int threads = static_cast<int>((s_ + 31) / 32 * 32);
        const long long estride = (kInvRows * x + 7) & ~7LL;
        const size_t ysm = sizeof(double) * 2 * kInvCols * kInvRows + sizeof(short) * 2 * estride +
                           (aug ? sizeof(double) * s_ * kInvCols : 0);
        APC_CUDA(cudaFuncSetAttribute(sketch_ss_dense_inv_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                      static_cast<int>(ysm)));
        sketch_ss_dense_inv_kernel<<<static_cast<unsigned>((n_ + kInvCols - 1) / kInvCols), threads, ysm, st>>>(
            a.dense.p, ml, n_, static_cast<int>(s_), static_cast<int>(x), cptr.p, ent.p, srow, ssg, scale,
            mu_scale, aug, carry, Y_.p);
        ctx_->launches += 6;
        APC_CUDA(cudaGetLastError());
        APC_CUDA(cudaStreamSynchronize(st));  // temporaries go back to the pool
      } else if (!a.sparse) {
        sketch_ss_dense_kernel<<<g, kSketchWarps * 32, smem, st>>>(a.dense.p, ml, n_, (int)s_, (int)x, srow, ssg,
                                                                  scale, mu_scale, aug, carry, Y_.p);
      } else {
        // columns longer than kHeavy go to the row-parallel kernel
        constexpr int kHeavy = 8192;
        std::vector<int> cp(static_cast<size_t>(n_ + 1));
        copy_sync(st, cp.data(), a.at.ptr.p, sizeof(int) * (n_ + 1), cudaMemcpyDeviceToHost);
        std::vector<int> heavy;
        for (i64 j = 0; j < n_; ++j)
          if (cp[j + 1] - cp[j] > kHeavy) heavy.push_back(static_cast<int>(j));
        sketch_ss_csc_kernel<<<g, kSketchWarps * 32, smem, st>>>(a.at.ptr.p, a.at.idx.p, a.at.val.p, ml, n_, (int)s_,
                                                                (int)x, srow, ssg, scale, mu_scale, aug, kHeavy,
                                                                carry, Y_.p);
        if (!heavy.empty()) {
          // inverted-index pass over the long columns, in batches of <= 2^28 pairs
          require(static_cast<double>(a.at.nnz) * x < 4.0e9, APC_INVALID_ARGUMENT,
                  "sketch: nnz * xi exceeds the 32-bit pair encoding");
          constexpr long long kMaxPairs = 1LL << 28;
          size_t h0 = 0;
          while (h0 < heavy.size()) {
            std::vector<int> bcols;
            std::vector<long long> boff;
            long long tot = 0;
            while (h0 < heavy.size()) {
              const long long len = cp[heavy[h0] + 1] - cp[heavy[h0]];
              if (!bcols.empty() && (tot + len) * x > kMaxPairs) break;
              bcols.push_back(heavy[h0]);
              boff.push_back(tot);
              tot += len;
              ++h0;
            }
            const long long npairs = tot * x;
            const int nbc = static_cast<int>(bcols.size());
            DBuf<int> d_bcols;
            DBuf<long long> d_boff;
            upload(ctx_, d_bcols, bcols.data(), nbc);
            upload(ctx_, d_boff, boff.data(), nbc);
            DBuf<unsigned> kin(npairs), kout(npairs), vin(npairs), vout(npairs);
            heavy_pairs_kernel<<<nb(tot), kT, 0, st>>>(a.at.ptr.p, a.at.idx.p, d_bcols.p, d_boff.p, nbc, tot,
                                                       (int)s_, (int)x, srow, kin.p, vin.p);
            int end_bit = 1;
            while ((1LL << end_bit) < static_cast<long long>(nbc) * s_ && end_bit < 32) ++end_bit;
            size_t tmp_bytes = 0;
            cub::DeviceRadixSort::SortPairs(nullptr, tmp_bytes, kin.p, kout.p, vin.p, vout.p,
                                            static_cast<std::int64_t>(npairs), 0, end_bit, st);
            DBuf<char> tmp(static_cast<i64>(tmp_bytes));
            APC_CUDA(cub::DeviceRadixSort::SortPairs(tmp.p, tmp_bytes, kin.p, kout.p, vin.p, vout.p,
                                                     static_cast<std::int64_t>(npairs), 0, end_bit, st));
            heavy_walk_kernel<<<nb(static_cast<long long>(nbc) * s_), kT, 0, st>>>(
                kout.p, vout.p, npairs, d_bcols.p, nbc, (int)s_, (int)x, a.at.idx.p, a.at.val.p, ssg, srow,
                scale, mu_scale, aug, ml, carry, Y_.p);
            ctx_->launches += 3;
            APC_CUDA(cudaStreamSynchronize(st));
          }
        }
      }
    };
    run_carried(sketch_rows);
    ctx_->launches++;
    APC_CUDA(cudaEventRecord(ev1, st));
    APC_CUDA(cudaStreamSynchronize(st));
  } else {
    // GaussianEmbedding (sketch.hpp:173-182): entries scale * gaussian() in storage order
    std::vector<double> S(static_cast<size_t>(s_ * m_));
    HostRng rng(emb_seed);
    const double scale = 1.0 / std::sqrt(static_cast<double>(s_));
    fill_gaussians(rng, S.data(), s_ * m_, scale, true);  // scale * gaussian() in storage order
    embed_ms_ = std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now() - th0).count();
    DBuf<double> d_S;
    const i64 ml = mloc_;
    upload(ctx_, d_S, S.data() + row0_ * s_, s_ * ml);  // S(:, this rank's rows)
    APC_CUDA(cudaEventRecord(ev0, st));
    run_carried([&](int carry) {
      if (ml == 0) return;
      if (!a.sparse && sketch_kind == 2 && !dist_) {  // DMMA: not a carried chain (sharded: the exact kernel)
        launch_sketch_gauss_dmma(ctx_, d_S.p, (int)s_, a.dense.p, ml, n_, Y_.p);
      } else if (!a.sparse) {
        launch_sketch_gauss_exact(st, ctx_->num_sms, d_S.p, (int)s_, a.dense.p, ml, n_, Y_.p, carry);
      } else {
        sketch_gauss_csc_kernel<<<nb(n_ * 32), kT, 0, st>>>(d_S.p, (int)s_, a.at.ptr.p, a.at.idx.p, a.at.val.p, n_,
                                                            carry, Y_.p);
      }
      ctx_->launches++;
    });
    APC_CUDA(cudaEventRecord(ev1, st));
    APC_CUDA(cudaStreamSynchronize(st));
  }
  {
    float ms = 0.f;
    APC_CUDA(cudaEventElapsedTime(&ms, ev0, ev1));
    sketch_ms_ = ms;
    cudaEventDestroy(ev0);
    cudaEventDestroy(ev1);
  }
  APC_CUDA(cudaGetLastError());
  APC_CUDA(cudaMemcpyAsync(E_.p, Y_.p, sizeof(double) * s_ * n_, cudaMemcpyDeviceToDevice, st));
  // ztol = 1e-14 ||Y||_F (frob_norm: sequential over storage order,
  // cur.hpp:224).  The exact sequential sum needs Y on the host; it is read in
  // chunks on a side stream (copy engine) by a host thread while the device
  // goes on with the first augment, and joined when ztol is first used.
  {
    APC_CUDA(cudaEventCreateWithFlags(&ev_sketch_, cudaEventDisableTiming));
    APC_CUDA(cudaEventRecord(ev_sketch_, st));
    const double* y = Y_.p;
    const i64 total = s_ * n_;
    cudaEvent_t ready = ev_sketch_;
    const int dev = ctx_->device;
    ztol_future_ = std::async(std::launch::async, [y, total, ready, dev]() {
      APC_CUDA(cudaSetDevice(dev));
      cudaStream_t cs;
      APC_CUDA(cudaStreamCreateWithFlags(&cs, cudaStreamNonBlocking));
      APC_CUDA(cudaStreamWaitEvent(cs, ready, 0));
      // small chunks: the main thread's short synchronous copies share the
      // copy engine and must not queue behind a long one
      static const i64 kChunk = std::getenv("APC_ZTOL_CHUNK") ? std::atoll(std::getenv("APC_ZTOL_CHUNK")) : (1 << 17);
      double* stage[2] = {nullptr, nullptr};
      const i64 cap = std::min<i64>(kChunk, std::max<i64>(1, total));
      APC_CUDA(cudaMallocHost(&stage[0], sizeof(double) * cap));
      APC_CUDA(cudaMallocHost(&stage[1], sizeof(double) * cap));
      cudaEvent_t done[2];
      APC_CUDA(cudaEventCreateWithFlags(&done[0], cudaEventDisableTiming));
      APC_CUDA(cudaEventCreateWithFlags(&done[1], cudaEventDisableTiming));
      double f2 = 0.0;
      const i64 nch = (total + cap - 1) / cap;
      auto issue = [&](i64 c) {
        const i64 b = c * cap, len = std::min(cap, total - b);
        APC_CUDA(cudaMemcpyAsync(stage[c & 1], y + b, sizeof(double) * len, cudaMemcpyDeviceToHost, cs));
        APC_CUDA(cudaEventRecord(done[c & 1], cs));
      };
      if (nch > 0) issue(0);
      for (i64 c = 0; c < nch; ++c) {
        if (c + 1 < nch) issue(c + 1);  // double-buffered: the next chunk streams while this one is summed
        APC_CUDA(cudaEventSynchronize(done[c & 1]));
        const i64 b = c * cap, len = std::min(cap, total - b);
        const double* h = stage[c & 1];
        for (i64 i = 0; i < len; ++i) f2 += h[i] * h[i];
      }
      cudaEventDestroy(done[0]);
      cudaEventDestroy(done[1]);
      cudaFreeHost(stage[0]);
      cudaFreeHost(stage[1]);
      cudaStreamDestroy(cs);
      return 1e-14 * std::sqrt(f2);
    });
  }
  rowsel_.alloc(std::max<i64>(1, rowsel_len()));
  colsel_.alloc(std::max<i64>(1, n_));
  APC_CUDA(cudaMemsetAsync(rowsel_.p, 0, rowsel_.bytes(), st));
  APC_CUDA(cudaMemsetAsync(colsel_.p, 0, colsel_.bytes(), st));
  SetupProf::add("init.embed", embed_ms_);
  SetupProf::add("init.sketch_kernel", sketch_ms_);
}

DeviceCur::~DeviceCur() {
  if (ztol_future_.valid()) ztol_future_.wait();  // the reader thread still streams Y_
  if (ev_sketch_) cudaEventDestroy(ev_sketch_);
}

std::vector<double> DeviceCur::draw_probes() {
  // probe p = the p-th block of n consecutive Gaussians of the probe stream
  std::vector<double> w(static_cast<size_t>(probes_ * n_));
  fill_gaussians(probe_rng_, w.data(), probes_ * n_);
  return w;
}

void DeviceCur::compute_rho() {
  // spectral_norm_estimate (sketch.hpp:209-223): probes drawn on the host
  const i64 r = probes_;
  std::unique_ptr<ProfScope> ps(new ProfScope("rho.gauss"));
  std::vector<double> w = next_probes_.valid() ? next_probes_.get() : draw_probes();
  static const bool sync_probes = std::getenv("APC_SYNC_PROBES") != nullptr;
  if (!sync_probes) next_probes_ = std::async(std::launch::async, [this] { return draw_probes(); });
  ps.reset(new ProfScope("rho.upload"));
  DBuf<double> d_w, d_out(std::max<i64>(1, s_ * r));
  upload(ctx_, d_w, w.data(), r * n_);
  APC_CUDA(cudaStreamSynchronize(ctx_->stream));
  ps.reset(new ProfScope("rho.kernel"));
  // one warp per CTA: (32 rows of E) x (one probe), spread over the SMs
  dim3 grid(static_cast<unsigned>((s_ + 31) / 32), static_cast<unsigned>(r));
  probe_kernel<<<grid, 32, 0, ctx_->stream>>>(E_.p, s_, n_, d_w.p, d_out.p);
  ctx_->launches++;
  std::vector<double> ew = download(ctx_, d_out.p, s_ * r);
  ps.reset();
  double best = 0.0;
  for (i64 p = 0; p < r; ++p) {
    double nrm2 = 0.0;
    for (i64 i = 0; i < s_; ++i) nrm2 += ew[p * s_ + i] * ew[p * s_ + i];
    best = std::max(best, std::sqrt(nrm2));
  }
  rho_ = 10.0 * std::sqrt(2.0 / 3.14159265358979323846) * best;
  rho_hist_.push_back(rho_);
}

static std::vector<i64> admissible(const LuppOut& piv, i64 cap, double ztol) {  // cur.hpp:341-348
  std::vector<i64> out;
  for (size_t k = 0; k < piv.order.size() && static_cast<i64>(out.size()) < cap; ++k) {
    if (piv.mags[k] <= ztol) break;
    out.push_back(piv.order[k]);
  }
  return out;
}

AugmentResult DeviceCur::augment() {
  cudaStream_t st = ctx_->stream;
  i64 want = block_size_;
  const i64 room = std::min(mt_, n_) - rank();
  require(room > 0, APC_INVALID_ARGUMENT, "CurState::augment: rank at capacity");
  want = std::min(want, room);

  // column pivots: LUPP over (E^row with J zeroed)^T  (n x s)
  work_.ensure(std::max<i64>(1, s_ * n_));
  transpose_zero_kernel<<<nb(s_ * n_), kT, 0, st>>>(E_.p, s_, n_, colsel_.p, work_.p);
  ctx_->launches++;
  std::unique_ptr<ProfScope> ps(new ProfScope("aug.col_lupp"));
  LuppOut col_piv = device_lupp(ctx_, work_.p, n_, s_, want);
  ps.reset(new ProfScope("aug.ecol"));
  std::vector<i64> jplus = admissible(col_piv, want, ztol());
  if (jplus.empty()) {
    if (rank() == 0) compute_rho();
    return {0, true};
  }
  const i64 b = static_cast<i64>(jplus.size()), l = rank();
  DBuf<long long> d_jp, d_J;
  upload(ctx_, d_jp, reinterpret_cast<const long long*>(jplus.data()), b);
  upload(ctx_, d_J, reinterpret_cast<const long long*>(J_.data()), l);

  // urj = U R(:, J+) (l x b col-major), the core solve on the device (same
  // exact-order kernels as the refresh's U R)
  DBuf<double> d_urj;
  if (l > 0) {
    DBuf<double> d_rj(l * b), d_hj(l * b);
    gather_rcols_rm_kernel<<<nb(l * b), kT, 0, st>>>(Rrm_.p, n_, l, d_jp.p, b, d_rj.p);
    // b columns only: warp per column (a thread per column left b threads
    // running l^2-long chains: ~5 ms per augment at C1's l = 500)
    launch_core_solve(d_rj.p, d_hj.p, b);
    d_urj.alloc(l * b);
    rm_to_cm_kernel<<<nb(l * b), kT, 0, st>>>(d_hj.p, l, b, d_urj.p);
    ctx_->launches += 2;
  }
  // E^col = A(:, J+) - C urj, rows I zeroed (m x b; sharded: this rank's rows)
  const i64 ml = mloc_, eld = rowsel_len();
  DBuf<double> ecol(std::max<i64>(1, eld * b));
  DBuf<int> colpos(n_);
  APC_CUDA(cudaMemsetAsync(colpos.p, 0xff, colpos.bytes(), st));
  if (l > 0) set_colpos_kernel<<<nb(l), kT, 0, st>>>(colpos.p, d_J.p, l);
  if (amu_ > 0.0) {  // rows m..m+n-1 of the augmented stack
    ecol_tail_kernel<<<nb(n_), kT, 0, st>>>(m_, n_, eld, colpos.p, l, d_jp.p, b, d_urj.p, rowsel_.p, amu_, ecol.p);
    ctx_->launches++;
  }
  if (ml == 0) {
    // an empty row block: no local rows of E^col
  } else if (!a_.sparse) {
    dim3 grid(nb(ml), static_cast<unsigned>((b + kEcolTile - 1) / kEcolTile));
    ecol_dense_kernel<<<grid, kT, 0, st>>>(a_.dense.p, ml, eld, d_J.p, l, d_jp.p, b, d_urj.p, rowsel_.p, ecol.p);
    ctx_->launches++;
  } else {
    DBuf<int> ccnt(ml + 1), cptr(ml + 1);
    crow_count_kernel<<<nb(ml), kT, 0, st>>>(a_.a.ptr.p, a_.a.idx.p, ml, colpos.p, ccnt.p);
    APC_CUDA(cudaMemsetAsync(ccnt.p + ml, 0, sizeof(int), st));
    size_t tmp = 0;
    cub::DeviceScan::ExclusiveSum(nullptr, tmp, ccnt.p, cptr.p, static_cast<int>(ml + 1), st);
    DBuf<char> tbuf(static_cast<i64>(tmp));
    APC_CUDA(cub::DeviceScan::ExclusiveSum(tbuf.p, tmp, ccnt.p, cptr.p, static_cast<int>(ml + 1), st));
    int total = 0;
    APC_CUDA(cudaMemcpyAsync(&total, cptr.p + ml, sizeof(int), cudaMemcpyDeviceToHost, st));
    APC_CUDA(cudaStreamSynchronize(st));
    DBuf<int> ct(std::max(1, total));
    DBuf<double> cv(std::max(1, total));
    crow_fill_kernel<<<nb(ml), kT, 0, st>>>(a_.a.ptr.p, a_.a.idx.p, a_.a.val.p, ml, colpos.p, cptr.p, ct.p, cv.p);
    ecol_sparse_kernel<<<nb(ml), kT, 0, st>>>(a_.a.ptr.p, a_.a.idx.p, a_.a.val.p, ml, eld, cptr.p, ct.p, cv.p, l,
                                              d_jp.p, b, d_urj.p, rowsel_.p, ecol.p);
    ctx_->launches += 4;
    APC_CUDA(cudaStreamSynchronize(st));
  }
  APC_CUDA(cudaGetLastError());
  ps.reset(new ProfScope("aug.row_lupp"));
  LuppOut row_piv = dist_ ? device_lupp_dist(ctx_, ecol.p, ml, row0_, m_, b, b) : device_lupp(ctx_, ecol.p, mt_, b, b);
  ps.reset();
  std::vector<i64> iplus = admissible(row_piv, b, ztol());
  if (iplus.empty()) return {0, true};
  const bool exhausted = static_cast<i64>(iplus.size()) < want;
  jplus.resize(iplus.size());
  I_.insert(I_.end(), iplus.begin(), iplus.end());
  J_.insert(J_.end(), jplus.begin(), jplus.end());
  last_added_ = static_cast<i64>(iplus.size());
  upload(ctx_, d_jp, reinterpret_cast<const long long*>(jplus.data()), last_added_);
  set_row_flags(iplus, 1);
  set_flags_kernel<<<nb(last_added_), kT, 0, st>>>(colsel_.p, d_jp.p, last_added_, 1);
  ctx_->launches++;
  APC_CUDA(cudaStreamSynchronize(st));
  return {last_added_, exhausted};
}

// rows of the target flagged in rowsel_ (sharded: only this rank's rows, local ids)
void DeviceCur::set_row_flags(const std::vector<i64>& rows, int value) {
  std::vector<long long> loc;
  for (i64 i : rows)
    if (i >= row0_ && i - row0_ < rowsel_len()) loc.push_back(i - row0_);
  if (loc.empty()) return;
  DBuf<long long> d;
  upload(ctx_, d, loc.data(), static_cast<i64>(loc.size()));
  set_flags_kernel<<<nb(static_cast<i64>(loc.size())), kT, 0, ctx_->stream>>>(rowsel_.p, d.p,
                                                                            static_cast<i64>(loc.size()), value);
  ctx_->launches++;
  APC_CUDA(cudaStreamSynchronize(ctx_->stream));
}

// Sharded setup: rows I[first..l) of R = A(I, :) from their owners.  Rank p
// packs the new rows it owns (row-major) and broadcasts them; every rank
// places them in Rrm_.  Exact copies, so R is one rank's R bit for bit.
void DeviceCur::gather_r_rows_dist(i64 first) {
  cudaStream_t st = ctx_->stream;
  const i64 l = rank();
  if (Rrm_.n < l * n_) {  // grow (contents discarded): room for max_rank rows, all rows gathered again
    const i64 cap = std::max(l, std::min(max_rank_ > 0 ? max_rank_ : l, std::min(m_, n_)));
    Rrm_.alloc(std::max<i64>(1, cap * n_));
    first = 0;
  }
  for (int p = 0; p < ctx_->nranks; ++p) {
    std::vector<long long> q, loc;  // slots in R and (on the owner) local rows
    for (i64 t = first; t < l; ++t)
      if (I_[t] >= bounds_[p] && I_[t] < bounds_[p + 1]) {
        q.push_back(t);
        loc.push_back(I_[t] - bounds_[p]);
      }
    const i64 cnt = static_cast<i64>(q.size());
    if (cnt == 0) continue;
    DBuf<double> pk(cnt * n_);
    if (p == ctx_->rank) {
      DBuf<long long> d_loc;
      upload(ctx_, d_loc, loc.data(), cnt);
      if (!a_.sparse) {
        gather_rows_dense_kernel<<<nb(cnt * n_), kT, 0, st>>>(a_.dense.p, mloc_, n_, d_loc.p, cnt, 0.0, pk.p);
      } else {
        APC_CUDA(cudaMemsetAsync(pk.p, 0, pk.bytes(), st));
        scatter_rows_csr_kernel<<<static_cast<unsigned>(cnt), 128, 0, st>>>(a_.a.ptr.p, a_.a.idx.p, a_.a.val.p,
                                                                           mloc_, n_, d_loc.p, cnt, 0.0, pk.p);
      }
      ctx_->launches++;
    }
    comm_bcast(ctx_, pk.p, cnt * n_, p);
    DBuf<long long> d_q;
    upload(ctx_, d_q, q.data(), cnt);
    place_rows_kernel<<<nb(cnt * n_), kT, 0, st>>>(pk.p, d_q.p, cnt, n_, Rrm_.p);
    ctx_->launches++;
    APC_CUDA(cudaStreamSynchronize(st));  // pk and the index buffers go back to the pool
  }
  rvalid_ = l;
}

void DeviceCur::rollback_last_augment() {
  require(last_added_ > 0 && last_added_ <= rank(), APC_INVALID_ARGUMENT,
          "CurState::rollback_last_augment: nothing to roll back");
  cudaStream_t st = ctx_->stream;
  std::vector<i64> di(I_.end() - last_added_, I_.end()), dj(J_.end() - last_added_, J_.end());
  DBuf<long long> d_j;
  upload(ctx_, d_j, reinterpret_cast<const long long*>(dj.data()), last_added_);
  set_row_flags(di, 0);
  set_flags_kernel<<<nb(last_added_), kT, 0, st>>>(colsel_.p, d_j.p, last_added_, 0);
  ctx_->launches++;
  APC_CUDA(cudaStreamSynchronize(st));
  I_.resize(I_.size() - last_added_);
  J_.resize(J_.size() - last_added_);
  rvalid_ = std::min(rvalid_, rank());
  last_added_ = 0;
}

void DeviceCur::refresh() {
  require(rank() > 0, APC_INVALID_ARGUMENT, "CurState::refresh: empty index sets");
  cudaStream_t st = ctx_->stream;
  const i64 l = rank();
  DBuf<long long> d_I, d_J;
  upload(ctx_, d_I, reinterpret_cast<const long long*>(I_.data()), l);
  upload(ctx_, d_J, reinterpret_cast<const long long*>(J_.data()), l);
  // intersection block A(I, J) -> host factor (sharded: R's columns J, after
  // the new rows of R arrived from their owners)
  DBuf<double> d_blk(l * l);
  if (dist_) {
    gather_r_rows_dist(rvalid_);
    gather_rcols_kernel<<<nb(l * l), kT, 0, st>>>(Rrm_.p, n_, l, d_J.p, l, d_blk.p);
  } else {
    gather_block_kernel<<<nb(l * l), kT, 0, st>>>(a_.dense.p, m_, a_.a.ptr.p, a_.a.idx.p, a_.a.val.p,
                                                  a_.sparse ? 1 : 0, d_I.p, d_J.p, l, l, amu_, d_blk.p);
  }
  ctx_->launches++;
  std::unique_ptr<ProfScope> ps(new ProfScope("ref.core_build"));
  static const bool host_core = std::getenv("APC_HOST_CORE") != nullptr;
  if (host_core || (kCoreCols * (l + 1) + l) * 8 > 227 * 1024) {
    block_ = download(ctx_, d_blk.p, l * l);
    core_ = CoreFactorH::build(l, block_, core_kind_);  // throws singular
    host_core_stale_ = false;
    core_l_ = l;
    upload_core();
  } else {
    block_d_ = std::move(d_blk);
    build_core_device(l);  // throws singular
  }
  ps.reset(new ProfScope("ref.rows_H_eres"));
  // R = A(I, :) row-major (all rows re-gathered: I may have changed after a rollback)
  Rrm_.ensure(l * n_);
  if (dist_) {
    // gathered above
  } else if (!a_.sparse) {
    gather_rows_dense_kernel<<<nb(l * n_), kT, 0, st>>>(a_.dense.p, m_, n_, d_I.p, l, amu_, Rrm_.p);
  } else {
    APC_CUDA(cudaMemsetAsync(Rrm_.p, 0, sizeof(double) * l * n_, st));
    scatter_rows_csr_kernel<<<static_cast<unsigned>(l), 128, 0, st>>>(a_.a.ptr.p, a_.a.idx.p, a_.a.val.p, m_,
                                                                     n_, d_I.p, l, amu_, Rrm_.p);
  }
  ctx_->launches++;
  // H = U R (core solve per column)
  H_.ensure(l * n_);
  launch_core_solve(Rrm_.p, H_.p, n_);
  // E^row = Y - Y(:, J) H
  DBuf<double> d_sc(s_ * l);
  gather_sc_kernel<<<nb(s_ * l), kT, 0, st>>>(Y_.p, s_, d_J.p, l, d_sc.p);
  eres_kernel<<<nb(n_ * 32), kT, 0, st>>>(Y_.p, d_sc.p, H_.p, s_, n_, l, E_.p);
  ctx_->launches += 3;
  APC_CUDA(cudaGetLastError());
  APC_CUDA(cudaStreamSynchronize(st));
  ps.reset(new ProfScope("ref.rho"));
  compute_rho();
}

// out = U rhs for the ncols columns of a row-major l x ncols block (CoreFactor
// solve, cur.hpp:119-144): warp per column when there are few columns
// (latency-bound chains, C1: n = 500); with many columns the FP64 pipe is the
// limit and a thread per column issues 32x fewer predicated instructions
void DeviceCur::launch_core_solve(const double* rhs_rm, double* out_rm, i64 ncols) const {
  cudaStream_t st = ctx_->stream;
  const i64 l = core_l_;
  static const bool force_warp = std::getenv("APC_CORE_SOLVE_WARP") != nullptr;
  if (l <= 1024 && (ncols <= 4096 || force_warp) && !std::getenv("APC_CORE_SOLVE_THREAD")) {
    const unsigned g = static_cast<unsigned>((ncols * 32 + 127) / 128);
    const int li = static_cast<int>(l);
    if (l <= 128)
      core_solve_warp_kernel<4><<<g, 128, 0, st>>>(rhs_rm, out_rm, li, ncols, core_kind_, core_h_.p, core_at_.p,
                                                  core_perm_.p);
    else if (l <= 256)
      core_solve_warp_kernel<8><<<g, 128, 0, st>>>(rhs_rm, out_rm, li, ncols, core_kind_, core_h_.p, core_at_.p,
                                                  core_perm_.p);
    else if (l <= 512)
      core_solve_warp_kernel<16><<<g, 128, 0, st>>>(rhs_rm, out_rm, li, ncols, core_kind_, core_h_.p, core_at_.p,
                                                   core_perm_.p);
    else
      core_solve_warp_kernel<32><<<g, 128, 0, st>>>(rhs_rm, out_rm, li, ncols, core_kind_, core_h_.p, core_at_.p,
                                                   core_perm_.p);
  } else {
    core_solve_cols_kernel<<<nb(ncols, 128), 128, 0, st>>>(rhs_rm, out_rm, l, ncols, core_kind_, core_h_.p,
                                                           core_a_.p, core_perm_.p);
  }
  ctx_->launches++;
  APC_CUDA(cudaGetLastError());
}

Vec DeviceCur::core_solve_rm(const Vec& rhs_rm, i64 ncols) const {
  const i64 l = core_l_;
  DBuf<double> b(std::max<i64>(1, l * ncols)), o(std::max<i64>(1, l * ncols));
  APC_CUDA(cudaMemcpyAsync(b.p, rhs_rm.data(), sizeof(double) * l * ncols, cudaMemcpyHostToDevice, ctx_->stream));
  launch_core_solve(b.p, o.p, ncols);
  return download(ctx_, o.p, l * ncols);
}

void DeviceCur::build_core_device(i64 l) {
  cudaStream_t st = ctx_->stream;
  core_a_.ensure(l * l);
  core_at_.ensure(l * l);
  core_h_.ensure(l * l);
  core_perm_.ensure(l);
  DBuf<double> vbuf(2 * l), sbuf(8);
  DBuf<int> flag(1);
  APC_CUDA(cudaMemsetAsync(core_h_.p, 0, sizeof(double) * l * l, st));
  const int smem = static_cast<int>((kCoreCols * (l + 1) + l) * sizeof(double));
  static int attr = 0;
  if (smem > attr) {
    APC_CUDA(cudaFuncSetAttribute(core_build_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, smem));
    attr = smem;
  }
  CoreBuildArgs args{block_d_.p, l, core_kind_, core_a_.p, core_at_.p, core_h_.p, core_perm_.p, vbuf.p, sbuf.p, flag.p};
  void* kargs[] = {&args};
  const unsigned grid = static_cast<unsigned>((l + kCoreCols - 1) / kCoreCols);
  APC_CUDA(cudaLaunchCooperativeKernel(reinterpret_cast<const void*>(core_build_kernel), dim3(grid), dim3(kCoreCols),
                                       kargs, smem, st));
  ctx_->launches++;
  int singular = 0;
  APC_CUDA(cudaMemcpyAsync(&singular, flag.p, sizeof(int), cudaMemcpyDeviceToHost, st));
  APC_CUDA(cudaStreamSynchronize(st));
  core_l_ = l;
  host_core_stale_ = true;
  if (singular) fail(APC_SINGULAR, "CoreFactor: intersection block numerically singular");
}

const CoreFactorH& DeviceCur::core() const {
  if (host_core_stale_) {
    const i64 l = core_l_;
    CoreFactorH f;
    f.l = l;
    f.kind = core_kind_;
    if (core_kind_ == 0) {
      f.qr.m = f.qr.k = l;
      f.qr.a = download(ctx_, core_a_.p, l * l);
      f.qr.hh = download(ctx_, core_h_.p, l * l);
    } else {
      f.lu = download(ctx_, core_a_.p, l * l);
      auto pm = download(ctx_, core_perm_.p, l);
      f.perm.assign(pm.begin(), pm.end());
    }
    core_ = std::move(f);
    block_ = download(ctx_, block_d_.p, l * l);
    host_core_stale_ = false;
  }
  return core_;
}

const Vec& DeviceCur::intersection() const {
  (void)core();
  return block_;
}

void DeviceCur::upload_core() {
  const i64 l = core_.l;
  if (core_.kind == 0) {
    upload(ctx_, core_h_, core_.qr.hh.data(), l * l);
    upload(ctx_, core_a_, core_.qr.a.data(), l * l);
    core_at_host_ = transpose(l, l, core_.qr.a);
  } else {
    upload(ctx_, core_a_, core_.lu.data(), l * l);
    upload(ctx_, core_perm_, reinterpret_cast<const long long*>(core_.perm.data()), l);
    core_at_host_ = transpose(l, l, core_.lu);
  }
  upload(ctx_, core_at_, core_at_host_.data(), l * l);
}

// G = C^T C of the target's selected columns (l x l, full), on the device:
// gather + DSYRK for dense A, row blocks densified + DSYRK accumulated in
// fixed order for sparse A; + amu^2 I for the augmented stack.
Vec DeviceCur::c_gram() const {
  const i64 l = rank();
  cudaStream_t st = ctx_->stream;
  DBuf<long long> d_J;
  upload(ctx_, d_J, reinterpret_cast<const long long*>(J_.data()), l);
  DBuf<double> G(l * l);
  const i64 ml = mloc_;  // sharded: this rank's rows, then a sum over the ranks
  APC_CUDA(cudaMemsetAsync(G.p, 0, G.bytes(), st));
  if (ml == 0) {
    // no local rows: a zero partial
  } else if (!a_.sparse) {
    DBuf<double> C(ml * l);
    gather_cols_kernel<<<nb(ml * l), kT, 0, st>>>(a_.dense.p, ml, d_J.p, l, C.p);
    // exact chol_gram order: T_C then equals the reference's factor bit for bit
    dim3 grid(static_cast<unsigned>((l + 63) / 64), static_cast<unsigned>((l + 63) / 64));
    gram_exact_kernel<<<grid, 256, 0, st>>>(C.p, ml, l, G.p);
    ctx_->launches += 2;
  } else {
    DBuf<int> colpos(n_);
    APC_CUDA(cudaMemsetAsync(colpos.p, 0xff, colpos.bytes(), st));
    set_colpos_kernel<<<nb(l), kT, 0, st>>>(colpos.p, d_J.p, l);
    const i64 rb = std::min<i64>(ml, std::max<i64>(1, (1LL << 28) / std::max<i64>(1, l)));  // <= 2 GB blocks
    DBuf<double> D(rb * l);
    for (i64 r0 = 0; r0 < ml; r0 += rb) {
      const i64 cnt = std::min(rb, ml - r0);
      APC_CUDA(cudaMemsetAsync(D.p, 0, sizeof(double) * cnt * l, st));
      densify_rows_kernel<<<nb(cnt), kT, 0, st>>>(a_.a.ptr.p, a_.a.idx.p, a_.a.val.p, r0, cnt, colpos.p, D.p);
      dsyrk_t(ctx_, l, cnt, 1.0, D.p, cnt, r0 == 0 ? 0.0 : 1.0, G.p, l);
      ctx_->launches++;
    }
  }
  // sharded: the ranks' partial Grams summed (identical on every rank; the
  // single-rank chol_gram sum order is not kept across the row blocks)
  if (dist_) comm_allreduce(ctx_, G.p, l * l);
  Vec g = download(ctx_, G.p, l * l);
  for (i64 j = 0; j < l; ++j)
    for (i64 i = j + 1; i < l; ++i) g[j * l + i] = g[i * l + j];  // mirror the upper triangle
  if (amu_ > 0.0)
    for (i64 t = 0; t < l; ++t) g[t * l + t] += amu_ * amu_;
  return g;
}

Vec DeviceCur::r_dense_rows(i64 first, i64 count) const {
  return download(ctx_, Rrm_.p + first * n_, count * n_);
}

Vec DeviceCur::c_dense() const {
  require(!a_.sparse, APC_INVALID_ARGUMENT, "c_dense: dense A only");
  require(!dist_, APC_NOT_APPLICABLE, "c_dense: the sharded setup holds no whole column of A");
  const i64 l = rank();
  Vec out(static_cast<size_t>(mt_ * l), 0.0);
  for (i64 t = 0; t < l; ++t)
    APC_CUDA(cudaMemcpyAsync(out.data() + t * mt_, a_.dense.p + J_[t] * m_, sizeof(double) * m_,
                             cudaMemcpyDeviceToHost, ctx_->stream));
  APC_CUDA(cudaStreamSynchronize(ctx_->stream));
  if (amu_ > 0.0)  // AugmentedOperator::extract_cols (matrix.hpp:428-438)
    for (i64 t = 0; t < l; ++t) out[t * mt_ + m_ + J_[t]] = amu_;
  return out;
}

// warp per row: nonzeros of each row of a row-major l x n matrix
__global__ void row_nnz_kernel(const double* __restrict__ R, long long l, long long n, int* __restrict__ cnt) {
  const long long i = (static_cast<long long>(blockIdx.x) * blockDim.x + threadIdx.x) >> 5;
  const int lane = threadIdx.x & 31;
  if (i >= l) return;
  int c = 0;
  for (long long j = lane; j < n; j += 32) c += R[i * n + j] != 0.0;
  for (int o = 16; o > 0; o >>= 1) c += __shfl_xor_sync(0xffffffffu, c, o);
  if (lane == 0) cnt[i] = c;
}
// warp per row: (column, value) of the nonzeros in column order from ptr[i]
__global__ void row_compact_kernel(const double* __restrict__ R, long long l, long long n,
                                   const long long* __restrict__ ptr, int* __restrict__ idx,
                                   double* __restrict__ val) {
  const long long i = (static_cast<long long>(blockIdx.x) * blockDim.x + threadIdx.x) >> 5;
  const int lane = threadIdx.x & 31;
  if (i >= l) return;
  long long q = ptr[i];
  for (long long j0 = 0; j0 < n; j0 += 32) {
    const long long j = j0 + lane;
    const double v = j < n ? R[i * n + j] : 0.0;
    const unsigned mask = __ballot_sync(0xffffffffu, v != 0.0);
    if (v != 0.0) {
      const long long at = q + __popc(mask & ((1u << lane) - 1u));
      idx[at] = static_cast<int>(j);
      val[at] = v;
    }
    q += __popc(mask);
  }
}

namespace {
// nonzeros of the rows of a device row-major l x n matrix as a host CSC-like
// triple (column t = row t)
void dense_rows_to_host_csr(apc_ctx* ctx, const double* R, i64 l, i64 n, std::vector<i64>& ptr,
                            std::vector<i64>& idx, Vec& val) {
  cudaStream_t st = ctx->stream;
  DBuf<int> cnt(std::max<i64>(1, l));
  row_nnz_kernel<<<nb(l * 32), kT, 0, st>>>(R, l, n, cnt.p);
  std::vector<int> hc = download(ctx, cnt.p, l);
  std::vector<long long> hp(static_cast<size_t>(l + 1), 0);
  for (i64 i = 0; i < l; ++i) hp[i + 1] = hp[i] + hc[i];
  const i64 nnz = hp[l];
  DBuf<long long> d_ptr;
  upload(ctx, d_ptr, hp.data(), l + 1);
  DBuf<int> d_idx(std::max<i64>(1, nnz));
  DBuf<double> d_val(std::max<i64>(1, nnz));
  row_compact_kernel<<<nb(l * 32), kT, 0, st>>>(R, l, n, d_ptr.p, d_idx.p, d_val.p);
  ctx->launches += 2;
  std::vector<int> hi = download(ctx, d_idx.p, nnz);
  val = download(ctx, d_val.p, nnz);
  ptr.assign(hp.begin(), hp.end());
  idx.assign(hi.begin(), hi.end());
}

// rows `which` of a device CSR as a host CSC-like triple (columns = which order)
void csr_rows_to_host(apc_ctx* ctx, const Csr& c, const std::vector<i64>& which, std::vector<i64>& ptr,
                      std::vector<i64>& idx, Vec& val) {
  ptr.assign(1, 0);
  idx.clear();
  val.clear();
  std::vector<int> hp(2), hi;
  std::vector<double> hv;
  for (i64 r : which) {
    copy_sync(ctx->stream, hp.data(), c.ptr.p + r, sizeof(int) * 2, cudaMemcpyDeviceToHost);
    const int len = hp[1] - hp[0];
    hi.resize(len);
    hv.resize(len);
    if (len > 0) {
      APC_CUDA(cudaMemcpyAsync(hi.data(), c.idx.p + hp[0], sizeof(int) * len, cudaMemcpyDeviceToHost, ctx->stream));
      copy_sync(ctx->stream, hv.data(), c.val.p + hp[0], sizeof(double) * len, cudaMemcpyDeviceToHost);
    }
    for (int q = 0; q < len; ++q) {
      idx.push_back(hi[q]);
      val.push_back(hv[q]);
    }
    ptr.push_back(static_cast<i64>(idx.size()));
  }
}
}  // namespace

void DeviceCur::c_csc(std::vector<i64>& ptr, std::vector<i64>& idx, Vec& val) const {
  require(!dist_, APC_NOT_APPLICABLE, "c_csc: the sharded setup holds no whole column of A");
  csr_rows_to_host(ctx_, a_.at, J_, ptr, idx, val);  // CSR(A^T) row j == column j of A
  if (amu_ > 0.0) {  // + amu at row m + J[t] of column t (matrix.hpp:439-446)
    std::vector<i64> p2(1, 0), i2;
    Vec v2;
    for (size_t t = 0; t + 1 < ptr.size(); ++t) {
      for (i64 q = ptr[t]; q < ptr[t + 1]; ++q) {
        i2.push_back(idx[q]);
        v2.push_back(val[q]);
      }
      i2.push_back(m_ + J_[t]);
      v2.push_back(amu_);
      p2.push_back(static_cast<i64>(i2.size()));
    }
    ptr.swap(p2);
    idx.swap(i2);
    val.swap(v2);
  }
}

void DeviceCur::rt_csc(std::vector<i64>& ptr, std::vector<i64>& idx, Vec& val) const {
  if (dist_) {  // from the replicated dense rows of R: their nonzeros, compacted on the device
    dense_rows_to_host_csr(ctx_, Rrm_.p, rank(), n_, ptr, idx, val);
    return;
  }
  // row i of the target == column of R^T; augmented rows are amu e_{i-m}
  std::vector<i64> base;
  for (i64 i : I_)
    if (i < m_) base.push_back(i);
  std::vector<i64> bp, bi;
  Vec bv;
  csr_rows_to_host(ctx_, a_.a, base, bp, bi, bv);
  ptr.assign(1, 0);
  idx.clear();
  val.clear();
  size_t k = 0;
  for (i64 i : I_) {
    if (i < m_) {
      for (i64 q = bp[k]; q < bp[k + 1]; ++q) {
        idx.push_back(bi[q]);
        val.push_back(bv[q]);
      }
      ++k;
    } else {
      idx.push_back(i - m_);
      val.push_back(amu_);
    }
    ptr.push_back(static_cast<i64>(idx.size()));
  }
}

}  // namespace apc

// ---------------------------------------------------------------------------
// C-ABI: CurState stepping and the LUPP pivot order
// ---------------------------------------------------------------------------
struct apc_cur {
  apc::DeviceCur* cur;
  apc_ctx* ctx;
};

namespace apc {
int capi_guard(apc_ctx* ctx, const std::function<void()>& f);
}

extern "C" {

int apc_cur_create(apc_mat* a, int64_t block, uint64_t seed, int64_t xi, int64_t probe_count, int core_kind,
                   int sketch_kind, apc_cur** out) {
  *out = nullptr;
  return apc::capi_guard(a->ctx, [&] {
    auto* c = new apc_cur{nullptr, a->ctx};
    try {
      c->cur = new apc::DeviceCur(*a, block, seed, xi, probe_count, core_kind, sketch_kind, 0);
    } catch (...) {
      delete c;
      throw;
    }
    *out = c;
  });
}

int apc_cur_free(apc_cur* c) {
  if (c) {
    delete c->cur;
    delete c;
  }
  return APC_OK;
}

int apc_cur_augment(apc_cur* c, int64_t* added, int* exhausted) {
  return apc::capi_guard(c->ctx, [&] {
    apc::AugmentResult r = c->cur->augment();
    *added = r.added;
    *exhausted = r.exhausted ? 1 : 0;
  });
}

int apc_cur_refresh(apc_cur* c) { return apc::capi_guard(c->ctx, [&] { c->cur->refresh(); }); }

int apc_cur_rollback_last_augment(apc_cur* c) {
  return apc::capi_guard(c->ctx, [&] { c->cur->rollback_last_augment(); });
}

int apc_cur_state(const apc_cur* c, int64_t* rank, double* rho, int64_t* sketch_rows, int64_t* n_rho) {
  if (rank) *rank = c->cur->rank();
  if (rho) *rho = c->cur->rho();
  if (sketch_rows) *sketch_rows = c->cur->sketch_rows();
  if (n_rho) *n_rho = static_cast<int64_t>(c->cur->rho_history().size());
  return APC_OK;
}

int apc_cur_indices(const apc_cur* c, int64_t* rows, int64_t* cols) {
  std::copy(c->cur->rows().begin(), c->cur->rows().end(), rows);
  std::copy(c->cur->cols().begin(), c->cur->cols().end(), cols);
  return APC_OK;
}

int apc_cur_timing(const apc_cur* c, double* embedding_host_ms, double* sketch_device_ms) {
  if (embedding_host_ms) *embedding_host_ms = c->cur->embedding_ms();
  if (sketch_device_ms) *sketch_device_ms = c->cur->sketch_ms();
  return APC_OK;
}

int apc_cur_rho_history(const apc_cur* c, double* rho) {
  std::copy(c->cur->rho_history().begin(), c->cur->rho_history().end(), rho);
  return APC_OK;
}

int apc_cur_sketch(const apc_cur* c, double* y) {
  return apc::capi_guard(c->ctx, [&] {
    const apc::i64 cnt = c->cur->sketch_rows() * c->cur->n();
    apc::copy_sync(c->ctx->stream, y, c->cur->y_dev(), sizeof(double) * cnt, cudaMemcpyDeviceToHost);
  });
}

int apc_cur_residual(const apc_cur* c, double* e) {
  return apc::capi_guard(c->ctx, [&] {
    const apc::i64 cnt = c->cur->sketch_rows() * c->cur->n();
    apc::copy_sync(c->ctx->stream, e, c->cur->eres_dev(), sizeof(double) * cnt, cudaMemcpyDeviceToHost);
  });
}

int apc_lupp(apc_ctx* ctx, const double* w, int64_t rows, int64_t cols, int64_t max_pivots, int64_t* order,
             double* mags, int64_t* steps) {
  return apc::capi_guard(ctx, [&] {
    apc::DBuf<double> d(std::max<apc::i64>(1, rows * cols));
    if (rows * cols > 0)
      apc::copy_sync(ctx->stream, d.p, w, sizeof(double) * rows * cols, cudaMemcpyHostToDevice);
    apc::LuppOut o = apc::device_lupp(ctx, d.p, rows, cols, max_pivots);
    *steps = static_cast<int64_t>(o.order.size());
    std::copy(o.order.begin(), o.order.end(), order);
    std::copy(o.mags.begin(), o.mags.end(), mags);
  });
}

}  // extern "C"
