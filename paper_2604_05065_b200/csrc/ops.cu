// Operator kernels and matrix upload (see ops.cuh for the design notes).
#include <cub/device/device_radix_sort.cuh>
#include <cub/device/device_scan.cuh>

#include <algorithm>
#include <cstdlib>
#include <cstdio>
#include <cstring>
#include <map>
#include <memory>
#include <mutex>
#include <utility>

#include "host_rng.hpp"
#include "ops.cuh"

namespace apc {

// ---------------------------------------------------------------------------
// Dense A^T u
// ---------------------------------------------------------------------------
__global__ void __launch_bounds__(kDenseAdjThreads)
dense_adj_kernel(const double* __restrict__ A, long long ld, long long mloc, long long n,
                 const double* __restrict__ u, long long rows_per_split,
                 double* __restrict__ part, unsigned* __restrict__ grp_ctr,
                 double* __restrict__ out, const int* done) {
  if (done && *done) return;
  const int w = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const long long cA = static_cast<long long>(blockIdx.x) * kDenseAdjCols + w;
  const long long cB = cA + 8;
  const long long rb = static_cast<long long>(blockIdx.y) * rows_per_split;
  const long long re = rb + rows_per_split < mloc ? rb + rows_per_split : mloc;
  const bool okA = cA < n, okB = cB < n;
  const double* pa = A + (okA ? cA : 0) * ld;
  const double* pb = A + (okB ? cB : 0) * ld;
  double sa0 = 0.0, sa1 = 0.0, sb0 = 0.0, sb1 = 0.0;
  long long r = rb + lane;
  if (okA && okB) {
    for (; r + 32 < re; r += 64) {
      double u0 = __ldg(u + r), u1 = __ldg(u + r + 32);
      sa0 += __ldg(pa + r) * u0;
      sb0 += __ldg(pb + r) * u0;
      sa1 += __ldg(pa + r + 32) * u1;
      sb1 += __ldg(pb + r + 32) * u1;
    }
    for (; r < re; r += 32) {
      double u0 = __ldg(u + r);
      sa0 += __ldg(pa + r) * u0;
      sb0 += __ldg(pb + r) * u0;
    }
  } else if (okA) {
    for (; r < re; r += 32) sa0 += __ldg(pa + r) * __ldg(u + r);
  }
  double sa = warp_sum(sa0 + sa1), sb = warp_sum(sb0 + sb1);
  const int msplit = gridDim.y;
  if (msplit == 1) {
    if (lane == 0) {
      if (okA) out[cA] = sa;
      if (okB) out[cB] = sb;
    }
    return;
  }
  if (lane == 0) {
    if (okA) part[blockIdx.y * n + cA] = sa;
    if (okB) part[blockIdx.y * n + cB] = sb;
  }
  if (!elect_last_block(grp_ctr + blockIdx.x, msplit)) return;
  if (lane == 0) {
    double ta = 0.0, tb = 0.0;
    for (int s = 0; s < msplit; ++s) {
      if (okA) ta += ((volatile double*)part)[s * n + cA];
      if (okB) tb += ((volatile double*)part)[s * n + cB];
    }
    if (okA) out[cA] = ta;
    if (okB) out[cB] = tb;
  }
}

// ---------------------------------------------------------------------------
// CSR over work units (transpose products)
// ---------------------------------------------------------------------------
#ifndef APC_UNITS_PRED
#define APC_UNITS_PRED 1
#endif
// lanes per work unit: units are at most kCsrUnitMax entries and most rows of
// A^T are short, so a half warp per unit doubles the units in flight
#ifndef APC_UNITS_G
#define APC_UNITS_G 32
#endif
__global__ void __launch_bounds__(kCsrUnitThreads)
csr_units_kernel(const int* __restrict__ ptr, const int* __restrict__ idx,
                 const double* __restrict__ val, const double* __restrict__ u, long long n_units,
                 const int* __restrict__ urow, const int* __restrict__ ustart,
                 const int* __restrict__ uend, const int* __restrict__ uslot,
                 double* __restrict__ out, double* __restrict__ upart, const int* done) {
  constexpr int G = APC_UNITS_G;
  if (done && *done) return;
  const long long unit = (static_cast<long long>(blockIdx.x) * kCsrUnitThreads + threadIdx.x) / G;
  const int lane = threadIdx.x % G;
  const bool ok = unit < n_units;
  if (G == 32 && !ok) return;
  const int b = ok ? __ldg(ustart + unit) : 0, e = ok ? __ldg(uend + unit) : 0;
  double s0 = 0.0, s1 = 0.0, s2 = 0.0, s3 = 0.0;
  int q = b + lane;
  // CSR(A^T) streamed with evict-first loads so the gathered u stays in L2
  for (; q + 3 * G < e; q += 4 * G) {
    const int i0 = __ldcs(idx + q), i1 = __ldcs(idx + q + G), i2 = __ldcs(idx + q + 2 * G),
              i3 = __ldcs(idx + q + 3 * G);
    s0 += __ldcs(val + q) * __ldg(u + i0);
    s1 += __ldcs(val + q + G) * __ldg(u + i1);
    s2 += __ldcs(val + q + 2 * G) * __ldg(u + i2);
    s3 += __ldcs(val + q + 3 * G) * __ldg(u + i3);
  }
#if APC_UNITS_PRED
  // the remainder (< 4 G entries) as one predicated block: its index loads, then
  // its u gathers, all in flight together (short rows: the common case of the
  // tail rows of a head-split A^T)
  if (q < e) {
    const bool o1 = q + G < e, o2 = q + 2 * G < e;
    const int i0 = __ldcs(idx + q);
    const int i1 = o1 ? __ldcs(idx + q + G) : 0;
    const int i2 = o2 ? __ldcs(idx + q + 2 * G) : 0;
    const double v0 = __ldcs(val + q);
    const double v1 = o1 ? __ldcs(val + q + G) : 0.0;
    const double v2 = o2 ? __ldcs(val + q + 2 * G) : 0.0;
    const double g0 = __ldg(u + i0);
    const double g1 = o1 ? __ldg(u + i1) : 0.0;
    const double g2 = o2 ? __ldg(u + i2) : 0.0;
    s0 += v0 * g0;
    if (o1) s1 += v1 * g1;
    if (o2) s2 += v2 * g2;
  }
#else
  for (; q < e; q += G) s0 += __ldcs(val + q) * __ldg(u + __ldcs(idx + q));
#endif
  s0 += s2;
  s1 += s3;
  double s = s0 + s1;
#pragma unroll
  for (int o = G / 2; o > 0; o >>= 1) s += __shfl_xor_sync(0xffffffffu, s, o);
  if (ok && lane == 0) {
    const int slot = __ldg(uslot + unit);
    if (slot < 0) out[__ldg(urow + unit)] = s;
    else upart[slot] = s;
  }
  (void)ptr;
}

namespace {

__global__ void unit_fixup_kernel(const double* out_raw, long long n, double mu, const double* tail, double* y) {
  long long j = static_cast<long long>(blockIdx.x) * blockDim.x + threadIdx.x;
  if (j >= n) return;
  double v = out_raw[j];
  if (tail) v += mu * tail[j];
  y[j] = v;
}

__global__ void tail_fwd_kernel(const double* x, long long n, double mu, double* y) {
  long long j = static_cast<long long>(blockIdx.x) * blockDim.x + threadIdx.x;
  if (j < n) y[j] = mu * x[j];
}

__global__ void add_tail_kernel(const double* t, long long n, double mu, double* y) {
  long long j = static_cast<long long>(blockIdx.x) * blockDim.x + threadIdx.x;
  if (j < n) y[j] += mu * t[j];
}

// ---- CSC -> CSR(A) build (stable radix sort by row keeps columns ascending)
// colof[k] = column of entry k (thread per entry, binary search in colptr:
// balanced even when a few columns hold most entries, as C5's Zipf head does)
__global__ void expand_cols_kernel(const int* colptr, long long ncols, long long nnz, int* colof) {
  const long long k = static_cast<long long>(blockIdx.x) * blockDim.x + threadIdx.x;
  if (k >= nnz) return;
  long long lo = 0, hi = ncols;  // last j with colptr[j] <= k
  while (hi - lo > 1) {
    const long long mid = (lo + hi) >> 1;
    if (colptr[mid] <= k) lo = mid;
    else hi = mid;
  }
  colof[k] = static_cast<int>(lo);
}
__global__ void fill_int_kernel(int* p, long long n, int v) {
  long long k = static_cast<long long>(blockIdx.x) * blockDim.x + threadIdx.x;
  if (k < n) p[k] = v;
}
__global__ void iota_kernel(int* p, long long n) {
  long long k = static_cast<long long>(blockIdx.x) * blockDim.x + threadIdx.x;
  if (k < n) p[k] = static_cast<int>(k);
}
__global__ void gather_csr_kernel(const int* perm, const int* colof, const double* val,
                                  long long nnz, int* oidx, double* oval) {
  long long k = static_cast<long long>(blockIdx.x) * blockDim.x + threadIdx.x;
  if (k >= nnz) return;
  int p = perm[k];
  oidx[k] = colof[p];
  oval[k] = val[p];
}
__global__ void row_ptr_kernel(const int* sorted_rows, long long nnz, long long rows, int* ptr) {
  // ptr[r] = first k with sorted_rows[k] >= r (lower bound), ptr[rows] = nnz
  long long r = static_cast<long long>(blockIdx.x) * blockDim.x + threadIdx.x;
  if (r > rows) return;
  long long lo = 0, hi = nnz;
  while (lo < hi) {
    long long mid = (lo + hi) >> 1;
    if (sorted_rows[mid] < r) lo = mid + 1;
    else hi = mid;
  }
  ptr[r] = static_cast<int>(lo);
}

inline unsigned nblk(long long n, int t) { return static_cast<unsigned>((n + t - 1) / t); }

// ---- hot-relabelled SELL-32 build (HotSell, apc_internal.hpp)
__device__ __forceinline__ long long upper_slot(const int* ptr, long long n, long long p) {
  long long lo = 0, hi = n;  // last k with ptr[k] <= p
  while (hi - lo > 1) {
    const long long mid = (lo + hi) >> 1;
    if (ptr[mid] <= p) lo = mid;
    else hi = mid;
  }
  return lo;
}
// entry p of the relabelled column order: key = its row, value = p
__global__ void hot_keys_kernel(const int* nptr, const int* hot, const int* tptr, const int* trow, long long n,
                                long long nnz, int* keys, int* vals) {
  const long long p = static_cast<long long>(blockIdx.x) * blockDim.x + threadIdx.x;
  if (p >= nnz) return;
  const long long k = upper_slot(nptr, n, p);
  keys[p] = trow[tptr[hot[k]] + (p - nptr[k])];
  vals[p] = static_cast<int>(p);
}
__global__ void hot_width_kernel(const int* __restrict__ ptr, long long rows, long long chunks, int* __restrict__ width) {
  const long long ch = static_cast<long long>(blockIdx.x) * blockDim.x + threadIdx.x;
  if (ch > chunks) return;
  int w = 0;
  if (ch < chunks) {
    const long long rend = ch * 32 + 32 < rows ? ch * 32 + 32 : rows;
    for (long long r = ch * 32; r < rend; ++r) w = max(w, ptr[r + 1] - ptr[r]);
  }
  width[ch] = 32 * w;
}
// sorted entry q (row-major, relabelled column order within rows) -> its SELL slot
__global__ void hot_fill_kernel(const int* sorted_vals, const int* rptr, const int* off, const int* nptr,
                                const int* hot, const int* tptr, const double* tval, long long n, long long rows,
                                int* sidx, double* sval) {
  const long long r = static_cast<long long>(blockIdx.x) * blockDim.x + threadIdx.x;
  if (r >= rows) return;
  const long long base = off[r >> 5] + (r & 31);
  const int b = rptr[r], e = rptr[r + 1];
  for (int q = b; q < e; ++q) {
    const long long p = sorted_vals[q];
    const long long k = upper_slot(nptr, n, p);
    sidx[base + 32LL * (q - b)] = static_cast<int>(k);
    sval[base + 32LL * (q - b)] = tval[tptr[hot[k]] + (p - nptr[k])];
  }
}

// sum of the partials of every split row (rows longer than one work unit),
// block per split row, fixed order: written to out[row] so every consumer of
// op_adj_raw (LSQR epilogue, NCCL allreduce, op_adj) reads plain values
// split rows of a units CSR: warp per row adds its partials in slot order
__global__ void __launch_bounds__(256)
split_fixup_kernel(const int* __restrict__ srows, const int* __restrict__ rfirst, const int* __restrict__ rcount,
                   long long n_split, const double* __restrict__ upart, double* __restrict__ out, const int* done) {
  if (done && *done) return;
  const long long r = (static_cast<long long>(blockIdx.x) * 256 + threadIdx.x) >> 5;
  const int lane = threadIdx.x & 31;
  if (r >= n_split) return;
  const int j = srows[r];
  const int f = rfirst[j], cnt = rcount[j];
  double s = 0.0;
  for (int k = lane; k < cnt; k += 32) s += upart[f + k];
  s = warp_sum(s);
  if (lane == 0) out[j] = s;
}

// ---- segmented A^T u over key-sorted entry streams (HeadAdj, apc_internal.hpp)
// Two streams share one kernel body (SegAdj policies below):
//  * head: the entries of the long (Zipf-head) rows of A^T, cut into blocks
//    of kHeadRows rows of A; block b's entries sorted by (head column, row),
//    key = column << 16 | row in block; the CTA stages block b's u in shared
//    memory; a closed (column, block) piece is a partial part[k * nb + b].
//  * tail: the remaining rows of A^T, whole columns grouped (in column order)
//    into groups of <= 2^(32-rb) - 1 columns; key = column in group << rb | row
//    (rb = bits of the local row count); u gathered from global memory (L2);
//    a closed piece is a whole column sum, stored to out[tcol[...]] directly.
// Work item = (block or group g, part p): a contiguous, 128-aligned range of
// g's entries.  Each warp walks a contiguous sub-range, 128 entries per step
// (lane = 4 consecutive entries, vector loads, next step prefetched), and
// closes pieces with a lane-local segmented prefix + one warp segmented scan.
// Pieces interior to a warp range are complete and stored directly; the first
// and the last piece of each range are chained across the warps in order (one
// thread), then across the parts of g (seg_bnd_kernel).  Every sum has a fixed
// order, so results are bit-identical run to run.  The tail stream replaces a
// warp-per-column walk whose dependent metadata -> entries -> gather chain per
// ~74-entry column left it latency-bound.
// warp sum in a fixed order, lane 0's value broadcast (identical in every lane)
__device__ __forceinline__ double warp_allsum(double v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  return __shfl_sync(0xffffffffu, v, 0);
}

struct HeadPiece {
  int fk, lk;  // first / last piece column (-1: none)
  double fs, ls;
};

struct HeadPolicy {
  __device__ __forceinline__ void begin() {}
  __device__ __forceinline__ void begin_item(int) {}
  double* part;
  int nb;    // blocks (ncols x nblocks < 2^31, build_head_adj)
  int rows;  // rows of A per block (<= 65536: the key's row field)
  static constexpr bool kStage = true;
  static constexpr bool kFast = true;  // single-column steps skip the scan (long Zipf-head runs)
  static constexpr int kMinBlocks = 2;  // 2 x 512 threads: <= 64 registers
  __device__ __forceinline__ int col(unsigned key) const { return static_cast<int>(key >> 16); }
  __device__ __forceinline__ int row(unsigned key) const { return static_cast<int>(key & 0xffffu); }
  __device__ __forceinline__ int block_rows() const { return rows; }
  __device__ __forceinline__ int pad() const { return kHeadPad; }
  __device__ __forceinline__ void store(int k, long long g, double s) const { part[k * nb + static_cast<int>(g)] = s; }
  __device__ __forceinline__ void zero(int k, long long g) const { part[k * nb + static_cast<int>(g)] = 0.0; }
};

struct TailPolicy {
  const int* __restrict__ gcol0;  // per group: index of its first column in tcol
  const int* __restrict__ tcol;   // per (group, column in group): destination index in out
  double* out;                    // A^T u (one row superblock) or the superblock partials
  int rb;                         // bits of the row field
  AdjEpi e;                       // e.n2top != nullptr: out = (raw + mu u_t) / beta (lsqr_epi_kernel)
  double beta;
  double* outc;  // non-null: column sums in tail order (outc[gcol0[g] + k]); tail_scatter_kernel maps them
  int gbase;
  __device__ __forceinline__ void begin() {
    if (e.n2top) beta = sqrt(*e.n2top + (e.n2tail ? *e.n2tail : 0.0));
  }
  // the group's first tail-order slot, once per work item: a closed piece's
  // store then needs no dependent tcol lookup (which stalled the warp's
  // in-order issue on every step that closed a column)
  __device__ __forceinline__ void begin_item(int g) {
    if (outc) gbase = __ldg(gcol0 + g);
  }
  static constexpr bool kStage = false;
  static constexpr bool kFast = false;  // tail runs are short: no single-column steps to speak of
#ifndef APC_TAIL_MINB
#define APC_TAIL_MINB 2
#endif
  static constexpr int kMinBlocks = APC_TAIL_MINB;
  __device__ __forceinline__ int col(unsigned key) const { return static_cast<int>(key >> rb); }
  __device__ __forceinline__ int row(unsigned key) const { return static_cast<int>(key & ((1u << rb) - 1u)); }
  __device__ __forceinline__ int pad() const { return static_cast<int>((1u << (32 - rb)) - 1u); }
  __device__ __forceinline__ int block_rows() const { return 0; }
  __device__ __forceinline__ void store(int k, long long g, double s) const {
    if (outc) {
      outc[gbase + k] = s;
      return;
    }
    const int j = __ldg(tcol + __ldg(gcol0 + g) + k);
    if (e.n2top) {
      const double raw = e.ut ? s + e.mu * e.ut[j] : s;
      s = beta > 0.0 ? raw / beta : raw;
    }
    out[j] = s;
  }
  __device__ __forceinline__ void zero(int k, long long g) const { store(k, g, 0.0); }
};

// chain step: piece (pk, ps) follows the open piece (k, s)
template <class Pol>
__device__ __forceinline__ void head_chain(int& k, double& s, int pk, double ps, int& fk, double& fs, bool& first,
                                           const Pol& pol, long long blk) {
  if (pk < 0) return;
  if (pk == k) {
    s += ps;
    return;
  }
  if (k >= 0) {
    if (first) {
      fk = k;
      fs = s;
      first = false;
    } else {
      pol.store(k, blk, s);
    }
  }
  k = pk;
  s = ps;
}

#ifndef APC_HEAD_MINB
#define APC_HEAD_MINB 1
#endif
#ifndef APC_TAIL_PF2
#define APC_TAIL_PF2 0
#endif
// one work item (CTA `bid`) of a segmented stream
template <class Pol>
__device__ __forceinline__ void seg_adj_body(int bid, const int* __restrict__ bptr, const int* __restrict__ hkey,
                                             const double* __restrict__ hval, const double* __restrict__ u,
                                             long long mloc, int parts, const int* __restrict__ zptr,
                                             const int* __restrict__ zcol, Pol pol, HeadPiece* __restrict__ bnd) {
  constexpr int NW = kHeadThreads / 32;
  constexpr unsigned FULL = 0xffffffffu;
  extern __shared__ double us[];
  __shared__ HeadPiece pc[NW];
  const int blk = bid / parts;
  const int prt = bid % parts;
  pol.begin();
  pol.begin_item(blk);
  const int PAD = pol.pad();
  const double* ub = u;
  if (Pol::kStage) {
    const int R = pol.block_rows();
    const long long r0 = static_cast<long long>(blk) * R;
    const int nr = static_cast<int>(mloc - r0 < R ? mloc - r0 : R);
    for (int i = threadIdx.x; i < nr; i += kHeadThreads) us[i] = __ldcg(u + r0 + i);
  }
  if (prt == 0)
    for (int z = __ldg(zptr + blk) + threadIdx.x; z < __ldg(zptr + blk + 1); z += kHeadThreads)
      pol.zero(__ldg(zcol + z), blk);
  if (Pol::kStage) __syncthreads();
  constexpr int KL = kHeadPerLane, STEP = 32 * KL;
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  const int b0 = __ldg(bptr + blk), b1 = __ldg(bptr + blk + 1);  // multiples of STEP
  const int pper = ((b1 - b0) / STEP + parts - 1) / parts * STEP;
  const int p0 = min(b1, b0 + prt * pper), p1 = min(b1, p0 + pper);
  const int wper = ((p1 - p0) / STEP + NW - 1) / NW * STEP;
  const int rb = min(p1, p0 + w * wper), re = min(p1, rb + wper);
  int ck = -1, fk = -1;  // open (carried) piece, first closed piece (warp-uniform)
  double cs = 0.0, fs = 0.0;
  double la = 0.0;    // lane partials of the carried piece from single-column steps
  bool lact = false;  // la holds unfolded partials (warp-uniform)
  const int4* kp = reinterpret_cast<const int4*>(hkey) + (KL / 4) * lane;
  const double2* vp = reinterpret_cast<const double2*>(hval) + (KL / 2) * lane;
  // software pipeline: the next step's entries (and, for a global u, its
  // gathers) are in flight while this one is scanned
  // a global u (tail): the keys run two steps ahead, so the gathers of step
  // e + STEP are issued on keys that arrived during the previous step instead
  // of stalling on keys loaded in the same step (long-scoreboard bound)
  int4 nkq[KL / 4], nk2[KL / 4];
  double2 nvq[KL / 2];
  double nug[KL];
  if (rb < re) {
#pragma unroll
    for (int i = 0; i < KL / 4; ++i) nkq[i] = __ldcs(kp + (rb >> 2) + i);
#pragma unroll
    for (int i = 0; i < KL / 2; ++i) nvq[i] = __ldcs(vp + (rb >> 1) + i);
    if (!Pol::kStage) {
      if (APC_TAIL_PF2 && rb + STEP < re) {
#pragma unroll
        for (int i = 0; i < KL / 4; ++i) nk2[i] = __ldcs(kp + ((rb + STEP) >> 2) + i);
      }
#pragma unroll
      for (int i = 0; i < KL / 4; ++i) {
        nug[4 * i] = __ldg(ub + pol.row(nkq[i].x));
        nug[4 * i + 1] = __ldg(ub + pol.row(nkq[i].y));
        nug[4 * i + 2] = __ldg(ub + pol.row(nkq[i].z));
        nug[4 * i + 3] = __ldg(ub + pol.row(nkq[i].w));
      }
    }
  }
  for (int e = rb; e < re; e += STEP) {
    int key[KL];
    double vv[KL], ug[KL];
#pragma unroll
    for (int i = 0; i < KL / 4; ++i) {
      key[4 * i] = nkq[i].x;
      key[4 * i + 1] = nkq[i].y;
      key[4 * i + 2] = nkq[i].z;
      key[4 * i + 3] = nkq[i].w;
    }
#pragma unroll
    for (int i = 0; i < KL / 2; ++i) {
      vv[2 * i] = nvq[i].x;
      vv[2 * i + 1] = nvq[i].y;
    }
    if (!Pol::kStage) {
#pragma unroll
      for (int i = 0; i < KL; ++i) ug[i] = nug[i];
    }
    if (e + STEP < re) {
      if (Pol::kStage || !APC_TAIL_PF2) {
#pragma unroll
        for (int i = 0; i < KL / 4; ++i) nkq[i] = __ldcs(kp + ((e + STEP) >> 2) + i);
      } else {
#pragma unroll
        for (int i = 0; i < KL / 4; ++i) nkq[i] = nk2[i];
        if (e + 2 * STEP < re) {
#pragma unroll
          for (int i = 0; i < KL / 4; ++i) nk2[i] = __ldcs(kp + ((e + 2 * STEP) >> 2) + i);
        }
      }
#pragma unroll
      for (int i = 0; i < KL / 2; ++i) nvq[i] = __ldcs(vp + ((e + STEP) >> 1) + i);
      if (!Pol::kStage) {
#pragma unroll
        for (int i = 0; i < KL / 4; ++i) {
          nug[4 * i] = __ldg(ub + pol.row(nkq[i].x));
          nug[4 * i + 1] = __ldg(ub + pol.row(nkq[i].y));
          nug[4 * i + 2] = __ldg(ub + pol.row(nkq[i].z));
          nug[4 * i + 3] = __ldg(ub + pol.row(nkq[i].w));
        }
      }
    }
    // padding keys carry column PAD and row 0 (value 0): a run that is never stored
    int k[KL];
    double x[KL];
#pragma unroll
    for (int i = 0; i < KL; ++i) {
      k[i] = pol.col(static_cast<unsigned>(key[i]));
      x[i] = vv[i] * (Pol::kStage ? us[pol.row(static_cast<unsigned>(key[i]))] : ug[i]);
    }
    const int kl0 = __shfl_sync(FULL, k[0], 0);
    const int kl31 = Pol::kFast ? __shfl_sync(FULL, k[KL - 1], 31) : -1;
    if (Pol::kFast && kl0 == kl31 && kl0 != PAD) {
      // the whole step is one column (keys are sorted): no scan.  Lane-local
      // partials accumulate in `la` across such steps and are folded into the
      // carried sum (cs + a fixed-order warp sum) only when the run goes on
      // into a mixed step or ends -- the long Zipf-head runs skip the
      // shuffles of the segmented scan entirely
      double t = x[0];
#pragma unroll
      for (int i = 1; i < KL; ++i) t += x[i];
      if (kl0 != ck) {
        if (ck >= 0) {
          if (lact) cs += warp_allsum(la);
          if (fk < 0) {
            fk = ck;
            fs = cs;
          } else if (lane == 0) {
            pol.store(ck, blk, cs);
          }
        }
        ck = kl0;
        cs = 0.0;
        la = t;
      } else {
        la = lact ? la + t : t;
      }
      lact = true;
      continue;
    }
    if (Pol::kFast && lact) {
      cs += warp_allsum(la);
      lact = false;
    }
    if (ck >= 0 && kl0 != ck) {  // the carried piece ended with the previous step
      if (fk < 0) {
        fk = ck;
        fs = cs;
      } else if (lane == 0) {
        pol.store(ck, blk, cs);
      }
      ck = -1;
    }
    if (lane == 0 && k[0] == ck) x[0] = cs + x[0];  // carried sum first
    const int kprev = __shfl_up_sync(FULL, k[KL - 1], 1);
    bool hd[KL];  // entry i starts a run within the lane (entry 0: relative to the previous lane)
    hd[0] = lane == 0 || k[0] != kprev;
#pragma unroll
    for (int i = 1; i < KL; ++i) hd[i] = k[i] != k[i - 1];
    double q[KL];
    q[0] = x[0];
#pragma unroll
    for (int i = 1; i < KL; ++i) q[i] = hd[i] ? x[i] : q[i - 1] + x[i];
    // warp segmented inclusive scan of (head seen, open-run sum) over lanes
    bool F0 = false;
#pragma unroll
    for (int i = 0; i < KL; ++i) F0 = F0 || hd[i];
    // lanes holding a run start; before the step of offset d a lane's segment
    // flag covers lanes [lane - d + 1, lane], read off this mask instead of
    // being shuffled along with the sums (shuffles share the L1TEX pipe)
    const unsigned Hm = __ballot_sync(FULL, F0);
    const unsigned upto = (2u << lane) - 1u;  // bits [0, lane]
    double A = q[KL - 1];
#pragma unroll
    for (int d = 1; d < 32; d <<= 1) {
      const double Au = __shfl_up_sync(FULL, A, d);
      const int lo = lane - d + 1;
      const unsigned win = lo > 0 ? upto & ~((1u << lo) - 1u) : upto;
      const bool F = (Hm & win) != 0u;
      A = (lane >= d && !F) ? Au + A : A;
    }
    const double E = __shfl_up_sync(FULL, A, 1);  // sum carried into this lane's first run
    double y[KL];
    bool seen = false;
#pragma unroll
    for (int i = 0; i < KL; ++i) {
      seen = seen || hd[i];
      y[i] = seen ? q[i] : E + q[i];
    }
    const int knext = __shfl_down_sync(FULL, k[0], 1);
    bool en[KL];
#pragma unroll
    for (int i = 0; i < KL - 1; ++i) en[i] = k[i] != PAD && k[i] != k[i + 1];
    en[KL - 1] = k[KL - 1] != PAD && lane < 31 && k[KL - 1] != knext;  // lane 31's last entry stays open
    bool anyen = false;
#pragma unroll
    for (int i = 0; i < KL; ++i) anyen = anyen || en[i];
    const unsigned m = __ballot_sync(FULL, anyen);
    // this lane's first closed piece (used when it is the range's first piece)
    int jk = k[KL - 1];
    double js = y[KL - 1];
#pragma unroll
    for (int i = KL - 2; i >= 0; --i) {
      jk = en[i] ? k[i] : jk;
      js = en[i] ? y[i] : js;
    }
    if (m != 0 && fk < 0) {  // warp-uniform; taken once per range
      const int fl = __ffs(m) - 1;
      fk = __shfl_sync(FULL, jk, fl);
      fs = __shfl_sync(FULL, js, fl);
      if (lane == fl) {
        bool cleared = false;
#pragma unroll
        for (int i = 0; i < KL; ++i) {
          const bool c = en[i] && !cleared;
          cleared = cleared || en[i];
          en[i] = en[i] && !c;
        }
      }
    }
#pragma unroll
    for (int i = 0; i < KL; ++i)
      if (en[i]) pol.store(k[i], blk, y[i]);
    ck = __shfl_sync(FULL, k[KL - 1], 31);
    cs = __shfl_sync(FULL, y[KL - 1], 31);
    if (ck == PAD) ck = -1;
  }
  if (Pol::kFast && lact) cs += warp_allsum(la);
  if (lane == 0) pc[w] = fk < 0 ? HeadPiece{ck, -1, cs, 0.0} : HeadPiece{fk, ck, fs, cs};
  __syncthreads();
  if (threadIdx.x == 0) {
    int k = -1, f = -1;
    double sum = 0.0, fsum = 0.0;
    bool first = parts > 1;  // with one part per block the CTA's pieces are all complete
    for (int i = 0; i < NW; ++i) {
      const HeadPiece P = pc[i];
      head_chain(k, sum, P.fk, P.fs, f, fsum, first, pol, blk);
      head_chain(k, sum, P.lk, P.ls, f, fsum, first, pol, blk);
    }
    if (parts > 1) {
      bnd[bid] = first ? HeadPiece{k, -1, sum, 0.0} : HeadPiece{f, k, fsum, sum};
    } else if (k >= 0) {
      pol.store(k, blk, sum);
    }
  }
}

template <class Pol>
__global__ void __launch_bounds__(kHeadThreads, Pol::kMinBlocks)
seg_adj_kernel(const int* __restrict__ bptr, const int* __restrict__ hkey, const double* __restrict__ hval,
               const double* __restrict__ u, long long mloc, int parts, const int* __restrict__ zptr,
               const int* __restrict__ zcol, Pol pol, HeadPiece* __restrict__ bnd, const int* done) {
  if (done && *done) return;
  seg_adj_body<Pol>(blockIdx.x, bptr, hkey, hval, u, mloc, parts, zptr, zcol, pol, bnd);
}


// pieces at the part boundaries of each block (group), chained in part order
template <class Pol>
__global__ void seg_bnd_kernel(const HeadPiece* __restrict__ bnd, int parts, long long nblocks, Pol pol,
                               const int* done) {
  if (done && *done) return;
  pol.begin();
  const long long blk = static_cast<long long>(blockIdx.x) * blockDim.x + threadIdx.x;
  if (blk >= nblocks) return;
  pol.begin_item(static_cast<int>(blk));
  int k = -1, f = -1;
  double sum = 0.0, fsum = 0.0;
  bool first = false;
  for (int i = 0; i < parts; ++i) {
    const HeadPiece P = bnd[blk * parts + i];
    head_chain(k, sum, P.fk, P.fs, f, fsum, first, pol, blk);
    head_chain(k, sum, P.lk, P.ls, f, fsum, first, pol, blk);
  }
  if (k >= 0) pol.store(k, blk, sum);
}

// out[col] = sum of the column's superblock partials, superblock order
__global__ void tail_combine_kernel(const double* __restrict__ part, const int* __restrict__ cols, long long ncols,
                                    int S, double* __restrict__ out, const int* done, AdjEpi e) {
  if (done && *done) return;
  const long long t = static_cast<long long>(blockIdx.x) * blockDim.x + threadIdx.x;
  if (t >= ncols) return;
  double s = part[t * S];
  for (int sb = 1; sb < S; ++sb) s += part[t * S + sb];
  const int j = cols[t];
  if (e.n2top) {
    const double beta = sqrt(*e.n2top + (e.n2tail ? *e.n2tail : 0.0));
    const double raw = e.ut ? s + e.mu * e.ut[j] : s;
    s = beta > 0.0 ? raw / beta : raw;
  }
  out[j] = s;
}

// tail-order column sums -> out[original column]
__global__ void tail_scatter_kernel(const double* __restrict__ outc, const int* __restrict__ tcol, long long ncols,
                                    double* __restrict__ out, const int* done, AdjEpi e) {
  if (done && *done) return;
  const long long i = static_cast<long long>(blockIdx.x) * blockDim.x + threadIdx.x;
  if (i >= ncols) return;
  const int j = __ldg(tcol + i);
  double s = __ldg(outc + i);
  if (e.n2top) {  // the LSQR epilogue (lsqr_epi_kernel), fused: same operations, same bits
    const double beta = sqrt(*e.n2top + (e.n2tail ? *e.n2tail : 0.0));
    const double raw = e.ut ? s + e.mu * e.ut[j] : s;
    s = beta > 0.0 ? raw / beta : raw;
  }
  out[j] = s;
}

// warp per head column: its partials in block order -> out[col]
__global__ void __launch_bounds__(256)
head_combine_kernel(const double* __restrict__ part, long long nblocks, const int* __restrict__ hcol,
                    long long ncols, double* __restrict__ out, const int* done, AdjEpi e) {
  if (done && *done) return;
  const long long k = (static_cast<long long>(blockIdx.x) * 256 + threadIdx.x) >> 5;
  const int lane = threadIdx.x & 31;
  if (k >= ncols) return;
  const double* pk = part + k * nblocks;
  // a lane's partials loaded 8 at a time before their in-order adds (a load per
  // add stalls the warp once per partial: 28 round trips at C5's 888 blocks);
  // same order of additions, same bits
  double s = 0.0;
  for (long long q = lane; q < nblocks; q += 256) {
    double t[8];
#pragma unroll
    for (int k = 0; k < 8; ++k) t[k] = q + 32 * k < nblocks ? pk[q + 32 * k] : 0.0;
#pragma unroll
    for (int k = 0; k < 8; ++k)
      if (q + 32 * k < nblocks) s += t[k];
  }
  s = warp_sum(s);
  if (lane == 0) {
    const int j = __ldg(hcol + k);
    if (e.n2top) {  // the LSQR epilogue (lsqr_epi_kernel), fused
      const double beta = sqrt(*e.n2top + (e.n2tail ? *e.n2tail : 0.0));
      const double raw = e.ut ? s + e.mu * e.ut[j] : s;
      s = beta > 0.0 ? raw / beta : raw;
    }
    out[j] = s;
  }
}

}  // namespace

__global__ void hot_permute_kernel(const int* __restrict__ hot, long long n, const double* __restrict__ x,
                                   double* __restrict__ xr) {
  const long long k = static_cast<long long>(blockIdx.x) * blockDim.x + threadIdx.x;
  if (k < n) xr[k] = __ldg(x + __ldg(hot + k));
}

void build_hot_sell(apc_mat& a, const std::vector<long long>& col_nnz) {
  apc_ctx* ctx = a.ctx;
  cudaStream_t st = ctx->stream;
  const long long n = a.n, rows = a.a.rows, nnz = a.a.nnz;
  HotSell& h = a.hot;
  h.s = Sell();
  if (rows == 0 || nnz == 0) return;
  {
    // SELL slots (chunk width = its longest row) must stay in int32: very
    // ragged rows keep the CSR forward instead
    std::vector<int> rp(static_cast<size_t>(rows + 1));
    copy_sync(st, rp.data(), a.a.ptr.p, sizeof(int) * rp.size(), cudaMemcpyDeviceToHost);
    long long slots = 0;
    for (long long c = 0; c * 32 < rows; ++c) {
      int w = 0;
      for (long long r = c * 32; r < std::min(rows, c * 32 + 32); ++r) w = std::max(w, rp[r + 1] - rp[r]);
      slots += 32LL * w;
    }
    if (slots >= (1LL << 31)) return;
  }
  // relabel: descending column length, ties by original id
  std::vector<int> hot(n), nptr(n + 1);
  for (long long j = 0; j < n; ++j) hot[j] = static_cast<int>(j);
  std::stable_sort(hot.begin(), hot.end(), [&](int x, int y) { return col_nnz[x] > col_nnz[y]; });
  nptr[0] = 0;
  for (long long k = 0; k < n; ++k) nptr[k + 1] = nptr[k] + static_cast<int>(col_nnz[hot[k]]);
  std::vector<int> inv(n);
  for (long long k = 0; k < n; ++k) inv[hot[k]] = static_cast<int>(k);
  h.n = n;
  h.hot.alloc(n);
  h.inv.alloc(n);
  h.xr.alloc(n);
  APC_CUDA(cudaMemcpyAsync(h.inv.p, inv.data(), sizeof(int) * n, cudaMemcpyHostToDevice, st));
  DBuf<int> dn(n + 1), keys(nnz), vals(nnz), kout(nnz), vout(nnz);
  APC_CUDA(cudaMemcpyAsync(h.hot.p, hot.data(), sizeof(int) * n, cudaMemcpyHostToDevice, st));
  APC_CUDA(cudaMemcpyAsync(dn.p, nptr.data(), sizeof(int) * (n + 1), cudaMemcpyHostToDevice, st));
  hot_keys_kernel<<<nblk(nnz, 256), 256, 0, st>>>(dn.p, h.hot.p, a.at.ptr.p, a.at.idx.p, n, nnz, keys.p, vals.p);
  int end_bit = 1;
  while ((1LL << end_bit) < rows + 1 && end_bit < 31) ++end_bit;
  size_t tmp_bytes = 0;
  cub::DeviceRadixSort::SortPairs(nullptr, tmp_bytes, keys.p, kout.p, vals.p, vout.p, static_cast<int>(nnz), 0,
                                  end_bit, st);
  DBuf<char> tmp(static_cast<long long>(std::max<size_t>(tmp_bytes, 1)));
  APC_CUDA(cub::DeviceRadixSort::SortPairs(tmp.p, tmp_bytes, keys.p, kout.p, vals.p, vout.p, static_cast<int>(nnz),
                                           0, end_bit, st));
  Sell& s = h.s;
  s.rows = rows;
  s.chunks = (rows + 31) / 32;
  s.off.alloc(s.chunks + 1);
  DBuf<int> width(s.chunks + 1);
  hot_width_kernel<<<nblk(s.chunks + 1, 256), 256, 0, st>>>(a.a.ptr.p, rows, s.chunks, width.p);
  size_t stmp = 0;
  cub::DeviceScan::ExclusiveSum(nullptr, stmp, width.p, s.off.p, static_cast<int>(s.chunks + 1), st);
  DBuf<char> sbuf(static_cast<long long>(std::max<size_t>(stmp, 1)));
  APC_CUDA(cub::DeviceScan::ExclusiveSum(sbuf.p, stmp, width.p, s.off.p, static_cast<int>(s.chunks + 1), st));
  int slots = 0;
  copy_sync(st, &slots, s.off.p + s.chunks, sizeof(int), cudaMemcpyDeviceToHost);
  s.slots = slots;
  s.idx.alloc(std::max(1, slots));
  s.val.alloc(std::max(1, slots));
  if (slots > nnz) {  // padding of ragged chunks (never read: rows stop at their length)
    APC_CUDA(cudaMemsetAsync(s.idx.p, 0, s.idx.bytes(), st));
    APC_CUDA(cudaMemsetAsync(s.val.p, 0, s.val.bytes(), st));
  }
  hot_fill_kernel<<<nblk(rows, 256), 256, 0, st>>>(vout.p, a.a.ptr.p, s.off.p, dn.p, h.hot.p, a.at.ptr.p, a.at.val.p,
                                                  n, rows, s.idx.p, s.val.p);
  ctx->launches += 4;
  APC_CUDA(cudaGetLastError());
  APC_CUDA(cudaStreamSynchronize(st));
}

bool hot_sell_wanted(long long nnz) {
  const char* e = std::getenv("APC_HOT_SELL");
  if (e) return std::atoi(e) != 0;
  return nnz * 12 > (96LL << 20);  // HBM-streamed (the persistent kernel takes the L2-resident ones)
}

unsigned fwd_gs_grid(apc_ctx* ctx, const void* kfn, int threads) {
  static std::mutex mu;
  static std::map<std::pair<int, const void*>, unsigned> cache;
  std::lock_guard<std::mutex> lk(mu);
  const auto key = std::make_pair(ctx->device, kfn);
  auto it = cache.find(key);
  if (it != cache.end()) return it->second;
  int per_sm = 0;
  APC_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kfn, threads, 0));
  const unsigned g = static_cast<unsigned>(ctx->num_sms * std::max(1, per_sm));
  cache[key] = g;
  return g;
}

// ---------------------------------------------------------------------------
// plans
// ---------------------------------------------------------------------------
DenseFwdPlan dense_fwd_plan(const apc_mat& a) { return dense_fwd_plan(a.mloc(), a.n, a.ctx->num_sms); }

// columns per split at least APC_DENSE_FWD_MINCOLS: short, wide operands (the
// explicit preconditioner basis B, n x l) need many splits to fill the GPU
#ifndef APC_DENSE_FWD_MINCOLS
#define APC_DENSE_FWD_MINCOLS 16
#endif
DenseFwdPlan dense_fwd_plan(long long mloc, long long ncols, int num_sms) {
  DenseFwdPlan p;
  p.ntiles = (mloc + kDenseFwdTile - 1) / kDenseFwdTile;
  if (p.ntiles < 1) p.ntiles = 1;
  // aim for >= 6 CTAs per SM, but keep >= APC_DENSE_FWD_MINCOLS columns per split
  const long long want = 6LL * num_sms;
  long long ns = (want + p.ntiles - 1) / p.ntiles;
  long long maxs = std::max<long long>(1, ncols / APC_DENSE_FWD_MINCOLS);
  ns = std::max<long long>(1, std::min(ns, maxs));
  p.nsplit = std::min<long long>(ns, 65535);
  p.cols_per_split = (ncols + p.nsplit - 1) / p.nsplit;
  if (p.cols_per_split < 1) p.cols_per_split = 1;
  p.nsplit = (ncols + p.cols_per_split - 1) / p.cols_per_split;
  if (p.nsplit < 1) p.nsplit = 1;
  return p;
}

DenseAdjPlan dense_adj_plan(const apc_mat& a) { return dense_adj_plan(a.mloc(), a.n, a.ctx->num_sms); }

DenseAdjPlan dense_adj_plan(long long mloc, long long n, int num_sms) {
  DenseAdjPlan p;
  p.ngroups = (n + kDenseAdjCols - 1) / kDenseAdjCols;
  if (p.ngroups < 1) p.ngroups = 1;
  const long long want = 6LL * num_sms;
  long long ms = (want + p.ngroups - 1) / p.ngroups;
  long long maxs = std::max<long long>(1, mloc / 512);
  ms = std::max<long long>(1, std::min(ms, maxs));
  p.rows_per_split = (mloc + ms - 1) / ms;
  p.rows_per_split = std::max<long long>(32, (p.rows_per_split + 31) / 32 * 32);
  p.msplit = (mloc + p.rows_per_split - 1) / p.rows_per_split;
  if (p.msplit < 1) p.msplit = 1;
  return p;
}

int csr_group_size(double avg) {
  if (avg <= 5.0) return 4;
  if (avg <= 10.0) return 8;
  if (avg <= 24.0) return 16;
  return 32;
}

double* ctx_scratch(apc_ctx* ctx, long long count) {
  ctx->scratch_d.ensure(count);
  return ctx->scratch_d.p;
}

unsigned* ctx_counters(apc_ctx* ctx, long long count) {
  if (count > ctx->counters.n) {
    ctx->counters.alloc(count);
    APC_CUDA(cudaMemsetAsync(ctx->counters.p, 0, ctx->counters.bytes(), ctx->stream));
  }
  return ctx->counters.p;
}

// ---------------------------------------------------------------------------
// operator products
// ---------------------------------------------------------------------------
void op_fwd(apc_mat& a, double mu, bool augmented, const double* x, double* y) {
  cudaStream_t st = a.ctx->stream;
  if (a.mloc() > 0) launch_fwd(a, x, nullptr, FwdStore{y}, st);
  if (augmented && a.n > 0) {
    tail_fwd_kernel<<<nblk(a.n, 256), 256, 0, st>>>(x, a.n, mu, y + a.mloc());
    a.ctx->launches++;
  }
  APC_CUDA(cudaGetLastError());
}

namespace {
// head + tail-stream adjoint; e.n2top != nullptr fuses the LSQR epilogue
void seg_adjoint(apc_mat& a, const double* u, double* out, const int* done, const AdjEpi& e) {
  cudaStream_t st = a.ctx->stream;
  const HeadAdj& h = a.head;
  const HeadAdj::Seg& t = h.seg;
  // tail-order stores (then one scatter) unless superblock partials are in use; a fused
  // epilogue rides on the scatter (inside the stream's stores its u_t gather and division
  // cost ~20 us per C5 iteration)
  const bool compact = t.sb == 1 && t.outc.p;
  const TailPolicy pol{t.gcol0.p, t.tcol.p, t.sb > 1 ? t.part.p : out, t.rb, t.sb > 1 || compact ? AdjEpi{} : e, 0.0,
                       compact ? t.outc.p : nullptr, 0};
  const HeadPolicy hp{h.part.p, static_cast<int>(h.nblocks), h.rows};
  // APC_ADJ_OVERLAP=1: the tail stream (latency-bound on its u gathers) on a
  // side stream beside the head stream (HBM-bound, 2 CTAs per SM by its shared
  // memory): fork / join by events, also inside graph capture.  The two write
  // disjoint columns of `out`.
  static const int overlap_mode = std::getenv("APC_ADJ_OVERLAP") ? std::atoi(std::getenv("APC_ADJ_OVERLAP")) : 0;
  const bool overlap_env = overlap_mode != 0;  // 1: head launched first, 2: tail first
  cudaStream_t ts = st;
  if (overlap_env) {
    apc_ctx* c = a.ctx;
    if (!c->side) {
      APC_CUDA(cudaStreamCreateWithFlags(&c->side, cudaStreamNonBlocking));
      APC_CUDA(cudaEventCreateWithFlags(&c->ev_fork, cudaEventDisableTiming));
      APC_CUDA(cudaEventCreateWithFlags(&c->ev_join, cudaEventDisableTiming));
    }
    ts = c->side;
    APC_CUDA(cudaEventRecord(c->ev_fork, st));
    APC_CUDA(cudaStreamWaitEvent(ts, c->ev_fork, 0));
  }
  auto head = [&] {
    seg_adj_kernel<HeadPolicy><<<static_cast<unsigned>(h.nblocks * h.parts), kHeadThreads, sizeof(double) * h.rows,
                                 st>>>(h.bptr.p, h.hkey.p, h.hval.p, u, a.mloc(), h.parts, h.zptr.p, h.zcol.p, hp,
                                       reinterpret_cast<HeadPiece*>(h.bnd.p), done);
    a.ctx->launches++;
    if (h.parts > 1) {
      seg_bnd_kernel<HeadPolicy><<<nblk(h.nblocks, 128), 128, 0, st>>>(reinterpret_cast<const HeadPiece*>(h.bnd.p),
                                                                       h.parts, h.nblocks, hp, done);
      a.ctx->launches++;
    }
    head_combine_kernel<<<nblk(h.ncols * 32, 256), 256, 0, st>>>(h.part.p, h.nblocks, h.hcol.p, h.ncols, out, done, e);
    a.ctx->launches++;
  };
  if (overlap_mode == 1) head();  // first: its CTAs take their 2 slots per SM, the tail fills the rest
  seg_adj_kernel<TailPolicy><<<static_cast<unsigned>(t.ngroups * t.parts), kHeadThreads, 0, ts>>>(
      t.gptr.p, t.tkey.p, t.tval.p, u, a.mloc(), t.parts, t.zptr.p, t.zcol.p, pol,
      reinterpret_cast<HeadPiece*>(t.bnd.p), done);
  a.ctx->launches++;
  if (t.parts > 1) {
    seg_bnd_kernel<TailPolicy><<<nblk(t.ngroups, 128), 128, 0, ts>>>(reinterpret_cast<const HeadPiece*>(t.bnd.p),
                                                                     t.parts, t.ngroups, pol, done);
    a.ctx->launches++;
  }
  if (t.sb > 1) {
    tail_combine_kernel<<<nblk(t.ncols, 256), 256, 0, ts>>>(t.part.p, t.cols.p, t.ncols, t.sb, out, done, e);
    a.ctx->launches++;
  }
  if (compact) {
    tail_scatter_kernel<<<nblk(t.ncols, 256), 256, 0, ts>>>(t.outc.p, t.tcol.p, t.ncols, out, done, e);
    a.ctx->launches++;
  }
  if (overlap_mode != 1) head();
  if (overlap_env) {
    APC_CUDA(cudaEventRecord(a.ctx->ev_join, ts));
    APC_CUDA(cudaStreamWaitEvent(st, a.ctx->ev_join, 0));
  }
}
}  // namespace

bool op_adj_epi(apc_mat& a, const double* u, double* h, const int* done, const AdjEpi& e) {
  if (!a.sparse || !a.head.built() || !a.head.seg.built()) return false;
  seg_adjoint(a, u, h, done, e);
  return true;
}

void op_adj_raw(apc_mat& a, const double* u, double* out, const int* done) {
  cudaStream_t st = a.ctx->stream;
  if (!a.sparse) {
    if (a.mloc() == 0) {
      APC_CUDA(cudaMemsetAsync(out, 0, sizeof(double) * a.n, st));
      return;
    }
    DenseAdjPlan p = dense_adj_plan(a);
    double* part = p.msplit > 1 ? ctx_scratch(a.ctx, p.msplit * a.n) : nullptr;
    unsigned* ctr = p.msplit > 1 ? ctx_counters(a.ctx, p.ngroups) : nullptr;
    launch_dense_adj(a.ctx, a.dense.p, a.mloc(), a.n, u, out, done, part, ctr);
    return;
  }
  const Csr& c = a.at;
  if (a.head.built()) {
    if (a.head.seg.built()) {
      seg_adjoint(a, u, out, done, AdjEpi{});
      return;
    }
    const HeadAdj& h = a.head;
    launch_units(a.ctx, c, h.tail, u, out, done);
    const HeadPolicy hp{h.part.p, static_cast<int>(h.nblocks), h.rows};
    seg_adj_kernel<HeadPolicy><<<static_cast<unsigned>(h.nblocks * h.parts), kHeadThreads,
                                 sizeof(double) * h.rows, st>>>(h.bptr.p, h.hkey.p, h.hval.p, u, a.mloc(),
                                                                   h.parts, h.zptr.p, h.zcol.p, hp,
                                                                   reinterpret_cast<HeadPiece*>(h.bnd.p), done);
    if (h.parts > 1) {
      seg_bnd_kernel<HeadPolicy><<<nblk(h.nblocks, 128), 128, 0, st>>>(reinterpret_cast<const HeadPiece*>(h.bnd.p),
                                                                       h.parts, h.nblocks, hp, done);
      a.ctx->launches++;
    }
    head_combine_kernel<<<nblk(h.ncols * 32, 256), 256, 0, st>>>(h.part.p, h.nblocks, h.hcol.p, h.ncols, out, done,
                                                                AdjEpi{});
    a.ctx->launches += 2;
    return;
  }
  launch_units(a.ctx, c, c, u, out, done);
}

void launch_units(apc_ctx* ctx, const Csr& c, const Units& un, const double* u, double* out, const int* done) {
  cudaStream_t st = ctx->stream;
  if (un.n_units == 0) return;
  unsigned nb = nblk(un.n_units * APC_UNITS_G, kCsrUnitThreads);
  csr_units_kernel<<<nb, kCsrUnitThreads, 0, st>>>(c.ptr.p, c.idx.p, c.val.p, u, un.n_units,
                                                   un.urow.p, un.ustart.p, un.uend.p, un.uslot.p, out,
                                                   un.upart.p, done);
  ctx->launches++;
  if (un.n_split > 0) {
    split_fixup_kernel<<<nblk(un.n_split * 32, 256), 256, 0, st>>>(un.srows.p, un.rfirst.p, un.rcount.p, un.n_split,
                                                                    un.upart.p, out, done);
    ctx->launches++;
  }
}

void launch_dense_adj(apc_ctx* ctx, const double* A, long long mloc, long long n, const double* u,
                      double* out, const int* done, double* part, unsigned* ctr) {
  DenseAdjPlan p = dense_adj_plan(mloc, n, ctx->num_sms);
  dim3 grid(static_cast<unsigned>(p.ngroups), static_cast<unsigned>(p.msplit));
  dense_adj_kernel<<<grid, kDenseAdjThreads, 0, ctx->stream>>>(A, mloc, mloc, n, u, p.rows_per_split,
                                                               part, ctr, out, done);
  ctx->launches++;
}

void op_adj(apc_mat& a, double mu, bool augmented, const double* u, double* y) {
  cudaStream_t st = a.ctx->stream;
  if (!a.sparse) {
    op_adj_raw(a, u, y, nullptr);
    if (augmented && a.n > 0) {
      add_tail_kernel<<<nblk(a.n, 256), 256, 0, st>>>(u + a.mloc(), a.n, mu, y);
      a.ctx->launches++;
    }
  } else {
    double* raw = ctx_scratch(a.ctx, a.n);
    op_adj_raw(a, u, raw, nullptr);
    unit_fixup_kernel<<<nblk(a.n, 256), 256, 0, st>>>(raw, a.n, mu, augmented ? u + a.mloc() : nullptr, y);
    a.ctx->launches++;
  }
  APC_CUDA(cudaGetLastError());
}

// ---------------------------------------------------------------------------
// work units for a CSR (host-built from the row lengths)
// ---------------------------------------------------------------------------
void build_units(apc_ctx* ctx, Csr& c, const std::vector<long long>& row_nnz) {
  std::vector<long long> off(c.rows + 1, 0);
  long long maxr = 0;
  for (long long r = 0; r < c.rows; ++r) {
    off[r + 1] = off[r] + row_nnz[r];
    maxr = std::max(maxr, row_nnz[r]);
  }
  c.max_row_nnz = maxr;
  c.avg_row_nnz = c.rows > 0 ? static_cast<double>(off[c.rows]) / static_cast<double>(c.rows) : 0.0;
  build_units_sel(ctx, c, c.rows, off, row_nnz, nullptr);
}

void build_units_sel(apc_ctx* ctx, Units& c, long long rows, const std::vector<long long>& off,
                     const std::vector<long long>& row_nnz, const std::vector<char>* skip, const int* colidx,
                     long long ncols_local, int superblocks) {
  // Row r of the CSR is cut into units of <= kCsrUnitMax entries.  With
  // superblocks > 1 (colidx = the host column indices) the entries of each row
  // are also cut at every boundary of `superblocks` equal ranges of the column
  // space, and the units are emitted superblock-major: the gathered vector's
  // active range at any time is 1/superblocks of it (L2-resident).  A row with
  // more than one unit gets consecutive partial slots in entry order, so the
  // split fix-up adds its pieces in the same order for any superblock count.
  std::vector<int> urow, ustart, uend, uslot, rfirst(rows, -1), rcount(rows, 0);
  urow.reserve(rows);
  const int S = colidx && superblocks > 1 ? superblocks : 1;
  const long long span = (ncols_local + S - 1) / std::max(1, S);
  // pieces of row r in superblock sb: [cut[r*(S+1)+sb], cut[r*(S+1)+sb+1])
  std::vector<long long> cut;
  if (S > 1) {
    cut.resize(static_cast<size_t>(rows * (S + 1)));
    for (long long r = 0; r < rows; ++r) {
      long long q = off[r];
      const long long e = off[r] + row_nnz[r];
      for (int sb = 0; sb < S; ++sb) {
        cut[r * (S + 1) + sb] = q;
        const long long lim = (sb + 1) * span;
        while (q < e && colidx[q] < lim) ++q;
      }
      cut[r * (S + 1) + S] = e;
    }
  }
  auto pieces_units = [&](long long len) { return (len + kCsrUnitMax - 1) / kCsrUnitMax; };
  long long nparts = 0;
  for (long long r = 0; r < rows; ++r) {  // slots first (entry order within each row)
    if (skip && (*skip)[r]) continue;
    long long k = 0;
    if (S > 1) {
      for (int sb = 0; sb < S; ++sb) k += pieces_units(cut[r * (S + 1) + sb + 1] - cut[r * (S + 1) + sb]);
    } else {
      k = pieces_units(row_nnz[r]);
    }
    if (k > 1) {
      rfirst[r] = static_cast<int>(nparts);
      rcount[r] = static_cast<int>(k);
      nparts += k;
    }
  }
  std::vector<int> next_slot(rfirst);
  for (int sb = 0; sb < S; ++sb) {
    for (long long r = 0; r < rows; ++r) {
      if (skip && (*skip)[r]) continue;
      const long long b0 = S > 1 ? cut[r * (S + 1) + sb] : off[r];
      const long long e0 = S > 1 ? cut[r * (S + 1) + sb + 1] : off[r] + row_nnz[r];
      if (row_nnz[r] == 0 && sb == 0) {  // an empty row still writes its 0
        urow.push_back(static_cast<int>(r));
        ustart.push_back(static_cast<int>(b0));
        uend.push_back(static_cast<int>(b0));
        uslot.push_back(-1);
        continue;
      }
      for (long long b = b0; b < e0; b += kCsrUnitMax) {
        urow.push_back(static_cast<int>(r));
        ustart.push_back(static_cast<int>(b));
        uend.push_back(static_cast<int>(std::min(e0, b + kCsrUnitMax)));
        uslot.push_back(rfirst[r] >= 0 ? next_slot[r]++ : -1);
      }
    }
  }
  c.n_units = static_cast<long long>(urow.size());
  c.n_parts = nparts;
  std::vector<int> srows;
  for (long long r = 0; r < rows; ++r)
    if (rfirst[r] >= 0) srows.push_back(static_cast<int>(r));
  c.n_split = static_cast<long long>(srows.size());
  auto up = [&](DBuf<int>& d, const std::vector<int>& h) {
    d.alloc(static_cast<long long>(h.size()));
    if (!h.empty())
      APC_CUDA(cudaMemcpyAsync(d.p, h.data(), h.size() * sizeof(int), cudaMemcpyHostToDevice, ctx->stream));
  };
  up(c.urow, urow);
  up(c.ustart, ustart);
  up(c.uend, uend);
  up(c.uslot, uslot);
  up(c.rfirst, rfirst);
  up(c.rcount, rcount);
  up(c.srows, srows);
  c.upart.alloc(std::max<long long>(1, nparts));
  APC_CUDA(cudaStreamSynchronize(ctx->stream));  // host vectors go out of scope
}

// Head/tail split of CSR(A^T) for the row-blocked adjoint (HeadAdj).  Host
// inputs: CSR(A^T) row offsets and int32 local row indices (the upload's
// staging copy) and the row lengths.  A row of A^T (column of A) is "head"
// when it averages >= APC_HEAD_MIN (default 2) entries per block of kHeadRows.
struct HeadSegs {  // per head column: entry offsets of its segment in each block
  const int* tptr;
  const int* hidx;
  const std::vector<int>* hc;
  long long nblocks, rows;
  std::vector<int>* seg;  // ncols x (nblocks + 1)
  void operator()(long long k0, long long k1) const {
    for (long long k = k0; k < k1; ++k) {
      const int j = (*hc)[k];
      int* sg = seg->data() + k * (nblocks + 1);
      long long q = tptr[j];
      const long long e = tptr[j + 1];
      for (long long b = 0; b < nblocks; ++b) {
        sg[b] = static_cast<int>(q);
        const long long lim = (b + 1) * rows;
        while (q < e && hidx[q] < lim) ++q;
      }
      sg[nblocks] = static_cast<int>(e);
    }
  }
};

// copy of the head entries, block-major: warp per (head column, block) segment
__global__ void head_pack_kernel(const int* __restrict__ seg, const int* __restrict__ dst, long long ncols,
                                 long long nblocks, int rows, const int* __restrict__ tidx,
                                 const double* __restrict__ tval, int* __restrict__ hkey, double* __restrict__ hval) {
  const long long t = (static_cast<long long>(blockIdx.x) * 256 + threadIdx.x) >> 5;
  const int lane = threadIdx.x & 31;
  if (t >= ncols * nblocks) return;
  const long long k = t / nblocks, b = t % nblocks;
  const int s0 = seg[k * (nblocks + 1) + b], s1 = seg[k * (nblocks + 1) + b + 1];
  const int d = dst[b * ncols + k];
  const int rb = static_cast<int>(b * rows);
  for (int q = s0 + lane; q < s1; q += 32) {
    hkey[d + q - s0] = static_cast<int>(k << 16) | (tidx[q] - rb);  // k < kHeadPad
    hval[d + q - s0] = tval[q];
  }
}

// tail stream: warp per (column, superblock) piece copies its entries with packed keys
__global__ void tail_pack_kernel(const int* __restrict__ src, const int* __restrict__ len, const int* __restrict__ kin,
                                 const int* __restrict__ dst, long long nitems, const int* __restrict__ tidx,
                                 const double* __restrict__ tv, int rb, int* __restrict__ tkey,
                                 double* __restrict__ tval) {
  const long long t = (static_cast<long long>(blockIdx.x) * 256 + threadIdx.x) >> 5;
  const int lane = threadIdx.x & 31;
  if (t >= nitems) return;
  const int s0 = src[t], L = len[t], d = dst[t];
  const unsigned hi = static_cast<unsigned>(kin[t]) << rb;
  for (int q = lane; q < L; q += 32) {
    tkey[d + q] = static_cast<int>(hi | static_cast<unsigned>(tidx[s0 + q]));
    tval[d + q] = tv[s0 + q];
  }
}

void build_tail_seg(apc_mat& a, const std::vector<int>& tptr, const int* hidx, const std::vector<long long>& tlen,
                    const std::vector<char>& is_head) {
  apc_ctx* ctx = a.ctx;
  cudaStream_t st = ctx->stream;
  HeadAdj::Seg& t = a.head.seg;
  t = HeadAdj::Seg();
  const long long n = a.n, mloc = a.mloc();
  int rb = 1;
  while ((1LL << rb) < mloc) ++rb;
  if (rb > 26) return;  // fewer than 64 columns per group: keep the work units
  const long long kcap = (1LL << (32 - rb)) - 2;  // column-in-group ids stay below the padding id
  const char* ee = std::getenv("APC_TAIL_ECAP");
  const long long ecap = ee ? std::max(1, std::atoi(ee)) : 16384;
  // row superblocks: the stream holds superblock 0's entries of every tail
  // column, then superblock 1's, ...  CTAs run roughly in stream order, so the
  // u rows being gathered at a time are one superblock (L2-resident on each
  // die); each (column, superblock) piece is a partial added in order after.
  const char* se = std::getenv("APC_TAIL_SB");
  const int S = se ? std::max(1, std::atoi(se)) : 1;
  const long long span = (mloc + S - 1) / S;
  std::vector<int> tc;  // tail columns
  for (long long j = 0; j < n; ++j)
    if (!is_head[j]) tc.push_back(static_cast<int>(j));
  const long long T = static_cast<long long>(tc.size());
  if (T == 0) return;
  // cut[t * (S + 1) + sb]: first entry of tail column t in superblock sb
  std::vector<int> cut(static_cast<size_t>(T * (S + 1)));
  for (long long q = 0; q < T; ++q) {
    const int j = tc[q];
    long long e = tptr[j];
    for (int sb = 0; sb < S; ++sb) {
      cut[q * (S + 1) + sb] = static_cast<int>(e);
      const long long lim = (sb + 1) * span;
      while (e < tptr[j + 1] && hidx[e] < lim) ++e;
    }
    cut[q * (S + 1) + S] = tptr[j + 1];
  }
  std::vector<int> dix, src, kin, dst, gptr(1, 0), gcol0(1, 0), zptr(1, 0), zcol;
  long long tot = 0, gcols = 0, gents = 0;
  auto close_group = [&]() {
    tot = (tot + kHeadStep - 1) / kHeadStep * kHeadStep;
    gptr.push_back(static_cast<int>(tot));
    gcol0.push_back(static_cast<int>(dix.size()));
    zptr.push_back(static_cast<int>(zcol.size()));
    gcols = gents = 0;
  };
  for (int sb = 0; sb < S; ++sb) {
    for (long long q = 0; q < T; ++q) {
      const long long b = cut[q * (S + 1) + sb], L = cut[q * (S + 1) + sb + 1] - b;
      if (gcols > 0 && (gcols >= kcap || gents + L > ecap)) close_group();
      if (L == 0) zcol.push_back(static_cast<int>(gcols));
      dix.push_back(S > 1 ? static_cast<int>(q * S + sb) : tc[q]);
      src.push_back(static_cast<int>(b));
      kin.push_back(static_cast<int>(L));
      dst.push_back(static_cast<int>(tot));
      tot += L;
      gents += L;
      ++gcols;
      if (tot >= (1LL << 31) - kHeadStep) return;
    }
    if (gcols > 0) close_group();  // groups never span superblocks
  }
  const long long G = static_cast<long long>(gptr.size()) - 1;
  gcol0.pop_back();
  std::vector<int> kk(dix.size());  // column in group of each (group, column) item
  for (long long g = 0; g < G; ++g)
    for (int i = gcol0[g]; i < (g + 1 < G ? gcol0[g + 1] : static_cast<int>(dix.size())); ++i) kk[i] = i - gcol0[g];
  auto up = [&](DBuf<int>& d, const std::vector<int>& v) {
    d.alloc(std::max<long long>(1, static_cast<long long>(v.size())));
    if (!v.empty()) APC_CUDA(cudaMemcpyAsync(d.p, v.data(), v.size() * sizeof(int), cudaMemcpyHostToDevice, st));
  };
  t.rb = rb;
  t.ngroups = G;
  t.nnz = tot;
  t.sb = S;
  t.ncols = T;
  up(t.gptr, gptr);
  up(t.gcol0, gcol0);
  up(t.tcol, dix);
  up(t.zptr, zptr);
  up(t.zcol, zcol);
  up(t.cols, tc);
  if (S > 1) t.part.alloc(T * S);
  static const bool compact_env = !std::getenv("APC_TAIL_COMPACT") || std::atoi(std::getenv("APC_TAIL_COMPACT")) != 0;
  if (S == 1 && compact_env) t.outc.alloc(std::max<long long>(1, static_cast<long long>(dix.size())));
  t.tkey.alloc(std::max<long long>(kHeadStep, tot));
  t.tval.alloc(std::max<long long>(kHeadStep, tot));
  fill_int_kernel<<<nblk(t.tkey.n, 256), 256, 0, st>>>(t.tkey.p, t.tkey.n,
                                                       static_cast<int>(static_cast<unsigned>(kcap + 1) << rb));
  APC_CUDA(cudaMemsetAsync(t.tval.p, 0, t.tval.bytes(), st));
  t.bnd.alloc(std::max<long long>(1, G * t.parts * 3));
  {
    DBuf<int> dsrc, dlen, dk, dd;
    up(dsrc, src);
    up(dlen, kin);
    up(dk, kk);
    up(dd, dst);
    const long long ni = static_cast<long long>(dix.size());
    tail_pack_kernel<<<nblk(ni * 32, 256), 256, 0, st>>>(dsrc.p, dlen.p, dk.p, dd.p, ni, a.at.idx.p, a.at.val.p, rb,
                                                         t.tkey.p, t.tval.p);
    ctx->launches += 2;
    APC_CUDA(cudaGetLastError());
    APC_CUDA(cudaStreamSynchronize(st));
  }
}

void build_head_adj(apc_mat& a, const std::vector<int>& tptr, const int* hidx, const std::vector<long long>& tlen) {
  apc_ctx* ctx = a.ctx;
  cudaStream_t st = ctx->stream;
  HeadAdj& h = a.head;
  h = HeadAdj();
  const long long n = a.n, mloc = a.mloc();
  if (mloc == 0 || n == 0) return;
  // block rows: kHeadRows, or -- once there is more than a wave of blocks --
  // the size that makes the block count a whole number of waves of the
  // co-resident CTAs (2 per SM: 64 registers x 512 threads).  977 blocks of
  // 8192 rows ran as 3.3 waves on 148 SMs; 888 blocks of 9010 rows run as 3
  const long long slots = 2LL * ctx->num_sms;
  long long rows = kHeadRows;
  const char* re = std::getenv("APC_HEAD_BLOCK_ROWS");
  if (re && *re) {
    rows = std::max(256, std::min(12288, std::atoi(re)));
  } else if (mloc > slots * kHeadRows) {
    const long long waves = std::max<long long>(1, std::llround(static_cast<double>(mloc) / (slots * kHeadRows)));
    rows = std::min<long long>(12288, (mloc + slots * waves - 1) / (slots * waves));
  }
  const long long nblocks = (mloc + rows - 1) / rows;
  const char* env = std::getenv("APC_HEAD_MIN");
  const double per_block = env ? std::atof(env) : 2.0;
  // the head threshold stays tied to kHeadRows-row blocks (independent of the wave fit)
  const long long thr = std::max<long long>(
      64, static_cast<long long>(per_block * static_cast<double>((mloc + kHeadRows - 1) / kHeadRows)));
  std::vector<int> hc;
  std::vector<char> is_head(n, 0);
  // head column ids fit below kHeadPad, and the (column, block) partial index in int32
  const long long hmax = std::min<long long>(kHeadPad, ((1LL << 31) - 1) / nblocks);
  for (long long j = 0; j < n && static_cast<long long>(hc.size()) < hmax; ++j)
    if (tlen[j] >= thr) {
      hc.push_back(static_cast<int>(j));
      is_head[j] = 1;
    }
  if (hc.empty()) return;
  const char* pe = std::getenv("APC_SETUP_PROF");
  const long long H = static_cast<long long>(hc.size());
  std::vector<int> seg(static_cast<size_t>(H * (nblocks + 1)));
  host_parallel_for(H, HeadSegs{tptr.data(), hidx, &hc, nblocks, rows, &seg}, 1);
  // destination of segment (k, b): block-major, columns ascending within a block
  std::vector<int> dst(static_cast<size_t>(H * nblocks)), bptr(nblocks + 1, 0), zptr(nblocks + 1, 0), zcol;
  long long tot = 0;
  for (long long b = 0; b < nblocks; ++b) {
    bptr[b] = static_cast<int>(tot);
    for (long long k = 0; k < H; ++k) {
      const int len = seg[k * (nblocks + 1) + b + 1] - seg[k * (nblocks + 1) + b];
      dst[b * H + k] = static_cast<int>(tot);
      tot += len;
      if (len == 0) zcol.push_back(static_cast<int>(k));
    }
    tot = (tot + kHeadStep - 1) / kHeadStep * kHeadStep;  // step-aligned blocks (padding: column kHeadPad)
    zptr[b + 1] = static_cast<int>(zcol.size());
  }
  require(tot < (1LL << 31), APC_INVALID_ARGUMENT, "build_head_adj: head entries exceed int32 range");
  bptr[nblocks] = static_cast<int>(tot);
  const char* penv = std::getenv("APC_HEAD_PARTS");
  h.parts = penv ? std::max(1, std::atoi(penv)) : 1;
  h.ncols = H;
  h.nblocks = nblocks;
  h.rows = static_cast<int>(rows);
  h.nnz = tot;
  auto up = [&](DBuf<int>& d, const std::vector<int>& v) {
    d.alloc(std::max<long long>(1, static_cast<long long>(v.size())));
    if (!v.empty()) APC_CUDA(cudaMemcpyAsync(d.p, v.data(), v.size() * sizeof(int), cudaMemcpyHostToDevice, st));
  };
  up(h.bptr, bptr);
  up(h.zptr, zptr);
  up(h.zcol, zcol);
  up(h.hcol, hc);
  h.hkey.alloc(std::max<long long>(kHeadStep, tot));
  h.hval.alloc(std::max<long long>(kHeadStep, tot));
  fill_int_kernel<<<nblk(h.hkey.n, 256), 256, 0, st>>>(h.hkey.p, h.hkey.n, kHeadPad << 16);
  ctx->launches++;
  APC_CUDA(cudaMemsetAsync(h.hval.p, 0, h.hval.bytes(), st));
  h.part.alloc(H * nblocks);
  h.bnd.alloc(nblocks * h.parts * 3);  // HeadPiece = 24 bytes
  {
    DBuf<int> dseg(static_cast<long long>(seg.size())), ddst(static_cast<long long>(dst.size()));
    APC_CUDA(cudaMemcpyAsync(dseg.p, seg.data(), seg.size() * sizeof(int), cudaMemcpyHostToDevice, st));
    APC_CUDA(cudaMemcpyAsync(ddst.p, dst.data(), dst.size() * sizeof(int), cudaMemcpyHostToDevice, st));
    head_pack_kernel<<<nblk(H * nblocks * 32, 256), 256, 0, st>>>(dseg.p, ddst.p, H, nblocks, h.rows, a.at.idx.p,
                                                                  a.at.val.p, h.hkey.p, h.hval.p);
    ctx->launches++;
    APC_CUDA(cudaGetLastError());
    APC_CUDA(cudaStreamSynchronize(st));
  }
  APC_CUDA(cudaFuncSetAttribute(seg_adj_kernel<HeadPolicy>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                static_cast<int>(sizeof(double) * rows)));
  const char* tse = std::getenv("APC_TAIL_SEG");
  if (!tse || std::atoi(tse) != 0) {
    build_tail_seg(a, tptr, hidx, tlen, is_head);
    if (h.seg.built()) {
      if (pe && std::atoi(pe) != 0)
        std::fprintf(stderr, "[apc] head adjoint: %lld head columns (>= %lld nnz), %lld blocks, %lld head nnz; "
                     "tail stream: %lld groups, %lld entries, rb %d\n", H, thr, nblocks, tot, h.seg.ngroups,
                     h.seg.nnz, h.seg.rb);
      return;
    }
  }
  std::vector<long long> off(n + 1);
  for (long long j = 0; j <= n; ++j) off[j] = tptr[j];
  // tail units superblock-major over the rows of A: the gathered u range at a
  // time is 1/APC_TAIL_SB of u, so the gathers hit L2 instead of DRAM
  const char* sbe = std::getenv("APC_TAIL_SB");
  const int sbs = sbe ? std::max(1, std::atoi(sbe)) : 1;
  build_units_sel(ctx, h.tail, n, off, tlen, &is_head, hidx, mloc, sbs);  // synchronizes: host vectors may go
  if (pe && std::atoi(pe) != 0)
    std::fprintf(stderr, "[apc] head adjoint: %lld head columns (>= %lld nnz), %lld blocks, %lld head nnz, %lld tail units\n",
                 H, thr, nblocks, tot, h.tail.n_units);
}

// ---------------------------------------------------------------------------
// CSC (int64, reference layout) -> device CSR(A^T) (= CSC arrays, local rows
// only) and CSR(A) via a stable radix sort by row.
// ---------------------------------------------------------------------------
struct StageCsc {  // narrow row indices to int32 and copy values into pinned staging
  const long long* rowidx;
  const double* val;
  int* hidx;
  double* hval;
  void operator()(long long b, long long e) const {
    for (long long k = b; k < e; ++k) {
      hidx[k] = static_cast<int>(rowidx[k]);
      hval[k] = val[k];
    }
  }
};

void upload_csc(apc_mat& a, const long long* colptr, const long long* rowidx, const double* val) {
  apc_ctx* ctx = a.ctx;
  cudaStream_t st = ctx->stream;
  const long long n = a.n, r0 = a.r0, r1 = a.r1, mloc = a.mloc();
  // host: filter to local rows and narrow indices to int32 (pinned staging)
  std::unique_ptr<ProfScope> ps(new ProfScope("upload.host"));
  std::vector<int> tptr(n + 1);
  std::vector<long long> tlen(n);
  int* hidx = nullptr;
  double* hval = nullptr;
  long long nnz = 0;
  if (r0 == 0 && r1 == a.m) {
    // whole matrix: no filtering; narrow and stage on the host cores
    nnz = n > 0 ? colptr[n] - colptr[0] : 0;
    require(nnz < (1LL << 31), APC_INVALID_ARGUMENT, "upload_csc: nnz exceeds int32 range");
    for (long long j = 0; j <= n; ++j) tptr[j] = static_cast<int>(colptr[j] - colptr[0]);
    for (long long j = 0; j < n; ++j) tlen[j] = tptr[j + 1] - tptr[j];
    hidx = static_cast<int*>(ctx_pinned(ctx, 0, sizeof(int) * std::max<long long>(1, nnz)));
    hval = static_cast<double*>(ctx_pinned(ctx, 1, sizeof(double) * std::max<long long>(1, nnz)));
    host_parallel_for(nnz, StageCsc{rowidx + colptr[0], val + colptr[0], hidx, hval}, 4);
  } else {
    long long cnt = 0;
    for (long long j = 0; j < n; ++j) {
      tptr[j] = static_cast<int>(cnt);
      for (long long k = colptr[j]; k < colptr[j + 1]; ++k)
        if (rowidx[k] >= r0 && rowidx[k] < r1) ++cnt;
    }
    tptr[n] = static_cast<int>(cnt);
    require(cnt < (1LL << 31), APC_INVALID_ARGUMENT, "upload_csc: nnz exceeds int32 range");
    nnz = cnt;
    hidx = static_cast<int*>(ctx_pinned(ctx, 0, sizeof(int) * std::max<long long>(1, nnz)));
    hval = static_cast<double*>(ctx_pinned(ctx, 1, sizeof(double) * std::max<long long>(1, nnz)));
    long long q = 0;
    for (long long j = 0; j < n; ++j) {
      for (long long k = colptr[j]; k < colptr[j + 1]; ++k) {
        long long r = rowidx[k];
        if (r >= r0 && r < r1) {
          hidx[q] = static_cast<int>(r - r0);
          hval[q] = val[k];
          ++q;
        }
      }
      tlen[j] = tptr[j + 1] - tptr[j];
    }
  }
  ps.reset(new ProfScope("upload.csc_units"));
  Csr& t = a.at;
  t.rows = n;
  t.cols = mloc;
  t.nnz = nnz;
  t.ptr.alloc(n + 1);
  t.idx.alloc(std::max<long long>(1, nnz));
  t.val.alloc(std::max<long long>(1, nnz));
  APC_CUDA(cudaMemcpyAsync(t.ptr.p, tptr.data(), sizeof(int) * (n + 1), cudaMemcpyHostToDevice, st));
  if (nnz > 0) {
    APC_CUDA(cudaMemcpyAsync(t.idx.p, hidx, sizeof(int) * nnz, cudaMemcpyHostToDevice, st));
    APC_CUDA(cudaMemcpyAsync(t.val.p, hval, sizeof(double) * nnz, cudaMemcpyHostToDevice, st));
  }
  build_units(ctx, t, tlen);  // synchronizes the stream (the staging buffers are free again)

  ps.reset(new ProfScope("upload.csr_build"));
  // CSR(A): sort entries by row (stable), keeping column order within rows
  Csr& c = a.a;
  c.rows = mloc;
  c.cols = n;
  c.nnz = nnz;
  c.ptr.alloc(mloc + 1);
  c.idx.alloc(std::max<long long>(1, nnz));
  c.val.alloc(std::max<long long>(1, nnz));
  if (nnz > 0) {
    DBuf<int> colof(nnz), perm_in(nnz), perm_out(nnz), keys_out(nnz);
    expand_cols_kernel<<<nblk(nnz, 256), 256, 0, st>>>(t.ptr.p, n, nnz, colof.p);
    iota_kernel<<<nblk(nnz, 256), 256, 0, st>>>(perm_in.p, nnz);
    int end_bit = 1;
    while ((1LL << end_bit) < mloc + 1 && end_bit < 31) ++end_bit;
    size_t tmp_bytes = 0;
    cub::DeviceRadixSort::SortPairs(nullptr, tmp_bytes, t.idx.p, keys_out.p, perm_in.p, perm_out.p,
                                    static_cast<int>(nnz), 0, end_bit, st);
    DBuf<char> tmp(static_cast<long long>(tmp_bytes));
    APC_CUDA(cub::DeviceRadixSort::SortPairs(tmp.p, tmp_bytes, t.idx.p, keys_out.p, perm_in.p,
                                             perm_out.p, static_cast<int>(nnz), 0, end_bit, st));
    gather_csr_kernel<<<nblk(nnz, 256), 256, 0, st>>>(perm_out.p, colof.p, t.val.p, nnz, c.idx.p,
                                                      c.val.p);
    row_ptr_kernel<<<nblk(mloc + 1, 256), 256, 0, st>>>(keys_out.p, nnz, mloc, c.ptr.p);
    ctx->launches += 4;
    APC_CUDA(cudaStreamSynchronize(st));
  } else {
    APC_CUDA(cudaMemsetAsync(c.ptr.p, 0, sizeof(int) * (mloc + 1), st));
  }
  c.avg_row_nnz = mloc > 0 ? static_cast<double>(nnz) / static_cast<double>(mloc) : 0.0;
  APC_CUDA(cudaGetLastError());
  if (hot_sell_wanted(nnz)) {
    ps.reset(new ProfScope("upload.hot_sell"));
    build_hot_sell(a, tlen);
    ps.reset(new ProfScope("upload.head_adj"));
    build_head_adj(a, tptr, hidx, tlen);
  }
}

}  // namespace apc
