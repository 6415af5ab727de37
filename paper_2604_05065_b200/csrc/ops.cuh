// Operator kernels for A_mu*x and A_mu^T*u on sm_100a (fp64, HBM-bound).
//
// Reference semantics: Matrix::matvec / matvec_transpose
// (/root/reference/proj/include/aplicur/matrix.hpp:151-195) and the
// AugmentedOperator tail (matrix.hpp:377-392).  Summation order differs from
// the reference's sequential loops (parallel, but fixed: reruns are
// bit-identical); LSQR parity is judged at the x / iteration level, never on
// CUR indices.
//
// Forward kernels take an epilogue functor so the LSQR vector update
// (u <- A z - alpha*u, ||u||^2 partials, lsqr.hpp:139-145) is fused into the
// pass that produces A z.  Transpose kernels only produce the raw A^T u; the
// LSQR epilogue runs in a light n-length kernel after the (optional) NCCL
// allreduce, which is where partial A_p^T u_p from row shards meet.
#pragma once

#include <algorithm>

#include "apc_internal.hpp"
#include "dev_common.cuh"
#include "ops_host.hpp"

namespace apc {

constexpr int kDenseFwdThreads = 256;
#ifndef APC_DENSE_FWD_R
#define APC_DENSE_FWD_R 8
#endif
constexpr int kDenseFwdRowsPerThread = APC_DENSE_FWD_R;
constexpr int kDenseFwdTile = kDenseFwdThreads * kDenseFwdRowsPerThread;
constexpr int kDenseAdjThreads = 256;
constexpr int kDenseAdjCols = 16;  // 8 warps x 2 columns
constexpr int kCsrFwdThreads = 256;
constexpr int kCsrFwdRowsPerBlock = 256;
constexpr int kCsrUnitThreads = 256;
constexpr int kCsrUnitMax = 2048;  // max nnz per work unit of the transpose SpMV
#ifndef APC_HEAD_ROWS
#define APC_HEAD_ROWS 8192
#endif
#ifndef APC_HEAD_THREADS
#define APC_HEAD_THREADS 512
#endif
constexpr int kHeadRows = APC_HEAD_ROWS;  // rows of A per block of the head adjoint (u block in shared memory)
constexpr int kHeadThreads = APC_HEAD_THREADS;
constexpr int kHeadPad = 0x7fff;
#ifndef APC_HEAD_PER_LANE
#define APC_HEAD_PER_LANE 4
#endif
#ifndef APC_HEAD_PREFETCH
#define APC_HEAD_PREFETCH 1
#endif
constexpr int kHeadPerLane = APC_HEAD_PER_LANE;       // consecutive entries per lane (4 or 8)
constexpr int kHeadStep = 32 * kHeadPerLane;          // entries per warp step   // column of the padding entries (head columns are below it)

// ---------------------------------------------------------------------------
// forward epilogue interface:
//   __device__ void begin();                       // load scalars
//   __device__ double load(i64 r);                 // epilogue input of row r (issued early)
//   __device__ double row(i64 r, double v, double pre); // consume (A x)_r, return ||.||^2 term
//   __device__ void tile_done(unsigned tile, unsigned ntiles, double sum_sq);
// ---------------------------------------------------------------------------
struct FwdStore {  // y = A x
  double* y;
  __device__ void begin() {}
  __device__ double load(long long) { return 0.0; }
  __device__ double row(long long r, double v, double) { y[r] = v; return 0.0; }
  __device__ void tile_done(unsigned, unsigned, double) {}
};

// ---------------------------------------------------------------------------
// Dense A x (column-major, ld = mloc), split over columns.
// grid = (ntiles, nsplit); part: nsplit x mloc partials; tile_ctr: ntiles counters
// ---------------------------------------------------------------------------
template <class Epi>
__global__ void __launch_bounds__(kDenseFwdThreads, 4)
dense_fwd_kernel(const double* __restrict__ A, long long ld, long long mloc, long long n,
                 const double* __restrict__ x, long long cols_per_split,
                 double* __restrict__ part, unsigned* __restrict__ tile_ctr, const int* done,
                 Epi epi) {
  constexpr int R = kDenseFwdRowsPerThread;
  __shared__ double red[32];
  if (done && *done) return;
  const int nsplit = gridDim.y;
  const long long tile = blockIdx.x;
  const long long c0 = blockIdx.y * cols_per_split;
  const long long c1 = c0 + cols_per_split < n ? c0 + cols_per_split : n;
  // R rows per thread, kDenseFwdThreads apart: per column the CTA reads one
  // contiguous R x 2 KB segment
  long long r[R];
  bool ok[R];
  double acc[R];
#pragma unroll
  for (int k = 0; k < R; ++k) {
    r[k] = tile * kDenseFwdTile + threadIdx.x + k * kDenseFwdThreads;
    ok[k] = r[k] < mloc;
    acc[k] = 0.0;
  }
  const double* ab = A + tile * kDenseFwdTile + threadIdx.x;
  long long c = c0;
  if (ok[R - 1]) {
    for (; c + 4 <= c1; c += 4) {
      double xv[4], av[4][R];
#pragma unroll
      for (int u = 0; u < 4; ++u) xv[u] = __ldg(x + c + u);
#pragma unroll
      for (int u = 0; u < 4; ++u)
#pragma unroll
        for (int k = 0; k < R; ++k) av[u][k] = __ldg(ab + (c + u) * ld + k * kDenseFwdThreads);
#pragma unroll
      for (int u = 0; u < 4; ++u)
#pragma unroll
        for (int k = 0; k < R; ++k) acc[k] += av[u][k] * xv[u];
    }
    for (; c < c1; ++c) {
      const double xc = __ldg(x + c);
#pragma unroll
      for (int k = 0; k < R; ++k) acc[k] += __ldg(ab + c * ld + k * kDenseFwdThreads) * xc;
    }
  } else {
    for (; c < c1; ++c) {
      const double xc = __ldg(x + c);
#pragma unroll
      for (int k = 0; k < R; ++k)
        if (ok[k]) acc[k] += __ldg(ab + c * ld + k * kDenseFwdThreads) * xc;
    }
  }
  if (nsplit > 1) {  // partials only: dense_split_epi_kernel sums them and runs the epilogue
#pragma unroll
    for (int k = 0; k < R; ++k)
      if (ok[k]) part[blockIdx.y * mloc + r[k]] = acc[k];
    return;
  }
  double pre[R];
#pragma unroll
  for (int k = 0; k < R; ++k) pre[k] = ok[k] ? epi.load(r[k]) : 0.0;
  epi.begin();
  double sq = 0.0;
#pragma unroll
  for (int k = 0; k < R; ++k)
    if (ok[k]) sq += epi.row(r[k], acc[k], pre[k]);
  sq = block_sum<kDenseFwdThreads>(sq, red);
  epi.tile_done(static_cast<unsigned>(tile), gridDim.x, sq);
}

// the split partials of dense_fwd_kernel summed in split order, thread per
// row (the loads of one row are independent and in flight together), then the
// epilogue; one norm partial per CTA.  A separate launch: the last CTA of a
// tile used to sum every split of its 2048 rows with one dependent load after
// another (~60 us for the 62 splits of an explicit basis B, n x l = 1e4 x 1000)
template <class Epi>
__global__ void __launch_bounds__(256)
dense_split_epi_kernel(const double* __restrict__ part, int nsplit, long long mloc, const int* done, Epi epi) {
  __shared__ double red[32];
  if (done && *done) return;
  const long long r = static_cast<long long>(blockIdx.x) * 256 + threadIdx.x;
  double pre = 0.0, acc = 0.0;
  if (r < mloc) {
    pre = epi.load(r);
    // the loads of a row issued 8 at a time before their (in-order) adds: a load
    // per add stalled the warp on every split (29 us for the 62 splits of C3's
    // explicit basis); same order of additions, same bits
    for (int sp = 0; sp < nsplit; sp += 8) {
      double t[8];
#pragma unroll
      for (int k = 0; k < 8; ++k) t[k] = sp + k < nsplit ? __ldcg(part + (sp + k) * mloc + r) : 0.0;
#pragma unroll
      for (int k = 0; k < 8; ++k)
        if (sp + k < nsplit) acc += t[k];
    }
  }
  epi.begin();
  double sq = r < mloc ? epi.row(r, acc, pre) : 0.0;
  sq = block_sum<256>(sq, red);
  epi.tile_done(blockIdx.x, gridDim.x, sq);
}

// ---------------------------------------------------------------------------
// Dense A^T u: CTA = 16 columns x one row split; warp-shuffle dot products.
// grid = (ceil(n/16), msplit); part: msplit x n; grp_ctr: ceil(n/16) counters.
// ---------------------------------------------------------------------------
__global__ void __launch_bounds__(kDenseAdjThreads)
dense_adj_kernel(const double* __restrict__ A, long long ld, long long mloc, long long n,
                 const double* __restrict__ u, long long rows_per_split,
                 double* __restrict__ part, unsigned* __restrict__ grp_ctr,
                 double* __restrict__ out, const int* done);

// ---------------------------------------------------------------------------
// CSR A x: G lanes per row, fixed rows per tile (deterministic tile slots).
// ---------------------------------------------------------------------------
// one tile of rows; returns this thread's share of the epilogue's ||.||^2
template <int G, class Epi, int U>
__device__ __forceinline__ double csr_fwd_tile(const int* __restrict__ ptr, const int* __restrict__ idx,
                                               const double* __restrict__ val, long long rows,
                                               const double* __restrict__ x, unsigned tile, Epi& epi) {
  constexpr int kGroups = kCsrFwdThreads / G;
  // U rows in flight per lane group: more memory-level parallelism for the
  // HBM-streaming case; U = 1 keeps small (L2-resident) matrices spread wide
  const int g = threadIdx.x / G, lane = threadIdx.x % G;
  const long long rbase = static_cast<long long>(tile) * kCsrFwdRowsPerBlock;
  double sq = 0.0;
  for (int k = 0; k < kCsrFwdRowsPerBlock; k += kGroups * U) {
    long long r[U];
    int b[U], len[U];
    // the epilogue of row uu runs on lane uu of the group (U <= G): its
    // input is fetched with the row pointers, off the critical path
    static_assert(U <= G, "one epilogue lane per row");
    double pre = 0.0;
    int maxlen = 0;
#pragma unroll
    for (int uu = 0; uu < U; ++uu) {
      r[uu] = rbase + k + uu * kGroups + g;
      b[uu] = 0;
      len[uu] = 0;
      if (k + uu * kGroups < kCsrFwdRowsPerBlock && r[uu] < rows) {
        b[uu] = __ldg(ptr + r[uu]);
        len[uu] = __ldg(ptr + r[uu] + 1) - b[uu];
        if (lane == uu) pre = epi.load(r[uu]);
      }
      maxlen = max(maxlen, len[uu]);
    }
    double s[U];
#pragma unroll
    for (int uu = 0; uu < U; ++uu) s[uu] = 0.0;
    // CSR arrays are streamed once (evict-first); x stays cached for the gathers
    for (int q = lane; q < maxlen; q += G) {
#pragma unroll
      for (int uu = 0; uu < U; ++uu)
        if (q < len[uu]) s[uu] += __ldcs(val + b[uu] + q) * __ldg(x + __ldcs(idx + b[uu] + q));
    }
    // butterfly: every lane of the group ends with the bit-identical row sum
#pragma unroll
    for (int uu = 0; uu < U; ++uu) {
#pragma unroll
      for (int o = G / 2; o > 0; o >>= 1) s[uu] += __shfl_xor_sync(0xffffffffu, s[uu], o, G);
      if (lane == uu && k + uu * kGroups < kCsrFwdRowsPerBlock && r[uu] < rows) sq += epi.row(r[uu], s[uu], pre);
    }
  }
  return sq;
}

template <int G, class Epi, int U = 1>
__global__ void __launch_bounds__(kCsrFwdThreads)
csr_fwd_kernel(const int* __restrict__ ptr, const int* __restrict__ idx,
               const double* __restrict__ val, long long rows, const double* __restrict__ x,
               const int* done, Epi epi) {
  __shared__ double red[32];
  if (done && *done) return;
  epi.begin();
  double sq = csr_fwd_tile<G, Epi, U>(ptr, idx, val, rows, x, blockIdx.x, epi);
  sq = block_sum<kCsrFwdThreads>(sq, red);
  epi.tile_done(blockIdx.x, gridDim.x, sq);
}

// Large CSR: exactly the co-resident CTAs walk the tiles grid-stride and the
// epilogue sees one slot per CTA -- a per-tile epilogue would make ~10^4-10^5
// CTAs serialise on the last-block counter (C5: +0.39 ms per product).
#ifndef APC_FWD_GS_MINB
#define APC_FWD_GS_MINB 4
#endif
template <int G, class Epi, int U>
__global__ void __launch_bounds__(kCsrFwdThreads, APC_FWD_GS_MINB)
csr_fwd_gs_kernel(const int* __restrict__ ptr, const int* __restrict__ idx, const double* __restrict__ val,
                  long long rows, const double* __restrict__ x, unsigned ntiles, const int* done, Epi epi) {
  __shared__ double red[32];
  if (done && *done) return;
  epi.begin();
  double sq = 0.0;
  for (unsigned t = blockIdx.x; t < ntiles; t += gridDim.x) sq += csr_fwd_tile<G, Epi, U>(ptr, idx, val, rows, x, t, epi);
  sq = block_sum<kCsrFwdThreads>(sq, red);
  epi.tile_done(blockIdx.x, gridDim.x, sq);
}

// ---------------------------------------------------------------------------
// Large CSR through the hot-relabelled SELL-32 copy (HotSell): lane = row, the
// co-resident CTAs walk 32-row chunks grid-stride (one epilogue slot per CTA).
// idx/val of entry k of the chunk's 32 rows are one coalesced 128 B / 256 B
// line each; each row is still summed sequentially (in relabelled column
// order), and the row's epilogue input (u_r) is a coalesced load too.
// ---------------------------------------------------------------------------
#ifndef APC_HOT_KU
#define APC_HOT_KU 16
#endif
#ifndef APC_HOT_MINB
#define APC_HOT_MINB 6
#endif
constexpr int kHotThreads = 256;

__global__ void hot_permute_kernel(const int* __restrict__ hot, long long n, const double* __restrict__ x,
                                   double* __restrict__ xr);

template <class Epi>
__global__ void __launch_bounds__(kHotThreads, APC_HOT_MINB)
hot_sell_fwd_kernel(const int* __restrict__ ptr, const int* __restrict__ off, const int* __restrict__ sidx,
                    const double* __restrict__ sval, long long rows, long long chunks,
                    const double* __restrict__ xr, const int* done, Epi epi) {
  constexpr int KU = APC_HOT_KU;
  __shared__ double red[32];
  if (done && *done) return;
  epi.begin();
  const int lane = threadIdx.x & 31;
  const long long wstride = static_cast<long long>(gridDim.x) * (kHotThreads / 32);
  double sq = 0.0;
  for (long long ch = static_cast<long long>(blockIdx.x) * (kHotThreads / 32) + (threadIdx.x >> 5); ch < chunks;
       ch += wstride) {
    const long long r = ch * 32 + lane;
    const bool ok = r < rows;
    int len = 0;
    double pre = 0.0;
    if (ok) {
      const int b = __ldg(ptr + r);
      len = __ldg(ptr + r + 1) - b;
      pre = epi.load(r);
    }
    const int o = __ldg(off + ch);
    const int w = (__ldg(off + ch + 1) - o) >> 5;
    const int* ip = sidx + o + lane;
    const double* vp = sval + o + lane;
    double s = 0.0;
    for (int k = 0; k < w; k += KU) {
      int id[KU];
      double v[KU];
#pragma unroll
      for (int q = 0; q < KU; ++q) {
        const bool on = k + q < len;
        id[q] = on ? __ldcs(ip + 32 * (k + q)) : 0;
        v[q] = on ? __ldcs(vp + 32 * (k + q)) : 0.0;
      }
#pragma unroll
      for (int q = 0; q < KU; ++q)
        if (k + q < len) s += v[q] * __ldg(xr + id[q]);
    }
    if (ok) sq += epi.row(r, s, pre);
  }
  sq = block_sum<kHotThreads>(sq, red);
  epi.tile_done(blockIdx.x, gridDim.x, sq);
}

// ---------------------------------------------------------------------------
// CSR A^T u over nnz-balanced work units (one warp per unit).
// ---------------------------------------------------------------------------
__global__ void __launch_bounds__(kCsrUnitThreads)
csr_units_kernel(const int* __restrict__ ptr, const int* __restrict__ idx,
                 const double* __restrict__ val, const double* __restrict__ u, long long n_units,
                 const int* __restrict__ urow, const int* __restrict__ ustart,
                 const int* __restrict__ uend, const int* __restrict__ uslot,
                 double* __restrict__ out, double* __restrict__ upart, const int* done);

// ---------------------------------------------------------------------------
// host-side launch helpers (ops.cu)
// ---------------------------------------------------------------------------
struct DenseFwdPlan {
  long long ntiles, nsplit, cols_per_split;
};
DenseFwdPlan dense_fwd_plan(const apc_mat& a);
DenseFwdPlan dense_fwd_plan(long long mloc, long long ncols, int num_sms);
struct DenseAdjPlan {
  long long ngroups, msplit, rows_per_split;
};
DenseAdjPlan dense_adj_plan(const apc_mat& a);
DenseAdjPlan dense_adj_plan(long long mloc, long long n, int num_sms);
// raw dense A^T u for an arbitrary column-major block (ld = mloc)
void launch_dense_adj(apc_ctx* ctx, const double* A, long long mloc, long long n, const double* u,
                      double* out, const int* done, double* part, unsigned* ctr);
int csr_group_size(double avg_row_nnz);

// scratch owned by the matrix-independent ctx
double* ctx_scratch(apc_ctx* ctx, long long count);
unsigned* ctx_counters(apc_ctx* ctx, long long count);

// A x -> y (local rows), optional mu-tail: y[mloc + j] = mu * x[j]
void op_fwd(apc_mat& a, double mu, bool augmented, const double* x, double* y);
// A^T u -> y (local contribution), optional + mu * u[mloc + j]
void op_adj(apc_mat& a, double mu, bool augmented, const double* u, double* y);
// raw A^T u into out[0..n) (units fix-up is left to the caller for CSR)
void op_adj_raw(apc_mat& a, const double* u, double* out, const int* done);
// LSQR epilogue applied where A^T u is finalised (single rank): h_j =
// (raw_j + mu u_t[j]) / beta, beta = sqrt(*n2top + *n2tail) (lsqr.cu lsqr_epi_kernel)
struct AdjEpi {
  const double* ut;      // mu-tail of u (nullptr: none)
  double mu;
  const double* n2top;   // ||u_top||^2
  const double* n2tail;  // ||u_tail||^2 (nullptr: 0)
};
// op_adj_raw with the epilogue fused into the kernels that finalise columns;
// returns false (nothing launched) when the layout has no fused path
bool op_adj_epi(apc_mat& a, const double* u, double* h, const int* done, const AdjEpi& e);
// true when launch_fwd may be given x already in the hot-relabelled order
inline bool fwd_takes_permuted(const apc_mat& a) { return a.sparse && a.hot.built(); }

// device CSR build from host CSC (matrix upload)
void upload_csc(apc_mat& a, const long long* colptr, const long long* rowidx, const double* val);
void build_units(apc_ctx* ctx, apc::Csr& c, const std::vector<long long>& row_nnz);
// units over the rows of a CSR with explicit row offsets, skipping rows with skip[r] != 0
void build_units_sel(apc_ctx* ctx, apc::Units& u, long long rows, const std::vector<long long>& off,
                     const std::vector<long long>& row_nnz, const std::vector<char>* skip,
                     const int* colidx = nullptr, long long ncols_local = 0, int superblocks = 1);
void launch_units(apc_ctx* ctx, const apc::Csr& c, const apc::Units& un, const double* u, double* out,
                  const int* done);
// head/tail split of CSR(A^T) for the row-blocked adjoint (called at upload)
void build_head_adj(apc_mat& a, const std::vector<int>& tptr, const int* hidx, const std::vector<long long>& tlen);

template <class Epi>
void launch_dense_fwd(apc_mat& a, const double* x, const int* done, Epi epi, cudaStream_t st) {
  DenseFwdPlan p = dense_fwd_plan(a);
  double* part = p.nsplit > 1 ? ctx_scratch(a.ctx, p.nsplit * a.mloc()) : nullptr;
  unsigned* ctr = p.nsplit > 1 ? ctx_counters(a.ctx, p.ntiles) : nullptr;
  dim3 grid(static_cast<unsigned>(p.ntiles), static_cast<unsigned>(p.nsplit));
  dense_fwd_kernel<Epi><<<grid, kDenseFwdThreads, 0, st>>>(a.dense.p, a.mloc(), a.mloc(), a.n, x,
                                                             p.cols_per_split, part, ctr, done, epi);
  a.ctx->launches++;
  if (p.nsplit > 1) {
    dense_split_epi_kernel<Epi><<<static_cast<unsigned>((a.mloc() + 255) / 256), 256, 0, st>>>(
        part, static_cast<int>(p.nsplit), a.mloc(), done, epi);
    a.ctx->launches++;
  }
}

// co-resident CTAs of a grid-stride forward kernel (cached occupancy)
unsigned fwd_gs_grid(apc_ctx* ctx, const void* kfn, int threads = kCsrFwdThreads);
// hot-relabelled SELL-32 copy of a large CSR (called at upload)
void build_hot_sell(apc_mat& a, const std::vector<long long>& col_nnz);

template <class Epi>
void launch_csr_fwd(apc_mat& a, const double* x, const int* done, Epi epi, cudaStream_t st,
                    bool x_permuted = false, double* xr_buf = nullptr) {
  const long long rows = a.a.rows;
  const unsigned nb = static_cast<unsigned>((rows + kCsrFwdRowsPerBlock - 1) / kCsrFwdRowsPerBlock);
  if (nb == 0) return;
  if (a.hot.built()) {
    // grid <= nb keeps the epilogue's slots within fwd_num_tiles(a)
    const unsigned grid =
        std::min<unsigned>(nb, fwd_gs_grid(a.ctx, reinterpret_cast<const void*>(hot_sell_fwd_kernel<Epi>), kHotThreads));
    // xr_buf: a private permuted copy (the observer's sample must not clobber
    // the z copy the fused n-space kernel left in a.hot.xr for the next forward)
    double* xr = xr_buf ? xr_buf : a.hot.xr.p;
    if (!x_permuted) {  // else the producer of x wrote a.hot.xr itself (pc_expand / lsqr_nspace_kernel)
      hot_permute_kernel<<<static_cast<unsigned>((a.n + 255) / 256), 256, 0, st>>>(a.hot.hot.p, a.n, x, xr);
      a.ctx->launches++;
    }
    hot_sell_fwd_kernel<Epi><<<grid, kHotThreads, 0, st>>>(a.a.ptr.p, a.hot.s.off.p, a.hot.s.idx.p, a.hot.s.val.p,
                                                           rows, a.hot.s.chunks, xr, done, epi);
    a.ctx->launches += 1;
    return;
  }
  const bool big = rows >= (1LL << 21);
#define APC_FWD_CASE(GG)                                                                                      \
  case GG:                                                                                                    \
    if (big) {                                                                                                \
      const unsigned grid = std::min<unsigned>(nb, fwd_gs_grid(a.ctx, reinterpret_cast<const void*>(         \
                                                       csr_fwd_gs_kernel<GG, Epi, 4>)));                      \
      csr_fwd_gs_kernel<GG, Epi, 4><<<grid, kCsrFwdThreads, 0, st>>>(a.a.ptr.p, a.a.idx.p, a.a.val.p, rows, x, \
                                                                     nb, done, epi);                          \
    } else {                                                                                                  \
      csr_fwd_kernel<GG, Epi, 1><<<nb, kCsrFwdThreads, 0, st>>>(a.a.ptr.p, a.a.idx.p, a.a.val.p, rows, x, done, \
                                                                epi);                                         \
    }                                                                                                         \
    break;
  switch (csr_group_size(a.a.avg_row_nnz)) {
    APC_FWD_CASE(4)
    APC_FWD_CASE(8)
    APC_FWD_CASE(16)
    APC_FWD_CASE(32)
  }
#undef APC_FWD_CASE
  a.ctx->launches++;
}

template <class Epi>
void launch_fwd(apc_mat& a, const double* x, const int* done, Epi epi, cudaStream_t st, bool x_permuted = false,
                double* xr_buf = nullptr) {
  if (a.sparse) launch_csr_fwd(a, x, done, epi, st, x_permuted, xr_buf);
  else launch_dense_fwd(a, x, done, epi, st);
}

inline unsigned fwd_num_tiles(const apc_mat& a) {
  if (a.sparse) return static_cast<unsigned>((a.a.rows + kCsrFwdRowsPerBlock - 1) / kCsrFwdRowsPerBlock);
  return static_cast<unsigned>(dense_fwd_plan(a).ntiles);
}

}  // namespace apc
