// Internal declarations shared by the host runtime (.cpp) and the sm_100a
// kernels (.cu) of libapc_b200.  Not part of the public C-ABI (include/apc_b200.h).
#pragma once

#include <cuda_runtime.h>

#include <cstdint>
#include <memory>
#include <stdexcept>
#include <string>
#include <vector>

#include "apc_b200.h"

namespace apc {

using i64 = std::int64_t;
using i32 = std::int32_t;

// Error carrying an APC_* status (1..9 mirror aplicur::ErrorKind + 1,
// /root/reference/proj/include/aplicur/error.hpp:10-20) and an index payload.
struct Status : std::runtime_error {
  int code;
  i64 index;
  Status(int c, const std::string& what, i64 idx = -1)
      : std::runtime_error(what), code(c), index(idx) {}
};

[[noreturn]] inline void fail(int code, const std::string& what, i64 idx = -1) {
  throw Status(code, what, idx);
}
inline void require(bool cond, int code, const std::string& what, i64 idx = -1) {
  if (!cond) fail(code, what, idx);
}
// literal messages: no std::string is built unless the check fails
inline void require(bool cond, int code, const char* what, i64 idx = -1) {
  if (!cond) fail(code, what, idx);
}

void cuda_check(cudaError_t e, const char* what);
#define APC_CUDA(call) ::apc::cuda_check((call), #call)

// Caching device allocator (per device, size-class free lists): the CUR and
// LSQR setup paths allocate many short-lived buffers; cudaMalloc/cudaFree
// (which synchronises the device) would dominate their wall time.
void* pool_alloc(size_t bytes);
void pool_free(void* p, size_t bytes);
void pool_trim();  // return every cached block to the driver

// Blocking copy ordered on the library stream (the ctx stream is created
// non-blocking, so plain cudaMemcpy on the legacy stream would not order
// against its kernels).
inline void copy_sync(cudaStream_t st, void* dst, const void* src, size_t bytes, cudaMemcpyKind kind) {
  if (bytes == 0) return;
  APC_CUDA(cudaMemcpyAsync(dst, src, bytes, kind, st));
  APC_CUDA(cudaStreamSynchronize(st));
}

// Host wall-time breakdown of the solve setup (APC_SETUP_PROF=1): named
// buckets, accumulated per thread, printed by the solver at the end.
struct SetupProf {
  static bool on();
  static void add(const char* name, double ms);
  static void dump_and_reset(const char* title);
};
struct ProfScope {
  const char* name;
  double t0;
  explicit ProfScope(const char* n);
  ~ProfScope();
};

// ---------------------------------------------------------------------------
// Device buffers
// ---------------------------------------------------------------------------
template <class T>
struct DBuf {
  T* p = nullptr;
  i64 n = 0;
  DBuf() = default;
  explicit DBuf(i64 count) { alloc(count); }
  DBuf(const DBuf&) = delete;
  DBuf& operator=(const DBuf&) = delete;
  DBuf(DBuf&& o) noexcept : p(o.p), n(o.n) { o.p = nullptr; o.n = 0; }
  DBuf& operator=(DBuf&& o) noexcept {
    if (this != &o) { release(); p = o.p; n = o.n; o.p = nullptr; o.n = 0; }
    return *this;
  }
  ~DBuf() { release(); }
  void alloc(i64 count) {
    release();
    if (count > 0) p = static_cast<T*>(pool_alloc(sizeof(T) * static_cast<size_t>(count)));
    n = count;
  }
  // grow-only reallocation (contents discarded)
  void ensure(i64 count) { if (count > n) alloc(count); }
  void release() {
    if (p) pool_free(p, sizeof(T) * static_cast<size_t>(n));
    p = nullptr;
    n = 0;
  }
  size_t bytes() const { return sizeof(T) * static_cast<size_t>(n); }
};

// ---------------------------------------------------------------------------
// Compressed sparse rows (int32 indices; values fp64)
// ---------------------------------------------------------------------------
// nnz-balanced work units over the rows of a CSR (one warp per unit): unit u
// covers [ustart[u], uend[u]) of row urow[u]; rows split in several units write
// partial sums to upart[slot] which a fix-up pass adds in order.
struct Units {
  i64 n_units = 0, n_parts = 0;
  DBuf<i32> urow, ustart, uend, uslot;  // per unit (uslot < 0: whole row)
  DBuf<i32> rfirst, rcount;             // per row: first partial slot (-1: not split), count
  i64 n_split = 0;
  DBuf<i32> srows;                      // the split rows (summed into the output by op_adj_raw)
  DBuf<double> upart;                   // n_parts partial sums
};

struct Csr : Units {
  i64 rows = 0, cols = 0, nnz = 0;
  DBuf<i32> ptr;  // rows+1
  DBuf<i32> idx;  // nnz
  DBuf<double> val;
  i64 max_row_nnz = 0;
  double avg_row_nnz = 0.0;
};

// Row-blocked A^T u for the long (Zipf-head) rows of CSR(A^T): the local rows
// of A are cut into blocks of kHeadRows.  The head entries of block b are
// stored contiguously at [bptr[b], bptr[b+1]), sorted by (head column, row),
// each with a packed key (head column << 16 | row within block).  A CTA stages
// its block of u in shared memory and streams the block's entries (warp steps
// of 32 coalesced entries, segmented scan by column), producing one partial per
// (head column, block) at part[k * nblocks + b]; a warp per head column adds its
// partials in block order.  The remaining (tail) rows of A^T go through `tail`
// work units gathering u from L2 as before.
struct HeadAdj {
  i64 ncols = 0, nblocks = 0, nnz = 0;
  int parts = 1;       // CTAs (work items) per block
  int rows = 0;        // rows of A per block (build_head_adj: a whole number of CTA waves)
  DBuf<i32> bptr;      // nblocks + 1 (multiples of 128; padding keys are -1)
  DBuf<i32> hkey;      // nnz: k << 16 | (row - block start)
  DBuf<double> hval;   // nnz
  DBuf<i32> zptr, zcol;  // per block: head columns absent from it (partial = 0)
  DBuf<i32> hcol;      // per head column: original column
  DBuf<double> part;   // ncols x nblocks
  DBuf<double> bnd;    // per work item: first / last piece (HeadPiece, ops.cu)
  Units tail;          // the other rows of A^T as warp-per-row work units (fallback)
  // ... or as a key-sorted entry stream (TailPolicy, ops.cu): whole columns
  // grouped in column order, key = column in group << rb | row, STEP-aligned
  struct Seg {
    i64 ngroups = 0, nnz = 0, ncols = 0;
    int rb = 0, parts = 1, sb = 1;       // sb: row superblocks (stream order)
    DBuf<i32> gptr, gcol0, tcol, zptr, zcol, tkey, cols;
    DBuf<double> tval, bnd, part;        // part: ncols x sb partials (sb > 1)
    DBuf<double> outc;                   // sb == 1: column sums in tail order, scattered by tcol
    bool built() const { return ngroups > 0; }
  } seg;
  bool built() const { return ncols > 0; }
};

// SELL-32 copy of a CSR (built on demand for L2-resident systems): rows in
// chunks of 32, entry k of the chunk's lane-th row at off[chunk] + 32 k + lane,
// so a warp walking 32 rows thread-per-row reads idx/val fully coalesced while
// every row is still summed sequentially in column order.
struct Sell {
  i64 rows = 0, chunks = 0, slots = 0;
  DBuf<i32> off;  // chunks + 1 (entries)
  DBuf<i32> idx;  // slots (padding never read)
  DBuf<double> val;
};

// Hot-relabelled SELL-32 copy of a large (HBM-streamed) CSR for the forward
// product: columns renumbered by descending nnz count (hot[k] = original id of
// relabelled column k), each row's entries sorted by the new id.  Lane l of a
// warp walks row 32c + l, so the k-th gather of the 32 rows of a chunk hits the
// few cache lines of x that hold the hottest columns (Zipf-headed matrices:
// ~40% fewer L1 wavefronts than gathering by original id).  x is permuted into
// xr (n doubles) before each product.
struct HotSell {
  Sell s;
  i64 n = 0;
  DBuf<i32> hot;    // n: relabelled -> original column
  DBuf<i32> inv;    // n: original -> relabelled column
  DBuf<double> xr;  // n: x in relabelled order (scratch of each product)
  bool built() const { return s.chunks > 0; }
};

// Panel copy of a dense A for the fused operator pair (dense_pair.cu): rows
// cut into panels of rb rows, panel p stored column-major on its own
// (ap[(p * n + c) * rb + r] = A(p * rb + r, c), rows past mloc zero), so the
// rb x W slice of one CTA (W consecutive columns) is ONE contiguous run: a
// single bulk (TMA) copy per tile whatever rb is.  The CTAs form ng groups of
// g; a group shares its panels (every CTA a column slice) and exchanges the
// rb partial row sums of each panel through `part` / `cnt`.
struct DensePanels {
  i64 mloc = 0, n = 0, npanels = 0;
  int rb = 0, W = 0, g = 0, gact = 0, ng = 0, stages = 0, nslot = 0;
  size_t smem = 0;
  int state = 0;        // 0: not tried, 1: built, -1: unsupported / disabled
  DBuf<double> ap;      // npanels * n * rb
  DBuf<double> part;    // ng * nslot * g * rb partial row sums (ring), two flagged 8-byte words each
  DBuf<double> gpart;   // ng * n column sums of the groups
  DBuf<double> nrmp;    // ng * g norm partials
  DBuf<unsigned> cnt;   // 2 finish counters (zero between launches) + the launch epoch of the exchange tags
};

}  // namespace apc

// ---------------------------------------------------------------------------
// Context (one per GPU / rank)
// ---------------------------------------------------------------------------
struct apc_ctx {
  int device = 0;
  int nranks = 1, rank = 0;
  cudaStream_t stream = nullptr;
  cudaStream_t side = nullptr;  // fork / join branch of the library stream (created on first use)
  cudaEvent_t ev_fork = nullptr, ev_join = nullptr;
  void* nccl = nullptr;  // ncclComm_t when nranks > 1 (NCCL backend)
  // host-staged backend (apc_ctx_create_host_comm): the caller's in-place sum
  // of a host buffer over the ranks, in rank order
  int (*host_allreduce)(double* buf, int64_t count, void* user) = nullptr;
  void* host_user = nullptr;
  void* blas = nullptr;  // cublasHandle_t (created lazily, bound to `stream`)
  std::string err;
  apc::i64 err_index = -1;
  int num_sms = 148;
  // scratch reused across calls
  apc::DBuf<double> scratch_d;
  apc::DBuf<unsigned int> counters;  // last-block counters (zeroed)
  // kernel launch counter (launches issued by this library on this ctx)
  std::uint64_t launches = 0;
  // grow-only pinned host staging buffers (cudaMallocHost takes driver locks
  // and costs milliseconds; uploads and solves reuse these): 0/1 CSC upload
  // index/value staging, 2 LSQR state readback
  struct Pinned {
    void* p = nullptr;
    size_t n = 0;
  } pinned[5];  // 3: host-staged collectives
};

// pinned host buffer `slot` of at least `bytes` (contents not preserved on growth)
inline void* ctx_pinned(apc_ctx* c, int slot, size_t bytes) {
  apc_ctx::Pinned& b = c->pinned[slot];
  if (b.n < bytes) {
    if (b.p) cudaFreeHost(b.p);
    b.p = nullptr;
    b.n = 0;
    APC_CUDA(cudaMallocHost(&b.p, bytes));
    b.n = bytes;
  }
  return b.p;
}

// Matrix handle: dense column-major (ld = local rows) or sparse stored twice
// as CSR(A) (for A*x) and CSR(A^T) (for A^T*x; the same arrays as the
// reference's CSC, matrix.hpp:31-34).  Row sharding keeps rows [r0, r1).
struct apc_mat {
  apc_ctx* ctx = nullptr;
  apc::i64 m = 0, n = 0;    // global shape
  apc::i64 r0 = 0, r1 = 0;  // local row shard [r0, r1)
  bool sparse = false;
  apc::DBuf<double> dense;  // local rows, column-major, ld = r1 - r0
  apc::Csr a;               // CSR of the local rows (mloc x n)
  apc::Csr at;              // CSR of their transpose (n x mloc)
  apc::Sell sell;           // SELL-32 copy of `a` (persistent LSQR, built lazily)
  apc::HotSell hot;         // hot-relabelled SELL-32 of `a` (large CSR forward, built at upload)
  apc::HeadAdj head;        // row-blocked A^T u of the long rows of `at` (built with `hot`)
  apc::DensePanels panels;  // panel copy of `dense` for the fused pair (built lazily by the LSQR phase)
  apc::i64 nnz_global = 0;
  apc::i64 mloc() const { return r1 - r0; }
};
