// Operator kernels and matrix upload (see ops.cuh for the design notes).
#include <cub/device/device_radix_sort.cuh>
#include <cub/device/device_scan.cuh>

#include <algorithm>
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
__global__ void __launch_bounds__(kCsrUnitThreads)
csr_units_kernel(const int* __restrict__ ptr, const int* __restrict__ idx,
                 const double* __restrict__ val, const double* __restrict__ u, long long n_units,
                 const int* __restrict__ urow, const int* __restrict__ ustart,
                 const int* __restrict__ uend, const int* __restrict__ uslot,
                 double* __restrict__ out, double* __restrict__ upart, const int* done) {
  if (done && *done) return;
  const long long unit = (static_cast<long long>(blockIdx.x) * kCsrUnitThreads + threadIdx.x) >> 5;
  const int lane = threadIdx.x & 31;
  if (unit >= n_units) return;
  const int b = __ldg(ustart + unit), e = __ldg(uend + unit);
  double s0 = 0.0, s1 = 0.0, s2 = 0.0, s3 = 0.0;
  int q = b + lane;
  // CSR(A^T) streamed with evict-first loads so the gathered u stays in L2
  for (; q + 96 < e; q += 128) {
    const int i0 = __ldcs(idx + q), i1 = __ldcs(idx + q + 32), i2 = __ldcs(idx + q + 64), i3 = __ldcs(idx + q + 96);
    s0 += __ldcs(val + q) * __ldg(u + i0);
    s1 += __ldcs(val + q + 32) * __ldg(u + i1);
    s2 += __ldcs(val + q + 64) * __ldg(u + i2);
    s3 += __ldcs(val + q + 96) * __ldg(u + i3);
  }
  for (; q < e; q += 32) s0 += __ldcs(val + q) * __ldg(u + __ldcs(idx + q));
  s0 += s2;
  s1 += s3;
  double s = warp_sum(s0 + s1);
  if (lane == 0) {
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

// sum of the partials of every split row (rows longer than one work unit),
// block per split row, fixed order: written to out[row] so every consumer of
// op_adj_raw (LSQR epilogue, NCCL allreduce, op_adj) reads plain values
__global__ void __launch_bounds__(256)
split_fixup_kernel(const int* __restrict__ srows, const int* __restrict__ rfirst, const int* __restrict__ rcount,
                   const double* __restrict__ upart, double* __restrict__ out, const int* done) {
  __shared__ double red[32];
  if (done && *done) return;
  const int j = srows[blockIdx.x];
  const int f = rfirst[j], cnt = rcount[j];
  double s = 0.0;
  for (int k = threadIdx.x; k < cnt; k += 256) s += upart[f + k];
  s = block_sum<256>(s, red);
  if (threadIdx.x == 0) out[j] = s;
}

}  // namespace

unsigned fwd_gs_grid(apc_ctx* ctx, const void* kfn) {
  static std::mutex mu;
  static std::map<std::pair<int, const void*>, unsigned> cache;
  std::lock_guard<std::mutex> lk(mu);
  const auto key = std::make_pair(ctx->device, kfn);
  auto it = cache.find(key);
  if (it != cache.end()) return it->second;
  int per_sm = 0;
  APC_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kfn, kCsrFwdThreads, 0));
  const unsigned g = static_cast<unsigned>(ctx->num_sms * std::max(1, per_sm));
  cache[key] = g;
  return g;
}

// ---------------------------------------------------------------------------
// plans
// ---------------------------------------------------------------------------
DenseFwdPlan dense_fwd_plan(const apc_mat& a) { return dense_fwd_plan(a.mloc(), a.n, a.ctx->num_sms); }

DenseFwdPlan dense_fwd_plan(long long mloc, long long ncols, int num_sms) {
  DenseFwdPlan p;
  p.ntiles = (mloc + kDenseFwdTile - 1) / kDenseFwdTile;
  if (p.ntiles < 1) p.ntiles = 1;
  // aim for >= 6 CTAs per SM, but keep >= 64 columns per split
  const long long want = 6LL * num_sms;
  long long ns = (want + p.ntiles - 1) / p.ntiles;
  long long maxs = std::max<long long>(1, ncols / 64);
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
  if (c.n_units == 0) return;
  unsigned nb = nblk(c.n_units * 32, kCsrUnitThreads);
  csr_units_kernel<<<nb, kCsrUnitThreads, 0, st>>>(c.ptr.p, c.idx.p, c.val.p, u, c.n_units,
                                                   c.urow.p, c.ustart.p, c.uend.p, c.uslot.p, out,
                                                   c.upart.p, done);
  a.ctx->launches++;
  if (c.n_split > 0) {
    split_fixup_kernel<<<static_cast<unsigned>(c.n_split), 256, 0, st>>>(c.srows.p, c.rfirst.p, c.rcount.p, c.upart.p,
                                                                         out, done);
    a.ctx->launches++;
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
  std::vector<int> urow, ustart, uend, uslot, rfirst(c.rows, -1), rcount(c.rows, 0);
  urow.reserve(c.rows);
  long long off = 0, nparts = 0, maxr = 0;
  for (long long r = 0; r < c.rows; ++r) {
    long long L = row_nnz[r];
    maxr = std::max(maxr, L);
    if (L <= kCsrUnitMax) {
      urow.push_back(static_cast<int>(r));
      ustart.push_back(static_cast<int>(off));
      uend.push_back(static_cast<int>(off + L));
      uslot.push_back(-1);
    } else {
      long long k = (L + kCsrUnitMax - 1) / kCsrUnitMax;
      rfirst[r] = static_cast<int>(nparts);
      rcount[r] = static_cast<int>(k);
      for (long long q = 0; q < k; ++q) {
        long long b = off + q * kCsrUnitMax, e = std::min(off + L, b + kCsrUnitMax);
        urow.push_back(static_cast<int>(r));
        ustart.push_back(static_cast<int>(b));
        uend.push_back(static_cast<int>(e));
        uslot.push_back(static_cast<int>(nparts + q));
      }
      nparts += k;
    }
    off += L;
  }
  c.n_units = static_cast<long long>(urow.size());
  c.n_parts = nparts;
  std::vector<int> srows;
  for (long long r = 0; r < c.rows; ++r)
    if (rfirst[r] >= 0) srows.push_back(static_cast<int>(r));
  c.n_split = static_cast<long long>(srows.size());
  c.max_row_nnz = maxr;
  c.avg_row_nnz = c.rows > 0 ? static_cast<double>(off) / static_cast<double>(c.rows) : 0.0;
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
}

}  // namespace apc
