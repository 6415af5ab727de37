// extern "C" entry points of libapc_b200.so (declared in include/apc_b200.h).
// Every call converts exceptions into APC_* status codes; nothing throws
// across the boundary.  There is no CPU fallback: without a CUDA device the
// device-facing calls fail with APC_NO_DEVICE.
#include <algorithm>
#include <cstring>
#include <functional>
#include <map>
#include <mutex>
#include <string>
#include <vector>

#include "apc_internal.hpp"
#include "blas.hpp"
#include "dense_pair.hpp"
#include "dense_small.hpp"
#include "host_rng.hpp"
#include "rng_dev.hpp"
#include "lsqr.hpp"
#include "ops_host.hpp"
#include "solver.hpp"

namespace apc {

apc_problem* generate_problem(int config, i64 m, i64 n, std::uint64_t seed);

void cuda_check(cudaError_t e, const char* what) {
  if (e != cudaSuccess) {
    cudaGetLastError();
    fail(APC_CUDA_ERROR, std::string(what) + ": " + cudaGetErrorString(e));
  }
}

// ---- caching device allocator ---------------------------------------------
namespace {
std::mutex g_pool_mu;
std::map<std::pair<int, size_t>, std::vector<void*>> g_pool;  // (device, class) -> blocks

size_t size_class(size_t bytes) {
  if (bytes <= 512) return 512;
  if (bytes >= (size_t{256} << 20)) return (bytes + 0xFFFFF) & ~size_t{0xFFFFF};  // 1 MB granules
  size_t c = 512;
  while (c < bytes) c <<= 1;
  return c;
}
}  // namespace

void* pool_alloc(size_t bytes) {
  int dev = 0;
  cudaGetDevice(&dev);
  const size_t c = size_class(bytes);
  {
    std::lock_guard<std::mutex> lk(g_pool_mu);
    auto it = g_pool.find({dev, c});
    if (it != g_pool.end() && !it->second.empty()) {
      void* p = it->second.back();
      it->second.pop_back();
      return p;
    }
  }
  void* p = nullptr;
  cudaError_t e = cudaMalloc(&p, c);
  if (e != cudaSuccess) {  // give cached blocks back and retry once
    cudaGetLastError();
    pool_trim();
    APC_CUDA(cudaMalloc(&p, c));
  }
  return p;
}

void pool_free(void* p, size_t bytes) {
  if (!p) return;
  int dev = 0;
  cudaGetDevice(&dev);
  std::lock_guard<std::mutex> lk(g_pool_mu);
  g_pool[{dev, size_class(bytes)}].push_back(p);
}

void pool_trim() {
  std::lock_guard<std::mutex> lk(g_pool_mu);
  cudaDeviceSynchronize();
  for (auto& kv : g_pool)
    for (void* p : kv.second) cudaFree(p);
  g_pool.clear();
}

namespace {

thread_local std::string t_err;
thread_local i64 t_err_index = -1;

template <class F>
int guard(apc_ctx* ctx, F&& f) {
  try {
    f();
    return APC_OK;
  } catch (const Status& s) {
    t_err = s.what();
    t_err_index = s.index;
    if (ctx) {
      ctx->err = s.what();
      ctx->err_index = s.index;
    }
    return s.code;
  } catch (const std::exception& e) {
    t_err = e.what();
    t_err_index = -1;
    if (ctx) ctx->err = e.what();
    return APC_INVALID_ARGUMENT;
  }
}

void need_device() {
  int n = 0;
  if (cudaGetDeviceCount(&n) != cudaSuccess || n == 0) {
    cudaGetLastError();
    fail(APC_NO_DEVICE, "no CUDA device visible: the APLICUR hot path has no CPU fallback");
  }
}

}  // namespace

int capi_guard(apc_ctx* ctx, const std::function<void()>& f) { return guard(ctx, f); }

}  // namespace apc

using namespace apc;

extern "C" {

int apc_abi_version(void) { return APC_ABI_VERSION; }

const char* apc_last_error(int64_t* index) {
  if (index) *index = t_err_index;
  return t_err.c_str();
}

int apc_device_count(int* count) {
  return guard(nullptr, [&] {
    int n = 0;
    if (cudaGetDeviceCount(&n) != cudaSuccess) {
      cudaGetLastError();
      n = 0;
    }
    *count = n;
  });
}

int apc_ctx_create(int device, int nranks, int rank, const void* uid, apc_ctx** out) {
  *out = nullptr;
  return guard(nullptr, [&] {
    need_device();
    require(nranks >= 1 && rank >= 0 && rank < nranks, APC_INVALID_ARGUMENT, "apc_ctx_create: bad rank");
    APC_CUDA(cudaSetDevice(device));
    auto* c = new apc_ctx();
    c->device = device;
    c->nranks = nranks;
    c->rank = rank;
    try {
      APC_CUDA(cudaStreamCreateWithFlags(&c->stream, cudaStreamNonBlocking));
      cudaDeviceProp prop{};
      APC_CUDA(cudaGetDeviceProperties(&prop, device));
      c->num_sms = prop.multiProcessorCount;
      comm_init(c, uid);
    } catch (...) {
      if (c->stream) cudaStreamDestroy(c->stream);
      delete c;
      throw;
    }
    *out = c;
  });
}

int apc_ctx_create_host_comm(int device, int nranks, int rank, apc_host_allreduce_fn fn, void* user,
                             apc_ctx** out) {
  *out = nullptr;
  return guard(nullptr, [&] {
    need_device();
    require(nranks >= 1 && rank >= 0 && rank < nranks, APC_INVALID_ARGUMENT, "apc_ctx_create: bad rank");
    require(fn != nullptr || nranks == 1, APC_INVALID_ARGUMENT, "apc_ctx_create_host_comm: callback required");
    APC_CUDA(cudaSetDevice(device));
    auto* c = new apc_ctx();
    c->device = device;
    c->nranks = nranks;
    c->rank = rank;
    c->host_allreduce = fn;
    c->host_user = user;
    try {
      APC_CUDA(cudaStreamCreateWithFlags(&c->stream, cudaStreamNonBlocking));
      cudaDeviceProp prop{};
      APC_CUDA(cudaGetDeviceProperties(&prop, device));
      c->num_sms = prop.multiProcessorCount;
    } catch (...) {
      if (c->stream) cudaStreamDestroy(c->stream);
      delete c;
      throw;
    }
    *out = c;
  });
}

int apc_ctx_destroy(apc_ctx* ctx) {
  if (!ctx) return APC_OK;
  return guard(nullptr, [&] {
    cudaSetDevice(ctx->device);
    cudaStreamSynchronize(ctx->stream);
    comm_destroy(ctx);
    blas_destroy(ctx);
    for (auto& b : ctx->pinned)
      if (b.p) cudaFreeHost(b.p);
    ctx->scratch_d.release();
    ctx->counters.release();
    if (ctx->side) {
      cudaStreamDestroy(ctx->side);
      cudaEventDestroy(ctx->ev_fork);
      cudaEventDestroy(ctx->ev_join);
    }
    cudaStreamDestroy(ctx->stream);
    delete ctx;
    pool_trim();
  });
}

void* apc_ctx_stream(apc_ctx* ctx) { return ctx ? static_cast<void*>(ctx->stream) : nullptr; }
uint64_t apc_ctx_launches(apc_ctx* ctx) { return ctx ? ctx->launches : 0; }

int apc_ctx_sync(apc_ctx* ctx) {
  return guard(ctx, [&] { APC_CUDA(cudaStreamSynchronize(ctx->stream)); });
}

int apc_mat_upload_dense(apc_ctx* ctx, int64_t m, int64_t n, const double* colmajor, int64_t r0,
                         int64_t r1, apc_mat** out) {
  *out = nullptr;
  return guard(ctx, [&] {
    require(m >= 0 && n >= 0, APC_INVALID_ARGUMENT, "negative matrix shape");
    require(0 <= r0 && r0 <= r1 && r1 <= m, APC_INVALID_ARGUMENT, "apc_mat_upload_dense: bad row range");
    APC_CUDA(cudaSetDevice(ctx->device));
    auto* a = new apc_mat();
    a->ctx = ctx;
    a->m = m;
    a->n = n;
    a->r0 = r0;
    a->r1 = r1;
    a->sparse = false;
    a->nnz_global = m * n;
    const i64 mloc = r1 - r0;
    try {
      a->dense.alloc(std::max<i64>(1, mloc * n));
      if (mloc > 0 && n > 0)
        APC_CUDA(cudaMemcpy2DAsync(a->dense.p, sizeof(double) * mloc, colmajor + r0, sizeof(double) * m,
                                   sizeof(double) * mloc, n, cudaMemcpyHostToDevice, ctx->stream));
      APC_CUDA(cudaStreamSynchronize(ctx->stream));
    } catch (...) {
      delete a;
      throw;
    }
    *out = a;
  });
}

int apc_mat_upload_csc(apc_ctx* ctx, int64_t m, int64_t n, const int64_t* colptr,
                       const int64_t* rowidx, const double* val, int64_t r0, int64_t r1,
                       apc_mat** out) {
  *out = nullptr;
  return guard(ctx, [&] {
    require(m >= 0 && n >= 0, APC_INVALID_ARGUMENT, "negative matrix shape");
    require(0 <= r0 && r0 <= r1 && r1 <= m, APC_INVALID_ARGUMENT, "apc_mat_upload_csc: bad row range");
    require(colptr[0] == 0, APC_INVALID_ARGUMENT, "apc_mat_upload_csc: colptr[0] != 0");
    // validation (messages built only on failure: a std::string per entry
    // would cost more than the whole upload)
    for (i64 j = 0; j < n; ++j) {
      if (colptr[j + 1] < colptr[j]) fail(APC_INVALID_ARGUMENT, "apc_mat_upload_csc: colptr not monotone", j);
      for (i64 k = colptr[j]; k < colptr[j + 1]; ++k) {
        if (rowidx[k] < 0 || rowidx[k] >= m) fail(APC_INVALID_ARGUMENT, "Matrix::sparse: entry out of range", k);
        if (k != colptr[j] && rowidx[k] <= rowidx[k - 1])
          fail(APC_INVALID_ARGUMENT, "Matrix::sparse: rows must be strictly increasing per column", k);
      }
    }
    APC_CUDA(cudaSetDevice(ctx->device));
    auto* a = new apc_mat();
    a->ctx = ctx;
    a->m = m;
    a->n = n;
    a->r0 = r0;
    a->r1 = r1;
    a->sparse = true;
    a->nnz_global = colptr[n];
    try {
      upload_csc(*a, reinterpret_cast<const long long*>(colptr), reinterpret_cast<const long long*>(rowidx), val);
    } catch (...) {
      delete a;
      throw;
    }
    *out = a;
  });
}

int apc_mat_free(apc_mat* a) {
  if (!a) return APC_OK;
  return guard(nullptr, [&] {
    cudaSetDevice(a->ctx->device);
    cudaStreamSynchronize(a->ctx->stream);
    delete a;
  });
}

int apc_mat_info(const apc_mat* a, int64_t* m, int64_t* n, int64_t* nnz, int* sparse, int64_t* r0,
                 int64_t* r1) {
  if (m) *m = a->m;
  if (n) *n = a->n;
  if (nnz) *nnz = a->nnz_global;
  if (sparse) *sparse = a->sparse ? 1 : 0;
  if (r0) *r0 = a->r0;
  if (r1) *r1 = a->r1;
  return APC_OK;
}

int apc_dgemm(apc_ctx* ctx, int ta, int tb, int64_t m, int64_t n, int64_t k, double alpha, const double* A,
              int64_t lda, const double* B, int64_t ldb, double beta, double* C, int64_t ldc) {
  return guard(ctx, [&] {
    require(m >= 0 && n >= 0 && k >= 0, APC_INVALID_ARGUMENT, "apc_dgemm: negative shape");
    dgemm(ctx, ta != 0, tb != 0, m, n, k, alpha, A, lda, B, ldb, beta, C, ldc);
    APC_CUDA(cudaStreamSynchronize(ctx->stream));
  });
}

int apc_dtrsm_right_upper(apc_ctx* ctx, int64_t m, int64_t n, const double* T, int64_t ldt, double* B, int64_t ldb) {
  return guard(ctx, [&] {
    require(m >= 0 && n >= 0, APC_INVALID_ARGUMENT, "apc_dtrsm_right_upper: negative shape");
    dtrsm_right_upper(ctx, m, n, T, ldt, B, ldb);
    APC_CUDA(cudaStreamSynchronize(ctx->stream));
  });
}

int apc_dpotrf_upper(apc_ctx* ctx, int64_t k, double* A, int64_t* bad) {
  return guard(ctx, [&] {
    require(k >= 0, APC_INVALID_ARGUMENT, "apc_dpotrf_upper: negative shape");
    const int b = k > 0 ? dpotrf_upper_dev(ctx, k, A) : -1;
    if (bad) *bad = b;
  });
}

int apc_dtrsm_rows(apc_ctx* ctx, int64_t k, const double* T, double* X, int64_t ncols, int transpose) {
  return guard(ctx, [&] {
    require(k >= 0 && ncols >= 0, APC_INVALID_ARGUMENT, "apc_dtrsm_rows: negative shape");
    dtrsm_rows_dev(ctx, k, T, X, ncols, transpose != 0);
    APC_CUDA(cudaStreamSynchronize(ctx->stream));
  });
}

int apc_op_apply_dev(apc_mat* a, double mu, int augmented, int transpose, const double* x, double* y) {
  return guard(a->ctx, [&] {
    require(!augmented || mu >= 0.0, APC_INVALID_ARGUMENT, "AugmentedOperator: mu < 0");
    if (!transpose) op_fwd(*a, mu, augmented != 0, x, y);
    else op_adj(*a, mu, augmented != 0, x, y);
  });
}

int apc_op_pair_dev(apc_mat* a, const double* x, double* y, double* g, int* fused) {
  return guard(a->ctx, [&] {
    const bool f = dense_pair_ready(*a);
    if (fused) *fused = f ? 1 : 0;
    if (f) {
      launch_dense_pair(*a, x, y, nullptr, g, nullptr);
    } else {
      op_fwd(*a, 0.0, false, x, y);
      op_adj(*a, 0.0, false, y, g);
      pair_norm2(a->ctx, y, a->mloc(), g + a->n);
    }
  });
}

int apc_op_apply_host(apc_mat* a, double mu, int augmented, int transpose, const double* x, double* y) {
  return guard(a->ctx, [&] {
    require(!augmented || mu >= 0.0, APC_INVALID_ARGUMENT, "AugmentedOperator: mu < 0");
    const i64 tail = augmented ? a->n : 0;
    const i64 xin = transpose ? a->mloc() + tail : a->n;
    const i64 yout = transpose ? a->n : a->mloc() + tail;
    DBuf<double> dx(std::max<i64>(1, xin)), dy(std::max<i64>(1, yout));
    cudaStream_t st = a->ctx->stream;
    if (xin > 0) APC_CUDA(cudaMemcpyAsync(dx.p, x, sizeof(double) * xin, cudaMemcpyHostToDevice, st));
    if (!transpose) op_fwd(*a, mu, augmented != 0, dx.p, dy.p);
    else op_adj(*a, mu, augmented != 0, dx.p, dy.p);
    if (yout > 0) APC_CUDA(cudaMemcpyAsync(y, dy.p, sizeof(double) * yout, cudaMemcpyDeviceToHost, st));
    APC_CUDA(cudaStreamSynchronize(st));
  });
}

int apc_partition_rows(int64_t m, const int64_t* row_nnz, int nranks, int64_t* bounds) {
  return guard(nullptr, [&] {
    require(nranks >= 1 && m >= 0, APC_INVALID_ARGUMENT, "apc_partition_rows: bad arguments");
    bounds[0] = 0;
    if (!row_nnz) {
      for (int p = 1; p <= nranks; ++p) bounds[p] = (m * p) / nranks;
      return;
    }
    i64 total = 0;
    for (i64 i = 0; i < m; ++i) total += row_nnz[i];
    // boundary p: first row whose prefix (inclusive of earlier rows) reaches p/nranks of nnz
    i64 acc = 0, row = 0;
    for (int p = 1; p < nranks; ++p) {
      const long double target = static_cast<long double>(total) * p / nranks;
      while (row < m && static_cast<long double>(acc) + row_nnz[row] / 2.0L < target) acc += row_nnz[row++];
      bounds[p] = std::max<i64>(row, bounds[p - 1]);
    }
    bounds[nranks] = m;
  });
}

int apc_rng_fill(uint64_t seed, int stream, uint64_t index, int kind, uint64_t bound, int64_t count,
                 void* out) {
  return guard(nullptr, [&] {
    HostRng r = stream < 0 ? HostRng(seed) : HostRng(seed, static_cast<Stream>(stream), index);
    for (int64_t i = 0; i < count; ++i) {
      switch (kind) {
        case 0: static_cast<uint64_t*>(out)[i] = r.bits(); break;
        case 1: static_cast<double*>(out)[i] = r.uniform(); break;
        case 2: static_cast<double*>(out)[i] = r.gaussian(); break;
        case 3: static_cast<uint64_t*>(out)[i] = r.below(bound); break;
        default: static_cast<double*>(out)[i] = r.sign(); break;
      }
    }
  });
}

uint64_t apc_mix64(uint64_t x) { return splitmix(x); }

int apc_rng_fill_device(apc_ctx* ctx, uint64_t seed, int stream, uint64_t index, int64_t count, uint64_t* out) {
  return guard(ctx, [&] {
    require(ctx && (out || count == 0) && count >= 0, APC_INVALID_ARGUMENT, "apc_rng_fill_device: bad arguments");
    require(mt64_device_ok(), APC_CUDA_ERROR, "apc_rng_fill_device: engine replica does not match the host library");
    // HostRng's engine seed (host_rng.hpp): splitmix(seed) or the stream derivation
    const std::uint64_t es = stream < 0 ? splitmix(seed)
                                        : splitmix(splitmix(seed ^ (0x51ed2701a3c5e1bdULL * static_cast<std::uint64_t>(stream))) + index);
    DBuf<std::uint64_t> d(std::max<int64_t>(1, count));
    mt64_stream_device(ctx, es, count, d.p);
    copy_sync(ctx->stream, out, d.p, sizeof(std::uint64_t) * count, cudaMemcpyDeviceToHost);
  });
}

int apc_problem_generate(int config, int64_t m, int64_t n, uint64_t seed, apc_problem** out) {
  *out = nullptr;
  return guard(nullptr, [&] { *out = generate_problem(config, m, n, seed); });
}

int apc_config_default(apc_solver_config* c) {
  std::memset(c, 0, sizeof(*c));
  c->block = 0;
  c->eps_cur = -1.0;
  c->eps_lsqr = 1e-10;
  c->nu_prec = 10.0;
  c->nu_lsqr = 100.0;
  c->mu = 0.0;
  c->variant = 0;
  c->core = 0;
  c->sketch_xi = 8;
  c->probe_count = 10;
  c->lsqr_cap = 0;
  c->max_rank = 0;
  c->seed = 0;
  c->trace_sample_stride = 1;
  c->outer_cap = 100000;
  c->sketch_kind = 0;
  return APC_OK;
}

int apc_solve(apc_mat* a, const double* b, const apc_solver_config* cfg, int plain, apc_result** out) {
  *out = nullptr;
  return guard(a->ctx, [&] {
    APC_CUDA(cudaSetDevice(a->ctx->device));
    *out = plain ? plain_solve(*a, b, *cfg) : aplicur_solve(*a, b, *cfg);
  });
}

int apc_solve_sharded(apc_mat* full, apc_mat* shard, const double* b, const apc_solver_config* cfg, int plain,
                      apc_result** out) {
  *out = nullptr;
  return guard(shard->ctx, [&] {
    APC_CUDA(cudaSetDevice(shard->ctx->device));
    if (plain) *out = plain_solve(*shard, b, *cfg);
    else {
      // rank 0 with `full`: root-only setup; NULL on rank 0: the sharded setup
      *out = aplicur_solve_sharded(full && shard->ctx->rank == 0 ? *full : *shard, *shard, b, *cfg);
    }
  });
}

int apc_solve_hooked(apc_mat* full, apc_mat* a, const double* b, const apc_solver_config* cfg,
                     const apc_hooks* hooks, apc_result** out) {
  *out = nullptr;
  return guard(a->ctx, [&] {
    APC_CUDA(cudaSetDevice(a->ctx->device));
    *out = aplicur_solve_sharded(full ? *full : *a, *a, b, *cfg, hooks);
  });
}

int apc_result_free(apc_result* r) {
  delete r;
  return APC_OK;
}

int apc_result_summary(const apc_result* r, int* status, double* final_rho, double* final_relres,
                       uint64_t* sketch_applications, uint64_t* system_matvecs, int64_t* n_phases,
                       int64_t* n_trace, int64_t* rank, int64_t* n_rho) {
  if (status) *status = r->status;
  if (final_rho) *final_rho = r->final_rho;
  if (final_relres) *final_relres = r->final_relres;
  if (sketch_applications) *sketch_applications = r->sketch_applications;
  if (system_matvecs) *system_matvecs = r->system_matvecs;
  if (n_phases) *n_phases = static_cast<int64_t>(r->phases.size());
  if (n_trace) *n_trace = static_cast<int64_t>(r->trace.size());
  if (rank) *rank = static_cast<int64_t>(r->rows.size());
  if (n_rho) *n_rho = static_cast<int64_t>(r->rho_history.size());
  return APC_OK;
}

int apc_result_x(const apc_result* r, double* x) {
  std::copy(r->x.begin(), r->x.end(), x);
  return APC_OK;
}

int apc_result_indices(const apc_result* r, int64_t* rows, int64_t* cols) {
  std::copy(r->rows.begin(), r->rows.end(), rows);
  std::copy(r->cols.begin(), r->cols.end(), cols);
  return APC_OK;
}

int apc_result_rho_history(const apc_result* r, double* rho) {
  std::copy(r->rho_history.begin(), r->rho_history.end(), rho);
  return APC_OK;
}

int apc_result_phases(const apc_result* r, apc_phase_report* phases) {
  std::copy(r->phases.begin(), r->phases.end(), phases);
  return APC_OK;
}

int apc_result_phase_spectrum(const apc_result* r, int64_t k, double* out, int64_t* n) {
  if (!r || !n || k < 0 || k >= static_cast<int64_t>(r->phases.size())) return APC_INVALID_ARGUMENT;
  static const std::vector<double> none;
  const auto& s = k < static_cast<int64_t>(r->spectra.size()) ? r->spectra[static_cast<size_t>(k)] : none;
  *n = static_cast<int64_t>(s.size());
  if (out) std::copy(s.begin(), s.end(), out);
  return APC_OK;
}

int apc_result_trace(const apc_result* r, apc_trace_row* rows) {
  std::copy(r->trace.begin(), r->trace.end(), rows);
  return APC_OK;
}

int apc_result_timing(const apc_result* r, double* total_ms, double* lsqr_ms, double* setup_ms) {
  if (total_ms) *total_ms = r->total_ms;
  if (lsqr_ms) *lsqr_ms = r->lsqr_ms;
  if (setup_ms) *setup_ms = r->setup_ms;
  return APC_OK;
}

int apc_problem_info(const apc_problem* p, int64_t* m, int64_t* n, int* sparse, int64_t* nnz);
const double* apc_problem_dense(const apc_problem* p);
int apc_problem_csc(const apc_problem* p, const int64_t** colptr, const int64_t** rowidx, const double** vals);
const double* apc_problem_b(const apc_problem* p);
int apc_problem_free(apc_problem* p);

}  // extern "C"
