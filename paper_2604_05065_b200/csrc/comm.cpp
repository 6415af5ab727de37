// Inter-GPU reduction for the row-partitioned solve: one
// allreduce(sum, fp64) of [A_p^T u_p (n) | ||u_p||^2 (1)] per LSQR iteration
// plus the residual norms.  Two backends behind one seam:
//  * NCCL (one process per GPU, unique id over torch.distributed): enqueued on
//    the ctx stream, so it is captured in the iteration graphs;
//  * host-staged (apc_ctx_create_host_comm): device -> pinned host buffer, the
//    caller's callback sums it over the ranks in rank order (every rank gets
//    the same bits), host -> device.  It synchronises the stream, so the LSQR
//    phase runs its kernels eagerly instead of from a graph.  It lets several
//    ranks share one GPU (tests) or use any host transport.
#include <nccl.h>

#include <cstdint>
#include <cstring>
#include <string>
#include <vector>

#include "lsqr.hpp"

namespace apc {

namespace {
void nccl_check(ncclResult_t r, const char* what) {
  if (r != ncclSuccess)
    fail(APC_NCCL_ERROR, std::string(what) + ": " + ncclGetErrorString(r));
}
}  // namespace

void comm_init(apc_ctx* ctx, const void* uid) {
  if (ctx->nranks <= 1 || ctx->host_allreduce) return;
  require(uid != nullptr, APC_INVALID_ARGUMENT, "apc_ctx_create: nccl unique id required for nranks > 1");
  ncclUniqueId id;
  static_assert(sizeof(id) == 128, "ncclUniqueId size");
  std::memcpy(&id, uid, sizeof(id));
  ncclComm_t comm;
  nccl_check(ncclCommInitRank(&comm, ctx->nranks, id, ctx->rank), "ncclCommInitRank");
  ctx->nccl = comm;
}

void comm_destroy(apc_ctx* ctx) {
  if (ctx->nccl) ncclCommDestroy(static_cast<ncclComm_t>(ctx->nccl));
  ctx->nccl = nullptr;
}

bool comm_graph_safe(const apc_ctx* ctx) { return ctx->host_allreduce == nullptr; }

void comm_allreduce(apc_ctx* ctx, double* buf, i64 count) {
  if (ctx->nranks <= 1 || count <= 0) return;
  if (ctx->host_allreduce) {
    auto* h = static_cast<double*>(ctx_pinned(ctx, 3, sizeof(double) * static_cast<size_t>(count)));
    APC_CUDA(cudaMemcpyAsync(h, buf, sizeof(double) * count, cudaMemcpyDeviceToHost, ctx->stream));
    APC_CUDA(cudaStreamSynchronize(ctx->stream));
    const int rc = ctx->host_allreduce(h, static_cast<int64_t>(count), ctx->host_user);
    require(rc == 0, APC_NCCL_ERROR, "host-staged allreduce callback failed");
    APC_CUDA(cudaMemcpyAsync(buf, h, sizeof(double) * count, cudaMemcpyHostToDevice, ctx->stream));
    APC_CUDA(cudaStreamSynchronize(ctx->stream));
    return;
  }
  nccl_check(ncclAllReduce(buf, buf, static_cast<size_t>(count), ncclDouble, ncclSum,
                           static_cast<ncclComm_t>(ctx->nccl), ctx->stream),
             "ncclAllReduce");
}

namespace {
// The host-staged backend only sums.  A sum with zeros off the owning rank
// returns the owner's value for every double but -0.0 (-0.0 + 0.0 = +0.0) and
// NaN payloads, so broadcasts and gathers travel as two exact integers per
// double (the 32-bit halves of its bit pattern, each < 2^32): the sum of one
// nonzero contribution and zeros is exact, the decoded bits are the owner's.
void host_encode(const double* v, i64 n, double* out) {
  for (i64 i = 0; i < n; ++i) {
    std::uint64_t b;
    std::memcpy(&b, v + i, 8);
    out[2 * i] = static_cast<double>(b >> 32);
    out[2 * i + 1] = static_cast<double>(b & 0xffffffffull);
  }
}
void host_decode(const double* in, i64 n, double* v) {
  for (i64 i = 0; i < n; ++i) {
    const std::uint64_t b = (static_cast<std::uint64_t>(in[2 * i]) << 32) | static_cast<std::uint64_t>(in[2 * i + 1]);
    std::memcpy(v + i, &b, 8);
  }
}
// out (nranks x count, rank-major on the host) = every rank's `mine` (or only
// root's when root >= 0, the other slots left zero), exactly
void host_exchange(apc_ctx* ctx, const double* mine_dev, i64 count, int root, std::vector<double>& out) {
  const int P = ctx->nranks;
  std::vector<double> mine(static_cast<size_t>(count)), enc(static_cast<size_t>(2 * count * P), 0.0);
  if (root < 0 || ctx->rank == root) {
    copy_sync(ctx->stream, mine.data(), mine_dev, sizeof(double) * count, cudaMemcpyDeviceToHost);
    host_encode(mine.data(), count, enc.data() + 2 * count * ctx->rank);
  }
  const int rc = ctx->host_allreduce(enc.data(), static_cast<int64_t>(enc.size()), ctx->host_user);
  require(rc == 0, APC_NCCL_ERROR, "host-staged collective callback failed");
  out.assign(static_cast<size_t>(count * P), 0.0);
  for (int p = 0; p < P; ++p) host_decode(enc.data() + 2 * count * p, count, out.data() + count * p);
}
}  // namespace

void comm_bcast(apc_ctx* ctx, double* buf, i64 count, int root) {
  if (ctx->nranks <= 1 || count <= 0) return;
  if (ctx->host_allreduce) {
    std::vector<double> all;
    host_exchange(ctx, buf, count, root, all);
    APC_CUDA(cudaMemcpyAsync(buf, all.data() + count * root, sizeof(double) * count, cudaMemcpyHostToDevice,
                             ctx->stream));
    APC_CUDA(cudaStreamSynchronize(ctx->stream));
    return;
  }
  nccl_check(ncclBroadcast(buf, buf, static_cast<size_t>(count), ncclDouble, root, static_cast<ncclComm_t>(ctx->nccl),
                           ctx->stream),
             "ncclBroadcast");
}

// recv (nranks x count, rank-major) = every rank's send (count doubles), bit-exact
void comm_allgather(apc_ctx* ctx, const double* send, i64 count, double* recv) {
  if (count <= 0) return;
  if (ctx->nranks <= 1) {
    if (recv != send)
      APC_CUDA(cudaMemcpyAsync(recv, send, sizeof(double) * count, cudaMemcpyDeviceToDevice, ctx->stream));
    return;
  }
  if (ctx->host_allreduce) {
    std::vector<double> all;
    host_exchange(ctx, send, count, -1, all);
    APC_CUDA(cudaMemcpyAsync(recv, all.data(), sizeof(double) * all.size(), cudaMemcpyHostToDevice, ctx->stream));
    APC_CUDA(cudaStreamSynchronize(ctx->stream));
    return;
  }
  nccl_check(ncclAllGather(send, recv, static_cast<size_t>(count), ncclDouble, static_cast<ncclComm_t>(ctx->nccl),
                           ctx->stream),
             "ncclAllGather");
}

}  // namespace apc

extern "C" int apc_nccl_unique_id(void* out128) {
  ncclUniqueId id;
  if (ncclGetUniqueId(&id) != ncclSuccess) return APC_NCCL_ERROR;
  std::memcpy(out128, &id, sizeof(id));
  return APC_OK;
}
