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

#include <cstring>
#include <string>

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

void comm_bcast(apc_ctx* ctx, double* buf, i64 count, int root) {
  if (ctx->nranks <= 1 || count <= 0) return;
  if (ctx->host_allreduce) {  // a sum with zeros everywhere but the root: the root's values, exactly
    if (ctx->rank != root) APC_CUDA(cudaMemsetAsync(buf, 0, sizeof(double) * count, ctx->stream));
    comm_allreduce(ctx, buf, count);
    return;
  }
  nccl_check(ncclBroadcast(buf, buf, static_cast<size_t>(count), ncclDouble, root, static_cast<ncclComm_t>(ctx->nccl),
                           ctx->stream),
             "ncclBroadcast");
}

}  // namespace apc

extern "C" int apc_nccl_unique_id(void* out128) {
  ncclUniqueId id;
  if (ncclGetUniqueId(&id) != ncclSuccess) return APC_NCCL_ERROR;
  std::memcpy(out128, &id, sizeof(id));
  return APC_OK;
}
