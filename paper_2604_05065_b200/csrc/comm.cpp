// Inter-GPU reduction for the row-partitioned solve: one
// ncclAllReduce(sum, fp64) of [A_p^T u_p (n) | ||u_p||^2 (1)] per LSQR
// iteration, enqueued on the ctx stream so it is captured in the iteration
// graph.  One process per GPU; the unique id travels over torch.distributed.
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
  if (ctx->nranks <= 1) return;
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

void comm_allreduce(apc_ctx* ctx, double* buf, i64 count) {
  if (ctx->nranks <= 1 || count <= 0) return;
  nccl_check(ncclAllReduce(buf, buf, static_cast<size_t>(count), ncclDouble, ncclSum,
                           static_cast<ncclComm_t>(ctx->nccl), ctx->stream),
             "ncclAllReduce");
}

}  // namespace apc

extern "C" int apc_nccl_unique_id(void* out128) {
  ncclUniqueId id;
  if (ncclGetUniqueId(&id) != ncclSuccess) return APC_NCCL_ERROR;
  std::memcpy(out128, &id, sizeof(id));
  return APC_OK;
}
