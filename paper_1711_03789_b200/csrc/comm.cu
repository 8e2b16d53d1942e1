// Multi-GPU plumbing: an NCCL communicator resolved at run time (dlopen), so
// libmdd.so loads and runs single-GPU without NCCL.
//
// Sharding: each rank factorises and solves only its block of
// subdomains (the small coarse space is replicated); the one-level output is
// a partial sum that one in-place ncclAllReduce completes (mdd_prec_set_comm).
// GMRES either replicates the Krylov vectors (MGS, no further collective) or
// shards them by contiguous row blocks (CGS2, gmres.cu): an allgather of the
// new basis vector feeds the preconditioner and the row-block SpMV, and three
// small allreduces per iteration complete the Gram-Schmidt coefficients and
// the norm.
#include <dlfcn.h>
#include <nccl.h>

#include <cstdlib>
#include <cstring>
#include <mutex>

#include "mdd_internal.h"

namespace mdd {

namespace {
struct NcclApi {
  void* h = nullptr;
  ncclResult_t (*getUniqueId)(ncclUniqueId*) = nullptr;
  ncclResult_t (*commInitRank)(ncclComm_t*, int, ncclUniqueId, int) = nullptr;
  ncclResult_t (*allReduce)(const void*, void*, size_t, ncclDataType_t, ncclRedOp_t, ncclComm_t,
                            cudaStream_t) = nullptr;
  ncclResult_t (*allGather)(const void*, void*, size_t, ncclDataType_t, ncclComm_t, cudaStream_t) = nullptr;
  ncclResult_t (*commDestroy)(ncclComm_t) = nullptr;
  const char* (*getErrorString)(ncclResult_t) = nullptr;
};

NcclApi& nccl() {
  static NcclApi api;
  static std::once_flag once;
  std::call_once(once, [] {
    const char* names[] = {"libnccl.so.2", "libnccl.so"};
    for (const char* n : names) {
      api.h = dlopen(n, RTLD_NOW | RTLD_GLOBAL);
      if (api.h) break;
    }
    if (!api.h) return;
    api.getUniqueId = reinterpret_cast<decltype(api.getUniqueId)>(dlsym(api.h, "ncclGetUniqueId"));
    api.commInitRank = reinterpret_cast<decltype(api.commInitRank)>(dlsym(api.h, "ncclCommInitRank"));
    api.allReduce = reinterpret_cast<decltype(api.allReduce)>(dlsym(api.h, "ncclAllReduce"));
    api.allGather = reinterpret_cast<decltype(api.allGather)>(dlsym(api.h, "ncclAllGather"));
    api.commDestroy = reinterpret_cast<decltype(api.commDestroy)>(dlsym(api.h, "ncclCommDestroy"));
    api.getErrorString =
        reinterpret_cast<decltype(api.getErrorString)>(dlsym(api.h, "ncclGetErrorString"));
  });
  if (!api.h || !api.getUniqueId || !api.commInitRank || !api.allReduce || !api.allGather || !api.commDestroy)
    fail(MDD_ENCCL, "NCCL (libnccl.so.2) is not available");
  return api;
}

void nccl_check(ncclResult_t r, const char* what) {
  if (r != ncclSuccess) {
    NcclApi& a = nccl();
    fail(MDD_ENCCL, std::string("NCCL error in ") + what + ": " +
                        (a.getErrorString ? a.getErrorString(r) : "unknown"));
  }
}
}  // namespace

}  // namespace mdd

namespace mdd {
void comm_allreduce_z(mdd_comm* c, double2* buf, int64_t n, cudaStream_t s) {
  if (!c || !c->comm) return;
  nccl_check(nccl().allReduce(buf, buf, (size_t)(2 * n), ncclFloat64, ncclSum,
                              static_cast<ncclComm_t>(c->comm), s),
             "ncclAllReduce");
}
void comm_allgather_z(mdd_comm* c, const double2* send, double2* recv, int64_t per_rank, cudaStream_t s) {
  if (!c || !c->comm) {
    double2* dst = recv + (c && c->emulated ? (int64_t)c->rank * per_rank : 0);
    if (send != dst) CK(cudaMemcpyAsync(dst, send, sizeof(double2) * per_rank, cudaMemcpyDeviceToDevice, s));
    return;
  }
  nccl_check(nccl().allGather(send, recv, (size_t)(2 * per_rank), ncclFloat64, static_cast<ncclComm_t>(c->comm), s),
             "ncclAllGather");
}
}  // namespace mdd

using namespace mdd;

extern "C" {

int mdd_comm_unique_id(char* out128) {
  MDD_API_BEGIN
  ncclUniqueId id;
  nccl_check(nccl().getUniqueId(&id), "ncclGetUniqueId");
  memcpy(out128, id.internal, NCCL_UNIQUE_ID_BYTES);
  MDD_API_END
}

int mdd_comm_create(mdd_ctx* ctx, int nranks, int rank, const char* id128, mdd_comm** out) {
  MDD_API_BEGIN
  if (nranks < 1 || rank < 0 || rank >= nranks) fail(MDD_EINVAL, "comm: bad rank/size");
  CK(cudaSetDevice(ctx->device));
  // id128 == NULL: a single-rank communicator without NCCL (all collectives
  // are identities); with an id, NCCL is initialised even for one rank
  const char* emu = getenv("MDD_COMM_EMULATE");
  const bool emulate = nranks > 1 && !id128 && emu && atoi(emu) != 0;
  if (nranks > 1 && !id128 && !emulate) fail(MDD_EINVAL, "comm: a unique id is required for more than one rank");
  std::unique_ptr<mdd_comm> c(new mdd_comm());
  c->ctx = ctx;
  c->nranks = nranks;
  c->rank = rank;
  c->emulated = emulate;
  if (id128) {
    ncclUniqueId id;
    memcpy(id.internal, id128, NCCL_UNIQUE_ID_BYTES);
    ncclComm_t nc = nullptr;
    nccl_check(nccl().commInitRank(&nc, nranks, id, rank), "ncclCommInitRank");
    c->comm = nc;
  }
  *out = c.release();
  MDD_API_END
}

void mdd_comm_destroy(mdd_comm* c) {
  if (!c) return;
  if (c->comm) nccl().commDestroy(static_cast<ncclComm_t>(c->comm));
  delete c;
}

int mdd_comm_info(const mdd_comm* c, int* nranks, int* rank) {
  MDD_API_BEGIN
  *nranks = c->nranks;
  *rank = c->rank;
  MDD_API_END
}

}  // extern "C"
