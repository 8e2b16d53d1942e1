/* A stand-in libnccl for PER-RANK TIMING on one GPU (tools/rank_emulation.py; not part of
 * the product).  libmdd resolves NCCL with dlopen at run time (MDD_NCCL_LIB selects the
 * file), so this library can take its place: rank r of N runs alone, and every collective
 * does only its local part -- allreduce and send are no-ops, recv zero-fills, allgather
 * places the caller's block.  The numbers such a run computes are NOT the solve's; what it
 * measures is the device time of one rank's share of the work, with the exchanges costed
 * separately from their byte counts. */
#include <cuda_runtime.h>
#include <stdlib.h>
#include <string.h>

typedef struct { int nranks, rank; } stub_comm;
typedef struct { char internal[128]; } ncclUniqueId;
typedef int ncclResult_t;
typedef int ncclDataType_t;
typedef int ncclRedOp_t;
typedef stub_comm* ncclComm_t;

static size_t type_bytes(ncclDataType_t t) { return t == 8 ? 8 : (t == 7 ? 4 : 8); } /* ncclFloat64 = 8 */

ncclResult_t ncclGetUniqueId(ncclUniqueId* id) { memset(id, 7, sizeof *id); return 0; }
ncclResult_t ncclCommInitRank(ncclComm_t* c, int n, ncclUniqueId id, int rank) {
  (void)id;
  *c = (stub_comm*)malloc(sizeof(stub_comm));
  (*c)->nranks = n;
  (*c)->rank = rank;
  return 0;
}
ncclResult_t ncclCommDestroy(ncclComm_t c) { free(c); return 0; }
const char* ncclGetErrorString(ncclResult_t r) { (void)r; return "stub"; }
ncclResult_t ncclGroupStart(void) { return 0; }
ncclResult_t ncclGroupEnd(void) { return 0; }
ncclResult_t ncclAllReduce(const void* s, void* r, size_t n, ncclDataType_t t, ncclRedOp_t op, ncclComm_t c,
                           cudaStream_t st) {
  (void)op; (void)c;
  if (s != r) cudaMemcpyAsync(r, s, n * type_bytes(t), cudaMemcpyDeviceToDevice, st);
  return 0;
}
ncclResult_t ncclAllGather(const void* s, void* r, size_t n, ncclDataType_t t, ncclComm_t c, cudaStream_t st) {
  char* dst = (char*)r + (size_t)c->rank * n * type_bytes(t);
  if (s != (void*)dst) cudaMemcpyAsync(dst, s, n * type_bytes(t), cudaMemcpyDeviceToDevice, st);
  return 0;
}
ncclResult_t ncclSend(const void* s, size_t n, ncclDataType_t t, int peer, ncclComm_t c, cudaStream_t st) {
  (void)s; (void)n; (void)t; (void)peer; (void)c; (void)st;
  return 0;
}
ncclResult_t ncclRecv(void* r, size_t n, ncclDataType_t t, int peer, ncclComm_t c, cudaStream_t st) {
  (void)peer; (void)c;
  cudaMemsetAsync(r, 0, n * type_bytes(t), st);
  return 0;
}
