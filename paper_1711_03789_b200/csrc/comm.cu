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

#include <chrono>
#include <condition_variable>
#include <cstdlib>
#include <cstring>
#include <mutex>

#include "mdd_internal.h"
#include "mdd_kernels.cuh"

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
  ncclResult_t (*send)(const void*, size_t, ncclDataType_t, int, ncclComm_t, cudaStream_t) = nullptr;
  ncclResult_t (*recv)(void*, size_t, ncclDataType_t, int, ncclComm_t, cudaStream_t) = nullptr;
  ncclResult_t (*groupStart)() = nullptr;
  ncclResult_t (*groupEnd)() = nullptr;
  const char* (*getErrorString)(ncclResult_t) = nullptr;
};

NcclApi& nccl() {
  static NcclApi api;
  static std::once_flag once;
  std::call_once(once, [] {
    // MDD_NCCL_LIB: the NCCL library file to load (a system build instead of a bundled one;
    // tools/rank_emulation.py points it at its timing stand-in)
    const char* names[] = {getenv("MDD_NCCL_LIB"), "libnccl.so.2", "libnccl.so"};
    for (const char* n : names) {
      if (!n || !*n) continue;
      api.h = dlopen(n, RTLD_NOW | RTLD_LOCAL);
      if (api.h) break;
    }
    if (!api.h) return;
    api.getUniqueId = reinterpret_cast<decltype(api.getUniqueId)>(dlsym(api.h, "ncclGetUniqueId"));
    api.commInitRank = reinterpret_cast<decltype(api.commInitRank)>(dlsym(api.h, "ncclCommInitRank"));
    api.allReduce = reinterpret_cast<decltype(api.allReduce)>(dlsym(api.h, "ncclAllReduce"));
    api.allGather = reinterpret_cast<decltype(api.allGather)>(dlsym(api.h, "ncclAllGather"));
    api.commDestroy = reinterpret_cast<decltype(api.commDestroy)>(dlsym(api.h, "ncclCommDestroy"));
    api.send = reinterpret_cast<decltype(api.send)>(dlsym(api.h, "ncclSend"));
    api.recv = reinterpret_cast<decltype(api.recv)>(dlsym(api.h, "ncclRecv"));
    api.groupStart = reinterpret_cast<decltype(api.groupStart)>(dlsym(api.h, "ncclGroupStart"));
    api.groupEnd = reinterpret_cast<decltype(api.groupEnd)>(dlsym(api.h, "ncclGroupEnd"));
    api.getErrorString =
        reinterpret_cast<decltype(api.getErrorString)>(dlsym(api.h, "ncclGetErrorString"));
  });
  if (!api.h || !api.getUniqueId || !api.commInitRank || !api.allReduce || !api.allGather || !api.commDestroy ||
      !api.send || !api.recv || !api.groupStart || !api.groupEnd)
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
namespace {
// Loopback group: host barrier + device copies between the ranks' buffers.
constexpr int kLoopMax = 8;
struct LoopGroup {
  int n = 0;
  std::mutex mu;
  std::condition_variable cv;
  int arrived = 0;
  uint64_t gen = 0;
  bool aborted = false;  // a rank failed: every waiter (now and later) fails fast
  const double2* bufs[kLoopMax] = {};
  int64_t count[kLoopMax] = {};  // per-rank element count of the current collective
  int kind[kLoopMax] = {};       // 1 allreduce, 2 allgather: every rank must be in the same collective
};
void loop_check(LoopGroup* g, int rank) {
  for (int k = 0; k < g->n; ++k)
    if (g->kind[k] != g->kind[rank] || g->count[k] != g->count[rank] || !g->bufs[k])
      fail(MDD_ENCCL, "loopback group: ranks " + std::to_string(rank) + " and " + std::to_string(k) +
                          " are in different collectives (kind " + std::to_string(g->kind[rank]) + "/" +
                          std::to_string(g->kind[k]) + ", count " + std::to_string(g->count[rank]) + "/" +
                          std::to_string(g->count[k]) + ")");
}
void loop_abort(LoopGroup* g) {
  std::lock_guard<std::mutex> l(g->mu);
  g->aborted = true;
  g->cv.notify_all();
}
void loop_barrier(LoopGroup* g) {
  std::unique_lock<std::mutex> l(g->mu);
  if (g->aborted) fail(MDD_ENCCL, "loopback group: another rank failed");
  const uint64_t my = g->gen;
  if (++g->arrived == g->n) {
    g->arrived = 0;
    ++g->gen;
    g->cv.notify_all();
  } else {
    const bool ok = g->cv.wait_for(l, std::chrono::seconds(300), [&] { return g->gen != my || g->aborted; });
    if (g->aborted) fail(MDD_ENCCL, "loopback group: another rank failed");
    if (!ok) {
      g->aborted = true;
      g->cv.notify_all();
      fail(MDD_ENCCL, "loopback group: a rank did not reach the collective within 300 s");
    }
  }
}
struct RankPtrs {
  const double2* p[kLoopMax];
};
__global__ void k_sum_ranks(RankPtrs r, int nr, int64_t n, double2* out) {
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
    double2 a = r.p[0][i];
    for (int k = 1; k < nr; ++k) a = cadd(a, r.p[k][i]);
    out[i] = a;
  }
}
void loop_allreduce(mdd_comm* c, double2* buf, int64_t n, cudaStream_t s) {
  auto* g = static_cast<LoopGroup*>(c->loop);
  CK(cudaStreamSynchronize(s));
  g->bufs[c->rank] = buf;
  g->count[c->rank] = n;
  g->kind[c->rank] = 1;
  loop_barrier(g);  // every rank's partial is final
  loop_check(g, c->rank);
  DevBuf<double2> tmp(n);
  RankPtrs rp{};
  for (int k = 0; k < g->n; ++k) rp.p[k] = g->bufs[k];
  const unsigned grid = (unsigned)std::max<int64_t>(1, std::min<int64_t>((n + 255) / 256, 4096));
  k_sum_ranks<<<grid, 256, 0, s>>>(rp, g->n, n, tmp.p);
  CK(cudaGetLastError());
  CK(cudaStreamSynchronize(s));
  loop_barrier(g);  // nobody reads the partials any more
  CK(cudaMemcpyAsync(buf, tmp.p, sizeof(double2) * n, cudaMemcpyDeviceToDevice, s));
  CK(cudaStreamSynchronize(s));
}
void loop_allgather(mdd_comm* c, const double2* send, double2* recv, int64_t per_rank, cudaStream_t s) {
  auto* g = static_cast<LoopGroup*>(c->loop);
  CK(cudaStreamSynchronize(s));
  g->bufs[c->rank] = send;
  g->count[c->rank] = per_rank;
  g->kind[c->rank] = 2;
  loop_barrier(g);
  loop_check(g, c->rank);
  for (int k = 0; k < g->n; ++k)
    CK(cudaMemcpyAsync(recv + (int64_t)k * per_rank, g->bufs[k], sizeof(double2) * per_rank,
                       cudaMemcpyDeviceToDevice, s));
  CK(cudaStreamSynchronize(s));
  loop_barrier(g);  // the send buffers may change again
}
// y[i] += x[i]
__global__ void k_add_into(int64_t n, const double2* __restrict__ x, double2* __restrict__ y) {
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
    y[i] = cadd(y[i], x[i]);
}
unsigned add_grid(int64_t n) { return (unsigned)std::max<int64_t>(1, std::min<int64_t>((n + 255) / 256, 4096)); }

void loop_halo_gather(mdd_comm* c, mdd_halo* h, double2* vec, cudaStream_t s) {
  auto* g = static_cast<LoopGroup*>(c->loop);
  CK(cudaStreamSynchronize(s));
  g->bufs[c->rank] = vec;
  g->count[c->rank] = h->n;
  g->kind[c->rank] = 3;
  loop_barrier(g);  // every rank's owned rows are final
  loop_check(g, c->rank);
  const int me = c->rank;
  for (int q = 0; q < g->n; ++q) {
    if (q == me) continue;
    const int64_t a = std::max(h->own_lo[q], h->need_lo[me]), b = std::min(h->own_hi[q], h->need_hi[me]);
    if (b > a)
      CK(cudaMemcpyAsync(vec + a, g->bufs[q] + a, sizeof(double2) * (b - a), cudaMemcpyDeviceToDevice, s));
  }
  CK(cudaStreamSynchronize(s));
  loop_barrier(g);  // the owned rows may change again
}
void loop_halo_reduce(mdd_comm* c, mdd_halo* h, double2* vec, cudaStream_t s) {
  auto* g = static_cast<LoopGroup*>(c->loop);
  CK(cudaStreamSynchronize(s));
  g->bufs[c->rank] = vec;
  g->count[c->rank] = h->n;
  g->kind[c->rank] = 4;
  loop_barrier(g);  // every rank's partial sums are final
  loop_check(g, c->rank);
  const int me = c->rank;
  const int64_t lo = h->own_lo[me], hi = h->own_hi[me];
  // ascending rank order, this rank's own partial in its place: the peers below me are summed
  // into the stage first, then my partial is added, then the peers above
  DevBuf<double2> acc(std::max<int64_t>(1, hi - lo));
  CK(cudaMemsetAsync(acc.p, 0, sizeof(double2) * std::max<int64_t>(1, hi - lo), s));
  for (int q = 0; q < g->n; ++q) {
    const int64_t a = std::max(lo, h->need_lo[q]), b = std::min(hi, h->need_hi[q]);
    if (b > a) {
      k_add_into<<<add_grid(b - a), 256, 0, s>>>(b - a, g->bufs[q] + a, acc.p + (a - lo));
      CK(cudaGetLastError());
    }
  }
  CK(cudaStreamSynchronize(s));
  loop_barrier(g);  // nobody reads the partials any more
  if (hi > lo) CK(cudaMemcpyAsync(vec + lo, acc.p, sizeof(double2) * (hi - lo), cudaMemcpyDeviceToDevice, s));
  CK(cudaStreamSynchronize(s));
}
}  // namespace

void comm_halo_setup(mdd_comm* c, mdd_halo* h, int64_t n, int64_t need_lo, int64_t need_hi, cudaStream_t s) {
  const int N = c ? c->nranks : 1, me = c ? c->rank : 0;
  const int64_t chunk = (n + N - 1) / N;
  h->n = n;
  h->own_lo.assign(N, 0);
  h->own_hi.assign(N, 0);
  for (int q = 0; q < N; ++q) {
    h->own_lo[q] = std::min<int64_t>(n, (int64_t)q * chunk);
    h->own_hi[q] = std::min<int64_t>(n, h->own_lo[q] + chunk);
  }
  need_lo = std::max<int64_t>(0, std::min(need_lo, h->own_lo[me]));
  need_hi = std::min<int64_t>(n, std::max(need_hi, h->own_hi[me]));
  // every rank learns every rank's needed range: one allgather of a (lo, hi) pair
  DevBuf<double2> mine(1), all(N);
  const double2 v = make_double2((double)need_lo, (double)need_hi);
  mine.upload(&v, 1, s);
  if (comm_active(c)) comm_allgather_z(c, mine.p, all.p, 1, s);
  else CK(cudaMemcpyAsync(all.p, mine.p, sizeof(double2), cudaMemcpyDeviceToDevice, s));
  std::vector<double2> hv(N);
  all.download(hv.data(), N, s);
  CK(cudaStreamSynchronize(s));
  h->need_lo.assign(N, 0);
  h->need_hi.assign(N, 0);
  int64_t stage = 0;
  for (int q = 0; q < N; ++q) {
    h->need_lo[q] = (int64_t)hv[q].x;
    h->need_hi[q] = (int64_t)hv[q].y;
    if (q != me)
      stage += std::max<int64_t>(0, std::min(h->own_hi[me], h->need_hi[q]) - std::max(h->own_lo[me], h->need_lo[q]));
  }
  h->stage = DevBuf<double2>(std::max<int64_t>(1, stage));
}

void comm_halo_gather(mdd_comm* c, mdd_halo* h, double2* vec, cudaStream_t s) {
  if (!comm_active(c)) return;
  if (c->loop) return loop_halo_gather(c, h, vec, s);
  NcclApi& a = nccl();
  const int me = c->rank;
  ncclComm_t nc = static_cast<ncclComm_t>(c->comm);
  nccl_check(a.groupStart(), "ncclGroupStart");
  for (int q = 0; q < c->nranks; ++q) {
    if (q == me) continue;
    // what q needs of mine; what I need of q's
    const int64_t sa = std::max(h->own_lo[me], h->need_lo[q]), sb = std::min(h->own_hi[me], h->need_hi[q]);
    const int64_t ra = std::max(h->own_lo[q], h->need_lo[me]), rb = std::min(h->own_hi[q], h->need_hi[me]);
    if (sb > sa) nccl_check(a.send(vec + sa, (size_t)(2 * (sb - sa)), ncclFloat64, q, nc, s), "ncclSend");
    if (rb > ra) nccl_check(a.recv(vec + ra, (size_t)(2 * (rb - ra)), ncclFloat64, q, nc, s), "ncclRecv");
  }
  nccl_check(a.groupEnd(), "ncclGroupEnd");
}

void comm_halo_reduce(mdd_comm* c, mdd_halo* h, double2* vec, cudaStream_t s) {
  if (!comm_active(c)) return;
  if (c->loop) return loop_halo_reduce(c, h, vec, s);
  NcclApi& a = nccl();
  const int me = c->rank;
  ncclComm_t nc = static_cast<ncclComm_t>(c->comm);
  const int64_t lo = h->own_lo[me], hi = h->own_hi[me];
  nccl_check(a.groupStart(), "ncclGroupStart");
  int64_t off = 0;
  for (int q = 0; q < c->nranks; ++q) {
    if (q == me) continue;
    // my partial sums on q's owned rows go to q; q's partial sums on my owned rows come here
    const int64_t sa = std::max(h->own_lo[q], h->need_lo[me]), sb = std::min(h->own_hi[q], h->need_hi[me]);
    const int64_t ra = std::max(lo, h->need_lo[q]), rb = std::min(hi, h->need_hi[q]);
    if (sb > sa) nccl_check(a.send(vec + sa, (size_t)(2 * (sb - sa)), ncclFloat64, q, nc, s), "ncclSend");
    if (rb > ra) {
      nccl_check(a.recv(h->stage.p + off, (size_t)(2 * (rb - ra)), ncclFloat64, q, nc, s), "ncclRecv");
      off += rb - ra;
    }
  }
  nccl_check(a.groupEnd(), "ncclGroupEnd");
  // owner adds, ascending rank order
  off = 0;
  for (int q = 0; q < c->nranks; ++q) {
    if (q == me) continue;
    const int64_t ra = std::max(lo, h->need_lo[q]), rb = std::min(hi, h->need_hi[q]);
    if (rb > ra) {
      k_add_into<<<add_grid(rb - ra), 256, 0, s>>>(rb - ra, h->stage.p + off, vec + ra);
      CK(cudaGetLastError());
      off += rb - ra;
    }
  }
}

void comm_allreduce_z(mdd_comm* c, double2* buf, int64_t n, cudaStream_t s) {
  if (c && c->loop) return loop_allreduce(c, buf, n, s);
  if (!c || !c->comm) return;
  nccl_check(nccl().allReduce(buf, buf, (size_t)(2 * n), ncclFloat64, ncclSum,
                              static_cast<ncclComm_t>(c->comm), s),
             "ncclAllReduce");
}
void comm_allgather_z(mdd_comm* c, const double2* send, double2* recv, int64_t per_rank, cudaStream_t s) {
  if (c && c->loop) return loop_allgather(c, send, recv, per_rank, s);
  if (!c || !c->comm) {
    if (send != recv) CK(cudaMemcpyAsync(recv, send, sizeof(double2) * per_rank, cudaMemcpyDeviceToDevice, s));
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
  if (nranks > 1 && !id128) fail(MDD_EINVAL, "comm: a unique id is required for more than one rank");
  std::unique_ptr<mdd_comm> c(new mdd_comm());
  c->ctx = ctx;
  c->nranks = nranks;
  c->rank = rank;
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

int mdd_comm_loopback_group(int nranks, void** group_out) {
  MDD_API_BEGIN
  if (nranks < 1 || nranks > kLoopMax) fail(MDD_EINVAL, "loopback group: 1..8 ranks");
  auto* g = new LoopGroup();
  g->n = nranks;
  *group_out = g;
  MDD_API_END
}

void mdd_comm_loopback_group_free(void* group) { delete static_cast<LoopGroup*>(group); }

int mdd_comm_create_loopback(mdd_ctx* ctx, void* group, int rank, mdd_comm** out) {
  MDD_API_BEGIN
  auto* g = static_cast<LoopGroup*>(group);
  if (!g || rank < 0 || rank >= g->n) fail(MDD_EINVAL, "loopback comm: bad group or rank");
  CK(cudaSetDevice(ctx->device));
  std::unique_ptr<mdd_comm> c(new mdd_comm());
  c->ctx = ctx;
  c->nranks = g->n;
  c->rank = rank;
  c->loop = g;
  *out = c.release();
  MDD_API_END
}

/* A rank that failed outside a collective (setup, a size check) tells the group, so the other
 * ranks' next or current barrier fails at once instead of waiting out the 300 s limit. */
int mdd_comm_abort(mdd_comm* c) {
  MDD_API_BEGIN
  if (c && c->loop) loop_abort(static_cast<LoopGroup*>(c->loop));
  MDD_API_END
}

int mdd_comm_info(const mdd_comm* c, int* nranks, int* rank) {
  MDD_API_BEGIN
  *nranks = c->nranks;
  *rank = c->rank;
  MDD_API_END
}

}  // extern "C"
