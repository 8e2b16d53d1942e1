// Internal definitions shared by the libmdd translation units.
#pragma once

#include <cuda_runtime.h>
#include <stdint.h>

#include <cstdio>
#include <memory>
#include <stdexcept>
#include <string>
#include <vector>

#include "../../include/mdd.h"

namespace mdd {

// ---------------------------------------------------------------- errors
struct Error : public std::exception {
  int code;
  std::string msg;
  int failed_ctx = -2;
  Error(int c, std::string m, int fctx = -2) : code(c), msg(std::move(m)), failed_ctx(fctx) {}
  const char* what() const noexcept override { return msg.c_str(); }
};

void set_last_error(const std::string& m);

[[noreturn]] inline void fail(int code, const std::string& m, int fctx = -2) {
  throw Error(code, m, fctx);
}

inline void cuda_check(cudaError_t e, const char* what, const char* file, int line) {
  if (e != cudaSuccess) {
    char buf[512];
    snprintf(buf, sizeof(buf), "CUDA error %s (%s) at %s:%d: %s", cudaGetErrorName(e),
             cudaGetErrorString(e), file, line, what);
    throw Error(e == cudaErrorMemoryAllocation ? MDD_ENOMEM : MDD_ECUDA, buf);
  }
}
#define CK(call) ::mdd::cuda_check((call), #call, __FILE__, __LINE__)
#define CK_LAUNCH(ctx)                                             \
  do {                                                             \
    ::mdd::cuda_check(cudaGetLastError(), "kernel launch", __FILE__, __LINE__); \
    (ctx)->launches++;                                             \
  } while (0)

// C-ABI wrapper: converts exceptions into codes + thread-local messages.
#define MDD_API_BEGIN try {
#define MDD_API_END                                \
  }                                                \
  catch (const ::mdd::Error& e) {                  \
    ::mdd::set_last_error(e.msg);                  \
    return e.code;                                 \
  }                                                \
  catch (const std::bad_alloc&) {                  \
    ::mdd::set_last_error("host allocation failed"); \
    return MDD_ENOMEM;                             \
  }                                                \
  catch (const std::exception& e) {                \
    ::mdd::set_last_error(e.what());               \
    return MDD_EINVAL;                             \
  }                                                \
  return MDD_OK;

// ----------------------------------------------------------- device memory
// Caching allocator: freed blocks go to size-bucketed free lists and are
// reused, so steady-state solves perform no cudaMalloc/cudaFree (cudaFree
// synchronises the device).  On allocation failure the cache is flushed and
// the allocation retried.
void* dev_alloc(size_t bytes);
void dev_free(void* p, size_t bytes);
void dev_cache_flush();

template <typename T>
struct DevBuf {
  T* p = nullptr;
  size_t n = 0;
  DevBuf() = default;
  explicit DevBuf(size_t count) { alloc(count); }
  DevBuf(const DevBuf&) = delete;
  DevBuf& operator=(const DevBuf&) = delete;
  DevBuf(DevBuf&& o) noexcept : p(o.p), n(o.n) { o.p = nullptr; o.n = 0; }
  DevBuf& operator=(DevBuf&& o) noexcept {
    if (this != &o) { release(); p = o.p; n = o.n; o.p = nullptr; o.n = 0; }
    return *this;
  }
  ~DevBuf() { release(); }
  void alloc(size_t count) {
    release();
    n = count;
    if (count) p = static_cast<T*>(dev_alloc(count * sizeof(T)));
  }
  void release() {
    if (p) dev_free(p, n * sizeof(T));
    p = nullptr;
    n = 0;
  }
  void upload(const T* h, size_t count, cudaStream_t s) {
    if (count > n) alloc(count);
    if (count) CK(cudaMemcpyAsync(p, h, count * sizeof(T), cudaMemcpyHostToDevice, s));
  }
  void upload(const std::vector<T>& h, cudaStream_t s) { upload(h.data(), h.size(), s); }
  void download(T* h, size_t count, cudaStream_t s) const {
    if (count) CK(cudaMemcpyAsync(h, p, count * sizeof(T), cudaMemcpyDeviceToHost, s));
  }
  void zero(cudaStream_t s) {
    if (n) CK(cudaMemsetAsync(p, 0, n * sizeof(T), s));
  }
};

template <typename T>
inline DevBuf<T> to_device(const std::vector<T>& h, cudaStream_t s) {
  DevBuf<T> d(h.size());
  d.upload(h, s);
  return d;
}

}  // namespace mdd

// --------------------------------------------------------- opaque objects
struct mdd_ctx {
  int device = 0;
  int nsm = 148;
  cudaStream_t stream = nullptr;
  int64_t launches = 0;
  bool timing = false;
  double timers[8] = {0, 0, 0, 0, 0, 0, 0, 0};
  int* mapped_status = nullptr;  // host-mapped GMRES status word
  // pinned staging used by host-pointer entry points
  void* pinned = nullptr;
  size_t pinned_bytes = 0;
  cudaEvent_t events[16] = {};
  void* pinned_buf(size_t bytes);
};

struct mdd_pattern {
  int64_t nrow = 0, ncol = 0, nnz = 0;
  mdd::DevBuf<int32_t> rowptr, cols;
  std::vector<int32_t> h_rowptr, h_cols;  // host copy (symbolic work)
};

struct mdd_csr {
  mdd_ctx* ctx = nullptr;
  std::shared_ptr<mdd_pattern> pat;
  bool is_complex = true;
  mdd::DevBuf<double> vals;  // nnz (real) or 2*nnz (complex, interleaved)
  int64_t nrow() const { return pat->nrow; }
  int64_t ncol() const { return pat->ncol; }
  int64_t nnz() const { return pat->nnz; }
};

// Device-resident mesh + edge space + CSR pattern of the kept DOFs.
struct mdd_space {
  mdd_ctx* ctx = nullptr;
  int32_t n = 0;  // cells per axis
  int64_t nv = 0, nt = 0, ne = 0, ndof = 0;
  // host copies (int32 unless noted)
  std::vector<double> h_verts;      // nv*3
  std::vector<int32_t> h_tets;      // nt*4
  std::vector<int32_t> h_tet_edges; // nt*6
  std::vector<int8_t> h_signs;      // nt*6
  std::vector<int32_t> h_e2d;       // ne
  // device copies
  mdd::DevBuf<double> verts;
  mdd::DevBuf<int32_t> tets, tet_edges, e2d;
  mdd::DevBuf<int8_t> signs;
  // kept-dof CSR pattern (shared by A, S, M, Dk)
  std::shared_ptr<mdd_pattern> pat;
  // cells grouped by parity colour (cx%2, cy%2, cz%2): no two cells of one
  // colour share an edge, so one thread per cell scatters without atomics
  mdd::DevBuf<int32_t> cells_by_color;
  int64_t color_off[9] = {0};
  // row window of a sharded solve (mdd_space_set_row_window): the colour lists restricted to
  // the cells that touch a row in [win_lo, win_hi); the lists stay cached while inactive
  bool win_active = false;
  int64_t win_lo = -1, win_hi = -1;
  mdd::DevBuf<int32_t> win_cells;
  int64_t win_off[9] = {0};
  // dof -> incident (tet*6 + local edge), ascending tet (rhs gather);
  // order 2: (tet*20 + local dof)
  mdd::DevBuf<int32_t> inc_ptr, inc;
  // order-2 spaces (nedelec2.cu): tets hold vertices sorted by global index,
  // tdofs (nt*20) the global DoF of each local basis function (-1: eliminated),
  // and the load-vector quadrature (nq barycentric points + weights)
  int32_t order = 1;
  mdd::DevBuf<int32_t> tdofs;
  int32_t nq = 0;
  mdd::DevBuf<double> qbary, qw;
};

// NCCL communicator (comm.cu); `comm` is an ncclComm_t (NCCL is dlopen'ed)
struct mdd_comm {
  mdd_ctx* ctx = nullptr;
  void* comm = nullptr;
  int nranks = 1, rank = 0;
  void* loop = nullptr;  // LoopGroup (mdd_comm_create_loopback)
};

// Row ranges of a sharded vector of length n (global numbering, every rank holds a
// full-length array of which only its ranges are meaningful).  Rank q OWNS rows
// [own_lo[q], own_hi[q]) (equal blocks of ceil(n/nranks) rows, gmres_cgs's layout) and
// NEEDS rows [need_lo[q], need_hi[q]) >= its owned rows: the unknowns of its subdomains
// (restriction, precond.py:220) and the columns of its rows of A (krylov.py:95-97).
// The reference numbering is x-major, the subdomain blocks of a rank are x-slabs, so both
// are contiguous ranges and a halo exchange is a set of in-place range copies.
struct mdd_halo {
  int64_t n = 0;
  std::vector<int64_t> own_lo, own_hi, need_lo, need_hi;
  mdd::DevBuf<double2> stage;  // overlap sums: the peers' contributions to my owned rows
};

namespace mdd {
// in-place sum of a complex vector over the communicator (stream-ordered)
void comm_allreduce_z(mdd_comm* c, double2* buf, int64_t n, cudaStream_t s);
// recv[r*per_rank ...] = send of rank r (stream-ordered); one rank: copy
void comm_allgather_z(mdd_comm* c, const double2* send, double2* recv, int64_t per_rank, cudaStream_t s);
// true when collectives go through NCCL (any rank count)
inline bool comm_active(const mdd_comm* c) { return c && (c->comm || c->loop); }
// Halo exchange (forward): on entry `vec` is valid on every rank's owned rows; on return it
// is valid on this rank's needed rows.  Grouped ncclSend/ncclRecv of sub-ranges, in place.
void comm_halo_gather(mdd_comm* c, mdd_halo* h, double2* vec, cudaStream_t s);
// Overlap sum (reverse halo): on entry `vec` holds this rank's partial sums on its needed
// rows; on return its owned rows hold the sum over all ranks (ascending rank order: fixed,
// bitwise reproducible).  Rows outside the owned range are left as they were.
void comm_halo_reduce(mdd_comm* c, mdd_halo* h, double2* vec, cudaStream_t s);
// fills own_*/need_* of every rank from this rank's needed range (one tiny allgather)
void comm_halo_setup(mdd_comm* c, mdd_halo* h, int64_t n, int64_t need_lo, int64_t need_hi, cudaStream_t s);

// element geometry + 6x6 stiffness / mass (fem.py:154-195); shared by the
// global assembly, the impras local assembly and the coarse Galerkin kernel
struct ElemMats {
  double s[6][6];
  double m[6][6];
  double vol;
};

// kernels shared across units ------------------------------------------
// y = A x (x, y device complex)
void spmv_dev(mdd_ctx* ctx, const mdd_csr* A, const double2* x, double2* y, cudaStream_t s);
// y[0..nrow) = A[row0:row0+nrow, :] x  (row block of a CSR, x full length)
void spmv_rows_dev(mdd_ctx* ctx, const mdd_csr* A, int64_t row0, int64_t nrow, const double2* x, double2* y,
                   cudaStream_t s);
// y = beta*y + alpha*A x on device; variants used by the preconditioner
void spmv_dev_axpby(mdd_ctx* ctx, const mdd_csr* A, const double2* x, double2* y,
                    double2 alpha, double2 beta, const double2* z, cudaStream_t s);
// out = a - b
void vec_sub(mdd_ctx* ctx, const double2* a, const double2* b, double2* out, int64_t n,
             cudaStream_t s);
void vec_add(mdd_ctx* ctx, const double2* a, const double2* b, double2* out, int64_t n,
             cudaStream_t s);
// assembly shared by the order-1 (assemble.cu) and order-2 (nedelec2.cu) spaces
struct GaussSrc {
  double cx, cy, cz, alpha, amp, dx, dy, dz;
};
__global__ void k_combine(int64_t nnz, const double* __restrict__ S, const double* __restrict__ M,
                          double2* __restrict__ A, double* __restrict__ Dk, double k2, double xi,
                          int write_a);
void assemble_system2(mdd_space* sp, const mdd_coeffs* co, mdd_csr** A, mdd_csr** S, mdd_csr** M,
                      mdd_csr** Dk);
void assemble_rhs2_dev(mdd_space* sp, const double2* fvals_host, const GaussSrc* gsrc, double2* rhs_dev);
// complex CSR with the given pattern, values zeroed
mdd_csr* new_csr(mdd_ctx* ctx, std::shared_ptr<mdd_pattern> pat, bool cplx);
std::shared_ptr<mdd_pattern> make_pattern(int64_t nrow, int64_t ncol,
                                          std::vector<int32_t>&& rowptr,
                                          std::vector<int32_t>&& cols, cudaStream_t s);
}  // namespace mdd
