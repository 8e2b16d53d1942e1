// Context, CSR storage, complex128 CSR SpMV and small vector kernels.
//
// SpMV replaces `a_mv = op @ v` (reference krylov.py:58-61, 95-97) and
// linalg.spmv (reference linalg.py:41-45).  HBM-bound: 16 B value + 4 B column
// per nonzero; a group of TPR lanes owns one row so the row's values and
// columns are read as contiguous 16 B / 4 B segments; the group reduces with
// shuffles (fixed order, so reruns are bitwise identical).
#include <cuda_runtime.h>

#include <cstdlib>
#include <cstring>
#include <mutex>

#include "mdd_internal.h"
#include "mdd_kernels.cuh"

#include <map>

namespace mdd {
static thread_local std::string g_last_error;

// ------------------------------------------------------- caching allocator
namespace {
struct DevCache {
  std::mutex mu;
  std::map<std::pair<int, size_t>, std::vector<void*>> free_blocks;  // (device, size) -> blocks
  size_t cached = 0;
  static constexpr size_t kCap = size_t(24) << 30;  // keep at most 24 GB cached
};
DevCache& cache() {
  static DevCache* c = new DevCache();  // never destroyed: outlives static DevBufs
  return *c;
}
size_t bucket(size_t bytes) {
  if (bytes <= 256) return 256;
  if (bytes < (size_t(1) << 20)) {
    size_t b = 256;
    while (b < bytes) b <<= 1;
    return b;
  }
  const size_t g = size_t(2) << 20;
  return (bytes + g - 1) / g * g;
}
}  // namespace

void* dev_alloc(size_t bytes) {
  const size_t b = bucket(bytes);
  int dev = 0;
  cudaGetDevice(&dev);
  DevCache& c = cache();
  {
    std::lock_guard<std::mutex> g(c.mu);
    auto it = c.free_blocks.find({dev, b});
    if (it != c.free_blocks.end() && !it->second.empty()) {
      void* p = it->second.back();
      it->second.pop_back();
      c.cached -= b;
      return p;
    }
  }
  void* p = nullptr;
  cudaError_t e = cudaMalloc(&p, b);
  if (e == cudaErrorMemoryAllocation) {
    cudaGetLastError();
    dev_cache_flush();
    e = cudaMalloc(&p, b);
  }
  CK(e);
  return p;
}

void dev_free(void* p, size_t bytes) {
  if (!p) return;
  const size_t b = bucket(bytes);
  int dev = 0;
  cudaGetDevice(&dev);
  DevCache& c = cache();
  {
    std::lock_guard<std::mutex> g(c.mu);
    if (c.cached + b <= DevCache::kCap) {
      c.free_blocks[{dev, b}].push_back(p);
      c.cached += b;
      return;
    }
  }
  cudaFree(p);
}

void dev_cache_flush() {
  DevCache& c = cache();
  std::lock_guard<std::mutex> g(c.mu);
  int cur = 0;
  cudaGetDevice(&cur);
  for (auto& kv : c.free_blocks) {
    cudaSetDevice(kv.first.first);
    for (void* p : kv.second) cudaFree(p);
  }
  cudaSetDevice(cur);
  c.free_blocks.clear();
  c.cached = 0;
}
void set_last_error(const std::string& m) { g_last_error = m; }

std::shared_ptr<mdd_pattern> make_pattern(int64_t nrow, int64_t ncol,
                                          std::vector<int32_t>&& rowptr,
                                          std::vector<int32_t>&& cols, cudaStream_t s) {
  auto p = std::make_shared<mdd_pattern>();
  p->nrow = nrow;
  p->ncol = ncol;
  p->nnz = (int64_t)cols.size();
  p->h_rowptr = std::move(rowptr);
  p->h_cols = std::move(cols);
  p->rowptr.upload(p->h_rowptr, s);
  p->cols.upload(p->h_cols, s);
  return p;
}

// ------------------------------------------------------------------ SpMV
template <bool CPLX, int TPR>
__global__ void __launch_bounds__(256) k_spmv(int64_t nrow, const int32_t* __restrict__ rowptr,
                                              const int32_t* __restrict__ cols,
                                              const double* __restrict__ vals,
                                              const double2* __restrict__ x,
                                              double2* __restrict__ y, double2 alpha,
                                              double2 beta, const double2* __restrict__ z) {
  const int64_t gid = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  const int64_t row = gid / TPR;
  const int lane = threadIdx.x % TPR;
  if (row >= nrow) return;  // TPR divides 32: whole groups exit together
  const int b = rowptr[row], e = rowptr[row + 1];
  double re = 0.0, im = 0.0;
  for (int j = b + lane; j < e; j += TPR) {
    const double2 xv = x[cols[j]];
    if (CPLX) {
      const double2 a = reinterpret_cast<const double2*>(vals)[j];
      re += a.x * xv.x - a.y * xv.y;
      im += a.x * xv.y + a.y * xv.x;
    } else {
      const double a = vals[j];
      re += a * xv.x;
      im += a * xv.y;
    }
  }
#pragma unroll
  for (int off = TPR / 2; off > 0; off >>= 1) {
    re += __shfl_down_sync(0xffffffffu, re, off, TPR);
    im += __shfl_down_sync(0xffffffffu, im, off, TPR);
  }
  if (lane == 0) {
    double2 r = make_double2(alpha.x * re - alpha.y * im, alpha.x * im + alpha.y * re);
    if (z) {
      const double2 zz = z[row];
      r.x += beta.x * zz.x - beta.y * zz.y;
      r.y += beta.x * zz.y + beta.y * zz.x;
    }
    y[row] = r;
  }
}

// Unrolled variant: each lane of a TPR-lane row group issues U column loads,
// then U value loads and U x gathers before any arithmetic (more loads in
// flight per thread than the loop above); longer rows continue in a loop.
template <bool CPLX, int TPR, int U>
__global__ void __launch_bounds__(256) k_spmv_u(int64_t nrow, const int32_t* __restrict__ rowptr,
                                                const int32_t* __restrict__ cols,
                                                const double* __restrict__ vals,
                                                const double2* __restrict__ x,
                                                double2* __restrict__ y, double2 alpha,
                                                double2 beta, const double2* __restrict__ z) {
  const int64_t gid = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  const int64_t row = gid / TPR;
  const int lane = threadIdx.x % TPR;
  if (row >= nrow) return;
  const int b = __ldg(rowptr + row), e = __ldg(rowptr + row + 1);
  double re = 0.0, im = 0.0;
  for (int j0 = b + lane; j0 < e; j0 += TPR * U) {
    int c[U];
    double2 a[U];
    double2 xv[U];
#pragma unroll
    for (int u = 0; u < U; ++u) c[u] = (j0 + u * TPR < e) ? __ldcs(cols + j0 + u * TPR) : -1;
#pragma unroll
    for (int u = 0; u < U; ++u) {
      // predicated on the index, not on the loaded column, so the value loads
      // issue together with the column loads (only the x gathers wait for them)
      const int j = j0 + u * TPR;
      if (CPLX) a[u] = j < e ? __ldcs(reinterpret_cast<const double2*>(vals) + j) : make_double2(0.0, 0.0);
      else a[u] = make_double2(j < e ? __ldcs(vals + j) : 0.0, 0.0);
    }
#pragma unroll
    for (int u = 0; u < U; ++u) xv[u] = c[u] >= 0 ? __ldg(x + c[u]) : make_double2(0.0, 0.0);
#pragma unroll
    for (int u = 0; u < U; ++u) {
      if (CPLX) {
        re += a[u].x * xv[u].x - a[u].y * xv[u].y;
        im += a[u].x * xv[u].y + a[u].y * xv[u].x;
      } else {
        re += a[u].x * xv[u].x;
        im += a[u].x * xv[u].y;
      }
    }
  }
#pragma unroll
  for (int off = TPR / 2; off > 0; off >>= 1) {
    re += __shfl_down_sync(0xffffffffu, re, off, TPR);
    im += __shfl_down_sync(0xffffffffu, im, off, TPR);
  }
  if (lane == 0) {
    double2 r = make_double2(alpha.x * re - alpha.y * im, alpha.x * im + alpha.y * re);
    if (z) {
      const double2 zz = z[row];
      r.x += beta.x * zz.x - beta.y * zz.y;
      r.y += beta.x * zz.y + beta.y * zz.x;
    }
    y[row] = r;
  }
}

// rows [row0, row0+nrow) of A (rowptr entries are absolute offsets into
// cols/vals, so a shifted rowptr is the row block).  Short rows (the
// edge-element operators: 7-19 nonzeros) use the unrolled kernel: 4 lanes per
// row, 16 nonzeros per pass (measured 4.4 TB/s on cfg1's A vs 3.0 for the
// plain loop); long rows a warp per row.
static void launch_spmv(mdd_ctx* ctx, const mdd_csr* A, int64_t row0, int64_t nrow, const double2* x,
                        double2* y, double2 alpha, double2 beta, const double2* z, cudaStream_t s) {
  if (nrow <= 0) return;
  const double avg = A->nrow() ? (double)A->nnz() / (double)A->nrow() : 0.0;
  const int32_t* rp = A->pat->rowptr.p + row0;
  const int32_t* cl = A->pat->cols.p;
  const double* va = A->vals.p;
  const bool cp = A->is_complex;
  auto grid = [&](int tpr) { return (unsigned)((nrow * tpr + 255) / 256); };
  if (avg > 48) {
    if (cp) k_spmv<true, 32><<<grid(32), 256, 0, s>>>(nrow, rp, cl, va, x, y, alpha, beta, z);
    else k_spmv<false, 32><<<grid(32), 256, 0, s>>>(nrow, rp, cl, va, x, y, alpha, beta, z);
  } else if (avg > 24) {
    if (cp) k_spmv_u<true, 8, 4><<<grid(8), 256, 0, s>>>(nrow, rp, cl, va, x, y, alpha, beta, z);
    else k_spmv_u<false, 8, 4><<<grid(8), 256, 0, s>>>(nrow, rp, cl, va, x, y, alpha, beta, z);
  } else {
    // 4 lanes x 5 nonzeros: the edge-element rows (7-19 nonzeros) take one
    // pass; 128-thread blocks (measured on cfg1's A inside GMRES: 8.52 -> 7.82 ms
    // per 201 calls, 56% -> 61% of HBM; standalone 4.42 -> 4.71 TB/s; swept
    // 2x8, 8x2, 4x4, 4x5)
    const unsigned g128 = (unsigned)((nrow * 4 + 127) / 128);
    if (cp) k_spmv_u<true, 4, 5><<<g128, 128, 0, s>>>(nrow, rp, cl, va, x, y, alpha, beta, z);
    else k_spmv_u<false, 4, 5><<<g128, 128, 0, s>>>(nrow, rp, cl, va, x, y, alpha, beta, z);
  }
  CK_LAUNCH(ctx);
}

void spmv_dev_axpby(mdd_ctx* ctx, const mdd_csr* A, const double2* x, double2* y,
                    double2 alpha, double2 beta, const double2* z, cudaStream_t s) {
  launch_spmv(ctx, A, 0, A->nrow(), x, y, alpha, beta, z, s);
}

void spmv_rows_dev(mdd_ctx* ctx, const mdd_csr* A, int64_t row0, int64_t nrow, const double2* x, double2* y,
                   cudaStream_t s) {
  if (nrow <= 0) return;
  if (row0 < 0 || row0 + nrow > A->nrow()) fail(MDD_EINVAL, "spmv: row block out of range");
  launch_spmv(ctx, A, row0, nrow, x, y, make_double2(1.0, 0.0), make_double2(0.0, 0.0), nullptr, s);
}

void spmv_dev(mdd_ctx* ctx, const mdd_csr* A, const double2* x, double2* y, cudaStream_t s) {
  spmv_dev_axpby(ctx, A, x, y, make_double2(1.0, 0.0), make_double2(0.0, 0.0), nullptr, s);
}

// ---------------------------------------------------------- vector kernels
__global__ void k_vec_sub(const double2* a, const double2* b, double2* out, int64_t n) {
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x) {
    const double2 u = a[i], v = b[i];
    out[i] = make_double2(u.x - v.x, u.y - v.y);
  }
}
__global__ void k_vec_add(const double2* a, const double2* b, double2* out, int64_t n) {
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x) {
    const double2 u = a[i], v = b[i];
    out[i] = make_double2(u.x + v.x, u.y + v.y);
  }
}
static unsigned grid_for(int64_t n, int bs, int nsm) {
  int64_t g = (n + bs - 1) / bs;
  const int64_t cap = (int64_t)nsm * 16;
  if (g > cap) g = cap;
  return (unsigned)(g < 1 ? 1 : g);
}
void vec_sub(mdd_ctx* ctx, const double2* a, const double2* b, double2* out, int64_t n,
             cudaStream_t s) {
  k_vec_sub<<<grid_for(n, 256, ctx->nsm), 256, 0, s>>>(a, b, out, n);
  CK_LAUNCH(ctx);
}
void vec_add(mdd_ctx* ctx, const double2* a, const double2* b, double2* out, int64_t n,
             cudaStream_t s) {
  k_vec_add<<<grid_for(n, 256, ctx->nsm), 256, 0, s>>>(a, b, out, n);
  CK_LAUNCH(ctx);
}
}  // namespace mdd

using namespace mdd;

void* mdd_ctx::pinned_buf(size_t bytes) {
  if (bytes > pinned_bytes) {
    if (pinned) cudaFreeHost(pinned);
    pinned = nullptr;
    size_t nb = bytes < (1u << 20) ? (1u << 20) : bytes;
    CK(cudaMallocHost(&pinned, nb));
    pinned_bytes = nb;
  }
  return pinned;
}

extern "C" {

const char* mdd_last_error(void) { return g_last_error.c_str(); }
int mdd_version(void) { return 1; }

int mdd_device_count(int* n) {
  MDD_API_BEGIN
  int c = 0;
  cudaError_t e = cudaGetDeviceCount(&c);
  if (e != cudaSuccess) {
    cudaGetLastError();
    c = 0;
  }
  *n = c;
  MDD_API_END
}

int mdd_ctx_create(int device, mdd_ctx** out) {
  MDD_API_BEGIN
  int count = 0;
  cudaError_t e = cudaGetDeviceCount(&count);
  if (e != cudaSuccess || count == 0) {
    cudaGetLastError();
    fail(MDD_ECUDA, "no CUDA device available: libmdd has no CPU fallback");
  }
  if (device < 0 || device >= count) fail(MDD_EINVAL, "device index out of range");
  CK(cudaSetDevice(device));
  auto c = new mdd_ctx();
  c->device = device;
  cudaDeviceProp prop;
  CK(cudaGetDeviceProperties(&prop, device));
  c->nsm = prop.multiProcessorCount;
  CK(cudaStreamCreateWithFlags(&c->stream, cudaStreamNonBlocking));
  *out = c;
  MDD_API_END
}

void mdd_ctx_destroy(mdd_ctx* ctx) {
  if (!ctx) return;
  cudaSetDevice(ctx->device);
  cudaStreamSynchronize(ctx->stream);
  for (auto& e : ctx->events)
    if (e) cudaEventDestroy(e);
  if (ctx->pinned) cudaFreeHost(ctx->pinned);
  if (ctx->mapped_status) cudaFreeHost(ctx->mapped_status);
  cudaStreamDestroy(ctx->stream);
  delete ctx;
}

int mdd_ctx_synchronize(mdd_ctx* ctx) {
  MDD_API_BEGIN
  CK(cudaStreamSynchronize(ctx->stream));
  MDD_API_END
}

int64_t mdd_ctx_kernel_launches(const mdd_ctx* ctx) { return ctx ? ctx->launches : 0; }

int mdd_ctx_timers(const mdd_ctx* ctx, double* out8) {
  MDD_API_BEGIN
  for (int i = 0; i < 8; ++i) out8[i] = ctx->timers[i];
  MDD_API_END
}

int mdd_ctx_set_timing(mdd_ctx* ctx, int enable) {
  MDD_API_BEGIN
  ctx->timing = enable != 0;
  MDD_API_END
}

int mdd_ctx_event_record(mdd_ctx* ctx, int slot) {
  MDD_API_BEGIN
  if (slot < 0 || slot >= 16) fail(MDD_EINVAL, "event slot out of range");
  CK(cudaSetDevice(ctx->device));
  if (!ctx->events[slot]) CK(cudaEventCreate(&ctx->events[slot]));
  CK(cudaEventRecord(ctx->events[slot], ctx->stream));
  MDD_API_END
}

int mdd_ctx_event_elapsed(mdd_ctx* ctx, int s0, int s1, double* ms) {
  MDD_API_BEGIN
  if (s0 < 0 || s0 >= 16 || s1 < 0 || s1 >= 16 || !ctx->events[s0] || !ctx->events[s1])
    fail(MDD_EINVAL, "event slot not recorded");
  CK(cudaEventSynchronize(ctx->events[s1]));
  float f = 0;
  CK(cudaEventElapsedTime(&f, ctx->events[s0], ctx->events[s1]));
  *ms = f;
  MDD_API_END
}

int mdd_dev_alloc(mdd_ctx* ctx, int64_t bytes, void** out) {
  MDD_API_BEGIN
  CK(cudaSetDevice(ctx->device));
  CK(cudaMalloc(out, bytes > 0 ? (size_t)bytes : 16));
  MDD_API_END
}

int mdd_dev_free(mdd_ctx* ctx, void* p) {
  MDD_API_BEGIN
  CK(cudaSetDevice(ctx->device));
  if (p) CK(cudaFree(p));
  MDD_API_END
}

int mdd_memcpy(mdd_ctx* ctx, void* dst, const void* src, int64_t bytes, int kind) {
  MDD_API_BEGIN
  CK(cudaSetDevice(ctx->device));
  const cudaMemcpyKind k = kind == 1 ? cudaMemcpyHostToDevice
                           : kind == 2 ? cudaMemcpyDeviceToHost : cudaMemcpyDeviceToDevice;
  CK(cudaMemcpyAsync(dst, src, (size_t)bytes, k, ctx->stream));
  CK(cudaStreamSynchronize(ctx->stream));
  MDD_API_END
}

int mdd_csr_from_host(mdd_ctx* ctx, int64_t nrow, int64_t ncol, int64_t nnz,
                      const int32_t* indptr, const int32_t* indices, const void* values,
                      int is_complex, mdd_csr** out) {
  MDD_API_BEGIN
  if (nrow < 0 || ncol < 0 || nnz < 0) fail(MDD_EINVAL, "negative CSR dimensions");
  if (nnz > INT32_MAX) fail(MDD_EINVAL, "CSR with more than 2^31 nonzeros");
  CK(cudaSetDevice(ctx->device));
  std::vector<int32_t> rp(indptr, indptr + nrow + 1);
  std::vector<int32_t> cl(indices, indices + nnz);
  if (rp[0] != 0 || rp[nrow] != nnz) fail(MDD_EINVAL, "inconsistent CSR indptr");
  auto A = new mdd_csr();
  A->ctx = ctx;
  A->pat = make_pattern(nrow, ncol, std::move(rp), std::move(cl), ctx->stream);
  A->is_complex = is_complex != 0;
  const size_t nv = (size_t)nnz * (A->is_complex ? 2 : 1);
  A->vals.upload(reinterpret_cast<const double*>(values), nv, ctx->stream);
  CK(cudaStreamSynchronize(ctx->stream));
  *out = A;
  MDD_API_END
}

int mdd_csr_info(const mdd_csr* A, int64_t* nrow, int64_t* ncol, int64_t* nnz, int* is_complex) {
  MDD_API_BEGIN
  *nrow = A->nrow();
  *ncol = A->ncol();
  *nnz = A->nnz();
  *is_complex = A->is_complex ? 1 : 0;
  MDD_API_END
}

int mdd_csr_to_host(const mdd_csr* A, int32_t* indptr, int32_t* indices, void* values) {
  MDD_API_BEGIN
  CK(cudaSetDevice(A->ctx->device));
  if (indptr) memcpy(indptr, A->pat->h_rowptr.data(), sizeof(int32_t) * (A->nrow() + 1));
  if (indices) memcpy(indices, A->pat->h_cols.data(), sizeof(int32_t) * A->nnz());
  if (values) {
    A->vals.download(reinterpret_cast<double*>(values),
                     (size_t)A->nnz() * (A->is_complex ? 2 : 1), A->ctx->stream);
    CK(cudaStreamSynchronize(A->ctx->stream));
  }
  MDD_API_END
}

void mdd_csr_destroy(mdd_csr* A) {
  if (!A) return;
  cudaSetDevice(A->ctx->device);
  delete A;
}

int mdd_spmv(mdd_ctx* ctx, const mdd_csr* A, const mdd_complex* x, mdd_complex* y) {
  MDD_API_BEGIN
  CK(cudaSetDevice(ctx->device));
  DevBuf<double2> dx(A->ncol()), dy(A->nrow());
  dx.upload(reinterpret_cast<const double2*>(x), A->ncol(), ctx->stream);
  spmv_dev(ctx, A, dx.p, dy.p, ctx->stream);
  dy.download(reinterpret_cast<double2*>(y), A->nrow(), ctx->stream);
  CK(cudaStreamSynchronize(ctx->stream));
  MDD_API_END
}

int mdd_spmv_bench(mdd_ctx* ctx, const mdd_csr* A, int reps, double* ms_per_call) {
  MDD_API_BEGIN
  CK(cudaSetDevice(ctx->device));
  DevBuf<double2> dx(A->ncol()), dy(A->nrow());
  CK(cudaMemsetAsync(dx.p, 0, sizeof(double2) * dx.n, ctx->stream));
  for (int i = 0; i < 3; ++i) spmv_dev(ctx, A, dx.p, dy.p, ctx->stream);
  cudaEvent_t e0, e1;
  CK(cudaEventCreate(&e0));
  CK(cudaEventCreate(&e1));
  CK(cudaEventRecord(e0, ctx->stream));
  for (int i = 0; i < reps; ++i) spmv_dev(ctx, A, dx.p, dy.p, ctx->stream);
  CK(cudaEventRecord(e1, ctx->stream));
  CK(cudaEventSynchronize(e1));
  float ms = 0;
  CK(cudaEventElapsedTime(&ms, e0, e1));
  cudaEventDestroy(e0);
  cudaEventDestroy(e1);
  *ms_per_call = reps > 0 ? ms / reps : 0.0;
  MDD_API_END
}

}  // extern "C"
