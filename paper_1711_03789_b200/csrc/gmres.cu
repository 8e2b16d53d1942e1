// Unrestarted GMRES on the device (reference krylov.gmres, krylov.py:64-209).
//
// One iteration = operator/preconditioner kernels + ONE cooperative
// persistent Arnoldi kernel that performs, exactly in the reference order
// (krylov.py:134-187):
//   2 passes x m modified Gram-Schmidt steps  h_j = <V_j, dw>, col[j] += h_j,
//       w -= h_j V_j, dw -= h_j DV_j          (krylov.py:137-143)
//   hnorm2 = Re vdot(w, dw), breakdown test, normalisation (krylov.py:144-151)
//   orthogonality drift max_j |vdot(V_j, DV_m)|               (krylov.py:153)
//   stored + new complex Givens rotations, history clamp     (krylov.py:162-187)
// Each MGS step costs one grid barrier: the axpy of step j and the partial
// dot of step j+1 are fused into one sweep over the CTA's slice, so w is read
// and written once per step and V_j once (the slice of V_j is L2-resident for
// the axpy).  Cross-CTA sums use a fixed order: reruns are bitwise identical.
#include <cooperative_groups.h>

#include <chrono>
#include <cmath>

#include "mdd_internal.h"
#include "mdd_kernels.cuh"

namespace cg = cooperative_groups;

namespace mdd {

void prec_apply_dev(mdd_prec* P, const double2* v, double2* out, cudaStream_t s);

struct ArnoldiArgs {
  int64_t n;
  int m;      // iteration (1-based); w = V[m]
  int maxit;
  double2* V;   // (maxit+1) x n
  double2* DV;  // weighted basis or nullptr (then dw == w)
  double2* partials;  // 2*G
  double2* dpart;     // maxit*G (drift partials)
  double2* H;         // (maxit+1) x maxit, column j at H + j*(maxit+1)
  double2* cs;
  double2* sn;
  double2* g;
  double* hist;       // maxit+1
  double* drift;      // maxit+1 (nan when not computed)
  const double* beta;
  double tol;
  int check_drift;
  volatile int* status;  // [done, breakdown, iterations] (host-mapped)
};

// Deterministic sum of partials[0..G) (all threads of the CTA get it).
__device__ __forceinline__ double2 reduce_partials(const double2* p, int G, double2* sh) {
  __syncthreads();
  if (threadIdx.x < 32) {
    double2 a = make_double2(0.0, 0.0);
    for (int b = threadIdx.x; b < G; b += 32) {
      const double2 v = __ldcg(p + b);
      a.x += v.x;
      a.y += v.y;
    }
    a = warp_sum2(a);
    if (threadIdx.x == 0) sh[0] = a;
  }
  __syncthreads();
  return sh[0];
}

__global__ void __launch_bounds__(256) k_arnoldi(ArnoldiArgs a) {
  cg::grid_group grid = cg::this_grid();
  extern __shared__ double2 col[];  // m+1 entries, identical in every CTA
  __shared__ double2 red[8];
  __shared__ double2 bcast[1];
  const int G = gridDim.x;
  const int64_t n = a.n;
  const int m = a.m;
  const int64_t stride = (int64_t)G * blockDim.x;
  const int64_t tid0 = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  double2* w = a.V + (int64_t)m * n;
  double2* dw = a.DV ? a.DV + (int64_t)m * n : w;
  const bool weighted = a.DV != nullptr;

  for (int j = threadIdx.x; j <= m; j += blockDim.x) col[j] = make_double2(0.0, 0.0);

  // first partial: <V_0, dw>
  {
    const double2* v0 = a.V;
    double2 acc = make_double2(0.0, 0.0);
    for (int64_t i = tid0; i < n; i += stride) {
      const double2 x = v0[i], y = dw[i];
      acc.x += x.x * y.x + x.y * y.y;
      acc.y += x.x * y.y - x.y * y.x;
    }
    acc = block_sum2(acc, red);
    if (threadIdx.x == 0) a.partials[blockIdx.x] = acc;
  }
  grid.sync();
  const int nsteps = 2 * m;
  for (int s = 0; s < nsteps; ++s) {
    const int j = s % m;
    const double2 h = reduce_partials(a.partials + (s & 1) * G, G, bcast);
    if (threadIdx.x == 0) col[j] = cadd(col[j], h);
    const double2* vj = a.V + (int64_t)j * n;
    const double2* dvj = weighted ? a.DV + (int64_t)j * n : nullptr;
    const bool last = (s + 1 == nsteps);
    const double2* vn = last ? w : a.V + (int64_t)((s + 1) % m) * n;
    double2 acc = make_double2(0.0, 0.0);
    for (int64_t i = tid0; i < n; i += stride) {
      const double2 v = vj[i];
      double2 wi = w[i];
      wi = make_double2(wi.x - (h.x * v.x - h.y * v.y), wi.y - (h.x * v.y + h.y * v.x));
      w[i] = wi;
      double2 dwi = wi;
      if (weighted) {
        const double2 dv = dvj[i];
        dwi = dw[i];
        dwi = make_double2(dwi.x - (h.x * dv.x - h.y * dv.y), dwi.y - (h.x * dv.y + h.y * dv.x));
        dw[i] = dwi;
      }
      const double2 x = last ? wi : vn[i];
      acc.x += x.x * dwi.x + x.y * dwi.y;
      acc.y += x.x * dwi.y - x.y * dwi.x;
    }
    acc = block_sum2(acc, red);
    if (threadIdx.x == 0) a.partials[((s + 1) & 1) * G + blockIdx.x] = acc;
    grid.sync();
  }
  const double hnorm2 = reduce_partials(a.partials + (nsteps & 1) * G, G, bcast).x;
  const double hlast = sqrt(fmax(hnorm2, 0.0));
  __syncthreads();
  if (threadIdx.x == 0) col[m] = make_double2(hlast, 0.0);
  __syncthreads();
  double cmax = 0.0;
  for (int j = 0; j <= m; ++j) cmax = fmax(cmax, hypot(col[j].x, col[j].y));
  const bool breakdown = hlast <= 1e-13 * cmax;
  if (!breakdown) {
    for (int64_t i = tid0; i < n; i += stride) {
      const double2 wi = w[i];
      w[i] = make_double2(wi.x / hlast, wi.y / hlast);
      if (weighted) {
        const double2 d = dw[i];
        dw[i] = make_double2(d.x / hlast, d.y / hlast);
      }
    }
    if (a.check_drift) {
      // partial vdot(V_j, DV_m) for all j < m over this thread's slice
      for (int j = 0; j < m; ++j) {
        const double2* vj = a.V + (int64_t)j * n;
        double2 acc = make_double2(0.0, 0.0);
        for (int64_t i = tid0; i < n; i += stride) {
          const double2 x = vj[i], y = dw[i];
          acc.x += x.x * y.x + x.y * y.y;
          acc.y += x.x * y.y - x.y * y.x;
        }
        acc = block_sum2(acc, red);
        if (threadIdx.x == 0) a.dpart[(int64_t)j * G + blockIdx.x] = acc;
      }
      grid.sync();
    }
  }
  if (blockIdx.x != 0) return;
  // ---- CTA 0: drift reduction + Givens (krylov.py:153, 162-187) ----
  if (!breakdown && a.check_drift) {
    double dmax = 0.0;
    for (int j = threadIdx.x >> 5; j < m; j += blockDim.x >> 5) {
      double2 s2 = make_double2(0.0, 0.0);
      for (int b = threadIdx.x & 31; b < G; b += 32) {
        const double2 v = __ldcg(a.dpart + (int64_t)j * G + b);
        s2.x += v.x;
        s2.y += v.y;
      }
      s2 = warp_sum2(s2);
      dmax = fmax(dmax, hypot(s2.x, s2.y));
    }
    dmax = warp_max(dmax);
    __syncthreads();
    if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5].x = dmax;
    __syncthreads();
    if (threadIdx.x == 0) {
      double d = 0.0;
      for (int k = 0; k < (int)(blockDim.x >> 5); ++k) d = fmax(d, red[k].x);
      a.drift[m] = d;
    }
  }
  if (threadIdx.x != 0) return;
  for (int j = 0; j < m - 1; ++j) {
    const double2 csj = a.cs[j], snj = a.sn[j];
    const double2 t = cadd(cmul(csj, col[j]), cmul(snj, col[j + 1]));
    col[j + 1] = cadd(cmul(cneg(cconj(snj)), col[j]), cmul(csj, col[j + 1]));
    col[j] = t;
  }
  const double am1 = hypot(col[m - 1].x, col[m - 1].y);
  const double am = hypot(col[m].x, col[m].y);
  const double denom = hypot(am1, am);
  double2 csm, snm;
  if (denom == 0.0) {
    csm = make_double2(1.0, 0.0);
    snm = make_double2(0.0, 0.0);
  } else {
    csm = make_double2(am1 / denom, 0.0);
    const double2 phase = am1 > 0 ? make_double2(col[m - 1].x / am1, col[m - 1].y / am1)
                                  : make_double2(1.0, 0.0);
    const double2 p = cmul(phase, cconj(col[m]));
    snm = make_double2(p.x / denom, p.y / denom);
  }
  a.cs[m - 1] = csm;
  a.sn[m - 1] = snm;
  double2* Hc = a.H + (int64_t)(m - 1) * (a.maxit + 1);
  for (int j = 0; j <= m; ++j) Hc[j] = col[j];
  Hc[m - 1] = cadd(cmul(csm, col[m - 1]), cmul(snm, col[m]));
  Hc[m] = make_double2(0.0, 0.0);
  const double2 gm1 = a.g[m - 1];
  a.g[m] = cmul(cneg(cconj(snm)), gm1);
  a.g[m - 1] = cmul(csm, gm1);
  const double rel = fmin(hypot(a.g[m].x, a.g[m].y) / *a.beta, a.hist[m - 1]);
  a.hist[m] = rel;
  const int done = (breakdown || rel <= a.tol) ? 1 : 0;
  a.status[1] = breakdown ? 1 : 0;
  a.status[2] = m;
  __threadfence_system();
  a.status[0] = done;
  __threadfence_system();
}

// beta = sqrt(Re vdot(r, dr)); V0 = r/beta, DV0 = dr/beta, g[0]=beta, hist[0]=1
__global__ void k_init_basis(int64_t n, const double2* r, const double2* dr, double2* V0,
                             double2* DV0, double* beta_out, double2* g, double* hist,
                             double2* part, int phase) {
  __shared__ double2 red[32];
  if (phase == 0) {
    double2 acc = make_double2(0.0, 0.0);
    for (int64_t i = threadIdx.x; i < n; i += blockDim.x) {
      const double2 x = r[i], y = dr[i];
      acc.x += x.x * y.x + x.y * y.y;
      acc.y += x.x * y.y - x.y * y.x;
    }
    acc = block_sum2(acc, red);
    if (threadIdx.x == 0) {
      const double beta = sqrt(acc.x);
      *beta_out = beta;
      g[0] = make_double2(beta, 0.0);
      hist[0] = 1.0;
    }
    return;
  }
  const double beta = *beta_out;
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x) {
    const double2 x = r[i];
    V0[i] = make_double2(x.x / beta, x.y / beta);
    if (DV0) {
      const double2 d = dr[i];
      DV0[i] = make_double2(d.x / beta, d.y / beta);
    }
  }
}

// update[e] = sum_i y[i] V_i[e], sequential in i (krylov.py:193-195)
__global__ void k_combine_basis(int64_t n, int m, const double2* V, const double2* y,
                                double2* out) {
  for (int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; e < n;
       e += (int64_t)gridDim.x * blockDim.x) {
    double2 acc = make_double2(0.0, 0.0);
    for (int i = 0; i < m; ++i) acc = cadd(acc, cmul(y[i], V[(int64_t)i * n + e]));
    out[e] = acc;
  }
}

// y[i] = (g[i] - H[i, i+1:m] @ y[i+1:m]) / H[i,i]   (krylov.py:190-192)
__global__ void k_backsub(int m, int maxit, const double2* H, const double2* g, double2* y) {
  if (threadIdx.x != 0 || blockIdx.x != 0) return;
  const int ld = maxit + 1;
  for (int i = m - 1; i >= 0; --i) {
    double2 s = make_double2(0.0, 0.0);
    for (int j = i + 1; j < m; ++j) s = cadd(s, cmul(H[(int64_t)j * ld + i], y[j]));
    y[i] = cdiv(csub(g[i], s), H[(int64_t)i * ld + i]);
  }
}

__global__ void k_axpy_out(int64_t n, const double2* x0, const double2* u, double2* x) {
  for (int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; e < n;
       e += (int64_t)gridDim.x * blockDim.x)
    x[e] = x0 ? cadd(x0[e], u[e]) : u[e];
}

struct OpRunner {
  mdd_ctx* ctx;
  const mdd_gmres_ops* ops;
  int64_t n;
  cudaStream_t s;
  mdd_complex* hin = nullptr;
  mdd_complex* hout = nullptr;
  void host_call(mdd_host_op fn, void* user, const double2* in, double2* out) {
    CK(cudaMemcpyAsync(hin, in, sizeof(double2) * n, cudaMemcpyDeviceToHost, s));
    CK(cudaStreamSynchronize(s));
    const int rc = fn(user, n, hin, hout);
    if (rc != 0) fail(MDD_EINVAL, "host operator callback failed");
    CK(cudaMemcpyAsync(out, hout, sizeof(double2) * n, cudaMemcpyHostToDevice, s));
  }
  void A(const double2* in, double2* out) {
    if (ops->A) spmv_dev(ctx, ops->A, in, out, s);
    else host_call(ops->a_fn, ops->a_user, in, out);
  }
  bool has_M() const { return ops->P || ops->m_fn || ops->Mcsr; }
  void M(const double2* in, double2* out) {
    if (ops->P) prec_apply_dev(ops->P, in, out, s);
    else if (ops->Mcsr) spmv_dev(ctx, ops->Mcsr, in, out, s);
    else host_call(ops->m_fn, ops->m_user, in, out);
  }
};

}  // namespace mdd

using namespace mdd;

extern "C" int mdd_gmres(mdd_ctx* ctx, const mdd_gmres_ops* ops, int64_t n, const mdd_complex* b,
                         const mdd_complex* x0, const mdd_gmres_cfg* cfg, mdd_complex* x,
                         double* history, double* drift, mdd_complex* basis,
                         int32_t* iterations, int32_t* converged, double* seconds) {
  MDD_API_BEGIN
  CK(cudaSetDevice(ctx->device));
  auto t0 = std::chrono::steady_clock::now();
  cudaStream_t s = ctx->stream;
  const int maxit = cfg->maxit;
  if (maxit < 1) fail(MDD_EINVAL, "maxit must be >= 1");
  if (maxit > 8000) fail(MDD_EINVAL, "maxit too large for the device Arnoldi (<= 8000)");
  if (!ops->A && !ops->a_fn) fail(MDD_EINVAL, "gmres: no operator");
  if (ops->A && (ops->A->nrow() != n || ops->A->ncol() != n))
    fail(MDD_EINVAL, "gmres: operator dimension mismatch");
  OpRunner op{ctx, ops, n, s};
  if (ops->a_fn || ops->m_fn) {
    CK(cudaMallocHost(&op.hin, sizeof(double2) * (n ? n : 1)));
    CK(cudaMallocHost(&op.hout, sizeof(double2) * (n ? n : 1)));
  }
  struct HostFree {
    OpRunner& o;
    ~HostFree() {
      if (o.hin) cudaFreeHost(o.hin);
      if (o.hout) cudaFreeHost(o.hout);
    }
  } hf{op};
  const bool weighted = ops->D != nullptr;
  const bool right = cfg->side == 0;
  DevBuf<double2> V((size_t)(maxit + 1) * n), DV, db(n), dx0, r(n), dr, z(n), t(n);
  if (weighted) {
    DV.alloc((size_t)(maxit + 1) * n);
    dr.alloc(n);
  }
  const bool dio = cfg->device_io != 0;
  if (dio) {
    CK(cudaMemcpyAsync(db.p, b, sizeof(double2) * n, cudaMemcpyDeviceToDevice, s));
    if (x0) {
      dx0.alloc(n);
      CK(cudaMemcpyAsync(dx0.p, x0, sizeof(double2) * n, cudaMemcpyDeviceToDevice, s));
    }
  } else {
    db.upload(reinterpret_cast<const double2*>(b), n, s);
    if (x0) dx0.upload(reinterpret_cast<const double2*>(x0), n, s);
  }

  // r0 (krylov.py:94-106)
  if (x0) {
    op.A(dx0.p, t.p);
    vec_sub(ctx, db.p, t.p, r.p, n, s);
  } else {
    CK(cudaMemcpyAsync(r.p, db.p, sizeof(double2) * n, cudaMemcpyDeviceToDevice, s));
  }
  if (!right && op.has_M()) {
    op.M(r.p, t.p);
    CK(cudaMemcpyAsync(r.p, t.p, sizeof(double2) * n, cudaMemcpyDeviceToDevice, s));
  }
  if (weighted) spmv_dev(ctx, ops->D, r.p, dr.p, s);

  DevBuf<double2> H((size_t)(maxit + 1) * maxit), cs(maxit), sn(maxit), g(maxit + 1), y(maxit);
  DevBuf<double> hist(maxit + 1), dbeta(1), ddrift(maxit + 1);
  H.zero(s);
  cs.zero(s);
  sn.zero(s);
  g.zero(s);
  {
    std::vector<double> nanv(maxit + 1, NAN);
    ddrift.upload(nanv, s);
  }
  // grid for the cooperative kernel
  const int bs = 256;
  int per_sm = 0;
  const size_t shmem = sizeof(double2) * (maxit + 1);
  CK(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, k_arnoldi, bs, shmem));
  if (per_sm < 1) fail(MDD_ECUDA, "arnoldi kernel cannot be resident");
  int G = ctx->nsm * std::min(per_sm, 4);
  const int64_t need = (n + bs - 1) / bs;
  if (need < G) G = (int)std::max<int64_t>(1, need);
  DevBuf<double2> partials(2 * G), dpart(cfg->check_drift ? (size_t)maxit * G : 1);

  k_init_basis<<<1, 1024, 0, s>>>(n, r.p, weighted ? dr.p : r.p, V.p, nullptr, dbeta.p, g.p,
                                  hist.p, nullptr, 0);
  CK_LAUNCH(ctx);
  double beta = 0.0;
  dbeta.download(&beta, 1, s);
  CK(cudaStreamSynchronize(s));
  if (beta == 0.0) {
    // zero residual: 0 iterations (krylov.py:110-118)
    if (dio) {
      if (x0) CK(cudaMemcpyAsync(x, x0, sizeof(double2) * n, cudaMemcpyDeviceToDevice, s));
      else CK(cudaMemsetAsync(x, 0, sizeof(double2) * n, s));
      CK(cudaStreamSynchronize(s));
    } else if (x0) {
      memcpy(x, x0, sizeof(mdd_complex) * n);
    } else {
      memset(x, 0, sizeof(mdd_complex) * n);
    }
    history[0] = 0.0;
    *iterations = 0;
    *converged = 1;
    *seconds = std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
    return MDD_OK;
  }
  k_init_basis<<<std::max<unsigned>(1, (unsigned)std::min<int64_t>((n + 255) / 256, 4096)), 256, 0,
                 s>>>(n, r.p, weighted ? dr.p : r.p, V.p, weighted ? DV.p : nullptr, dbeta.p, g.p,
                      hist.p, nullptr, 1);
  CK_LAUNCH(ctx);

  int* status = nullptr;
  CK(cudaHostAlloc(&status, sizeof(int) * 4, cudaHostAllocMapped));
  struct StFree {
    int* p;
    ~StFree() { cudaFreeHost(p); }
  } sf{status};
  int* status_dev = nullptr;
  CK(cudaHostGetDevicePointer(&status_dev, status, 0));

  cudaEvent_t ev[4];
  for (auto& e : ev) CK(cudaEventCreate(&e));
  double t_op = 0, t_prec = 0, t_arn = 0;
  int m = 0;
  bool done = false;
  for (m = 1; m <= maxit; ++m) {
    double2* vprev = V.p + (int64_t)(m - 1) * n;
    double2* w = V.p + (int64_t)m * n;
    if (ctx->timing) CK(cudaEventRecord(ev[0], s));
    if (right) {
      if (op.has_M()) {
        op.M(vprev, z.p);
        if (ctx->timing) CK(cudaEventRecord(ev[1], s));
        op.A(z.p, w);
      } else {
        if (ctx->timing) CK(cudaEventRecord(ev[1], s));
        op.A(vprev, w);
      }
    } else {
      if (op.has_M()) {
        op.A(vprev, t.p);
        if (ctx->timing) CK(cudaEventRecord(ev[1], s));
        op.M(t.p, w);
      } else {
        if (ctx->timing) CK(cudaEventRecord(ev[1], s));
        op.A(vprev, w);
      }
    }
    if (weighted) spmv_dev(ctx, ops->D, w, DV.p + (int64_t)m * n, s);
    if (ctx->timing) CK(cudaEventRecord(ev[2], s));
    status[0] = 0;
    ArnoldiArgs aa{n,       m,      maxit,  V.p,    weighted ? DV.p : nullptr,
                   partials.p, dpart.p, H.p, cs.p,   sn.p,
                   g.p,     hist.p, ddrift.p, dbeta.p, cfg->tol,
                   cfg->check_drift, status_dev};
    void* args[] = {&aa};
    CK(cudaLaunchCooperativeKernel((void*)k_arnoldi, dim3(G), dim3(bs), args, shmem, s));
    CK_LAUNCH(ctx);
    if (ctx->timing) CK(cudaEventRecord(ev[3], s));
    CK(cudaStreamSynchronize(s));
    if (ctx->timing) {
      float a = 0, b2 = 0, c = 0;
      CK(cudaEventElapsedTime(&a, ev[0], ev[1]));
      CK(cudaEventElapsedTime(&b2, ev[1], ev[2]));
      CK(cudaEventElapsedTime(&c, ev[2], ev[3]));
      if (right) { t_prec += a; t_op += b2; } else { t_op += a; t_prec += b2; }
      t_arn += c;
    }
    if (((volatile int*)status)[0]) {
      done = true;
      break;
    }
  }
  if (m > maxit) m = maxit;
  const bool breakdown = done && status[1];
  // solution (krylov.py:189-198)
  k_backsub<<<1, 32, 0, s>>>(m, maxit, H.p, g.p, y.p);
  CK_LAUNCH(ctx);
  k_combine_basis<<<std::max<unsigned>(1, (unsigned)std::min<int64_t>((n + 255) / 256, 8192)), 256,
                    0, s>>>(n, m, V.p, y.p, t.p);
  CK_LAUNCH(ctx);
  double2* upd = t.p;
  if (right && op.has_M()) {
    op.M(t.p, z.p);
    upd = z.p;
  }
  DevBuf<double2> dxo(dio ? 0 : n);
  double2* xout = dio ? reinterpret_cast<double2*>(x) : dxo.p;
  k_axpy_out<<<std::max<unsigned>(1, (unsigned)std::min<int64_t>((n + 255) / 256, 8192)), 256, 0,
               s>>>(n, x0 ? dx0.p : nullptr, upd, xout);
  CK_LAUNCH(ctx);
  if (!dio) dxo.download(reinterpret_cast<double2*>(x), n, s);
  hist.download(history, m + 1, s);
  if (drift) ddrift.download(drift, m + 1, s);
  if (basis) {
    const int nb = breakdown ? m : m + 1;
    V.download(reinterpret_cast<double2*>(basis), (size_t)nb * n, s);
  }
  CK(cudaStreamSynchronize(s));
  for (auto& e : ev) cudaEventDestroy(e);
  if (ctx->timing) {
    ctx->timers[0] = t_op;
    ctx->timers[1] = t_prec;
    ctx->timers[2] = t_arn;
  }
  *iterations = m;
  *converged = done ? (breakdown ? 2 : 1) : 0;  // 2: happy breakdown
  *seconds = std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
  MDD_API_END
}
