// Second-order Nedelec (first kind, 20 DoFs per tet) fine space: CSR pattern,
// coloured device assembly and load vector.
//
// No reference counterpart: the reference implements lowest-order Whitney
// elements only (reference fem.py:1-7).  BASELINE.json config 2
// asks for a second-order fine space with a lowest-order coarse space; this
// file is its device assembly (SURVEY.md §8f rank 2, §8c "cfg2: no oracle").
//
// Hierarchical basis, defined on each tet with its vertices sorted by global
// index (so every orientation is the global one and neighbouring tets agree
// on shared edges and faces):
//   k = 0..5   Whitney      w_ab = l_a grad l_b - l_b grad l_a   (a<b, LOCAL_EDGES order)
//   k = 6..11  edge grads   grad(l_a l_b)
//   k = 12+2f  face         l_c w_ab     (face f = sorted (a,b,c), LOCAL_FACES order)
//   k = 13+2f  face         l_a w_bc
// The Whitney block is exactly the lowest-order element, so the lowest-order
// coarse space is nested in the fine space with the order-1 R0 on the Whitney
// DoFs and zeros elsewhere, and R0 A R0^T equals the order-1 Galerkin matrix.
//
// Each basis function is phi_k = sum_i p_ki(l) grad l_i with p_ki of degree
// <= 2, and curl phi_k = sum_{a<b} q_k,ab(l) (grad l_a x grad l_b) with
// q_ab = d p_b/d l_a - d p_a/d l_b.  Hence
//   M_kl = |T| sum_{i<=j} (grad l_i . grad l_j) CM[kl][ij]
//   S_kl = |T| sum_{P<=Q} (X_P . X_Q)            CS[kl][PQ],   X_ab = grad l_a x grad l_b
// with CM, CS universal rationals (exact integrals of barycentric monomials,
// int_T l^alpha = 6|T| alpha! / (|alpha|+3)!) computed once on the host.
#include <algorithm>
#include <array>
#include <cmath>
#include <map>
#include <mutex>
#include <numeric>
#include <thread>

#include "fem_device.cuh"
#include "mdd_internal.h"
#include "mdd_kernels.cuh"

namespace mdd {

constexpr int kL2 = 20;            // local DoFs per tet
constexpr int kP2 = kL2 * (kL2 + 1) / 2;  // upper-triangle entries (210)
constexpr int kMon = 15;           // monomials of degree <= 2 in 4 variables

// ------------------------------------------------------------ host tables
namespace {
using Expo = std::array<int, 4>;
using Poly = std::map<Expo, double>;

Poly mono(std::initializer_list<int> vars, double c = 1.0) {
  Expo e{0, 0, 0, 0};
  for (int v : vars) e[v]++;
  return Poly{{e, c}};
}
Poly add(const Poly& a, const Poly& b, double sb = 1.0) {
  Poly r = a;
  for (auto& kv : b) r[kv.first] += sb * kv.second;
  return r;
}
Poly mul(const Poly& a, const Poly& b) {
  Poly r;
  for (auto& x : a)
    for (auto& y : b) {
      Expo e;
      for (int i = 0; i < 4; ++i) e[i] = x.first[i] + y.first[i];
      r[e] += x.second * y.second;
    }
  return r;
}
Poly deriv(const Poly& a, int v) {
  Poly r;
  for (auto& x : a)
    if (x.first[v] > 0) {
      Expo e = x.first;
      const double c = x.second * e[v];
      e[v]--;
      r[e] += c;
    }
  return r;
}
double fact(int n) {
  double f = 1;
  for (int i = 2; i <= n; ++i) f *= i;
  return f;
}
// int_T poly / |T|
double integ(const Poly& p) {
  double s = 0;
  for (auto& x : p) {
    const Expo& e = x.first;
    const int deg = e[0] + e[1] + e[2] + e[3];
    s += x.second * 6.0 * fact(e[0]) * fact(e[1]) * fact(e[2]) * fact(e[3]) / fact(deg + 3);
  }
  return s;
}

const int EA[6] = {0, 0, 0, 1, 1, 2}, EB[6] = {1, 2, 3, 2, 3, 3};
const int FV[4][3] = {{1, 2, 3}, {0, 2, 3}, {0, 1, 3}, {0, 1, 2}};

struct Tables {
  double cm[kP2][10];
  double cs[kP2][21];
  double ptab[kL2][4][kMon];  // p_ki as monomial coefficients (rhs)
  int16_t kl[kP2][2];
};

int mono_index(const Expo& e) {
  // 0: 1; 1..4: l_i; 5..14: l_i l_j (i<=j) in row-major order
  const int deg = e[0] + e[1] + e[2] + e[3];
  if (deg == 0) return 0;
  int idx[2], n = 0;
  for (int i = 0; i < 4; ++i)
    for (int r = 0; r < e[i]; ++r) idx[n++] = i;
  if (deg == 1) return 1 + idx[0];
  int k = 5;
  for (int i = 0; i < 4; ++i)
    for (int j = i; j < 4; ++j, ++k)
      if (i == idx[0] && j == idx[1]) return k;
  return -1;
}

Tables build_tables() {
  Tables T{};
  // p[k][i]
  std::vector<std::array<Poly, 4>> p(kL2);
  for (int e = 0; e < 6; ++e) {
    const int a = EA[e], b = EB[e];
    p[e][a] = mono({b}, -1.0);
    p[e][b] = mono({a}, 1.0);
    p[6 + e][a] = mono({b});
    p[6 + e][b] = mono({a});
  }
  for (int f = 0; f < 4; ++f) {
    const int a = FV[f][0], b = FV[f][1], c = FV[f][2];
    // l_c w_ab = l_c l_a grad l_b - l_c l_b grad l_a
    p[12 + 2 * f][a] = mono({b, c}, -1.0);
    p[12 + 2 * f][b] = mono({a, c}, 1.0);
    // l_a w_bc = l_a l_b grad l_c - l_a l_c grad l_b
    p[13 + 2 * f][b] = mono({a, c}, -1.0);
    p[13 + 2 * f][c] = mono({a, b}, 1.0);
  }
  // curls q[k][P], P over the 6 pairs
  std::vector<std::array<Poly, 6>> q(kL2);
  for (int k = 0; k < kL2; ++k)
    for (int P = 0; P < 6; ++P) q[k][P] = add(deriv(p[k][EB[P]], EA[P]), deriv(p[k][EA[P]], EB[P]), -1.0);
  int e = 0;
  for (int k = 0; k < kL2; ++k)
    for (int l = k; l < kL2; ++l, ++e) {
      T.kl[e][0] = (int16_t)k;
      T.kl[e][1] = (int16_t)l;
      int u = 0;
      for (int i = 0; i < 4; ++i)
        for (int j = i; j < 4; ++j, ++u)
          T.cm[e][u] = (i == j) ? integ(mul(p[k][i], p[l][i]))
                                : integ(add(mul(p[k][i], p[l][j]), mul(p[k][j], p[l][i])));
      u = 0;
      for (int P = 0; P < 6; ++P)
        for (int Q = P; Q < 6; ++Q, ++u)
          T.cs[e][u] = (P == Q) ? integ(mul(q[k][P], q[l][P]))
                                : integ(add(mul(q[k][P], q[l][Q]), mul(q[k][Q], q[l][P])));
    }
  for (int k = 0; k < kL2; ++k)
    for (int i = 0; i < 4; ++i)
      for (auto& x : p[k][i]) T.ptab[k][i][mono_index(x.first)] += x.second;
  return T;
}
}  // namespace

// device copies (per device, uploaded once)
__device__ double g_cm[kP2][10];
__device__ double g_cs[kP2][21];
__device__ double g_ptab[kL2][4][kMon];
__device__ int16_t g_kl[kP2][2];

static void ensure_tables(int device) {
  static std::mutex mu;
  static std::vector<int> done;
  std::lock_guard<std::mutex> g(mu);
  if (std::find(done.begin(), done.end(), device) != done.end()) return;
  static const Tables T = build_tables();
  CK(cudaMemcpyToSymbol(g_cm, T.cm, sizeof(T.cm)));
  CK(cudaMemcpyToSymbol(g_cs, T.cs, sizeof(T.cs)));
  CK(cudaMemcpyToSymbol(g_ptab, T.ptab, sizeof(T.ptab)));
  CK(cudaMemcpyToSymbol(g_kl, T.kl, sizeof(T.kl)));
  done.push_back(device);
}

// ------------------------------------------------------------ kernels
struct Geom2 {
  double G[10];  // grad l_i . grad l_j, i <= j
  double X[21];  // X_P . X_Q, P <= Q
  double vol;
  double g[4][3];
};

__device__ __forceinline__ void geom2(const double* __restrict__ verts, const int32_t* __restrict__ tets,
                                      int64_t t, Geom2& o, double (&c)[4][3]) {
#pragma unroll
  for (int i = 0; i < 4; ++i) {
    const int v = tets[t * 4 + i];
#pragma unroll
    for (int k = 0; k < 3; ++k) c[i][k] = verts[(int64_t)v * 3 + k];
  }
  TetGeom tg;
  tet_geometry(c, tg);
  o.vol = fabs(tg.det) / 6.0;
#pragma unroll
  for (int i = 0; i < 4; ++i)
#pragma unroll
    for (int k = 0; k < 3; ++k) o.g[i][k] = tg.g[i][k];
  int u = 0;
#pragma unroll
  for (int i = 0; i < 4; ++i)
#pragma unroll
    for (int j = i; j < 4; ++j, ++u)
      o.G[u] = tg.g[i][0] * tg.g[j][0] + tg.g[i][1] * tg.g[j][1] + tg.g[i][2] * tg.g[j][2];
  double X[6][3];
#pragma unroll
  for (int P = 0; P < 6; ++P) {
    const double* ga = tg.g[kEA[P]];
    const double* gb = tg.g[kEB[P]];
    X[P][0] = ga[1] * gb[2] - ga[2] * gb[1];
    X[P][1] = ga[2] * gb[0] - ga[0] * gb[2];
    X[P][2] = ga[0] * gb[1] - ga[1] * gb[0];
  }
  u = 0;
#pragma unroll
  for (int P = 0; P < 6; ++P)
#pragma unroll
    for (int Q = P; Q < 6; ++Q, ++u) o.X[u] = X[P][0] * X[Q][0] + X[P][1] * X[Q][1] + X[P][2] * X[Q][2];
}

__device__ __forceinline__ void entry2(const Geom2& g, int e, double& sv, double& mv) {
  double m = 0.0, s = 0.0;
#pragma unroll
  for (int u = 0; u < 10; ++u) m += g.G[u] * g_cm[e][u];
#pragma unroll
  for (int u = 0; u < 21; ++u) s += g.X[u] * g_cs[e][u];
  sv = g.vol * s;
  mv = g.vol * m;
}

struct Coef2 {
  const double* eps;
  const double* mu;
  const double* sigma;
  double eps0, mu0, sigma0;
  double k, xi;
};

// One warp per cell of one colour: for each of the cell's 6 tets the lanes
// take the 210 upper-triangle entries (k<=l) of the 20x20 element matrices
// and add them into the (k,l) and (l,k) CSR slots.  Slots of one tet are
// distinct, the tets of a cell follow in order, cells of one colour share no
// edge or face: no atomics, fixed summation order.
__global__ void __launch_bounds__(128) k_assemble2_cells(
    const int32_t* __restrict__ cells, int64_t ncells, const double* __restrict__ verts,
    const int32_t* __restrict__ tets, const int32_t* __restrict__ tdofs,
    const int32_t* __restrict__ rowptr, const int32_t* __restrict__ cols, double* __restrict__ S,
    double* __restrict__ M, double2* __restrict__ A, Coef2 co) {
  const int64_t ci = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const int lane = threadIdx.x & 31;
  if (ci >= ncells) return;
  const int64_t cell = cells[ci];
  for (int p = 0; p < 6; ++p) {
    const int64_t t = cell * 6 + p;
    Geom2 g;
    double c[4][3];
    geom2(verts, tets, t, g, c);
    double2 w = make_double2(0.0, 0.0);
    double imu = 1.0;
    if (A) {
      const double eps = co.eps ? co.eps[t] : co.eps0;
      const double mu = co.mu ? co.mu[t] : co.mu0;
      const double sig = co.sigma ? co.sigma[t] : co.sigma0;
      w = make_double2(co.k * co.k * eps, co.xi * eps + co.k * sig);
      imu = mu;
    }
    for (int e = lane; e < kP2; e += 32) {
      const int k = g_kl[e][0], l = g_kl[e][1];
      const int dk = tdofs[t * kL2 + k], dl = tdofs[t * kL2 + l];
      if (dk < 0 || dl < 0) continue;
      double sv, mv;
      entry2(g, e, sv, mv);
      const int nslot = (k == l) ? 1 : 2;
      for (int h = 0; h < nslot; ++h) {
        const int slot = h == 0 ? csr_find(rowptr, cols, dk, dl) : csr_find(rowptr, cols, dl, dk);
        S[slot] += sv;
        M[slot] += mv;
        if (A) {
          const double sm = sv / imu;
          double2 v = A[slot];
          v.x += sm - w.x * mv;
          v.y += -w.y * mv;
          A[slot] = v;
        }
      }
    }
    __syncwarp();
  }
}

__device__ __forceinline__ double mono_eval(int m, const double (&l)[4]) {
  if (m == 0) return 1.0;
  if (m < 5) return l[m - 1];
  int k = 5;
  for (int i = 0; i < 4; ++i)
    for (int j = i; j < 4; ++j, ++k)
      if (k == m) return l[i] * l[j];
  return 0.0;
}

// contrib[t*20 + k] = sum_q w_q |T| F(x_q) . phi_k(x_q)
// F from fvals (nq, nt, 3) or the device Gaussian when fvals == nullptr.
__global__ void __launch_bounds__(128) k_rhs2_contrib(int64_t nt, const double* __restrict__ verts,
                                                      const int32_t* __restrict__ tets, int nq,
                                                      const double* __restrict__ qbary,
                                                      const double* __restrict__ qw,
                                                      const double2* __restrict__ fvals, GaussSrc gs,
                                                      double2* __restrict__ contrib) {
  const int64_t t = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (t >= nt) return;
  Geom2 g;
  double c[4][3];
  geom2(verts, tets, t, g, c);
  double2 acc[kL2];
#pragma unroll
  for (int k = 0; k < kL2; ++k) acc[k] = make_double2(0.0, 0.0);
  for (int q = 0; q < nq; ++q) {
    double l[4];
#pragma unroll
    for (int i = 0; i < 4; ++i) l[i] = qbary[q * 4 + i];
    double2 F[3];
    if (fvals) {
#pragma unroll
      for (int k = 0; k < 3; ++k) F[k] = fvals[((int64_t)q * nt + t) * 3 + k];
    } else {
      double x[3];
#pragma unroll
      for (int k = 0; k < 3; ++k) x[k] = l[0] * c[0][k] + l[1] * c[1][k] + l[2] * c[2][k] + l[3] * c[3][k];
      const double r2 = (x[0] - gs.cx) * (x[0] - gs.cx) + (x[1] - gs.cy) * (x[1] - gs.cy) +
                        (x[2] - gs.cz) * (x[2] - gs.cz);
      const double f = gs.amp * exp(-gs.alpha * r2);
      F[0] = make_double2(f * gs.dx, 0.0);
      F[1] = make_double2(f * gs.dy, 0.0);
      F[2] = make_double2(f * gs.dz, 0.0);
    }
    // F . grad l_i, then phi_k . F = sum_i p_ki(l) (F . grad l_i)
    double2 fg[4];
#pragma unroll
    for (int i = 0; i < 4; ++i)
      fg[i] = make_double2(F[0].x * g.g[i][0] + F[1].x * g.g[i][1] + F[2].x * g.g[i][2],
                           F[0].y * g.g[i][0] + F[1].y * g.g[i][1] + F[2].y * g.g[i][2]);
    double mv[kMon];
#pragma unroll
    for (int m = 0; m < kMon; ++m) mv[m] = mono_eval(m, l);
    const double wq = qw[q] * g.vol;
    for (int k = 0; k < kL2; ++k) {
      double2 s = make_double2(0.0, 0.0);
#pragma unroll
      for (int i = 0; i < 4; ++i) {
        double pv = 0.0;
#pragma unroll
        for (int m = 0; m < kMon; ++m) pv += g_ptab[k][i][m] * mv[m];
        s.x += pv * fg[i].x;
        s.y += pv * fg[i].y;
      }
      acc[k].x += wq * s.x;
      acc[k].y += wq * s.y;
    }
  }
#pragma unroll
  for (int k = 0; k < kL2; ++k) contrib[t * kL2 + k] = acc[k];
}

// rhs[i] = sum over incident (t,k), ascending t (fixed order)
__global__ void k_rhs2_gather(int64_t ndof, const int32_t* __restrict__ inc_ptr,
                              const int32_t* __restrict__ inc, const double2* __restrict__ contrib,
                              double2* __restrict__ rhs) {
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < ndof;
       i += (int64_t)gridDim.x * blockDim.x) {
    double2 acc = make_double2(0.0, 0.0);
    for (int k = inc_ptr[i]; k < inc_ptr[i + 1]; ++k) {
      const double2 v = contrib[inc[k]];
      acc.x += v.x;
      acc.y += v.y;
    }
    rhs[i] = acc;
  }
}

// element matrices of single tets (sorted-frame basis), for tests
__global__ void k_element2_batch(int64_t nt, const double* __restrict__ coords, double* s_el,
                                 double* m_el) {
  const int64_t t = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (t >= nt) return;
  int32_t tv[4] = {0, 1, 2, 3};
  Geom2 g;
  double c[4][3];
  geom2(coords + t * 12, tv, 0, g, c);
  for (int e = 0; e < kP2; ++e) {
    const int k = g_kl[e][0], l = g_kl[e][1];
    double sv, mv;
    entry2(g, e, sv, mv);
    s_el[t * 400 + k * 20 + l] = s_el[t * 400 + l * 20 + k] = sv;
    m_el[t * 400 + k * 20 + l] = m_el[t * 400 + l * 20 + k] = mv;
  }
}

static unsigned nb2(int64_t n, int bs) { return (unsigned)std::max<int64_t>(1, (n + bs - 1) / bs); }

void assemble_system2(mdd_space* sp, const mdd_coeffs* co, mdd_csr** A, mdd_csr** S, mdd_csr** M,
                      mdd_csr** Dk) {
  mdd_ctx* ctx = sp->ctx;
  cudaStream_t s = ctx->stream;
  CK(cudaSetDevice(ctx->device));
  ensure_tables(ctx->device);
  std::unique_ptr<mdd_csr> cS(new_csr(ctx, sp->pat, false));
  std::unique_ptr<mdd_csr> cM(new_csr(ctx, sp->pat, false));
  std::unique_ptr<mdd_csr> cA(new_csr(ctx, sp->pat, true));
  std::unique_ptr<mdd_csr> cD;
  if (Dk) cD.reset(new_csr(ctx, sp->pat, false));
  const bool het = !co->homogeneous;
  DevBuf<double> deps, dmu, dsig;
  Coef2 cd{nullptr, nullptr, nullptr, co->eps0, co->mu0, co->sigma0, co->k, co->xi};
  if (het) {
    if (co->eps) { deps.upload(co->eps, sp->nt, s); cd.eps = deps.p; }
    if (co->mu) { dmu.upload(co->mu, sp->nt, s); cd.mu = dmu.p; }
    if (co->sigma) { dsig.upload(co->sigma, sp->nt, s); cd.sigma = dsig.p; }
  }
  for (int c = 0; c < 8; ++c) {
    const int64_t nc = sp->color_off[c + 1] - sp->color_off[c];
    if (!nc) continue;
    k_assemble2_cells<<<nb2(nc * 32, 128), 128, 0, s>>>(
        sp->cells_by_color.p + sp->color_off[c], nc, sp->verts.p, sp->tets.p, sp->tdofs.p,
        sp->pat->rowptr.p, sp->pat->cols.p, cS->vals.p, cM->vals.p,
        het ? reinterpret_cast<double2*>(cA->vals.p) : nullptr, cd);
    CK_LAUNCH(ctx);
  }
  const int64_t nnz = sp->pat->nnz;
  if (nnz) {
    k_combine<<<nb2(std::min<int64_t>(nnz, (int64_t)ctx->nsm * 16 * 256), 256), 256, 0, s>>>(
        nnz, cS->vals.p, cM->vals.p, reinterpret_cast<double2*>(cA->vals.p), cD ? cD->vals.p : nullptr,
        co->k * co->k, co->xi, het ? 0 : 1);
    CK_LAUNCH(ctx);
  }
  CK(cudaStreamSynchronize(s));
  if (A) *A = cA.release();
  if (S) *S = cS.release();
  if (M) *M = cM.release();
  if (Dk) *Dk = cD.release();
}

void assemble_rhs2_dev(mdd_space* sp, const double2* fvals_host, const GaussSrc* gsrc, double2* rhs_dev) {
  mdd_ctx* ctx = sp->ctx;
  cudaStream_t s = ctx->stream;
  ensure_tables(ctx->device);
  DevBuf<double2> contrib(std::max<int64_t>(1, sp->nt * kL2)), fv;
  if (fvals_host) fv.upload(fvals_host, (int64_t)sp->nq * sp->nt * 3, s);
  GaussSrc g = gsrc ? *gsrc : GaussSrc{0, 0, 0, 0, 0, 0, 0, 0};
  if (sp->nt) {
    k_rhs2_contrib<<<nb2(sp->nt, 128), 128, 0, s>>>(sp->nt, sp->verts.p, sp->tets.p, sp->nq, sp->qbary.p,
                                                    sp->qw.p, fvals_host ? fv.p : nullptr, g, contrib.p);
    CK_LAUNCH(ctx);
  }
  if (sp->ndof) {
    k_rhs2_gather<<<nb2(std::min<int64_t>(sp->ndof, (int64_t)ctx->nsm * 16 * 256), 256), 256, 0, s>>>(
        sp->ndof, sp->inc_ptr.p, sp->inc.p, contrib.p, rhs_dev);
    CK_LAUNCH(ctx);
  }
}

}  // namespace mdd

using namespace mdd;

extern "C" {

int mdd_space2_create(mdd_ctx* ctx, int32_t cells_per_axis, int64_t nv, const double* vertices, int64_t nt,
                      const int64_t* tets, const int64_t* tet_dofs, int64_t ndof, int32_t nq,
                      const double* qbary, const double* qweights, mdd_space** out) {
  MDD_API_BEGIN
  CK(cudaSetDevice(ctx->device));
  const int64_t n = cells_per_axis;
  if (n < 1 || nt != 6 * n * n * n) fail(MDD_EINVAL, "space: expected a Kuhn mesh with 6 n^3 tets");
  if (nv > INT32_MAX || nt * kL2 > INT32_MAX || ndof > INT32_MAX)
    fail(MDD_EINVAL, "space: mesh too large for int32 indexing");
  if (nq < 1 || !qbary || !qweights) fail(MDD_EINVAL, "space: order 2 needs a quadrature rule");
  ensure_tables(ctx->device);
  auto sp = std::make_unique<mdd_space>();
  sp->ctx = ctx;
  sp->order = 2;
  sp->n = cells_per_axis;
  sp->nv = nv;
  sp->nt = nt;
  sp->ne = 0;
  sp->ndof = ndof;
  sp->h_verts.assign(vertices, vertices + nv * 3);
  // vertices sorted by global index inside each tet (the basis frame)
  sp->h_tets.resize(nt * 4);
  for (int64_t t = 0; t < nt; ++t) {
    int64_t v[4] = {tets[t * 4], tets[t * 4 + 1], tets[t * 4 + 2], tets[t * 4 + 3]};
    std::sort(v, v + 4);
    for (int i = 0; i < 4; ++i) sp->h_tets[t * 4 + i] = (int32_t)v[i];
  }
  std::vector<int32_t> td(nt * kL2);
  for (int64_t i = 0; i < nt * kL2; ++i) {
    if (tet_dofs[i] >= ndof) fail(MDD_EINVAL, "space: tet_dofs out of range");
    td[i] = (int32_t)tet_dofs[i];
  }
  // cells by colour (cells of one parity colour share no edge or face)
  std::vector<int32_t> cbc;
  cbc.reserve(n * n * n);
  for (int col = 0; col < 8; ++col) {
    sp->color_off[col] = (int64_t)cbc.size();
    for (int64_t c = 0; c < n * n * n; ++c) {
      const int64_t cx = c / (n * n), cy = (c / n) % n, cz = c % n;
      if ((int)(((cx & 1) << 2) | ((cy & 1) << 1) | (cz & 1)) == col) cbc.push_back((int32_t)c);
    }
  }
  sp->color_off[8] = (int64_t)cbc.size();
  // dof -> incident (t*20 + k), ascending t
  std::vector<int32_t> iptr(ndof + 1, 0), iinc;
  for (int64_t i = 0; i < nt * kL2; ++i)
    if (td[i] >= 0) iptr[td[i] + 1]++;
  for (int64_t d = 0; d < ndof; ++d) {
    if (iptr[d + 1] == 0) fail(MDD_EINVAL, "space: dof without a tet");
    iptr[d + 1] += iptr[d];
  }
  iinc.resize(iptr[ndof]);
  {
    std::vector<int32_t> fp(iptr.begin(), iptr.end() - 1);
    for (int64_t i = 0; i < nt * kL2; ++i)
      if (td[i] >= 0) iinc[fp[td[i]]++] = (int32_t)i;
  }
  // CSR pattern: row d = sorted unique kept dofs of the tets incident to d
  auto row_of = [&](int64_t d, std::vector<int32_t>& buf) {
    buf.clear();
    int32_t last_t = -1;
    for (int32_t k = iptr[d]; k < iptr[d + 1]; ++k) {
      const int32_t t = iinc[k] / kL2;
      if (t == last_t) continue;
      last_t = t;
      for (int q = 0; q < kL2; ++q) {
        const int32_t dd = td[(int64_t)t * kL2 + q];
        if (dd >= 0) buf.push_back(dd);
      }
    }
    std::sort(buf.begin(), buf.end());
    buf.erase(std::unique(buf.begin(), buf.end()), buf.end());
  };
  std::vector<int32_t> rowcnt(ndof + 1, 0);
  const unsigned nth = std::max(1u, std::min(16u, std::thread::hardware_concurrency()));
  auto par = [&](auto&& f) {
    std::vector<std::thread> th;
    const int64_t chunk = (ndof + nth - 1) / nth;
    for (unsigned t = 0; t < nth; ++t) {
      const int64_t b = t * chunk, e = std::min<int64_t>(ndof, b + chunk);
      if (b >= e) break;
      th.emplace_back([&f, b, e] { f(b, e); });
    }
    for (auto& x : th) x.join();
  };
  par([&](int64_t b, int64_t e) {
    std::vector<int32_t> buf;
    for (int64_t d = b; d < e; ++d) {
      row_of(d, buf);
      rowcnt[d + 1] = (int32_t)buf.size();
    }
  });
  std::vector<int32_t> rowptr(ndof + 1, 0);
  for (int64_t d = 0; d < ndof; ++d) {
    if ((int64_t)rowptr[d] + rowcnt[d + 1] > INT32_MAX) fail(MDD_EINVAL, "space: nnz > 2^31");
    rowptr[d + 1] = rowptr[d] + rowcnt[d + 1];
  }
  std::vector<int32_t> cols(rowptr[ndof]);
  par([&](int64_t b, int64_t e) {
    std::vector<int32_t> buf;
    for (int64_t d = b; d < e; ++d) {
      row_of(d, buf);
      std::copy(buf.begin(), buf.end(), cols.begin() + rowptr[d]);
    }
  });
  cudaStream_t s = ctx->stream;
  sp->nq = nq;
  sp->qbary.upload(qbary, (int64_t)nq * 4, s);
  sp->qw.upload(qweights, nq, s);
  sp->verts.upload(sp->h_verts, s);
  sp->tets.upload(sp->h_tets, s);
  sp->tdofs.upload(td, s);
  sp->cells_by_color.upload(cbc, s);
  sp->inc_ptr.upload(iptr, s);
  sp->inc.upload(iinc, s);
  sp->pat = make_pattern(ndof, ndof, std::move(rowptr), std::move(cols), s);
  CK(cudaStreamSynchronize(s));
  *out = sp.release();
  MDD_API_END
}

int mdd_element2_matrices(mdd_ctx* ctx, int64_t nt, const double* coords, double* s_el, double* m_el) {
  MDD_API_BEGIN
  CK(cudaSetDevice(ctx->device));
  ensure_tables(ctx->device);
  cudaStream_t s = ctx->stream;
  DevBuf<double> dc, ds(std::max<int64_t>(1, nt * 400)), dm(std::max<int64_t>(1, nt * 400));
  dc.upload(coords, nt * 12, s);
  if (nt) {
    k_element2_batch<<<nb2(nt, 64), 64, 0, s>>>(nt, dc.p, ds.p, dm.p);
    CK_LAUNCH(ctx);
  }
  ds.download(s_el, nt * 400, s);
  dm.download(m_el, nt * 400, s);
  CK(cudaStreamSynchronize(s));
  MDD_API_END
}

}  // extern "C"
