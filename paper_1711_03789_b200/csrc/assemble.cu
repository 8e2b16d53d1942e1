// Device assembly of the Nedelec curl-curl system (reference fem.assemble,
// fem.py:233-279), the impedance boundary mass (fem.py:286-353) and the load
// vector (fem.py:367-390).
//
// The CSR pattern (all pairs of kept DOFs sharing a tetrahedron: the
// structural pattern scipy's COO->CSR produces, fem.py:225-230) is built once
// per space on the host; the numeric assembly is a coloured scatter: cells
// are split into 8 parity colours, one thread owns one cell (its 6 Kuhn
// tets), computes the 6x6 element matrices in registers and adds them into
// the CSR slots.  Cells of one colour share no edge, so no atomics are needed
// and the summation order is fixed (bitwise reproducible).
#include <algorithm>
#include <cstring>
#include <numeric>
#include <thread>

#include "fem_device.cuh"
#include "mdd_internal.h"
#include "mdd_kernels.cuh"

namespace mdd {

mdd_csr* new_csr(mdd_ctx* ctx, std::shared_ptr<mdd_pattern> pat, bool cplx) {
  auto A = new mdd_csr();
  A->ctx = ctx;
  A->pat = std::move(pat);
  A->is_complex = cplx;
  A->vals.alloc((size_t)A->nnz() * (cplx ? 2 : 1));
  A->vals.zero(ctx->stream);
  return A;
}

template <typename F>
static void parallel_for(int64_t n, F&& f) {
  unsigned nth = std::max(1u, std::min(16u, std::thread::hardware_concurrency()));
  if (n < 20000 || nth == 1) {
    f(0, n);
    return;
  }
  std::vector<std::thread> th;
  const int64_t chunk = (n + nth - 1) / nth;
  for (unsigned t = 0; t < nth; ++t) {
    const int64_t b = t * chunk, e = std::min(n, b + chunk);
    if (b >= e) break;
    th.emplace_back([&f, b, e] { f(b, e); });
  }
  for (auto& x : th) x.join();
}

// ------------------------------------------------------------- kernels
struct CoefDev {
  const double* eps;
  const double* mu;
  const double* sigma;
  double eps0, mu0, sigma0;
  double k, xi;
};

__device__ __forceinline__ void load_tet(const double* __restrict__ verts,
                                         const int32_t* __restrict__ tets,
                                         const int8_t* __restrict__ signs, int64_t t,
                                         double (&c)[4][3], double (&sg)[6]) {
#pragma unroll
  for (int i = 0; i < 4; ++i) {
    const int v = tets[t * 4 + i];
#pragma unroll
    for (int k = 0; k < 3; ++k) c[i][k] = verts[(int64_t)v * 3 + k];
  }
#pragma unroll
  for (int e = 0; e < 6; ++e) sg[e] = (double)signs[t * 6 + e];
}

// One warp per cell of one colour class: for each of the cell's 6 Kuhn tets
// the lanes compute the 36 entries of S_e, M_e (and, when heterogeneous, the
// complex a_e = S_e/mu - w M_e, fem.py:253-256) in parallel and add them into
// the CSR slots of the kept DOFs.  The 36 slots of one tet are distinct; the
// tets of a cell share slots and follow in order; cells of one colour share
// no edge -> no atomics, fixed summation order.
__global__ void __launch_bounds__(128) k_assemble_cells(
    const int32_t* __restrict__ cells, int64_t ncells, const double* __restrict__ verts,
    const int32_t* __restrict__ tets, const int32_t* __restrict__ tet_edges,
    const int8_t* __restrict__ signs, const int32_t* __restrict__ e2d,
    const int32_t* __restrict__ rowptr, const int32_t* __restrict__ cols, double* __restrict__ S,
    double* __restrict__ M, double2* __restrict__ A, CoefDev co) {
  const int64_t ci = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const int lane = threadIdx.x & 31;
  if (ci >= ncells) return;
  const int64_t cell = cells[ci];
  for (int p = 0; p < 6; ++p) {
    const int64_t t = cell * 6 + p;
    double c[4][3], sg[6];
    load_tet(verts, tets, signs, t, c, sg);
    TetGeom g;
    tet_geometry(c, g);
    double2 w = make_double2(0.0, 0.0);
    double imu = 1.0;
    if (A) {
      const double eps = co.eps ? co.eps[t] : co.eps0;
      const double mu = co.mu ? co.mu[t] : co.mu0;
      const double sig = co.sigma ? co.sigma[t] : co.sigma0;
      w = make_double2(co.k * co.k * eps, co.xi * eps + co.k * sig);
      imu = mu;
    }
    for (int e = lane; e < 36; e += 32) {
      const int a = e / 6, b = e % 6;
      const int da = e2d[tet_edges[t * 6 + a]], db = e2d[tet_edges[t * 6 + b]];
      if (da < 0 || db < 0) continue;
      double sv, mv;
      // (a,b) and (b,a) from the same evaluation: the assembled matrices are
      // bitwise complex symmetric (the factorisation's transpose path relies on it)
      element_entry(g, sg, min(a, b), max(a, b), sv, mv);
      const int slot = csr_find(rowptr, cols, da, db);
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
    __syncwarp();
  }
}

// Homogeneous: A = S - (k^2 + i xi) M entrywise (fem.py:248-252); Dk = S + k^2 M.
__global__ void k_combine(int64_t nnz, const double* __restrict__ S, const double* __restrict__ M,
                          double2* __restrict__ A, double* __restrict__ Dk, double k2, double xi,
                          int write_a) {
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < nnz;
       i += (int64_t)gridDim.x * blockDim.x) {
    const double s = S[i], m = M[i];
    if (write_a) A[i] = make_double2(s - k2 * m, -(xi * m));
    if (Dk) Dk[i] = s + k2 * m;
  }
}

// Boundary-face tangential masses (nf, 3, 3)
__global__ void k_face_mass(int64_t nf, const int32_t* __restrict__ faces,
                            const double* __restrict__ verts, double* __restrict__ out) {
  const int64_t f = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (f >= nf) return;
  double p[3][3];
  for (int i = 0; i < 3; ++i) {
    const int64_t v = faces[f * 3 + i];
    for (int k = 0; k < 3; ++k) p[i][k] = verts[v * 3 + k];
  }
  double m[3][3];
  triangle_tangential_mass(p, m);
  for (int a = 0; a < 3; ++a)
    for (int b = 0; b < 3; ++b) out[f * 9 + a * 3 + b] = m[a][b];
}

// Gather-form sum into slots: out[s] = sum_{k in [ptr[s],ptr[s+1])} src[idx[k]]
__global__ void k_slot_gather(int64_t ns, const int32_t* __restrict__ ptr,
                              const int32_t* __restrict__ idx, const double* __restrict__ src,
                              double* __restrict__ out) {
  for (int64_t s = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; s < ns;
       s += (int64_t)gridDim.x * blockDim.x) {
    double acc = 0.0;
    for (int k = ptr[s]; k < ptr[s + 1]; ++k) acc += src[idx[k]];
    out[s] = acc;
  }
}

// A[amap[s]] += coef * Mb[s]  (coef = -i*s_imp*k)
__global__ void k_imp_update(int64_t ns, const int32_t* __restrict__ amap,
                             const double* __restrict__ mb, double2* __restrict__ A, double2 coef) {
  for (int64_t s = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; s < ns;
       s += (int64_t)gridDim.x * blockDim.x) {
    const double v = mb[s];
    double2 a = A[amap[s]];
    a.x += coef.x * v;
    a.y += coef.y * v;
    A[amap[s]] = a;
  }
}

// ------------------------------------------------------------------ rhs
// degree-2 rule, 4 points, weights |T|/4 (fem.py:367-370)
__device__ __forceinline__ double qlam(int q, int i) {
  const double qa = (5.0 + 3.0 * sqrt(5.0)) / 20.0;
  const double qb = (5.0 - sqrt(5.0)) / 20.0;
  return q == i ? qa : qb;
}

// contrib[(q*nt + t)*6 + e] = (w_e(x_q) . F_q) * s_e * |T|/4   (fem.py:382-389)
// F from fvals (4,nt,3) or the device Gaussian when fvals == nullptr.
__global__ void k_rhs_contrib(int64_t nt, const double* __restrict__ verts,
                              const int32_t* __restrict__ tets, const int8_t* __restrict__ signs,
                              const double2* __restrict__ fvals, GaussSrc gs,
                              double2* __restrict__ contrib) {
  const int64_t t = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (t >= nt) return;
  double c[4][3], sg[6];
  load_tet(verts, tets, signs, t, c, sg);
  TetGeom g;
  tet_geometry(c, g);
  for (int q = 0; q < 4; ++q) {
    double2 F[3];
    if (fvals) {
      for (int k = 0; k < 3; ++k) F[k] = fvals[((int64_t)q * nt + t) * 3 + k];
    } else {
      double x[3];
      for (int k = 0; k < 3; ++k)
        x[k] = qlam(q, 0) * c[0][k] + qlam(q, 1) * c[1][k] + qlam(q, 2) * c[2][k] +
               qlam(q, 3) * c[3][k];
      const double r2 = (x[0] - gs.cx) * (x[0] - gs.cx) + (x[1] - gs.cy) * (x[1] - gs.cy) +
                        (x[2] - gs.cz) * (x[2] - gs.cz);
      const double f = gs.amp * exp(-gs.alpha * r2);
      F[0] = make_double2(f * gs.dx, 0.0);
      F[1] = make_double2(f * gs.dy, 0.0);
      F[2] = make_double2(f * gs.dz, 0.0);
    }
    for (int e = 0; e < 6; ++e) {
      const int a = kEA[e], b = kEB[e];
      double w[3];
      for (int k = 0; k < 3; ++k) w[k] = qlam(q, a) * g.g[b][k] - qlam(q, b) * g.g[a][k];
      double2 s = make_double2(w[0] * F[0].x + w[1] * F[1].x + w[2] * F[2].x,
                               w[0] * F[0].y + w[1] * F[1].y + w[2] * F[2].y);
      const double sc = sg[e] * (g.vol / 4.0);
      contrib[((int64_t)q * nt + t) * 6 + e] = make_double2(s.x * sc, s.y * sc);
    }
  }
}

// rhs[i] = sum_q sum_{(t,e) incident, ascending t} contrib  (np.add.at order)
__global__ void k_rhs_gather(int64_t ndof, int64_t nt, const int32_t* __restrict__ inc_ptr,
                             const int32_t* __restrict__ inc, const double2* __restrict__ contrib,
                             double2* __restrict__ rhs) {
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < ndof;
       i += (int64_t)gridDim.x * blockDim.x) {
    double2 acc = make_double2(0.0, 0.0);
    for (int q = 0; q < 4; ++q)
      for (int k = inc_ptr[i]; k < inc_ptr[i + 1]; ++k) {
        const int te = inc[k];
        const int64_t t = te / 6, e = te % 6;
        const double2 v = contrib[((int64_t)q * nt + t) * 6 + e];
        acc.x += v.x;
        acc.y += v.y;
      }
    rhs[i] = acc;
  }
}

__global__ void k_element_batch(int64_t nt, const double* __restrict__ coords,
                                const double* __restrict__ signs, double* s_el, double* m_el,
                                double* vol) {
  const int64_t t = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (t >= nt) return;
  double c[4][3], sg[6];
  for (int i = 0; i < 4; ++i)
    for (int k = 0; k < 3; ++k) c[i][k] = coords[t * 12 + i * 3 + k];
  for (int e = 0; e < 6; ++e) sg[e] = signs[t * 6 + e];
  ElemMats em;
  element_matrices(c, sg, em);
  for (int a = 0; a < 6; ++a)
    for (int b = 0; b < 6; ++b) {
      s_el[t * 36 + a * 6 + b] = em.s[a][b];
      m_el[t * 36 + a * 6 + b] = em.m[a][b];
    }
  vol[t] = em.vol;
}

static unsigned nblocks(int64_t n, int bs) { return (unsigned)std::max<int64_t>(1, (n + bs - 1) / bs); }
static unsigned gs_blocks(mdd_ctx* ctx, int64_t n) {
  return (unsigned)std::max<int64_t>(1, std::min<int64_t>((n + 255) / 256, (int64_t)ctx->nsm * 16));
}

// Host: boundary-mass pattern + slot lists for a set of faces (sorted vertex
// triples). Returns the n x n pattern, per-slot contribution lists into the
// (nf,3,3) face-mass array, and the map of each slot into `into` (A's pattern).
struct FaceAsm {
  std::shared_ptr<mdd_pattern> pat;
  DevBuf<int32_t> faces, slot_ptr, slot_idx, amap;
  int64_t nf = 0;
};

static void edge_lookup_build(const mdd_space* sp, std::vector<int64_t>& keys,
                              std::vector<int32_t>& ids) {
  const int64_t nv = sp->nv;
  // edges as (lo,hi) from tets: recover via tet_edges (global edge ids)
  keys.assign(sp->ne, -1);
  for (int64_t t = 0; t < sp->nt; ++t)
    for (int e = 0; e < 6; ++e) {
      static const int EA[6] = {0, 0, 0, 1, 1, 2}, EB[6] = {1, 2, 3, 2, 3, 3};
      int64_t a = sp->h_tets[t * 4 + EA[e]], b = sp->h_tets[t * 4 + EB[e]];
      if (a > b) std::swap(a, b);
      keys[sp->h_tet_edges[t * 6 + e]] = a * nv + b;
    }
  ids.resize(sp->ne);
  std::iota(ids.begin(), ids.end(), 0);
  std::sort(ids.begin(), ids.end(), [&](int32_t x, int32_t y) { return keys[x] < keys[y]; });
}

static FaceAsm build_face_asm(const mdd_space* sp, int64_t nf, const int64_t* faces,
                              const std::vector<int32_t>& e2d_local, int64_t nloc,
                              const mdd_pattern* into, cudaStream_t s) {
  FaceAsm fa;
  fa.nf = nf;
  std::vector<int64_t> keys;
  std::vector<int32_t> order;
  edge_lookup_build(sp, keys, order);
  const int64_t nv = sp->nv;
  auto find_edge = [&](int64_t a, int64_t b) -> int32_t {
    const int64_t key = a * nv + b;
    auto it = std::lower_bound(order.begin(), order.end(), key,
                               [&](int32_t id, int64_t k) { return keys[id] < k; });
    if (it == order.end() || keys[*it] != key) fail(MDD_EINVAL, "boundary face edge not in mesh");
    return *it;
  };
  std::vector<int32_t> fdof(nf * 3);
  const int tp[3][2] = {{0, 1}, {0, 2}, {1, 2}};
  for (int64_t f = 0; f < nf; ++f)
    for (int e = 0; e < 3; ++e)
      fdof[f * 3 + e] = e2d_local[find_edge(faces[f * 3 + tp[e][0]], faces[f * 3 + tp[e][1]])];
  // contributions (row, col, src)
  struct C { int32_t r, c, src; };
  std::vector<C> cs;
  cs.reserve(nf * 9);
  for (int64_t f = 0; f < nf; ++f)
    for (int a = 0; a < 3; ++a)
      for (int b = 0; b < 3; ++b) {
        const int32_t r = fdof[f * 3 + a], c = fdof[f * 3 + b];
        if (r >= 0 && c >= 0) cs.push_back({r, c, (int32_t)(f * 9 + a * 3 + b)});
      }
  std::stable_sort(cs.begin(), cs.end(), [](const C& x, const C& y) {
    return x.r != y.r ? x.r < y.r : x.c < y.c;
  });
  std::vector<int32_t> rowptr(nloc + 1, 0), cols, sptr{0}, sidx;
  for (size_t i = 0; i < cs.size(); ++i) {
    if (i == 0 || cs[i].r != cs[i - 1].r || cs[i].c != cs[i - 1].c) {
      if (i) sptr.push_back((int32_t)sidx.size());
      cols.push_back(cs[i].c);
      rowptr[cs[i].r + 1]++;
    }
    sidx.push_back(cs[i].src);
  }
  if (!cs.empty()) sptr.push_back((int32_t)sidx.size());
  for (int64_t r = 0; r < nloc; ++r) rowptr[r + 1] += rowptr[r];
  std::vector<int32_t> amap;
  if (into) {
    amap.resize(cols.size());
    for (int64_t r = 0; r < nloc; ++r)
      for (int32_t k = rowptr[r]; k < rowptr[r + 1]; ++k) {
        const int32_t* b = into->h_cols.data() + into->h_rowptr[r];
        const int32_t* e = into->h_cols.data() + into->h_rowptr[r + 1];
        const int32_t* it = std::lower_bound(b, e, cols[k]);
        if (it == e || *it != cols[k]) fail(MDD_EINVAL, "boundary mass entry outside A's pattern");
        amap[k] = (int32_t)(it - into->h_cols.data());
      }
  }
  std::vector<int32_t> fv(nf * 3);
  for (int64_t i = 0; i < nf * 3; ++i) fv[i] = (int32_t)faces[i];
  fa.faces.upload(fv, s);
  fa.slot_ptr.upload(sptr, s);
  fa.slot_idx.upload(sidx, s);
  fa.amap.upload(amap, s);
  fa.pat = make_pattern(nloc, nloc, std::move(rowptr), std::move(cols), s);
  return fa;
}

// Computes face masses and gathers them into an (nloc x nloc) real CSR.
static mdd_csr* assemble_face_mass(mdd_space* sp, FaceAsm& fa) {
  mdd_ctx* ctx = sp->ctx;
  cudaStream_t s = ctx->stream;
  mdd_csr* mb = new_csr(ctx, fa.pat, false);
  if (fa.nf > 0) {
    DevBuf<double> fm(fa.nf * 9);
    k_face_mass<<<nblocks(fa.nf, 128), 128, 0, s>>>(fa.nf, fa.faces.p, sp->verts.p, fm.p);
    CK_LAUNCH(ctx);
    const int64_t ns = fa.pat->nnz;
    if (ns) {
      k_slot_gather<<<gs_blocks(ctx, ns), 256, 0, s>>>(ns, fa.slot_ptr.p, fa.slot_idx.p, fm.p,
                                                       mb->vals.p);
      CK_LAUNCH(ctx);
    }
    CK(cudaStreamSynchronize(s));
  }
  return mb;
}

void assemble_system(mdd_space* sp, const mdd_coeffs* co, int impedance, int64_t nbf,
                     const int64_t* bfaces, mdd_csr** A, mdd_csr** S, mdd_csr** M,
                     mdd_csr** Dk, mdd_csr** Mb) {
  mdd_ctx* ctx = sp->ctx;
  cudaStream_t s = ctx->stream;
  CK(cudaSetDevice(ctx->device));
  std::unique_ptr<mdd_csr> cS(new_csr(ctx, sp->pat, false));
  std::unique_ptr<mdd_csr> cM(new_csr(ctx, sp->pat, false));
  std::unique_ptr<mdd_csr> cA(new_csr(ctx, sp->pat, true));
  std::unique_ptr<mdd_csr> cD;
  if (Dk) cD.reset(new_csr(ctx, sp->pat, false));
  const bool het = !co->homogeneous;
  DevBuf<double> deps, dmu, dsig;
  CoefDev cd{nullptr, nullptr, nullptr, co->eps0, co->mu0, co->sigma0, co->k, co->xi};
  if (het) {
    if (co->eps) { deps.upload(co->eps, sp->nt, s); cd.eps = deps.p; }
    if (co->mu) { dmu.upload(co->mu, sp->nt, s); cd.mu = dmu.p; }
    if (co->sigma) { dsig.upload(co->sigma, sp->nt, s); cd.sigma = dsig.p; }
  }
  // a row window (sharded solve) assembles the cells that touch the rank's rows only
  const bool win = sp->win_active;
  const int64_t* coff = win ? sp->win_off : sp->color_off;
  const int32_t* clist = win ? sp->win_cells.p : sp->cells_by_color.p;
  for (int c = 0; c < 8; ++c) {
    const int64_t nc = coff[c + 1] - coff[c];
    if (!nc) continue;
    k_assemble_cells<<<nblocks(nc * 32, 128), 128, 0, s>>>(
        clist + coff[c], nc, sp->verts.p, sp->tets.p, sp->tet_edges.p,
        sp->signs.p, sp->e2d.p, sp->pat->rowptr.p, sp->pat->cols.p, cS->vals.p, cM->vals.p,
        het ? reinterpret_cast<double2*>(cA->vals.p) : nullptr, cd);
    CK_LAUNCH(ctx);
  }
  const int64_t nnz = sp->pat->nnz;
  if (nnz) {
    k_combine<<<gs_blocks(ctx, nnz), 256, 0, s>>>(nnz, cS->vals.p, cM->vals.p,
                                                  reinterpret_cast<double2*>(cA->vals.p),
                                                  cD ? cD->vals.p : nullptr, co->k * co->k, co->xi,
                                                  het ? 0 : 1);
    CK_LAUNCH(ctx);
  }
  std::unique_ptr<mdd_csr> cMb;
  if (impedance) {
    FaceAsm fa = build_face_asm(sp, nbf, bfaces, sp->h_e2d, sp->ndof, sp->pat.get(), s);
    cMb.reset(assemble_face_mass(sp, fa));
    const double simp = co->xi >= 0 ? 1.0 : -1.0;
    const int64_t ns = fa.pat->nnz;
    if (ns) {
      k_imp_update<<<gs_blocks(ctx, ns), 256, 0, s>>>(
          ns, fa.amap.p, cMb->vals.p, reinterpret_cast<double2*>(cA->vals.p),
          make_double2(0.0, -simp * co->k));
      CK_LAUNCH(ctx);
    }
  }
  CK(cudaStreamSynchronize(s));
  if (A) *A = cA.release();
  if (S) *S = cS.release();
  if (M) *M = cM.release();
  if (Dk) *Dk = cD.release();
  if (Mb) *Mb = cMb.release();
}

void assemble_rhs_dev(mdd_space* sp, const double2* fvals_host, const GaussSrc* gsrc,
                      double2* rhs_dev) {
  mdd_ctx* ctx = sp->ctx;
  cudaStream_t s = ctx->stream;
  DevBuf<double2> contrib(sp->nt * 24), fv;
  if (fvals_host) fv.upload(fvals_host, sp->nt * 12, s);
  GaussSrc g = gsrc ? *gsrc : GaussSrc{0, 0, 0, 0, 0, 0, 0, 0};
  if (sp->nt) {
    k_rhs_contrib<<<nblocks(sp->nt, 128), 128, 0, s>>>(sp->nt, sp->verts.p, sp->tets.p,
                                                      sp->signs.p, fvals_host ? fv.p : nullptr, g,
                                                      contrib.p);
    CK_LAUNCH(ctx);
  }
  if (sp->ndof) {
    k_rhs_gather<<<gs_blocks(ctx, sp->ndof), 256, 0, s>>>(sp->ndof, sp->nt, sp->inc_ptr.p,
                                                          sp->inc.p, contrib.p, rhs_dev);
    CK_LAUNCH(ctx);
  }
}

}  // namespace mdd

using namespace mdd;

extern "C" {

int mdd_space_create(mdd_ctx* ctx, int32_t cells_per_axis, int64_t nv, const double* vertices,
                     int64_t nt, const int64_t* tets, const int64_t* tet_edges,
                     const int64_t* tet_edge_signs, int64_t ne, const int64_t* edge_to_dof,
                     int64_t ndof, mdd_space** out) {
  MDD_API_BEGIN
  CK(cudaSetDevice(ctx->device));
  const int64_t n = cells_per_axis;
  if (n < 1 || nt != 6 * n * n * n) fail(MDD_EINVAL, "space: expected a Kuhn mesh with 6 n^3 tets");
  if (nv > INT32_MAX || ne > INT32_MAX || nt * 6 > INT32_MAX)
    fail(MDD_EINVAL, "space: mesh too large for int32 indexing");
  auto sp = std::make_unique<mdd_space>();
  sp->ctx = ctx;
  sp->n = cells_per_axis;
  sp->nv = nv;
  sp->nt = nt;
  sp->ne = ne;
  sp->ndof = ndof;
  sp->h_verts.assign(vertices, vertices + nv * 3);
  sp->h_tets.resize(nt * 4);
  sp->h_tet_edges.resize(nt * 6);
  sp->h_signs.resize(nt * 6);
  sp->h_e2d.resize(ne);
  for (int64_t i = 0; i < nt * 4; ++i) sp->h_tets[i] = (int32_t)tets[i];
  for (int64_t i = 0; i < nt * 6; ++i) {
    sp->h_tet_edges[i] = (int32_t)tet_edges[i];
    sp->h_signs[i] = (int8_t)tet_edge_signs[i];
  }
  for (int64_t i = 0; i < ne; ++i) sp->h_e2d[i] = (int32_t)edge_to_dof[i];
  // structured check: tet 6c..6c+5 lie in cell c (first vertex = cell corner)
  const int64_t nv1 = n + 1;
  for (int64_t c = 0; c < n * n * n; ++c) {
    const int64_t cx = c / (n * n), cy = (c / n) % n, cz = c % n;
    const int64_t corner = (cx * nv1 + cy) * nv1 + cz;
    for (int p = 0; p < 6; ++p)
      if (sp->h_tets[(c * 6 + p) * 4] != corner)
        fail(MDD_EINVAL, "space: tets are not cell-major Kuhn tets");
  }
  // cells by colour
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
  // edge -> (tet*6+e) incidence, ascending tet
  std::vector<int32_t> eptr(ne + 1, 0), einc(nt * 6);
  for (int64_t i = 0; i < nt * 6; ++i) eptr[sp->h_tet_edges[i] + 1]++;
  for (int64_t e = 0; e < ne; ++e) eptr[e + 1] += eptr[e];
  {
    std::vector<int32_t> fillp(eptr.begin(), eptr.end() - 1);
    for (int64_t i = 0; i < nt * 6; ++i) einc[fillp[sp->h_tet_edges[i]]++] = (int32_t)i;
  }
  std::vector<int32_t> d2e(ndof, -1);
  for (int64_t e = 0; e < ne; ++e) {
    const int32_t d = sp->h_e2d[e];
    if (d >= ndof) fail(MDD_EINVAL, "space: edge_to_dof out of range");
    if (d >= 0) d2e[d] = (int32_t)e;
  }
  for (int64_t d = 0; d < ndof; ++d)
    if (d2e[d] < 0) fail(MDD_EINVAL, "space: dof without an edge");
  // dof incidence for the rhs gather
  std::vector<int32_t> iptr(ndof + 1, 0), iinc;
  iinc.reserve(nt * 6);
  for (int64_t d = 0; d < ndof; ++d) {
    const int32_t e = d2e[d];
    for (int32_t k = eptr[e]; k < eptr[e + 1]; ++k) iinc.push_back(einc[k]);
    iptr[d + 1] = (int32_t)iinc.size();
  }
  // CSR pattern: row d = sorted unique kept dofs of all tets incident to edge(d)
  std::vector<int32_t> rowcnt(ndof + 1, 0);
  auto row_of = [&](int64_t d, std::vector<int32_t>& buf) {
    buf.clear();
    const int32_t e = d2e[d];
    for (int32_t k = eptr[e]; k < eptr[e + 1]; ++k) {
      const int32_t t = einc[k] / 6;
      for (int q = 0; q < 6; ++q) {
        const int32_t dd = sp->h_e2d[sp->h_tet_edges[(int64_t)t * 6 + q]];
        if (dd >= 0) buf.push_back(dd);
      }
    }
    std::sort(buf.begin(), buf.end());
    buf.erase(std::unique(buf.begin(), buf.end()), buf.end());
  };
  parallel_for(ndof, [&](int64_t b, int64_t e) {
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
  parallel_for(ndof, [&](int64_t b, int64_t e) {
    std::vector<int32_t> buf;
    for (int64_t d = b; d < e; ++d) {
      row_of(d, buf);
      std::copy(buf.begin(), buf.end(), cols.begin() + rowptr[d]);
    }
  });
  cudaStream_t s = ctx->stream;
  sp->verts.upload(sp->h_verts, s);
  sp->tets.upload(sp->h_tets, s);
  sp->tet_edges.upload(sp->h_tet_edges, s);
  sp->signs.upload(sp->h_signs, s);
  sp->e2d.upload(sp->h_e2d, s);
  sp->cells_by_color.upload(cbc, s);
  sp->inc_ptr.upload(iptr, s);
  sp->inc.upload(iinc, s);
  sp->pat = make_pattern(ndof, ndof, std::move(rowptr), std::move(cols), s);
  CK(cudaStreamSynchronize(s));
  *out = sp.release();
  MDD_API_END
}

void mdd_space_destroy(mdd_space* sp) {
  if (!sp) return;
  cudaSetDevice(sp->ctx->device);
  delete sp;
}

int mdd_space_nnz(const mdd_space* sp, int64_t* nnz) {
  MDD_API_BEGIN
  *nnz = sp->pat->nnz;
  MDD_API_END
}

int mdd_assemble(mdd_space* sp, const mdd_coeffs* co, int impedance, int64_t nbf,
                 const int64_t* bfaces, mdd_csr** A, mdd_csr** S, mdd_csr** M, mdd_csr** Dk,
                 mdd_csr** Mb) {
  MDD_API_BEGIN
  if (sp->order == 2) {
    if (impedance) fail(MDD_EINVAL, "order-2 spaces support the PEC boundary only");
    if (Mb) *Mb = nullptr;
    assemble_system2(sp, co, A, S, M, Dk);
  } else {
    assemble_system(sp, co, impedance, nbf, bfaces, A, S, M, Dk, Mb);
  }
  MDD_API_END
}

int mdd_space_set_row_window(mdd_space* sp, int64_t row_lo, int64_t row_hi) {
  MDD_API_BEGIN
  if (row_lo < 0 || (row_lo == 0 && row_hi >= sp->ndof)) {  // reset: every cell
    sp->win_active = false;
    return MDD_OK;
  }
  if (sp->order != 1) fail(MDD_EINVAL, "row windows are implemented for lowest-order spaces");
  if (row_hi <= row_lo || row_hi > sp->ndof) fail(MDD_EINVAL, "row window out of range");
  if (sp->win_lo == row_lo && sp->win_hi == row_hi) {
    sp->win_active = true;
    return MDD_OK;
  }
  CK(cudaSetDevice(sp->ctx->device));
  const int64_t ncell = sp->nt / 6;
  // a cell is kept when one of its 36 (tet, edge) slots carries a kept unknown inside the window
  std::vector<uint8_t> keep(ncell, 0);
  for (int64_t c = 0; c < ncell; ++c) {
    const int32_t* te = sp->h_tet_edges.data() + c * 36;
    for (int q = 0; q < 36 && !keep[c]; ++q) {
      const int32_t d = sp->h_e2d[te[q]];
      keep[c] = d >= row_lo && d < row_hi;
    }
  }
  std::vector<int32_t> h_cbc((size_t)sp->color_off[8]), list;
  sp->cells_by_color.download(h_cbc.data(), h_cbc.size(), sp->ctx->stream);
  CK(cudaStreamSynchronize(sp->ctx->stream));
  list.reserve(h_cbc.size());
  for (int col = 0; col < 8; ++col) {
    sp->win_off[col] = (int64_t)list.size();
    for (int64_t i = sp->color_off[col]; i < sp->color_off[col + 1]; ++i)
      if (keep[h_cbc[i]]) list.push_back(h_cbc[i]);
  }
  sp->win_off[8] = (int64_t)list.size();
  sp->win_cells.upload(list, sp->ctx->stream);
  CK(cudaStreamSynchronize(sp->ctx->stream));
  sp->win_lo = row_lo;
  sp->win_hi = row_hi;
  sp->win_active = true;
  MDD_API_END
}

int mdd_assemble_rhs(mdd_space* sp, const mdd_complex* fvals, mdd_complex* rhs) {
  MDD_API_BEGIN
  mdd_ctx* ctx = sp->ctx;
  CK(cudaSetDevice(ctx->device));
  DevBuf<double2> r(sp->ndof);
  if (sp->order == 2) assemble_rhs2_dev(sp, reinterpret_cast<const double2*>(fvals), nullptr, r.p);
  else assemble_rhs_dev(sp, reinterpret_cast<const double2*>(fvals), nullptr, r.p);
  r.download(reinterpret_cast<double2*>(rhs), sp->ndof, ctx->stream);
  CK(cudaStreamSynchronize(ctx->stream));
  MDD_API_END
}

int mdd_assemble_rhs_gaussian(mdd_space* sp, const double* center, double alpha, double amp,
                              const double* dir, mdd_complex* rhs) {
  MDD_API_BEGIN
  mdd_ctx* ctx = sp->ctx;
  CK(cudaSetDevice(ctx->device));
  GaussSrc g{center[0], center[1], center[2], alpha, amp, dir[0], dir[1], dir[2]};
  DevBuf<double2> r(sp->ndof);
  if (sp->order == 2) assemble_rhs2_dev(sp, nullptr, &g, r.p);
  else assemble_rhs_dev(sp, nullptr, &g, r.p);
  r.download(reinterpret_cast<double2*>(rhs), sp->ndof, ctx->stream);
  CK(cudaStreamSynchronize(ctx->stream));
  MDD_API_END
}

int mdd_element_matrices(mdd_ctx* ctx, int64_t nt, const double* coords, const double* signs,
                         double* s_el, double* m_el, double* vol) {
  MDD_API_BEGIN
  CK(cudaSetDevice(ctx->device));
  cudaStream_t s = ctx->stream;
  DevBuf<double> c(nt * 12), sg(nt * 6), so(nt * 36), mo(nt * 36), vo(nt);
  c.upload(coords, nt * 12, s);
  sg.upload(signs, nt * 6, s);
  if (nt) {
    k_element_batch<<<nblocks(nt, 128), 128, 0, s>>>(nt, c.p, sg.p, so.p, mo.p, vo.p);
    CK_LAUNCH(ctx);
  }
  so.download(s_el, nt * 36, s);
  mo.download(m_el, nt * 36, s);
  vo.download(vol, nt, s);
  CK(cudaStreamSynchronize(s));
  MDD_API_END
}

}  // extern "C"
