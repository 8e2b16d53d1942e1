// Two-level overlapping Schwarz preconditioners on the device
// (reference precond.PreconditionerState, precond.py:147-247).
//
//  setup : subdomain blocks R_l A_prec R_l^T (exact minors, linalg.py:48-70)
//          are analysed by geometric nested dissection and factorised as one
//          batched multifrontal plan; the coarse block R0 A_prec R0^T is
//          formed element by element (each fine tet T lies in one coarse tet
//          C(T), so R0 A R0^T = sum_T Q_T A_T Q_T^T with Q_T the 6x6 values of
//          C(T)'s Whitney functions on T's edges) and factorised the same way.
//  apply : gather v[I_l] -> batched forward/backward solves -> owner-computes
//          scatter out[i] = sum_{l owning i} w_l(i) u_l(i) (subdomain order,
//          as precond.py:220-225), fused with the coarse prolongation for
//          the additive variant; hybrid / ADEF1 compose the same primitives
//          (precond.py:230-245).
#include <algorithm>
#include <chrono>
#include <cmath>
#include <cstring>
#include <numeric>
#include <atomic>
#include <thread>
#include <unordered_map>

#include "fem_device.cuh"
#include "frontal.h"
#include "mdd_kernels.cuh"

namespace mdd {

void assemble_system(mdd_space* sp, const mdd_coeffs* co, int impedance, int64_t nbf,
                     const int64_t* bfaces, mdd_csr** A, mdd_csr** S, mdd_csr** M, mdd_csr** Dk,
                     mdd_csr** Mb);

struct PrecCore {
  mdd_ctx* ctx = nullptr;
  int64_t ndof = 0;
  int local_kind = 0;  // 0: conducting minors (as/ras), 1: impedance (impras)
  int32_t nsub = 0;
  FrontPlan sub;
  DevBuf<int32_t> gidx;               // nloc
  DevBuf<int32_t> own_ptr, own_idx;   // ndof+1, nloc
  DevBuf<double> own_w;               // nloc (PoU weight of each ownership)
  bool have_coarse = false;
  int64_t ncs = 0;
  FrontPlan coarse;
  std::unique_ptr<mdd_csr> R0p, R0Tp;  // rows / columns in coarse ND order
  std::unique_ptr<mdd_csr> A0;         // assembled coarse Galerkin matrix (coarse pattern)
  // A_prec entry -> transposed entry (AS/RAS minors), symmetry flag of the last factorisation
  DevBuf<int32_t> tpos;
  DevBuf<int> symflag;
  bool sym_checked = false;
  // non-nested coarse mesh: A0[slot] = sum_t rap_c[t] * A_prec[rap_k[t]], t in [rap_ptr[slot], rap_ptr[slot+1])
  bool rap = false;
  DevBuf<int64_t> rap_ptr;
  DevBuf<int32_t> rap_k;
  DevBuf<double> rap_c;
  // Galerkin data
  const mdd_space* fine_space = nullptr;
  const mdd_space* coarse_space = nullptr;
  DevBuf<int32_t> tet_map, cfine_ptr, cfine_idx, face_tet, cface_ptr, cface_idx, gfaces;
  int64_t n_gfaces = 0;
  // impras local assembly data
  DevBuf<double2> loc_vals;
  DevBuf<int32_t> loc_tet, loc_tet_sub;          // (subdomain tet, subdomain) pairs by colour
  std::vector<int64_t> loc_color_off;
  DevBuf<int32_t> loc_rowptr, loc_cols;          // concatenated local patterns (local ids)
  DevBuf<int32_t> loc_sub_off;                   // entry offset per subdomain
  DevBuf<int32_t> loc_e2l;                       // per (pair, 6): local index or -1
  DevBuf<int32_t> loc_face, loc_face_sub, loc_face_l;  // boundary faces
  int64_t n_loc_faces = 0;
  DevBuf<int32_t> loc_row_off;                   // per subdomain: offset into loc_rowptr
  std::vector<int32_t> h_loc_row_off, h_loc_ent_off;  // host copies (mdd_prec_local_matrix)
  std::vector<double> stats = std::vector<double>(8, 0.0);
  DevBuf<double2> t1, t2, t3, t4;
  cudaStream_t s2 = nullptr;  // coarse-solve branch
  cudaEvent_t ev_fork = nullptr, ev_join = nullptr;
  ~PrecCore() {
    if (ev_fork) cudaEventDestroy(ev_fork);
    if (ev_join) cudaEventDestroy(ev_join);
    if (s2) cudaStreamDestroy(s2);
  }
};

}  // namespace mdd

struct mdd_prec {
  std::shared_ptr<mdd::PrecCore> core;
  int family = 0, levels = 1, correction = 0;
  const mdd_csr* A_corr = nullptr;
  mdd_comm* comm = nullptr;  // sharded: this rank holds a block of the subdomains
  // sharded data plane (mdd_prec_set_halo): row ranges of the overlap sum and of the halo
  // exchange, and R0 restricted to this rank's owned columns (the coarse restriction is a
  // local partial product completed by an allreduce of the ncs coarse values)
  std::shared_ptr<mdd_halo> halo;
  std::shared_ptr<mdd_csr> R0own;
};

namespace mdd {

// ---------------------------------------------------------------- kernels
// out[i] = (sum_k w_k x[own_idx[k]]) (+ add[i])
__global__ void k_scatter_owner(int64_t ndof, const int32_t* __restrict__ ptr,
                                const int32_t* __restrict__ idx, const double* __restrict__ w,
                                const double2* __restrict__ x, const double2* __restrict__ add,
                                double2* __restrict__ out) {
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < ndof;
       i += (int64_t)gridDim.x * blockDim.x) {
    double2 acc = make_double2(0.0, 0.0);
    for (int k = ptr[i]; k < ptr[i + 1]; ++k) {
      const double2 u = x[idx[k]];
      if (w) {
        const double ww = w[k];
        acc.x += ww * u.x;
        acc.y += ww * u.y;
      } else {
        acc.x += u.x;
        acc.y += u.y;
      }
    }
    if (add) acc = cadd(acc, add[i]);
    out[i] = acc;
  }
}

// out = (a - b) + c
__global__ void k_sub_add(int64_t n, const double2* a, const double2* b, const double2* c,
                          double2* out) {
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x)
    out[i] = cadd(csub(a[i], b[i]), c[i]);
}

// barycentric coordinates of x in a tet with vertex 0 at p0 and gradients g
__device__ __forceinline__ void bary(const TetGeom& g, const double* p0, const double* x,
                                     double (&l)[4]) {
  double d[3] = {x[0] - p0[0], x[1] - p0[1], x[2] - p0[2]};
  for (int i = 1; i < 4; ++i) l[i] = g.g[i][0] * d[0] + g.g[i][1] * d[1] + g.g[i][2] * d[2];
  l[0] = 1.0 - l[1] - l[2] - l[3];
}

struct GalArgs {
  // fine
  const double* fverts;
  const int32_t* ftets;
  const int32_t* ftet_edges;
  const int8_t* fsigns;
  const int32_t* fe2d;
  // coarse
  const double* cverts;
  const int32_t* ctets;
  const int8_t* csigns;
  const int32_t* tet_map;
};

// Q[c][e]: coarse local edge c of C (oriented by its sign) on fine edge
// (lo -> hi):  sc * (l_a(x0) l_b(x1) - l_a(x1) l_b(x0))   (exact line integral
// of the Whitney function, = decomp.coarse_restriction's 2-point Gauss value)
__device__ void coarse_Q_edges(const GalArgs& ga, int ct, const int64_t* lo, const int64_t* hi,
                               int ne, double (&Q)[6][6]) {
  double cc[4][3];
  for (int i = 0; i < 4; ++i) {
    const int v = ga.ctets[(int64_t)ct * 4 + i];
    for (int k = 0; k < 3; ++k) cc[i][k] = ga.cverts[(int64_t)v * 3 + k];
  }
  TetGeom g;
  tet_geometry(cc, g);
  for (int e = 0; e < ne; ++e) {
    double l0[4], l1[4];
    bary(g, cc[0], ga.fverts + lo[e] * 3, l0);
    bary(g, cc[0], ga.fverts + hi[e] * 3, l1);
    for (int c = 0; c < 6; ++c) {
      const int a = kEA[c], b = kEB[c];
      const double sc = (double)ga.csigns[(int64_t)ct * 6 + c];
      Q[c][e] = sc * (l0[a] * l1[b] - l1[a] * l0[b]);
    }
  }
}

// per fine tet: BS = Q S Q^T, BM = Q M Q^T (6x6 real each)
__global__ void __launch_bounds__(128) k_galerkin_tets(int64_t nt, GalArgs ga, double* __restrict__ BS,
                                                       double* __restrict__ BM) {
  const int64_t t = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (t >= nt) return;
  double c[4][3], sg[6];
  int32_t vid[4];
  for (int i = 0; i < 4; ++i) {
    vid[i] = ga.ftets[t * 4 + i];
    for (int k = 0; k < 3; ++k) c[i][k] = ga.fverts[(int64_t)vid[i] * 3 + k];
  }
  for (int e = 0; e < 6; ++e) sg[e] = (double)ga.fsigns[t * 6 + e];
  ElemMats em;
  element_matrices(c, sg, em);
  int64_t lo[6], hi[6];
  for (int e = 0; e < 6; ++e) {
    const int64_t a = vid[kEA[e]], b = vid[kEB[e]];
    lo[e] = a < b ? a : b;
    hi[e] = a < b ? b : a;
  }
  double Q[6][6];
  coarse_Q_edges(ga, ga.tet_map[t], lo, hi, 6, Q);
  for (int e = 0; e < 6; ++e)
    if (ga.fe2d[ga.ftet_edges[t * 6 + e]] < 0)
      for (int cc = 0; cc < 6; ++cc) Q[cc][e] = 0.0;
  // QS = Q S, then BS = QS Q^T  (same for M)
  for (int pass = 0; pass < 2; ++pass) {
    const double(*E)[6] = pass == 0 ? em.s : em.m;
    double* out = (pass == 0 ? BS : BM) + t * 36;
    double QE[6][6];
    for (int a = 0; a < 6; ++a)
      for (int b = 0; b < 6; ++b) {
        double s = 0.0;
        for (int k = 0; k < 6; ++k) s += Q[a][k] * E[k][b];
        QE[a][b] = s;
      }
    for (int a = 0; a < 6; ++a)
      for (int b = 0; b < 6; ++b) {
        double s = 0.0;
        for (int k = 0; k < 6; ++k) s += QE[a][k] * Q[b][k];
        out[a * 6 + b] = s;
      }
  }
}

// per global impedance face: BF = Q_f m_f Q_f^T (6x6 real)
__global__ void k_galerkin_faces(int64_t nf, GalArgs ga, const int32_t* __restrict__ faces,
                                 const int32_t* __restrict__ face_tet, double* __restrict__ BF) {
  const int64_t f = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (f >= nf) return;
  double p[3][3];
  int64_t v[3];
  for (int i = 0; i < 3; ++i) {
    v[i] = faces[f * 3 + i];
    for (int k = 0; k < 3; ++k) p[i][k] = ga.fverts[v[i] * 3 + k];
  }
  double mf[3][3];
  triangle_tangential_mass(p, mf);
  const int64_t lo[3] = {v[0], v[0], v[1]}, hi[3] = {v[1], v[2], v[2]};
  double Q[6][6];
  coarse_Q_edges(ga, ga.tet_map[face_tet[f]], lo, hi, 3, Q);
  for (int a = 0; a < 6; ++a)
    for (int b = 0; b < 6; ++b) {
      double s = 0.0;
      for (int x = 0; x < 3; ++x)
        for (int y = 0; y < 3; ++y) s += Q[a][x] * mf[x][y] * Q[b][y];
      BF[f * 36 + a * 6 + b] = s;
    }
}

struct CoefArr {
  const double* eps;
  const double* mu;
  const double* sigma;
  double eps0, mu0, sigma0, k, xi;
  int homogeneous;
  double2 face_coef;  // -i*s*k
};

// per (coarse tet, entry): sum over its fine tets (ascending) and faces
__global__ void k_galerkin_reduce(int64_t nct, const int32_t* __restrict__ fptr,
                                  const int32_t* __restrict__ fidx, const double* __restrict__ BS,
                                  const double* __restrict__ BM, const int32_t* __restrict__ gptr,
                                  const int32_t* __restrict__ gidx, const double* __restrict__ BF,
                                  CoefArr co, double2* __restrict__ blk) {
  const int64_t gid = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (gid >= nct * 36) return;
  const int64_t ct = gid / 36;
  const int e = (int)(gid % 36);
  double2 acc = make_double2(0.0, 0.0);
  for (int k = fptr[ct]; k < fptr[ct + 1]; ++k) {
    const int64_t t = fidx[k];
    const double s = BS[t * 36 + e], m = BM[t * 36 + e];
    if (co.homogeneous) {
      acc.x += s - co.k * co.k * m;
      acc.y += -co.xi * m;
    } else {
      const double eps = co.eps ? co.eps[t] : co.eps0;
      const double mu = co.mu ? co.mu[t] : co.mu0;
      const double sig = co.sigma ? co.sigma[t] : co.sigma0;
      const double wr = co.k * co.k * eps, wi = co.xi * eps + co.k * sig;
      acc.x += s / mu - wr * m;
      acc.y += -wi * m;
    }
  }
  if (gptr)
    for (int k = gptr[ct]; k < gptr[ct + 1]; ++k) {
      const double b = BF[(int64_t)gidx[k] * 36 + e];
      acc.x += co.face_coef.x * b;
      acc.y += co.face_coef.y * b;
    }
  blk[gid] = acc;
}

// coloured scatter of complex 6x6 element blocks into a complex CSR: one warp
// per cell of a colour; the lanes cover the 36 (distinct) slots of one tet and
// the cell's 6 tets follow in order (they share slots), so no atomics.
__global__ void __launch_bounds__(128) k_scatter_blocks(const int32_t* __restrict__ cells, int64_t ncells,
                                                        const int32_t* __restrict__ tet_edges,
                                                        const int32_t* __restrict__ e2d,
                                                        const int32_t* __restrict__ rowptr,
                                                        const int32_t* __restrict__ cols,
                                                        const double2* __restrict__ blk,
                                                        double2* __restrict__ A) {
  const int64_t ci = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const int lane = threadIdx.x & 31;
  if (ci >= ncells) return;
  const int64_t cell = cells[ci];
  for (int p = 0; p < 6; ++p) {
    const int64_t t = cell * 6 + p;
    for (int e = lane; e < 36; e += 32) {
      const int a = e / 6, b = e % 6;
      const int da = e2d[tet_edges[t * 6 + a]], db = e2d[tet_edges[t * 6 + b]];
      if (da >= 0 && db >= 0) {
        const int slot = csr_find(rowptr, cols, da, db);
        A[slot] = cadd(A[slot], blk[t * 36 + e]);
      }
    }
    __syncwarp();
  }
}

// impras local assembly: one thread per (subdomain, cell) pair of one colour;
// adds the subdomain tets of that cell into the subdomain's local CSR.
__global__ void __launch_bounds__(128) k_local_cells(
    int64_t npairs, const int32_t* __restrict__ pair_cell, const int32_t* __restrict__ pair_sub,
    const int32_t* __restrict__ pair_mask, const double* __restrict__ verts,
    const int32_t* __restrict__ tets, const int8_t* __restrict__ signs,
    const int32_t* __restrict__ e2l, const int32_t* __restrict__ row_off,
    const int32_t* __restrict__ rowptr, const int32_t* __restrict__ cols,
    const int32_t* __restrict__ ent_off, CoefArr co, double2* __restrict__ vals) {
  const int64_t pi = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (pi >= npairs) return;
  const int64_t cell = pair_cell[pi];
  const int sub = pair_sub[pi];
  const int mask = pair_mask[pi];
  const int32_t* rp = rowptr + row_off[sub];
  const int32_t* cl = cols + ent_off[sub];
  double2* vv = vals + ent_off[sub];
  for (int p = 0; p < 6; ++p) {
    if (!((mask >> p) & 1)) continue;
    const int64_t t = cell * 6 + p;
    double c[4][3], sg[6];
    for (int i = 0; i < 4; ++i) {
      const int v = tets[t * 4 + i];
      for (int k = 0; k < 3; ++k) c[i][k] = verts[(int64_t)v * 3 + k];
    }
    for (int e = 0; e < 6; ++e) sg[e] = (double)signs[t * 6 + e];
    ElemMats em;
    element_matrices(c, sg, em);
    const double eps = co.eps ? co.eps[t] : co.eps0;
    const double mu = co.mu ? co.mu[t] : co.mu0;
    const double sig = co.sigma ? co.sigma[t] : co.sigma0;
    const double wr = co.k * co.k * eps, wi = co.xi * eps + co.k * sig;
    int l[6];
    for (int e = 0; e < 6; ++e) l[e] = e2l[(pi * 6 + p) * 6 + e];
    for (int a = 0; a < 6; ++a) {
      if (l[a] < 0) continue;
      for (int b = 0; b < 6; ++b) {
        if (l[b] < 0) continue;
        const int slot = csr_find(rp, cl, l[a], l[b]);
        double2 v = vv[slot];
        v.x += em.s[a][b] / mu - wr * em.m[a][b];
        v.y += -wi * em.m[a][b];
        vv[slot] = v;
      }
    }
  }
}

// impras boundary faces: local boundary mass, -i*s*k times, added per face
// (faces of one subdomain processed sequentially by one thread: no races)
__global__ void k_local_faces(int32_t nsub, const int32_t* __restrict__ sub_face_ptr,
                              const int32_t* __restrict__ faces, const int32_t* __restrict__ face_l,
                              const double* __restrict__ verts, const int32_t* __restrict__ row_off,
                              const int32_t* __restrict__ rowptr, const int32_t* __restrict__ cols,
                              const int32_t* __restrict__ ent_off, double2 coef,
                              double2* __restrict__ vals) {
  const int sub = blockIdx.x * blockDim.x + threadIdx.x;
  if (sub >= nsub) return;
  const int32_t* rp = rowptr + row_off[sub];
  const int32_t* cl = cols + ent_off[sub];
  double2* vv = vals + ent_off[sub];
  for (int f = sub_face_ptr[sub]; f < sub_face_ptr[sub + 1]; ++f) {
    double p[3][3];
    for (int i = 0; i < 3; ++i) {
      const int64_t v = faces[(int64_t)f * 3 + i];
      for (int k = 0; k < 3; ++k) p[i][k] = verts[v * 3 + k];
    }
    double mf[3][3];
    triangle_tangential_mass(p, mf);
    for (int a = 0; a < 3; ++a) {
      const int la = face_l[(int64_t)f * 3 + a];
      if (la < 0) continue;
      for (int b = 0; b < 3; ++b) {
        const int lb = face_l[(int64_t)f * 3 + b];
        if (lb < 0) continue;
        const int slot = csr_find(rp, cl, la, lb);
        vv[slot] = cadd(vv[slot], make_double2(coef.x * mf[a][b], coef.y * mf[a][b]));
      }
    }
  }
}

static unsigned gsb(mdd_ctx* ctx, int64_t n) {
  return (unsigned)std::max<int64_t>(1, std::min<int64_t>((n + 255) / 256, (int64_t)ctx->nsm * 16));
}
static unsigned nb(int64_t n, int bs) { return (unsigned)std::max<int64_t>(1, (n + bs - 1) / bs); }

// ------------------------------------------------------------ apply
static void one_level_solve(mdd_prec* P, const double2* v, cudaStream_t s) {
  PrecCore& c = *P->core;
  const int64_t nl = c.sub.nloc;
  if (nl) {
    c.sub.solve(s, v, c.gidx.p);  // restriction v[I_l] fused into the solve
  }
}

static void one_level_scatter(mdd_prec* P, const double2* add, double2* out, cudaStream_t s) {
  PrecCore& c = *P->core;
  mdd_ctx* ctx = c.ctx;
  const bool weighted = P->family != 0;  // ras / impras (precond.py:218)
  k_scatter_owner<<<gsb(ctx, c.ndof), 256, 0, s>>>(c.ndof, c.own_ptr.p, c.own_idx.p,
                                                   weighted ? c.own_w.p : nullptr, c.sub.xloc.p,
                                                   add, out);
  CK_LAUNCH(ctx);
}

bool prec_is_distributed(const mdd_prec* P) { return P && comm_active(P->comm); }
mdd_comm* prec_comm(const mdd_prec* P) { return P ? P->comm : nullptr; }

// Scatter of the local solutions (+ add), one GPU.
static void one_level_finish(mdd_prec* P, const double2* add, double2* out, cudaStream_t s) {
  one_level_scatter(P, add, out, s);
}

static void one_level(mdd_prec* P, const double2* v, const double2* add, double2* out,
                      cudaStream_t s) {
  one_level_solve(P, v, s);
  one_level_finish(P, add, out, s);
}

// out = R0^T A0^{-1} R0 v   (precond.py:227-228)
static void coarse_solve(mdd_prec* P, const double2* v, double2* out, cudaStream_t s) {
  PrecCore& c = *P->core;
  spmv_dev(c.ctx, c.R0p.get(), v, c.coarse.bloc.p, s);
  c.coarse.solve(s);
  spmv_dev(c.ctx, c.R0Tp.get(), c.coarse.xloc.p, out, s);
}

// out[lo..hi) = (a - b) + c on a row range
__global__ void k_sub_add_rows(int64_t lo, int64_t hi, const double2* a, const double2* b, const double2* c,
                               double2* out) {
  for (int64_t i = lo + (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < hi; i += (int64_t)gridDim.x * blockDim.x) {
    double2 r = csub(a[i], b[i]);
    if (c) r = cadd(r, c[i]);
    out[i] = r;
  }
}

mdd_halo* prec_halo(const mdd_prec* P) { return P ? P->halo.get() : nullptr; }

// The sharded apply.  Contract: on entry `v` is valid on this rank's NEEDED
// rows (its subdomains' unknowns); on return `out` is valid on its OWNED rows only.  Exchanges:
//   restriction       - none here: the caller's halo gather made v[I_l] available (precond.py:220)
//   prolongation      - comm_halo_reduce: partial sums on ghost rows go to their owners (precond.py:224)
//   coarse restriction- local partial R0[:, owned] v, ncclAllReduce of ncs values, replicated solve
//   A_corr products   - halo gather of the operand, rows of this rank (precond.py:240-245)
void prec_apply_dist(mdd_prec* P, const double2* v, double2* out, cudaStream_t s) {
  PrecCore& c = *P->core;
  mdd_ctx* ctx = c.ctx;
  mdd_halo* h = P->halo.get();
  if (!h) fail(MDD_EINVAL, "sharded preconditioner without row ranges (mdd_prec_set_halo)");
  const int me = P->comm->rank;
  const int64_t lo = h->own_lo[me], hi = h->own_hi[me], nl = hi - lo;
  auto one = [&](const double2* in, double2* o) {
    one_level_solve(P, in, s);
    one_level_scatter(P, nullptr, o, s);
    comm_halo_reduce(P->comm, h, o, s);
  };
  auto coarse = [&](const double2* in, double2* o) {
    spmv_dev(ctx, P->R0own.get(), in, c.coarse.bloc.p, s);
    comm_allreduce_z(P->comm, c.coarse.bloc.p, c.coarse.nloc, s);
    c.coarse.solve(s);
    spmv_rows_dev(ctx, c.R0Tp.get(), lo, nl, c.coarse.xloc.p, o + lo, s);
  };
  auto rows_of_A = [&](double2* x, double2* y) {  // x: owned-valid on entry
    comm_halo_gather(P->comm, h, x, s);
    spmv_rows_dev(ctx, P->A_corr, lo, nl, x, y + lo, s);
  };
  auto combine = [&](const double2* a, const double2* b, const double2* cc, double2* o) {
    if (nl > 0) {
      k_sub_add_rows<<<gsb(ctx, nl), 256, 0, s>>>(lo, hi, a, b, cc, o);
      CK_LAUNCH(ctx);
    }
  };
  if (P->levels == 1) {
    one(v, out);
    return;
  }
  double2* gv = c.t1.p;
  coarse(v, gv);
  if (P->correction == 0) {  // additive: B1 v + G v
    one(v, out);
    if (nl > 0) vec_add(ctx, out + lo, gv + lo, out + lo, nl, s);
    return;
  }
  double2* t = c.t2.p;
  rows_of_A(gv, t);        // t = A_corr G v   (owned rows)
  combine(v, t, nullptr, t);  // t = v - A_corr G v
  comm_halo_gather(P->comm, h, t, s);
  if (P->correction == 2) {  // adef1: B1 (v - A G v) + G v
    one(t, out);
    if (nl > 0) vec_add(ctx, out + lo, gv + lo, out + lo, nl, s);
    return;
  }
  // hybrid: y = B1 t ; out = y - G (A_corr y) + G v
  double2* y = c.t3.p;
  one(t, y);
  rows_of_A(y, t);
  double2* cy = c.t4.p;
  coarse(t, cy);
  combine(y, cy, gv, out);
}

// owned rows of every rank -> the whole vector on every rank (equal blocks, zero padded)
void prec_gather_owned(mdd_prec* P, double2* vec, cudaStream_t s) {
  mdd_halo* h = P->halo.get();
  const int N = P->comm->nranks, me = P->comm->rank;
  const int64_t n = h->n, chunk = (n + N - 1) / N, lo = h->own_lo[me], nl = h->own_hi[me] - lo;
  DevBuf<double2> send(chunk), all((size_t)N * chunk);
  CK(cudaMemsetAsync(send.p, 0, sizeof(double2) * chunk, s));
  if (nl > 0) CK(cudaMemcpyAsync(send.p, vec + lo, sizeof(double2) * nl, cudaMemcpyDeviceToDevice, s));
  comm_allgather_z(P->comm, send.p, all.p, chunk, s);
  CK(cudaMemcpyAsync(vec, all.p, sizeof(double2) * n, cudaMemcpyDeviceToDevice, s));
  CK(cudaStreamSynchronize(s));  // the staging buffers go out of scope
}

void prec_apply_dev(mdd_prec* P, const double2* v, double2* out, cudaStream_t s) {
  PrecCore& c = *P->core;
  if (prec_is_distributed(P)) {
    // whole vector in, whole vector out (the Python-level apply and the replicated MGS loop);
    // the sharded Krylov loop calls prec_apply_dist directly and never completes the vector
    prec_apply_dist(P, v, out, s);
    prec_gather_owned(P, out, s);
    return;
  }
  if (P->levels == 1) {
    one_level(P, v, nullptr, out, s);
    return;
  }
  const int64_t n = c.ndof;
  double2* gv = c.t1.p;
  if (P->correction == 0) {  // additive: B1 v + G v
    // the coarse solve is independent of the subdomain solves: fork it onto a
    // second stream (a parallel branch when captured into the GMRES graph)
    CK(cudaEventRecord(c.ev_fork, s));
    CK(cudaStreamWaitEvent(c.s2, c.ev_fork, 0));
    coarse_solve(P, v, gv, c.s2);
    CK(cudaEventRecord(c.ev_join, c.s2));
    one_level_solve(P, v, s);
    CK(cudaStreamWaitEvent(s, c.ev_join, 0));
    one_level_finish(P, gv, out, s);
    return;
  }
  coarse_solve(P, v, gv, s);
  // t = v - A_corr G v
  double2* t = c.t2.p;
  spmv_dev_axpby(c.ctx, P->A_corr, gv, t, make_double2(-1.0, 0.0), make_double2(1.0, 0.0), v, s);
  if (P->correction == 2) {  // adef1: B1 (v - A G v) + G v
    one_level(P, t, gv, out, s);
    return;
  }
  // hybrid: y = B1 t ; out = y - G (A_corr y) + G v
  double2* y = c.t3.p;
  one_level(P, t, nullptr, y, s);
  spmv_dev(c.ctx, P->A_corr, y, t, s);
  double2* cy = c.t4.p;
  coarse_solve(P, t, cy, s);
  k_sub_add<<<gsb(c.ctx, n), 256, 0, s>>>(n, y, cy, gv, out);
  CK_LAUNCH(c.ctx);
}

// ------------------------------------------------------------- setup
static std::unique_ptr<mdd_csr> csr_host(mdd_ctx* ctx, int64_t nr, int64_t nc,
                                         std::vector<int32_t>&& rp, std::vector<int32_t>&& cl,
                                         const std::vector<double>& v) {
  std::unique_ptr<mdd_csr> A(new mdd_csr());
  A->ctx = ctx;
  A->is_complex = false;
  A->pat = make_pattern(nr, nc, std::move(rp), std::move(cl), ctx->stream);
  A->vals.upload(v, ctx->stream);
  return A;
}

static void galerkin_assemble(PrecCore& c, const mdd_coeffs* co, cudaStream_t s) {
  mdd_ctx* ctx = c.ctx;
  const mdd_space* fs = c.fine_space;
  const mdd_space* cs = c.coarse_space;
  GalArgs ga{fs->verts.p, fs->tets.p, fs->tet_edges.p, fs->signs.p, fs->e2d.p,
             cs->verts.p, cs->tets.p, cs->signs.p,     c.tet_map.p};
  DevBuf<double> BS(fs->nt * 36), BM(fs->nt * 36), BF;
  k_galerkin_tets<<<nb(fs->nt, 128), 128, 0, s>>>(fs->nt, ga, BS.p, BM.p);
  CK_LAUNCH(ctx);
  if (c.n_gfaces) {
    BF.alloc(c.n_gfaces * 36);
    k_galerkin_faces<<<nb(c.n_gfaces, 128), 128, 0, s>>>(c.n_gfaces, ga, c.gfaces.p, c.face_tet.p,
                                                        BF.p);
    CK_LAUNCH(ctx);
  }
  DevBuf<double> deps, dmu, dsig;
  CoefArr ca{nullptr, nullptr, nullptr, co->eps0, co->mu0, co->sigma0, co->k, co->xi,
             co->homogeneous, make_double2(0.0, -(co->xi >= 0 ? 1.0 : -1.0) * co->k)};
  if (!co->homogeneous) {
    if (co->eps) { deps.upload(co->eps, fs->nt, s); ca.eps = deps.p; }
    if (co->mu) { dmu.upload(co->mu, fs->nt, s); ca.mu = dmu.p; }
    if (co->sigma) { dsig.upload(co->sigma, fs->nt, s); ca.sigma = dsig.p; }
  }
  DevBuf<double2> blk(cs->nt * 36);
  k_galerkin_reduce<<<nb(cs->nt * 36, 256), 256, 0, s>>>(
      cs->nt, c.cfine_ptr.p, c.cfine_idx.p, BS.p, BM.p, c.n_gfaces ? c.cface_ptr.p : nullptr,
      c.n_gfaces ? c.cface_idx.p : nullptr, c.n_gfaces ? BF.p : nullptr, ca, blk.p);
  CK_LAUNCH(ctx);
  c.A0->vals.zero(s);
  for (int col = 0; col < 8; ++col) {
    const int64_t ncell = cs->color_off[col + 1] - cs->color_off[col];
    if (!ncell) continue;
    k_scatter_blocks<<<nb(ncell * 32, 128), 128, 0, s>>>(
        cs->cells_by_color.p + cs->color_off[col], ncell, cs->tet_edges.p, cs->e2d.p,
        cs->pat->rowptr.p, cs->pat->cols.p, blk.p, reinterpret_cast<double2*>(c.A0->vals.p));
    CK_LAUNCH(ctx);
  }
  CK(cudaStreamSynchronize(s));
}

static void impras_local_assemble(PrecCore& c, const mdd_coeffs* co, cudaStream_t s) {
  mdd_ctx* ctx = c.ctx;
  const mdd_space* fs = c.fine_space;
  c.loc_vals.zero(s);
  DevBuf<double> deps, dmu, dsig;
  CoefArr ca{nullptr, nullptr, nullptr, co->eps0, co->mu0, co->sigma0, co->k, co->xi,
             co->homogeneous, make_double2(0.0, 0.0)};
  if (co->eps) { deps.upload(co->eps, fs->nt, s); ca.eps = deps.p; }
  if (co->mu) { dmu.upload(co->mu, fs->nt, s); ca.mu = dmu.p; }
  if (co->sigma) { dsig.upload(co->sigma, fs->nt, s); ca.sigma = dsig.p; }
  for (int col = 0; col < 8; ++col) {
    const int64_t b = c.loc_color_off[col], e = c.loc_color_off[col + 1];
    if (e <= b) continue;
    // pair arrays are laid out [cell | sub | mask] consecutively per colour block
    k_local_cells<<<nb(e - b, 128), 128, 0, s>>>(
        e - b, c.loc_tet.p + b, c.loc_tet_sub.p + b, c.loc_tet.p + c.loc_color_off[8] + b,
        fs->verts.p, fs->tets.p, fs->signs.p, c.loc_e2l.p + b * 36, c.loc_row_off.p,
        c.loc_rowptr.p, c.loc_cols.p, c.loc_sub_off.p, ca,
        c.loc_vals.p);
    CK_LAUNCH(ctx);
  }
  if (c.n_loc_faces) {
    const double2 coef = make_double2(0.0, -(co->xi >= 0 ? 1.0 : -1.0) * co->k);
    k_local_faces<<<nb(c.nsub, 64), 64, 0, s>>>(c.nsub, c.loc_face_sub.p, c.loc_face.p,
                                                c.loc_face_l.p, fs->verts.p, c.loc_row_off.p,
                                                c.loc_rowptr.p, c.loc_cols.p, c.loc_sub_off.p,
                                                coef, c.loc_vals.p);
    CK_LAUNCH(ctx);
  }
}

// Generic Galerkin product for a coarse mesh that does not nest in the fine
// one (tet_map == NULL; extension, BASELINE config 2): A0 = R0 A_prec R0^T
// with R0 given entry by entry (decomp.coarse_restriction_nonnested).  The
// symbolic phase (host, once) lists for every A0 slot (p,q) its terms
// R0[p,i] R0[q,j] * A_prec[i,j] as (A entry index, coefficient), in a fixed
// order; the numeric phase (k_rap, one warp per slot) is a deterministic
// gather-reduce over the current A_prec values.  This is exact: no element
// integration, so it holds for any operator on the fine space.
static void build_rap(PrecCore& c, const mdd_csr& R0, const mdd_pattern& AP, cudaStream_t s) {
  const mdd_pattern& RP = *R0.pat;
  const int64_t ncs = RP.nrow, ndof = RP.ncol;
  std::vector<double> rv(RP.nnz);
  R0.vals.download(rv.data(), RP.nnz, s);
  CK(cudaStreamSynchronize(s));
  // R0^T rows: fine dof -> (coarse row, value), ascending coarse row
  std::vector<int32_t> tp(ndof + 1, 0), tc(RP.nnz);
  std::vector<double> tv(RP.nnz);
  for (int64_t k = 0; k < RP.nnz; ++k) tp[RP.h_cols[k] + 1]++;
  for (int64_t i = 0; i < ndof; ++i) tp[i + 1] += tp[i];
  {
    std::vector<int32_t> fp(tp.begin(), tp.end() - 1);
    for (int64_t r = 0; r < ncs; ++r)
      for (int32_t k = RP.h_rowptr[r]; k < RP.h_rowptr[r + 1]; ++k) {
        const int32_t pos = fp[RP.h_cols[k]]++;
        tc[pos] = (int32_t)r;
        tv[pos] = rv[k];
      }
  }
  struct Term {
    int32_t q, k;
    double c;
  };
  std::vector<std::vector<int32_t>> rq(ncs);
  std::vector<std::vector<int64_t>> rcnt(ncs);
  std::vector<std::vector<int32_t>> rk(ncs);
  std::vector<std::vector<double>> rc(ncs);
  const unsigned nth = std::max(1u, std::min(16u, std::thread::hardware_concurrency()));
  std::atomic<int64_t> next{0};
  std::vector<std::thread> th;
  for (unsigned t = 0; t < nth; ++t)
    th.emplace_back([&] {
      std::vector<Term> terms;
      for (int64_t p = next++; p < ncs; p = next++) {
        terms.clear();
        for (int32_t e = RP.h_rowptr[p]; e < RP.h_rowptr[p + 1]; ++e) {
          const int32_t i = RP.h_cols[e];
          const double rpi = rv[e];
          for (int32_t kk = AP.h_rowptr[i]; kk < AP.h_rowptr[i + 1]; ++kk) {
            const int32_t j = AP.h_cols[kk];
            for (int32_t u = tp[j]; u < tp[j + 1]; ++u) terms.push_back({tc[u], kk, rpi * tv[u]});
          }
        }
        std::stable_sort(terms.begin(), terms.end(), [](const Term& a, const Term& b) { return a.q < b.q; });
        for (size_t a = 0; a < terms.size(); ++a) {
          if (a == 0 || terms[a].q != terms[a - 1].q) {
            rq[p].push_back(terms[a].q);
            rcnt[p].push_back(0);
          }
          rcnt[p].back()++;
          rk[p].push_back(terms[a].k);
          rc[p].push_back(terms[a].c);
        }
      }
    });
  for (auto& x : th) x.join();
  std::vector<int32_t> rowptr(ncs + 1, 0), cols;
  std::vector<int64_t> tptr(1, 0);
  std::vector<int32_t> hk;
  std::vector<double> hc;
  for (int64_t p = 0; p < ncs; ++p) {
    if ((int64_t)rowptr[p] + (int64_t)rq[p].size() > INT32_MAX) fail(MDD_EINVAL, "coarse: nnz > 2^31");
    rowptr[p + 1] = rowptr[p] + (int32_t)rq[p].size();
    cols.insert(cols.end(), rq[p].begin(), rq[p].end());
    for (int64_t n : rcnt[p]) tptr.push_back(tptr.back() + n);
    hk.insert(hk.end(), rk[p].begin(), rk[p].end());
    hc.insert(hc.end(), rc[p].begin(), rc[p].end());
    std::vector<int32_t>().swap(rk[p]);
    std::vector<double>().swap(rc[p]);
  }
  auto pat = make_pattern(ncs, ncs, std::move(rowptr), std::move(cols), s);
  c.A0.reset(new_csr(c.ctx, pat, true));
  c.rap_ptr.upload(tptr, s);
  c.rap_k.upload(hk, s);
  c.rap_c.upload(hc, s);
  c.rap = true;
  CK(cudaStreamSynchronize(s));
}

__global__ void __launch_bounds__(256) k_rap(int64_t nslot, const int64_t* __restrict__ ptr,
                                             const int32_t* __restrict__ kidx, const double* __restrict__ coef,
                                             const double2* __restrict__ A, double2* __restrict__ A0) {
  const int64_t w = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const int lane = threadIdx.x & 31;
  if (w >= nslot) return;
  double2 acc = make_double2(0.0, 0.0);
  for (int64_t t = ptr[w] + lane; t < ptr[w + 1]; t += 32) {
    const double cf = __ldg(coef + t);
    const double2 a = __ldg(A + __ldg(kidx + t));
    acc.x += cf * a.x;
    acc.y += cf * a.y;
  }
  acc = warp_sum2(acc);
  if (lane == 0) A0[w] = acc;
}

static void rap_assemble(PrecCore& c, const mdd_csr* A_prec, cudaStream_t s) {
  const int64_t nslot = c.A0->pat->nnz;
  if (!nslot) return;
  k_rap<<<nb(nslot * 32, 256), 256, 0, s>>>(nslot, c.rap_ptr.p, c.rap_k.p, c.rap_c.p,
                                            reinterpret_cast<const double2*>(A_prec->vals.p),
                                            reinterpret_cast<double2*>(c.A0->vals.p));
  CK_LAUNCH(c.ctx);
}

// bitwise complex symmetry of A_prec (its minors then are too): flag != 0 on
// any A[i][j] != A[j][i]; tpos maps every entry to its transposed position
__global__ void k_symcheck(int64_t nnz, const int32_t* __restrict__ tpos, const double2* __restrict__ a,
                           int* __restrict__ flag) {
  for (int64_t k = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; k < nnz; k += (int64_t)gridDim.x * blockDim.x) {
    const int32_t t = tpos[k];
    if (t < 0) { atomicOr(flag, 1); continue; }
    const double2 x = a[k], y = a[t];
    if (__double_as_longlong(x.x) != __double_as_longlong(y.x) ||
        __double_as_longlong(x.y) != __double_as_longlong(y.y))
      atomicOr(flag, 1);
  }
}

// device-side symmetry flag for the factorisation (no host sync); null when
// the check does not apply (impras local matrices) or MDD_NO_SYM is set
static const int* prec_symmetric(PrecCore& c, const mdd_csr* A_prec, cudaStream_t s) {
  if (c.tpos.n == 0 || getenv("MDD_NO_SYM")) return nullptr;
  const int64_t nnz = A_prec->pat->nnz;
  c.symflag.zero(s);
  k_symcheck<<<nb(std::min<int64_t>(nnz, (int64_t)c.ctx->nsm * 16 * 256), 256), 256, 0, s>>>(
      nnz, c.tpos.p, reinterpret_cast<const double2*>(A_prec->vals.p), c.symflag.p);
  CK_LAUNCH(c.ctx);
  return c.symflag.p;
}

static void numeric_setup(mdd_prec* P, const mdd_csr* A_prec, const mdd_coeffs* pc,
                          int32_t* failed_ctx) {
  PrecCore& c = *P->core;
  mdd_ctx* ctx = c.ctx;
  cudaStream_t s = ctx->stream;
  cudaEvent_t e0, e1;
  CK(cudaEventCreate(&e0));
  CK(cudaEventCreate(&e1));
  CK(cudaEventRecord(e0, s));
  if (c.local_kind == 0) {
    c.sym_checked = prec_symmetric(c, A_prec, s) != nullptr;
    c.sub.factor(reinterpret_cast<const double2*>(A_prec->vals.p), s, c.sym_checked ? c.symflag.p : nullptr);
  } else {
    impras_local_assemble(c, pc, s);
    c.sub.factor(c.loc_vals.p, s);
  }
  if (c.have_coarse) {
    if (c.rap) rap_assemble(c, A_prec, s);
    else galerkin_assemble(c, pc, s);
    c.coarse.factor(reinterpret_cast<const double2*>(c.A0->vals.p), s);
  }
  CK(cudaEventRecord(e1, s));
  CK(cudaEventSynchronize(e1));
  float ms = 0;
  CK(cudaEventElapsedTime(&ms, e0, e1));
  cudaEventDestroy(e0);
  cudaEventDestroy(e1);
  c.stats[4] = ms;
  std::string msg;
  const int bad = c.sub.check_pivots(msg, s);
  if (bad >= 0) {
    if (failed_ctx) *failed_ctx = bad;
    fail(MDD_ESINGULAR, "subdomain " + std::to_string(bad) + ": " + msg, bad);
  }
  if (c.have_coarse) {
    if (c.coarse.check_pivots(msg, s) >= 0) {
      if (failed_ctx) *failed_ctx = -1;
      fail(MDD_ESINGULAR, "coarse space: " + msg, -1);
    }
  }
}

}  // namespace mdd

using namespace mdd;

extern "C" {

int mdd_prec_create(mdd_ctx* ctx, const mdd_prec_desc* d, mdd_prec** out, int32_t* failed_ctx) {
  MDD_API_BEGIN
  CK(cudaSetDevice(ctx->device));
  cudaStream_t s = ctx->stream;
  if (failed_ctx) *failed_ctx = -2;
  if (!d->A_prec || !d->A_prec->is_complex) fail(MDD_EINVAL, "prec: A_prec must be complex CSR");
  auto core = std::make_shared<PrecCore>();
  PrecCore& c = *core;
  c.ctx = ctx;
  c.ndof = d->A_prec->nrow();
  c.nsub = d->nsub;
  c.local_kind = d->family == 2 ? 1 : 0;
  c.fine_space = d->space;
  const int64_t ndof = c.ndof;
  const char* env_leaf = getenv("MDD_ND_LEAF");
  const int leaf = d->leaf_size > 0 ? d->leaf_size : (env_leaf ? std::max(4, atoi(env_leaf)) : 64);
  const mdd_pattern& AP = *d->A_prec->pat;
  // ---- size cap (linalg.py:80-84), checked in subdomain order
  for (int l = 0; l < d->nsub; ++l) {
    const int64_t nl = d->sub_ptr[l + 1] - d->sub_ptr[l];
    if (d->lu_cap > 0 && nl > d->lu_cap) {
      if (failed_ctx) *failed_ctx = l;
      fail(MDD_ECAP, "subdomain " + std::to_string(l) + ": dense factor of size " +
                         std::to_string(nl) + " exceeds cap " + std::to_string(d->lu_cap) +
                         "; raise the cap or shrink the block", l);
    }
  }
  // ---- local matrices (patterns + value sources)
  std::vector<MatrixInput> mats(d->nsub);
  if (c.local_kind == 0) {
    // transposed positions of A_prec's pattern (symmetry check per factorisation)
    std::vector<int32_t> tp(AP.nnz, -1);
    for (int64_t i = 0; i < AP.nrow; ++i)
      for (int32_t k = AP.h_rowptr[i]; k < AP.h_rowptr[i + 1]; ++k) {
        const int32_t j = AP.h_cols[k];
        const int32_t* b = AP.h_cols.data() + AP.h_rowptr[j];
        const int32_t* e = AP.h_cols.data() + AP.h_rowptr[j + 1];
        const int32_t* it = std::lower_bound(b, e, (int32_t)i);
        if (it != e && *it == i) tp[k] = (int32_t)(it - AP.h_cols.data());
      }
    c.tpos.upload(tp, s);
    c.symflag.alloc(1);
    // exact minors of A_prec on I_l (precond.py:166-171)
    const unsigned nth = std::max(1u, std::min(16u, std::thread::hardware_concurrency()));
    std::vector<std::thread> th;
    std::atomic<int> next{0};
    for (unsigned t = 0; t < nth; ++t)
      th.emplace_back([&] {
        std::vector<int32_t> g2l(ndof, -1);
        for (int l = next++; l < d->nsub; l = next++) {
          MatrixInput& mi = mats[l];
          const int64_t b = d->sub_ptr[l], e = d->sub_ptr[l + 1];
          mi.n = (int32_t)(e - b);
          for (int64_t i = b; i < e; ++i) g2l[d->sub_dofs[i]] = (int32_t)(i - b);
          mi.rowptr.assign(1, 0);
          mi.grid = d->dof_grid > 0 ? d->dof_grid : 2;
          mi.xyz.resize(3 * (size_t)mi.n);
          for (int64_t i = b; i < e; ++i) {
            const int64_t g = d->sub_dofs[i];
            for (int32_t k = AP.h_rowptr[g]; k < AP.h_rowptr[g + 1]; ++k) {
              const int32_t lc = g2l[AP.h_cols[k]];
              if (lc >= 0) {
                mi.cols.push_back(lc);
                mi.src.push_back(k);
              }
            }
            mi.rowptr.push_back((int32_t)mi.cols.size());
            for (int a = 0; a < 3; ++a) mi.xyz[3 * (i - b) + a] = d->dof_xyz[3 * g + a];
          }
          for (int64_t i = b; i < e; ++i) g2l[d->sub_dofs[i]] = -1;
        }
      });
    for (auto& x : th) x.join();
  } else {
    // impras: submesh assembly + boundary faces (precond.py:82-139)
    const mdd_space* fs = d->space;
    if (!fs || !d->sub_tet_ptr || !d->sub_tets) fail(MDD_EINVAL, "impras needs subdomain tets");
    const int64_t nv = fs->nv;
    std::vector<int32_t> h_cell, h_sub, h_mask, h_e2l;
    std::vector<std::vector<int64_t>> pairs_by_col(8);  // encoded index into per-sub lists
    std::vector<int32_t> row_off(d->nsub + 1, 0), ent_off(d->nsub + 1, 0);
    std::vector<int32_t> all_rowptr, all_cols;
    std::vector<std::vector<int32_t>> sub_e2l(d->nsub);
    // edge key lookup for faces
    std::vector<int64_t> ekeys(fs->ne);
    {
      static const int EA[6] = {0, 0, 0, 1, 1, 2}, EB[6] = {1, 2, 3, 2, 3, 3};
      for (int64_t t = 0; t < fs->nt; ++t)
        for (int e = 0; e < 6; ++e) {
          int64_t a = fs->h_tets[t * 4 + EA[e]], b = fs->h_tets[t * 4 + EB[e]];
          if (a > b) std::swap(a, b);
          ekeys[fs->h_tet_edges[t * 6 + e]] = a * nv + b;
        }
    }
    std::vector<int32_t> eorder(fs->ne);
    std::iota(eorder.begin(), eorder.end(), 0);
    std::sort(eorder.begin(), eorder.end(), [&](int32_t x, int32_t y) { return ekeys[x] < ekeys[y]; });
    auto find_edge = [&](int64_t a, int64_t b) {
      const int64_t key = a * nv + b;
      auto it = std::lower_bound(eorder.begin(), eorder.end(), key,
                                 [&](int32_t id, int64_t k) { return ekeys[id] < k; });
      if (it == eorder.end() || ekeys[*it] != key) fail(MDD_EINVAL, "face edge not in mesh");
      return *it;
    };
    std::vector<int32_t> face_flat, face_l, face_ptr(d->nsub + 1, 0);
    const int64_t ncell = (int64_t)fs->n * fs->n * fs->n;
    std::vector<int32_t> g2l(ndof, -1);
    for (int l = 0; l < d->nsub; ++l) {
      MatrixInput& mi = mats[l];
      const int64_t b = d->sub_ptr[l], e = d->sub_ptr[l + 1];
      mi.n = (int32_t)(e - b);
      for (int64_t i = b; i < e; ++i) g2l[d->sub_dofs[i]] = (int32_t)(i - b);
      // local pattern: pairs sharing a subdomain tet, plus boundary-face pairs (subset)
      std::vector<std::vector<int32_t>> rows(mi.n);
      const int64_t tb = d->sub_tet_ptr[l], te = d->sub_tet_ptr[l + 1];
      std::unordered_map<int64_t, int32_t> cellmask;
      for (int64_t k = tb; k < te; ++k) {
        const int64_t t = d->sub_tets[k];
        int32_t loc[6];
        for (int q = 0; q < 6; ++q) {
          const int32_t dd = fs->h_e2d[fs->h_tet_edges[t * 6 + q]];
          loc[q] = dd >= 0 ? g2l[dd] : -1;
        }
        for (int a = 0; a < 6; ++a)
          if (loc[a] >= 0)
            for (int q = 0; q < 6; ++q)
              if (loc[q] >= 0) rows[loc[a]].push_back(loc[q]);
        cellmask[t / 6] |= 1 << (t % 6);
      }
      row_off[l + 1] = row_off[l] + mi.n + 1;
      mi.rowptr.assign(1, 0);
      for (int32_t i = 0; i < mi.n; ++i) {
        auto& r = rows[i];
        std::sort(r.begin(), r.end());
        r.erase(std::unique(r.begin(), r.end()), r.end());
        for (int32_t cc : r) mi.cols.push_back(cc);
        mi.rowptr.push_back((int32_t)mi.cols.size());
      }
      mi.src.resize(mi.cols.size());
      for (size_t k = 0; k < mi.cols.size(); ++k) mi.src[k] = ent_off[l] + (int32_t)k;
      ent_off[l + 1] = ent_off[l] + (int32_t)mi.cols.size();
      all_rowptr.insert(all_rowptr.end(), mi.rowptr.begin(), mi.rowptr.end());
      all_cols.insert(all_cols.end(), mi.cols.begin(), mi.cols.end());
      mi.xyz.resize(3 * (size_t)mi.n);
      for (int64_t i = b; i < e; ++i)
        for (int a = 0; a < 3; ++a) mi.xyz[3 * (i - b) + a] = d->dof_xyz[3 * d->sub_dofs[i] + a];
      // (subdomain, cell) pairs by colour
      std::vector<int64_t> cells;
      for (auto& kv : cellmask) cells.push_back(kv.first);
      std::sort(cells.begin(), cells.end());
      for (int64_t cell : cells) {
        const int64_t n = fs->n;
        const int64_t cx = cell / (n * n), cy = (cell / n) % n, cz = cell % n;
        const int colr = (int)(((cx & 1) << 2) | ((cy & 1) << 1) | (cz & 1));
        pairs_by_col[colr].push_back((int64_t)h_cell.size());
        h_cell.push_back((int32_t)cell);
        h_sub.push_back(l);
        h_mask.push_back(cellmask[cell]);
        for (int p = 0; p < 6; ++p)
          for (int q = 0; q < 6; ++q) {
            const int64_t t = cell * 6 + p;
            const int32_t dd = fs->h_e2d[fs->h_tet_edges[t * 6 + q]];
            h_e2l.push_back(((cellmask[cell] >> p) & 1) && dd >= 0 ? g2l[dd] : -1);
          }
      }
      // boundary faces of the subdomain
      if (d->sub_bface_ptr) {
        for (int64_t f = d->sub_bface_ptr[l]; f < d->sub_bface_ptr[l + 1]; ++f) {
          const int64_t* fv = d->sub_bfaces + 3 * f;
          const int tp[3][2] = {{0, 1}, {0, 2}, {1, 2}};
          for (int q = 0; q < 3; ++q) face_flat.push_back((int32_t)fv[q]);
          for (int q = 0; q < 3; ++q) {
            const int32_t dd = fs->h_e2d[find_edge(fv[tp[q][0]], fv[tp[q][1]])];
            face_l.push_back(dd >= 0 ? g2l[dd] : -1);
          }
        }
        face_ptr[l + 1] = (int32_t)(face_flat.size() / 3);
      }
      for (int64_t i = b; i < e; ++i) g2l[d->sub_dofs[i]] = -1;
      (void)ncell;
    }
    // reorder pair arrays by colour
    std::vector<int32_t> pc, ps, pm, pe;
    c.loc_color_off.assign(9, 0);
    for (int col = 0; col < 8; ++col) {
      c.loc_color_off[col] = (int64_t)pc.size();
      for (int64_t k : pairs_by_col[col]) {
        pc.push_back(h_cell[k]);
        ps.push_back(h_sub[k]);
        pm.push_back(h_mask[k]);
        pe.insert(pe.end(), h_e2l.begin() + k * 36, h_e2l.begin() + k * 36 + 36);
      }
    }
    c.loc_color_off[8] = (int64_t)pc.size();
    std::vector<int32_t> cellmask_arr(pc);
    cellmask_arr.insert(cellmask_arr.end(), pm.begin(), pm.end());
    c.loc_tet.upload(cellmask_arr, s);  // [cells | masks]
    c.loc_tet_sub.upload(ps, s);
    c.loc_e2l.upload(pe, s);
    c.h_loc_row_off = row_off;
    c.h_loc_ent_off = ent_off;
    c.loc_row_off.upload(row_off, s);
    c.loc_rowptr.upload(all_rowptr, s);
    c.loc_cols.upload(all_cols, s);
    c.loc_sub_off.upload(ent_off, s);
    c.loc_vals.alloc(std::max<int64_t>(1, ent_off[d->nsub]));
    c.loc_face.upload(face_flat, s);
    c.loc_face_l.upload(face_l, s);
    c.loc_face_sub.upload(face_ptr, s);
    c.n_loc_faces = (int64_t)face_flat.size() / 3;
  }
  auto t0 = std::chrono::steady_clock::now();
  c.sub.build(ctx, mats, leaf);
  // gather indices + ownership (subdomain order)
  {
    std::vector<int32_t> gidx(c.sub.nloc);
    std::vector<double> wloc(c.sub.nloc, 1.0);
    for (int l = 0; l < d->nsub; ++l) {
      const int64_t b = d->sub_ptr[l];
      const auto& pm = c.sub.perm[l];
      for (int32_t a = 0; a < c.sub.mat_n[l]; ++a) {
        gidx[c.sub.mat_off[l] + a] = (int32_t)d->sub_dofs[b + pm[a]];
        if (d->sub_pou) wloc[c.sub.mat_off[l] + a] = d->sub_pou[b + pm[a]];
      }
    }
    std::vector<int32_t> optr(ndof + 1, 0), oidx(c.sub.nloc);
    std::vector<double> ow(c.sub.nloc);
    for (int64_t t = 0; t < c.sub.nloc; ++t) optr[gidx[t] + 1]++;
    for (int64_t i = 0; i < ndof; ++i) optr[i + 1] += optr[i];
    std::vector<int32_t> fillp(optr.begin(), optr.end() - 1);
    for (int64_t t = 0; t < c.sub.nloc; ++t) {  // ascending t == ascending subdomain
      const int32_t k = fillp[gidx[t]]++;
      oidx[k] = (int32_t)t;
      ow[k] = wloc[t];
    }
    c.gidx.upload(gidx, s);
    c.own_ptr.upload(optr, s);
    c.own_idx.upload(oidx, s);
    c.own_w.upload(ow, s);
  }
  // ---- coarse level
  if (d->levels == 2) {
    if (!d->R0 || !d->coarse_space || !d->coarse_dof_xyz)
      fail(MDD_EINVAL, "two-level preconditioner needs a coarse link");
    c.have_coarse = true;
    const mdd_space* cs = d->coarse_space;
    c.coarse_space = cs;
    c.ncs = cs->ndof;
    if (d->R0->nrow() != c.ncs || d->R0->ncol() != ndof) fail(MDD_EINVAL, "R0 has the wrong shape");
    if (d->lu_cap > 0 && c.ncs > d->lu_cap) {
      if (failed_ctx) *failed_ctx = -1;
      fail(MDD_ECAP, "coarse space: dense factor of size " + std::to_string(c.ncs) +
                         " exceeds cap " + std::to_string(d->lu_cap) +
                         "; raise the cap or shrink the block", -1);
    }
    std::vector<MatrixInput> cm(1);
    cm[0].n = (int32_t)c.ncs;
    if (d->tet_map) {  // nested meshes: element-wise Galerkin on the coarse mesh pattern
      c.A0.reset(new_csr(ctx, cs->pat, true));
    } else {           // non-nested: generic R0 A_prec R0^T plan (pattern of the product)
      build_rap(c, *d->R0, AP, s);
    }
    cm[0].rowptr = c.A0->pat->h_rowptr;
    cm[0].cols = c.A0->pat->h_cols;
    cm[0].src.resize(cm[0].cols.size());
    std::iota(cm[0].src.begin(), cm[0].src.end(), 0);
    cm[0].xyz.assign(d->coarse_dof_xyz, d->coarse_dof_xyz + 3 * c.ncs);
    c.coarse.build(ctx, cm, leaf);
    // R0 with rows in coarse ND order; R0^T with columns in coarse ND order
    const auto& pm = c.coarse.perm[0];
    std::vector<int32_t> ip(c.ncs);
    for (int64_t a = 0; a < c.ncs; ++a) ip[pm[a]] = (int32_t)a;
    const mdd_pattern& RP = *d->R0->pat;
    std::vector<double> rv(RP.nnz);
    d->R0->vals.download(rv.data(), RP.nnz, s);
    CK(cudaStreamSynchronize(s));
    std::vector<int32_t> rp(c.ncs + 1, 0), rc;
    std::vector<double> rvals;
    rc.reserve(RP.nnz);
    rvals.reserve(RP.nnz);
    for (int64_t a = 0; a < c.ncs; ++a) {
      const int32_t r = pm[a];
      for (int32_t k = RP.h_rowptr[r]; k < RP.h_rowptr[r + 1]; ++k) {
        rc.push_back(RP.h_cols[k]);
        rvals.push_back(rv[k]);
      }
      rp[a + 1] = (int32_t)rc.size();
    }
    c.R0p = csr_host(ctx, c.ncs, ndof, std::move(rp), std::move(rc), rvals);
    std::vector<int32_t> tp(ndof + 1, 0), tc(RP.nnz);
    std::vector<double> tv(RP.nnz);
    for (int64_t k = 0; k < RP.nnz; ++k) tp[RP.h_cols[k] + 1]++;
    for (int64_t i = 0; i < ndof; ++i) tp[i + 1] += tp[i];
    std::vector<int32_t> fp(tp.begin(), tp.end() - 1);
    for (int64_t r = 0; r < c.ncs; ++r)  // ascending original coarse index p
      for (int32_t k = RP.h_rowptr[r]; k < RP.h_rowptr[r + 1]; ++k) {
        const int32_t pos = fp[RP.h_cols[k]]++;
        tc[pos] = ip[r];
        tv[pos] = rv[k];
      }
    c.R0Tp = csr_host(ctx, ndof, c.ncs, std::move(tp), std::move(tc), tv);
    // Galerkin index data: fine tets per coarse tet (ascending)
    const mdd_space* fs = d->space;
    if (c.rap) goto coarse_done;
    if (!fs) fail(MDD_EINVAL, "two-level preconditioner needs the fine space");
    std::vector<int32_t> tm(fs->nt);
    for (int64_t t = 0; t < fs->nt; ++t) {
      if (d->tet_map[t] < 0 || d->tet_map[t] >= cs->nt) fail(MDD_EINVAL, "tet_map out of range");
      tm[t] = (int32_t)d->tet_map[t];
    }
    std::vector<int32_t> cptr(cs->nt + 1, 0), cidx(fs->nt);
    for (int64_t t = 0; t < fs->nt; ++t) cptr[tm[t] + 1]++;
    for (int64_t q = 0; q < cs->nt; ++q) cptr[q + 1] += cptr[q];
    {
      std::vector<int32_t> f2(cptr.begin(), cptr.end() - 1);
      for (int64_t t = 0; t < fs->nt; ++t) cidx[f2[tm[t]]++] = (int32_t)t;
    }
    c.tet_map.upload(tm, s);
    c.cfine_ptr.upload(cptr, s);
    c.cfine_idx.upload(cidx, s);
    // global impedance faces -> containing fine tet
    c.n_gfaces = d->nbf_global;
    if (c.n_gfaces) {
      const int64_t nv = fs->nv;
      std::unordered_map<int64_t, int32_t> fkey;
      fkey.reserve(c.n_gfaces * 2);
      for (int64_t f = 0; f < c.n_gfaces; ++f) {
        const int64_t* v = d->bfaces_global + 3 * f;
        fkey[(v[0] * nv + v[1]) * nv + v[2]] = (int32_t)f;
      }
      std::vector<int32_t> ftet(c.n_gfaces, -1), gf(3 * c.n_gfaces);
      static const int LF[4][3] = {{1, 2, 3}, {0, 2, 3}, {0, 1, 3}, {0, 1, 2}};
      for (int64_t t = 0; t < fs->nt; ++t)
        for (int q = 0; q < 4; ++q) {
          int64_t v[3] = {fs->h_tets[t * 4 + LF[q][0]], fs->h_tets[t * 4 + LF[q][1]],
                          fs->h_tets[t * 4 + LF[q][2]]};
          std::sort(v, v + 3);
          auto it = fkey.find((v[0] * nv + v[1]) * nv + v[2]);
          if (it != fkey.end()) ftet[it->second] = (int32_t)t;
        }
      for (int64_t f = 0; f < c.n_gfaces; ++f) {
        if (ftet[f] < 0) fail(MDD_EINVAL, "boundary face without a tet");
        for (int q = 0; q < 3; ++q) gf[3 * f + q] = (int32_t)d->bfaces_global[3 * f + q];
      }
      std::vector<int32_t> gptr(cs->nt + 1, 0), gidx2(c.n_gfaces);
      for (int64_t f = 0; f < c.n_gfaces; ++f) gptr[tm[ftet[f]] + 1]++;
      for (int64_t q = 0; q < cs->nt; ++q) gptr[q + 1] += gptr[q];
      std::vector<int32_t> f2(gptr.begin(), gptr.end() - 1);
      for (int64_t f = 0; f < c.n_gfaces; ++f) gidx2[f2[tm[ftet[f]]]++] = (int32_t)f;
      c.face_tet.upload(ftet, s);
      c.gfaces.upload(gf, s);
      c.cface_ptr.upload(gptr, s);
      c.cface_idx.upload(gidx2, s);
    }
  }
coarse_done:
  CK(cudaStreamCreateWithFlags(&c.s2, cudaStreamNonBlocking));
  CK(cudaEventCreateWithFlags(&c.ev_fork, cudaEventDisableTiming));
  CK(cudaEventCreateWithFlags(&c.ev_join, cudaEventDisableTiming));
  c.t1.alloc(ndof);
  c.t2.alloc(ndof);
  c.t3.alloc(ndof);
  c.t4.alloc(ndof);
  const double sym_ms =
      std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now() - t0).count();
  auto P = std::make_unique<mdd_prec>();
  P->core = core;
  P->family = d->family;
  P->levels = d->levels;
  P->correction = d->correction;
  P->A_corr = d->A_corr ? d->A_corr : d->A_prec;
  numeric_setup(P.get(), d->A_prec, d->prec_coeffs, failed_ctx);
  c.stats[0] = c.sub.nnodes + c.coarse.nnodes;
  c.stats[1] = std::max(c.sub.max_m, c.coarse.max_m);
  c.stats[2] = c.sub.factor_entries + c.coarse.factor_entries;
  c.stats[3] = c.sub.factor_flops + c.coarse.factor_flops;
  c.stats[5] = std::max(c.sub.nlevels, c.coarse.nlevels);
  c.stats[6] = (double)c.sub.nloc;
  c.stats[7] = (double)c.ncs;
  (void)sym_ms;
  *out = P.release();
  MDD_API_END
}

int mdd_prec_variant(const mdd_prec* base, int family, int levels, int correction,
                     const mdd_csr* A_corr, mdd_prec** out) {
  MDD_API_BEGIN
  const int kind_b = base->family == 2 ? 1 : 0, kind_n = family == 2 ? 1 : 0;
  if (kind_b != kind_n) fail(MDD_EINVAL, "variant would need different local factorizations");
  if (levels == 2 && !base->core->have_coarse)
    fail(MDD_EINVAL, "variant needs a coarse factor the state does not hold");
  auto P = std::make_unique<mdd_prec>();
  P->core = base->core;
  P->family = family;
  P->levels = levels;
  P->correction = correction;
  P->A_corr = A_corr ? A_corr : base->A_corr;
  P->comm = base->comm;
  P->halo = base->halo;
  P->R0own = base->R0own;
  *out = P.release();
  MDD_API_END
}

void mdd_prec_destroy(mdd_prec* P) {
  if (!P) return;
  cudaSetDevice(P->core->ctx->device);
  delete P;
}

int mdd_prec_apply(mdd_prec* P, const mdd_complex* v, mdd_complex* out) {
  MDD_API_BEGIN
  mdd_ctx* ctx = P->core->ctx;
  CK(cudaSetDevice(ctx->device));
  const int64_t n = P->core->ndof;
  DevBuf<double2> dv(n), dout(n);
  dv.upload(reinterpret_cast<const double2*>(v), n, ctx->stream);
  prec_apply_dev(P, dv.p, dout.p, ctx->stream);
  dout.download(reinterpret_cast<double2*>(out), n, ctx->stream);
  CK(cudaStreamSynchronize(ctx->stream));
  MDD_API_END
}

int mdd_prec_coarse_apply(mdd_prec* P, const mdd_complex* v, mdd_complex* out) {
  MDD_API_BEGIN
  mdd_ctx* ctx = P->core->ctx;
  CK(cudaSetDevice(ctx->device));
  if (!P->core->have_coarse) fail(MDD_EINVAL, "preconditioner has no coarse level");
  const int64_t n = P->core->ndof;
  DevBuf<double2> dv(n), dout(n);
  dv.upload(reinterpret_cast<const double2*>(v), n, ctx->stream);
  coarse_solve(P, dv.p, dout.p, ctx->stream);
  dout.download(reinterpret_cast<double2*>(out), n, ctx->stream);
  CK(cudaStreamSynchronize(ctx->stream));
  MDD_API_END
}

// Device-timed applies (CUDA events on the context stream, inputs resident):
// which = 0 full apply, 1 subdomain solves only (restriction + solves), 2 coarse solve only.
int mdd_prec_apply_bench(mdd_prec* P, int which, int reps, double* ms_per_call) {
  MDD_API_BEGIN
  mdd_ctx* ctx = P->core->ctx;
  CK(cudaSetDevice(ctx->device));
  if (which == 2 && !P->core->have_coarse) fail(MDD_EINVAL, "preconditioner has no coarse level");
  const int64_t n = P->core->ndof;
  DevBuf<double2> dv(n), dout(n);
  CK(cudaMemsetAsync(dv.p, 0, sizeof(double2) * n, ctx->stream));
  auto one = [&]() {
    if (which == 0) prec_apply_dev(P, dv.p, dout.p, ctx->stream);
    else if (which == 1) one_level_solve(P, dv.p, ctx->stream);
    else coarse_solve(P, dv.p, dout.p, ctx->stream);
  };
  for (int i = 0; i < 3; ++i) one();
  cudaEvent_t e0, e1;
  CK(cudaEventCreate(&e0));
  CK(cudaEventCreate(&e1));
  CK(cudaEventRecord(e0, ctx->stream));
  for (int i = 0; i < reps; ++i) one();
  CK(cudaEventRecord(e1, ctx->stream));
  CK(cudaEventSynchronize(e1));
  float ms = 0;
  CK(cudaEventElapsedTime(&ms, e0, e1));
  cudaEventDestroy(e0);
  cudaEventDestroy(e1);
  *ms_per_call = reps > 0 ? ms / reps : 0.0;
  MDD_API_END
}

int mdd_prec_set_comm(mdd_prec* P, mdd_comm* comm) {
  MDD_API_BEGIN
  if (comm && comm->ctx != P->core->ctx) fail(MDD_EINVAL, "comm: different context");
  P->comm = comm;
  MDD_API_END
}

int mdd_prec_set_halo(mdd_prec* P, int64_t need_lo, int64_t need_hi) {
  MDD_API_BEGIN
  if (!P->comm) fail(MDD_EINVAL, "set_halo: attach the communicator first (mdd_prec_set_comm)");
  PrecCore& c = *P->core;
  CK(cudaSetDevice(c.ctx->device));
  cudaStream_t s = c.ctx->stream;
  auto h = std::make_shared<mdd_halo>();
  comm_halo_setup(P->comm, h.get(), c.ndof, need_lo, need_hi, s);
  P->halo = h;
  P->R0own.reset();
  if (c.have_coarse) {
    // R0 (rows in coarse ND order, as the coarse plan expects) restricted to the owned columns
    const int me = P->comm->rank;
    const int64_t lo = h->own_lo[me], hi = h->own_hi[me];
    const mdd_pattern& RP = *c.R0p->pat;
    std::vector<double> rv(RP.nnz);
    c.R0p->vals.download(rv.data(), RP.nnz, s);
    CK(cudaStreamSynchronize(s));
    std::vector<int32_t> rp(c.ncs + 1, 0), rc;
    std::vector<double> vals;
    for (int64_t a = 0; a < c.ncs; ++a) {
      for (int32_t k = RP.h_rowptr[a]; k < RP.h_rowptr[a + 1]; ++k)
        if (RP.h_cols[k] >= lo && RP.h_cols[k] < hi) {
          rc.push_back(RP.h_cols[k]);
          vals.push_back(rv[k]);
        }
      rp[a + 1] = (int32_t)rc.size();
    }
    P->R0own = std::shared_ptr<mdd_csr>(csr_host(c.ctx, c.ncs, c.ndof, std::move(rp), std::move(rc), vals).release());
    CK(cudaStreamSynchronize(s));
  }
  MDD_API_END
}

int mdd_prec_halo_info(const mdd_prec* P, int64_t* own_lo, int64_t* own_hi, int64_t* need_lo, int64_t* need_hi,
                       int64_t* exchanged_rows) {
  MDD_API_BEGIN
  if (!P->halo) fail(MDD_EINVAL, "halo_info: no row ranges set");
  const mdd_halo& h = *P->halo;
  const int me = P->comm->rank;
  *own_lo = h.own_lo[me];
  *own_hi = h.own_hi[me];
  *need_lo = h.need_lo[me];
  *need_hi = h.need_hi[me];
  *exchanged_rows = (h.need_hi[me] - h.need_lo[me]) - (h.own_hi[me] - h.own_lo[me]);
  MDD_API_END
}

int mdd_prec_local_matrix_size(const mdd_prec* P, int32_t sub, int64_t* n, int64_t* nnz) {
  MDD_API_BEGIN
  const PrecCore& c = *P->core;
  if (c.h_loc_row_off.empty()) fail(MDD_EINVAL, "local matrices exist only for impras preconditioners");
  if (sub < 0 || sub + 1 >= (int32_t)c.h_loc_row_off.size()) fail(MDD_EINVAL, "local matrix: subdomain out of range");
  *n = c.h_loc_row_off[sub + 1] - c.h_loc_row_off[sub] - 1;
  *nnz = c.h_loc_ent_off[sub + 1] - c.h_loc_ent_off[sub];
  MDD_API_END
}

int mdd_prec_local_matrix(const mdd_prec* P, int32_t sub, int32_t* rowptr, int32_t* cols, mdd_complex* vals) {
  MDD_API_BEGIN
  const PrecCore& c = *P->core;
  if (c.h_loc_row_off.empty()) fail(MDD_EINVAL, "local matrices exist only for impras preconditioners");
  if (sub < 0 || sub + 1 >= (int32_t)c.h_loc_row_off.size()) fail(MDD_EINVAL, "local matrix: subdomain out of range");
  CK(cudaSetDevice(c.ctx->device));
  cudaStream_t s = c.ctx->stream;
  const int64_t n = c.h_loc_row_off[sub + 1] - c.h_loc_row_off[sub] - 1;
  const int64_t e0 = c.h_loc_ent_off[sub], nnz = c.h_loc_ent_off[sub + 1] - e0;
  CK(cudaMemcpyAsync(rowptr, c.loc_rowptr.p + c.h_loc_row_off[sub], sizeof(int32_t) * (n + 1), cudaMemcpyDeviceToHost, s));
  if (nnz > 0) {
    CK(cudaMemcpyAsync(cols, c.loc_cols.p + e0, sizeof(int32_t) * nnz, cudaMemcpyDeviceToHost, s));
    CK(cudaMemcpyAsync(vals, c.loc_vals.p + e0, sizeof(double2) * nnz, cudaMemcpyDeviceToHost, s));
  }
  CK(cudaStreamSynchronize(s));
  MDD_API_END
}

int mdd_prec_pivot_ratio(const mdd_prec* P, double* sub_ratio, double* coarse_ratio) {
  MDD_API_BEGIN
  *sub_ratio = P->core->sub.min_pivot_ratio;
  *coarse_ratio = P->core->have_coarse ? P->core->coarse.min_pivot_ratio : INFINITY;
  MDD_API_END
}

int mdd_prec_stats(const mdd_prec* P, double* out8) {
  MDD_API_BEGIN
  for (int i = 0; i < 8; ++i) out8[i] = P->core->stats[i];
  MDD_API_END
}

int mdd_prec_symmetric(const mdd_prec* P, int* sym) {
  MDD_API_BEGIN
  int f = 1;
  if (P->core->sym_checked) {
    P->core->symflag.download(&f, 1, P->core->ctx->stream);
    CK(cudaStreamSynchronize(P->core->ctx->stream));
  }
  *sym = f == 0 ? 1 : 0;
  MDD_API_END
}

int mdd_prec_flop_counts(const mdd_prec* P, double* out3) {
  MDD_API_BEGIN
  const PrecCore& c = *P->core;
  int f = 1;
  if (c.sym_checked) {
    c.symflag.download(&f, 1, c.ctx->stream);
    CK(cudaStreamSynchronize(c.ctx->stream));
  }
  out3[0] = c.sub.factor_flops + c.coarse.factor_flops;
  out3[1] = c.sub.lu_flops + c.coarse.lu_flops;
  // the coarse block and ImpRAS local matrices are never taken as symmetric
  out3[2] = (f == 0 ? c.sub.exec_flops_sym : c.sub.exec_flops_full) + c.coarse.exec_flops_full;
  MDD_API_END
}

int mdd_prec_refactor(mdd_prec* P, const mdd_csr* A_prec, const mdd_coeffs* pc) {
  MDD_API_BEGIN
  CK(cudaSetDevice(P->core->ctx->device));
  numeric_setup(P, A_prec, pc, nullptr);
  MDD_API_END
}

}  // extern "C"
