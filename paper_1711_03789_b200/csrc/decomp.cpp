// Host (C++) decomposition helpers: overlap growth, subdomain DoF sets, the
// fine->coarse nesting map and the nested coarse restriction R0.
//
// the reference builds these with per-edge Python loops
// (decomp.py:97-176, 212-297; mesh.py:231-263), 18 s at cfg0 and minutes at
// the larger configs.  They are setup-time inputs of the device path; here
// they are threaded C++ over the structured Kuhn mesh, with the reference's
// semantics (index sets bit-identical, R0 values equal to rounding; pinned by
// tests/test_host_mesh_decomp.py against the reference's golden fixtures).
// Output arrays are malloc'ed here and released with mdd_free.
#include <algorithm>
#include <atomic>
#include <cmath>
#include <cstdlib>
#include <cstring>
#include <exception>
#include <mutex>
#include <string>
#include <thread>
#include <vector>

#include "mdd_internal.h"

namespace mdd {
namespace {

const int LF[4][3] = {{1, 2, 3}, {0, 2, 3}, {0, 1, 3}, {0, 1, 2}};  // mesh.LOCAL_FACES
const int EA[6] = {0, 0, 0, 1, 1, 2}, EB[6] = {1, 2, 3, 2, 3, 3};  // mesh.LOCAL_EDGES
// local edge index of the vertex pair (a,b), a<b
int ledge(int a, int b) {
  static const int T[4][4] = {{-1, 0, 1, 2}, {0, -1, 3, 4}, {1, 3, -1, 5}, {2, 4, 5, -1}};
  return T[a][b];
}

template <typename F>
void par_items(int64_t n, F&& f) {
  const unsigned nth = std::max(1u, std::min(16u, std::thread::hardware_concurrency()));
  std::atomic<int64_t> next{0};
  std::exception_ptr err;
  std::mutex mu;
  auto body = [&](unsigned tid) {
    try {
      for (int64_t i = next++; i < n; i = next++) f(tid, i);
    } catch (...) {
      std::lock_guard<std::mutex> g(mu);
      if (!err) err = std::current_exception();
    }
  };
  std::vector<std::thread> th;
  const unsigned nt = (unsigned)std::min<int64_t>(nth, std::max<int64_t>(1, n));
  for (unsigned t = 1; t < nt; ++t) th.emplace_back(body, t);
  body(0);
  for (auto& x : th) x.join();
  if (err) std::rethrow_exception(err);
}

// ragged per-item outputs -> malloc'ed (ptr, idx)
void emit_ragged(std::vector<std::vector<int64_t>>& parts, int64_t** out_ptr, int64_t** out_idx) {
  const size_t n = parts.size();
  int64_t tot = 0;
  for (auto& p : parts) tot += (int64_t)p.size();
  int64_t* ptr = (int64_t*)malloc(sizeof(int64_t) * (n + 1));
  int64_t* idx = (int64_t*)malloc(sizeof(int64_t) * std::max<int64_t>(1, tot));
  if (!ptr || !idx) {
    free(ptr);
    free(idx);
    fail(MDD_ENOMEM, "decomposition: out of host memory");
  }
  ptr[0] = 0;
  for (size_t i = 0; i < n; ++i) {
    std::copy(parts[i].begin(), parts[i].end(), idx + ptr[i]);
    ptr[i + 1] = ptr[i] + (int64_t)parts[i].size();
  }
  *out_ptr = ptr;
  *out_idx = idx;
}

// barycentric map of a tet: lam_{1..3} = Binv (x - v0), lam_0 = 1 - sum
struct Bary {
  double v0[3], inv[3][3];
};
Bary bary_of(const double* verts, const int64_t* tv) {
  Bary b;
  double B[3][3];  // columns v_i - v_0
  for (int r = 0; r < 3; ++r) {
    b.v0[r] = verts[tv[0] * 3 + r];
    for (int i = 0; i < 3; ++i) B[r][i] = verts[tv[i + 1] * 3 + r] - b.v0[r];
  }
  const double c00 = B[1][1] * B[2][2] - B[1][2] * B[2][1];
  const double c01 = B[1][2] * B[2][0] - B[1][0] * B[2][2];
  const double c02 = B[1][0] * B[2][1] - B[1][1] * B[2][0];
  const double id = 1.0 / (B[0][0] * c00 + B[0][1] * c01 + B[0][2] * c02);
  b.inv[0][0] = c00 * id;
  b.inv[1][0] = c01 * id;
  b.inv[2][0] = c02 * id;
  b.inv[0][1] = (B[0][2] * B[2][1] - B[0][1] * B[2][2]) * id;
  b.inv[1][1] = (B[0][0] * B[2][2] - B[0][2] * B[2][0]) * id;
  b.inv[2][1] = (B[0][1] * B[2][0] - B[0][0] * B[2][1]) * id;
  b.inv[0][2] = (B[0][1] * B[1][2] - B[0][2] * B[1][1]) * id;
  b.inv[1][2] = (B[0][2] * B[1][0] - B[0][0] * B[1][2]) * id;
  b.inv[2][2] = (B[0][0] * B[1][1] - B[0][1] * B[1][0]) * id;
  return b;
}
void bary_eval(const Bary& b, const double* x, double (&lam)[4]) {
  double d[3] = {x[0] - b.v0[0], x[1] - b.v0[1], x[2] - b.v0[2]};
  double s = 0;
  for (int i = 0; i < 3; ++i) {
    lam[i + 1] = b.inv[i][0] * d[0] + b.inv[i][1] * d[1] + b.inv[i][2] * d[2];
    s += lam[i + 1];
  }
  lam[0] = 1.0 - s;
}

}  // namespace
}  // namespace mdd

using namespace mdd;

extern "C" {

void mdd_free(void* p) { free(p); }

// decomp.extend_overlap (reference decomp.py:97-110): grow each tet set by
// `layers` rings of vertex-touching tets.  A tet touching a vertex of a set
// tet lies within one cell of it, so each ring is searched in the window of
// cells around the set.  Output sets are ascending.
int mdd_extend_overlap(int32_t n, int64_t nv, const int64_t* tets, int32_t nsub, const int64_t* part_ptr,
                       const int64_t* part_idx, int32_t layers, int64_t** out_ptr, int64_t** out_idx) {
  MDD_API_BEGIN
  if (layers < 1) fail(MDD_EDECOMP, "layers must be >= 1");
  const int64_t nt = 6LL * n * n * n;
  std::vector<std::vector<int64_t>> res(nsub);
  const unsigned nth = std::max(1u, std::min(16u, std::thread::hardware_concurrency()));
  std::vector<std::vector<uint8_t>> tmask(nth), vmask(nth);
  par_items(nsub, [&](unsigned tid, int64_t s) {
    const int64_t b = part_ptr[s], e = part_ptr[s + 1];
    if (b == e) return;
    auto& tm = tmask[tid];
    auto& vm = vmask[tid];
    if (tm.empty()) {
      tm.assign(nt, 0);
      vm.assign(nv, 0);
    }
    int64_t lo[3] = {n, n, n}, hi[3] = {-1, -1, -1};
    for (int64_t k = b; k < e; ++k) {
      const int64_t t = part_idx[k], c = t / 6;
      const int64_t cc[3] = {c / ((int64_t)n * n), (c / n) % n, c % n};
      for (int a = 0; a < 3; ++a) {
        lo[a] = std::min(lo[a], cc[a]);
        hi[a] = std::max(hi[a], cc[a]);
      }
      tm[t] = 1;
    }
    for (int a = 0; a < 3; ++a) {
      lo[a] = std::max<int64_t>(0, lo[a] - layers);
      hi[a] = std::min<int64_t>(n - 1, hi[a] + layers);
    }
    std::vector<int64_t> win;
    for (int64_t x = lo[0]; x <= hi[0]; ++x)
      for (int64_t y = lo[1]; y <= hi[1]; ++y)
        for (int64_t z = lo[2]; z <= hi[2]; ++z) {
          const int64_t c = (x * n + y) * n + z;
          for (int p = 0; p < 6; ++p) win.push_back(c * 6 + p);
        }
    for (int L = 0; L < layers; ++L) {
      for (int64_t t : win)
        if (tm[t])
          for (int i = 0; i < 4; ++i) vm[tets[t * 4 + i]] = 1;
      for (int64_t t : win)
        if (!tm[t])
          for (int i = 0; i < 4; ++i)
            if (vm[tets[t * 4 + i]]) {
              tm[t] = 1;
              break;
            }
      for (int64_t t : win)
        for (int i = 0; i < 4; ++i) vm[tets[t * 4 + i]] = 0;
    }
    auto& out = res[s];
    for (int64_t t : win)  // ascending (window enumerated in tet order)
      if (tm[t]) {
        out.push_back(t);
        tm[t] = 0;
      }
  });
  emit_ragged(res, out_ptr, out_idx);
  MDD_API_END
}

// decomp.subdomain_dof_sets (reference decomp.py:140-176): the kept unknowns of
// the subdomain tets minus those with a trace on internal subdomain-boundary
// faces (faces incident to one subdomain tet and not on the domain boundary):
// the edges of those faces and, for the order-2 space (tet_faces != NULL), the
// faces themselves.  Order 2 DoFs: [e, e + ned, f + 2 ned, f + 2 ned + nfd].
int mdd_subdomain_dofs(int32_t n, int64_t nv, const int64_t* tets, const int64_t* tet_edges, int64_t ne,
                       const int64_t* edge_to_dof, int64_t ned, const int64_t* tet_faces, int64_t nf,
                       const int64_t* face_to_dof, int64_t nfd, int32_t nsub, const int64_t* sub_ptr,
                       const int64_t* sub_tets, int64_t** out_ptr, int64_t** out_dofs) {
  MDD_API_BEGIN
  const int64_t nv1 = n + 1;
  auto on_domain_boundary = [&](int64_t a, int64_t b, int64_t c) {
    for (int ax = 0; ax < 3; ++ax) {
      auto co = [&](int64_t v) { return ax == 0 ? v / (nv1 * nv1) : ax == 1 ? (v / nv1) % nv1 : v % nv1; };
      const int64_t x = co(a);
      if ((x == 0 || x == n) && co(b) == x && co(c) == x) return true;
    }
    return false;
  };
  std::vector<std::vector<int64_t>> res(nsub);
  const unsigned nth = std::max(1u, std::min(16u, std::thread::hardware_concurrency()));
  std::vector<std::vector<uint8_t>> emask(nth), fmask(nth);
  par_items(nsub, [&](unsigned tid, int64_t s) {
    const int64_t b = sub_ptr[s], e = sub_ptr[s + 1];
    auto& em = emask[tid];
    auto& fm = fmask[tid];
    if (em.empty()) {
      em.assign(ne, 0);
      if (tet_faces) fm.assign(nf, 0);
    }
    struct FK {
      int64_t key, t;
      int f;
    };
    std::vector<FK> fk;
    fk.reserve((size_t)(e - b) * 4);
    for (int64_t k = b; k < e; ++k) {
      const int64_t t = sub_tets[k];
      for (int f = 0; f < 4; ++f) {
        int64_t v[3] = {tets[t * 4 + LF[f][0]], tets[t * 4 + LF[f][1]], tets[t * 4 + LF[f][2]]};
        std::sort(v, v + 3);
        fk.push_back({(v[0] * nv + v[1]) * nv + v[2], t, f});
      }
      for (int q = 0; q < 6; ++q) em[tet_edges[t * 6 + q]] |= 1;
      if (tet_faces)
        for (int q = 0; q < 4; ++q) fm[tet_faces[t * 4 + q]] |= 1;
    }
    std::sort(fk.begin(), fk.end(), [](const FK& x, const FK& y) { return x.key < y.key; });
    for (size_t i = 0; i < fk.size();) {
      size_t j = i;
      while (j < fk.size() && fk[j].key == fk[i].key) ++j;
      if (j - i == 1) {
        const int64_t key = fk[i].key;
        const int64_t a = key / (nv * nv), bb = (key / nv) % nv, c = key % nv;
        if (!on_domain_boundary(a, bb, c)) {  // internal subdomain-boundary face
          const int64_t t = fk[i].t;
          const int f = fk[i].f;
          for (int p = 0; p < 3; ++p)
            for (int q = p + 1; q < 3; ++q) {
              const int la = std::min(LF[f][p], LF[f][q]), lb = std::max(LF[f][p], LF[f][q]);
              em[tet_edges[t * 6 + ledge(la, lb)]] |= 2;
            }
          if (tet_faces) fm[tet_faces[t * 4 + f]] |= 2;
        }
      }
      i = j;
    }
    std::vector<int64_t> ed, fd;
    for (int64_t k = b; k < e; ++k) {
      const int64_t t = sub_tets[k];
      for (int q = 0; q < 6; ++q) {
        const int64_t g = tet_edges[t * 6 + q];
        if (em[g] == 1 && edge_to_dof[g] >= 0) ed.push_back(edge_to_dof[g]);
        em[g] |= 4;  // visited
      }
      if (tet_faces)
        for (int q = 0; q < 4; ++q) {
          const int64_t g = tet_faces[t * 4 + q];
          if (fm[g] == 1 && face_to_dof[g] >= 0) fd.push_back(face_to_dof[g]);
          fm[g] |= 4;
        }
    }
    for (int64_t k = b; k < e; ++k) {  // reset scratch
      const int64_t t = sub_tets[k];
      for (int q = 0; q < 6; ++q) em[tet_edges[t * 6 + q]] = 0;
      if (tet_faces)
        for (int q = 0; q < 4; ++q) fm[tet_faces[t * 4 + q]] = 0;
    }
    std::sort(ed.begin(), ed.end());
    std::sort(fd.begin(), fd.end());
    auto& out = res[s];
    out = ed;
    if (tet_faces) {
      for (int64_t x : ed) out.push_back(x + ned);
      for (int64_t x : fd) out.push_back(x + 2 * ned);
      for (int64_t x : fd) out.push_back(x + 2 * ned + nfd);
    }
  });
  emit_ragged(res, out_ptr, out_dofs);
  MDD_API_END
}

// mesh.nesting_map (reference mesh.py:231-263): the coarse tet containing each
// fine tet.  Candidates are the 6 Kuhn tets of the coarse cell holding the
// fine barycentre; the one maximising the barycentre's smallest barycentric
// coordinate wins, and all 4 fine vertices must lie in it to `tol`.
int mdd_nesting_map(int32_t nc, const double* cverts, const int64_t* ctets, int32_t nf, const double* fverts,
                    const int64_t* ftets, double tol, int64_t* out) {
  MDD_API_BEGIN
  if (nf % nc != 0)
    fail(MDD_EINVAL, "fine resolution " + std::to_string(nf) + " is not a multiple of coarse resolution " +
                         std::to_string(nc));
  const int64_t ntc = 6LL * nc * nc * nc, ntf = 6LL * nf * nf * nf;
  std::vector<Bary> cb(ntc);
  for (int64_t t = 0; t < ntc; ++t) cb[t] = bary_of(cverts, ctets + t * 4);
  std::atomic<int64_t> bad{-1};
  const int64_t chunk = 4096;
  par_items((ntf + chunk - 1) / chunk, [&](unsigned, int64_t ck) {
    for (int64_t t = ck * chunk; t < std::min(ntf, (ck + 1) * chunk); ++t) {
      double x[3] = {0, 0, 0};
      for (int i = 0; i < 4; ++i)
        for (int r = 0; r < 3; ++r) x[r] += fverts[ftets[t * 4 + i] * 3 + r];
      int64_t cell[3];
      for (int r = 0; r < 3; ++r) {
        x[r] *= 0.25;
        cell[r] = std::min<int64_t>(nc - 1, std::max<int64_t>(0, (int64_t)(x[r] * nc)));
      }
      const int64_t cid = (cell[0] * nc + cell[1]) * nc + cell[2];
      int64_t best = -1;
      double bmin = -INFINITY;
      for (int p = 0; p < 6; ++p) {
        double lam[4];
        bary_eval(cb[cid * 6 + p], x, lam);
        const double mn = std::min(std::min(lam[0], lam[1]), std::min(lam[2], lam[3]));
        if (mn > bmin) {
          bmin = mn;
          best = cid * 6 + p;
        }
      }
      for (int i = 0; i < 4; ++i) {
        double lam[4];
        bary_eval(cb[best], fverts + ftets[t * 4 + i] * 3, lam);
        if (std::min(std::min(lam[0], lam[1]), std::min(lam[2], lam[3])) < -tol) {
          int64_t exp = -1;
          bad.compare_exchange_strong(exp, t);
        }
      }
      out[t] = best;
    }
  });
  if (bad.load() >= 0) fail(MDD_EINVAL, "meshes do not nest (fine tet " + std::to_string(bad.load()) + ")");
  MDD_API_END
}

// decomp.coarse_restriction for nested meshes (reference decomp.py:212-297):
// R0[p, j] = line integral of coarse basis p along kept fine edge j, by the
// exact closed form s_p (l_a(x0) l_b(x1) - l_a(x1) l_b(x0)) over every coarse
// tet holding a fine tet incident to the edge (ascending); repeated (j, p)
// values must agree to continuity_tol (first wins), zeros are dropped.  CSR
// output (ncs rows, columns ascending); on a discontinuity *bad_edge is the
// fine edge and MDD_EDECOMP is returned.
int mdd_coarse_restriction(int64_t nv, const double* fverts, int64_t ntf, const int64_t* ftet_edges,
                           const int64_t* fedges, int64_t nkept, const int64_t* kept_edges, const double* cverts,
                           int64_t ntc, const int64_t* ctets, const int64_t* ctet_edges, const int64_t* csigns,
                           const int64_t* cedge_to_dof, int64_t ncs, const int64_t* tet_map, double continuity_tol,
                           int64_t** out_rowptr, int64_t** out_cols, double** out_vals, int64_t* bad_edge) {
  MDD_API_BEGIN
  (void)nv;
  *bad_edge = -1;
  int64_t ne = 0;
  for (int64_t i = 0; i < ntf * 6; ++i) ne = std::max(ne, ftet_edges[i] + 1);
  std::vector<int64_t> eptr(ne + 1, 0), einc(ntf * 6);
  for (int64_t i = 0; i < ntf * 6; ++i) eptr[ftet_edges[i] + 1]++;
  for (int64_t e = 0; e < ne; ++e) eptr[e + 1] += eptr[e];
  {
    std::vector<int64_t> fp(eptr.begin(), eptr.end() - 1);
    for (int64_t i = 0; i < ntf * 6; ++i) einc[fp[ftet_edges[i]]++] = i / 6;
  }
  std::vector<Bary> cb(ntc);
  for (int64_t t = 0; t < ntc; ++t) cb[t] = bary_of(cverts, ctets + t * 4);
  struct Ent {
    int64_t p;
    double v;
  };
  std::vector<std::vector<Ent>> col(nkept);
  std::atomic<int64_t> bad{-1};
  const int64_t chunk = 2048;
  par_items((nkept + chunk - 1) / chunk, [&](unsigned, int64_t ck) {
    std::vector<int64_t> cts;
    for (int64_t j = ck * chunk; j < std::min(nkept, (ck + 1) * chunk); ++j) {
      const int64_t fe = kept_edges[j];
      cts.clear();
      for (int64_t k = eptr[fe]; k < eptr[fe + 1]; ++k) cts.push_back(tet_map[einc[k]]);
      std::sort(cts.begin(), cts.end());
      cts.erase(std::unique(cts.begin(), cts.end()), cts.end());
      const double* x0 = fverts + fedges[fe * 2] * 3;
      const double* x1 = fverts + fedges[fe * 2 + 1] * 3;
      auto& out = col[j];
      for (int64_t ct : cts) {
        double l0[4], l1[4];
        bary_eval(cb[ct], x0, l0);
        bary_eval(cb[ct], x1, l1);
        for (int le = 0; le < 6; ++le) {
          const int64_t p = cedge_to_dof[ctet_edges[ct * 6 + le]];
          if (p < 0) continue;
          const int a = EA[le], b = EB[le];
          const double v = (l0[a] * l1[b] - l1[a] * l0[b]) * (double)csigns[ct * 6 + le];
          bool seen = false;
          for (auto& en : out)
            if (en.p == p) {
              seen = true;
              if (std::fabs(v - en.v) > continuity_tol * std::max(1.0, std::fabs(en.v))) {
                int64_t exp = -1;
                bad.compare_exchange_strong(exp, fe);
              }
              break;
            }
          if (!seen) out.push_back({p, v});
        }
      }
    }
  });
  if (bad.load() >= 0) {
    *bad_edge = bad.load();
    fail(MDD_EDECOMP, "tangential trace discontinuity on fine edge " + std::to_string(bad.load()));
  }
  std::vector<int64_t> rp(ncs + 1, 0);
  for (int64_t j = 0; j < nkept; ++j)
    for (auto& en : col[j])
      if (en.v != 0.0) rp[en.p + 1]++;
  for (int64_t p = 0; p < ncs; ++p) rp[p + 1] += rp[p];
  int64_t* rowptr = (int64_t*)malloc(sizeof(int64_t) * (ncs + 1));
  int64_t* cols = (int64_t*)malloc(sizeof(int64_t) * std::max<int64_t>(1, rp[ncs]));
  double* vals = (double*)malloc(sizeof(double) * std::max<int64_t>(1, rp[ncs]));
  if (!rowptr || !cols || !vals) {
    free(rowptr);
    free(cols);
    free(vals);
    fail(MDD_ENOMEM, "coarse restriction: out of host memory");
  }
  std::copy(rp.begin(), rp.end(), rowptr);
  std::vector<int64_t> fill(rp.begin(), rp.end() - 1);
  for (int64_t j = 0; j < nkept; ++j)  // ascending j -> sorted columns per row
    for (auto& en : col[j])
      if (en.v != 0.0) {
        const int64_t q = fill[en.p]++;
        cols[q] = j;
        vals[q] = en.v;
      }
  *out_rowptr = rowptr;
  *out_cols = cols;
  *out_vals = vals;
  MDD_API_END
}

}  // extern "C"
