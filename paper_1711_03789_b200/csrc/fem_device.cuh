// Element-level finite-element math on the device.
//
// Restates reference fem._tet_geometry / fem._element_matrices_batch
// (fem.py:154-195): barycentric gradients are the rows of B^{-1} with
// B = [v1-v0, v2-v0, v3-v0] (columns), grad(l0) = -sum of rows; Whitney edge
// function of local edge (a,b) is l_a grad l_b - l_b grad l_a; its curl is
// 2 grad l_a x grad l_b; S_e = |T| curl_e . curl_f; M_e from the exact
// integrals of l_i l_j (|T| (1+delta_ij)/20, fem.py:171); orientation s_e s_f.
#pragma once
#include <cuda_runtime.h>

#include "mdd_internal.h"

namespace mdd {

__constant__ static const int kEA[6] = {0, 0, 0, 1, 1, 2};
__constant__ static const int kEB[6] = {1, 2, 3, 2, 3, 3};

struct TetGeom {
  double g[4][3];  // barycentric gradients
  double vol;
  double det;
};

__device__ __forceinline__ void tet_geometry(const double (&c)[4][3], TetGeom& t) {
  // B columns are v_i - v_0  => B[r][i-1] = c[i][r] - c[0][r]
  double b[3][3];
#pragma unroll
  for (int r = 0; r < 3; ++r)
#pragma unroll
    for (int i = 0; i < 3; ++i) b[r][i] = c[i + 1][r] - c[0][r];
  const double c00 = b[1][1] * b[2][2] - b[1][2] * b[2][1];
  const double c01 = b[1][2] * b[2][0] - b[1][0] * b[2][2];
  const double c02 = b[1][0] * b[2][1] - b[1][1] * b[2][0];
  const double det = b[0][0] * c00 + b[0][1] * c01 + b[0][2] * c02;
  const double id = 1.0 / det;
  // inverse = adj(B)/det ; row i of inv is grad(lambda_{i+1})
  double inv[3][3];
  inv[0][0] = c00 * id;
  inv[1][0] = c01 * id;
  inv[2][0] = c02 * id;
  inv[0][1] = (b[0][2] * b[2][1] - b[0][1] * b[2][2]) * id;
  inv[1][1] = (b[0][0] * b[2][2] - b[0][2] * b[2][0]) * id;
  inv[2][1] = (b[0][1] * b[2][0] - b[0][0] * b[2][1]) * id;
  inv[0][2] = (b[0][1] * b[1][2] - b[0][2] * b[1][1]) * id;
  inv[1][2] = (b[0][2] * b[1][0] - b[0][0] * b[1][2]) * id;
  inv[2][2] = (b[0][0] * b[1][1] - b[0][1] * b[1][0]) * id;
#pragma unroll
  for (int k = 0; k < 3; ++k) {
    t.g[1][k] = inv[0][k];
    t.g[2][k] = inv[1][k];
    t.g[3][k] = inv[2][k];
    t.g[0][k] = -(inv[0][k] + inv[1][k] + inv[2][k]);
  }
  t.det = det;
  t.vol = det / 6.0;
}

// S_e and M_e (6x6) for oriented edge functions; sgn[e] in {+1,-1}.
__device__ __forceinline__ void element_matrices(const double (&c)[4][3], const double (&sgn)[6],
                                                 ElemMats& em) {
  TetGeom t;
  tet_geometry(c, t);
  double curl[6][3];
#pragma unroll
  for (int e = 0; e < 6; ++e) {
    const double* ga = t.g[kEA[e]];
    const double* gb = t.g[kEB[e]];
    curl[e][0] = 2.0 * (ga[1] * gb[2] - ga[2] * gb[1]);
    curl[e][1] = 2.0 * (ga[2] * gb[0] - ga[0] * gb[2]);
    curl[e][2] = 2.0 * (ga[0] * gb[1] - ga[1] * gb[0]);
  }
  double dots[4][4];
#pragma unroll
  for (int i = 0; i < 4; ++i)
#pragma unroll
    for (int j = 0; j < 4; ++j)
      dots[i][j] = t.g[i][0] * t.g[j][0] + t.g[i][1] * t.g[j][1] + t.g[i][2] * t.g[j][2];
  const double v = t.vol;
#pragma unroll
  for (int e = 0; e < 6; ++e) {
#pragma unroll
    for (int f = 0; f < 6; ++f) {
      const int ia = kEA[e], ib = kEB[e], ja = kEA[f], jb = kEB[f];
      const double o = sgn[e] * sgn[f];
      const double s = (curl[e][0] * curl[f][0] + curl[e][1] * curl[f][1] +
                        curl[e][2] * curl[f][2]) * v;
      const double l_aa = (ia == ja ? 2.0 : 1.0) / 20.0;
      const double l_ab = (ia == jb ? 2.0 : 1.0) / 20.0;
      const double l_ba = (ib == ja ? 2.0 : 1.0) / 20.0;
      const double l_bb = (ib == jb ? 2.0 : 1.0) / 20.0;
      const double m = (dots[ib][jb] * l_aa - dots[ib][ja] * l_ab - dots[ia][jb] * l_ba +
                        dots[ia][ja] * l_bb) * v;
      em.s[e][f] = s * o;
      em.m[e][f] = m * o;
    }
  }
  em.vol = v;
}

// One entry (a, b) of the oriented S_e, M_e from precomputed geometry
// (same formulas as element_matrices; used by the warp-per-cell assembly).
__device__ __forceinline__ void element_entry(const TetGeom& t, const double (&sgn)[6], int e, int f,
                                              double& s_out, double& m_out) {
  const int ia = kEA[e], ib = kEB[e], ja = kEA[f], jb = kEB[f];
  double ce[3], cf[3];
  ce[0] = 2.0 * (t.g[ia][1] * t.g[ib][2] - t.g[ia][2] * t.g[ib][1]);
  ce[1] = 2.0 * (t.g[ia][2] * t.g[ib][0] - t.g[ia][0] * t.g[ib][2]);
  ce[2] = 2.0 * (t.g[ia][0] * t.g[ib][1] - t.g[ia][1] * t.g[ib][0]);
  cf[0] = 2.0 * (t.g[ja][1] * t.g[jb][2] - t.g[ja][2] * t.g[jb][1]);
  cf[1] = 2.0 * (t.g[ja][2] * t.g[jb][0] - t.g[ja][0] * t.g[jb][2]);
  cf[2] = 2.0 * (t.g[ja][0] * t.g[jb][1] - t.g[ja][1] * t.g[jb][0]);
  auto dot = [&](int i, int j) {
    return t.g[i][0] * t.g[j][0] + t.g[i][1] * t.g[j][1] + t.g[i][2] * t.g[j][2];
  };
  const double v = t.vol;
  const double o = sgn[e] * sgn[f];
  const double sv = (ce[0] * cf[0] + ce[1] * cf[1] + ce[2] * cf[2]) * v;
  const double l_aa = (ia == ja ? 2.0 : 1.0) / 20.0;
  const double l_ab = (ia == jb ? 2.0 : 1.0) / 20.0;
  const double l_ba = (ib == ja ? 2.0 : 1.0) / 20.0;
  const double l_bb = (ib == jb ? 2.0 : 1.0) / 20.0;
  const double mv = (dot(ib, jb) * l_aa - dot(ib, ja) * l_ab - dot(ia, jb) * l_ba + dot(ia, ja) * l_bb) * v;
  s_out = sv * o;
  m_out = mv * o;
}

// Tangential mass of the three edge functions of a boundary triangle whose
// vertices p0<p1<p2 are in ascending global order (fem.py:286-316): the
// three-midpoint rule, exact for the quadratic integrand.
__device__ __forceinline__ void triangle_tangential_mass(const double (&p)[3][3], double (&m)[3][3]) {
  double e1[3], e2[3], nv[3];
  for (int k = 0; k < 3; ++k) { e1[k] = p[1][k] - p[0][k]; e2[k] = p[2][k] - p[0][k]; }
  nv[0] = e1[1] * e2[2] - e1[2] * e2[1];
  nv[1] = e1[2] * e2[0] - e1[0] * e2[2];
  nv[2] = e1[0] * e2[1] - e1[1] * e2[0];
  const double a2 = sqrt(nv[0] * nv[0] + nv[1] * nv[1] + nv[2] * nv[2]);
  double nh[3] = {nv[0] / a2, nv[1] / a2, nv[2] / a2};
  double g[3][3];
  const int opp[3][2] = {{1, 2}, {2, 0}, {0, 1}};  // g_i = nhat x (p_b - p_a) / a2
  for (int i = 0; i < 3; ++i) {
    double d[3];
    for (int k = 0; k < 3; ++k) d[k] = p[opp[i][1]][k] - p[opp[i][0]][k];
    g[i][0] = (nh[1] * d[2] - nh[2] * d[1]) / a2;
    g[i][1] = (nh[2] * d[0] - nh[0] * d[2]) / a2;
    g[i][2] = (nh[0] * d[1] - nh[1] * d[0]) / a2;
  }
  const int te[3][2] = {{0, 1}, {0, 2}, {1, 2}};
  const double ql[3][3] = {{0.5, 0.5, 0.0}, {0.5, 0.0, 0.5}, {0.0, 0.5, 0.5}};
  for (int a = 0; a < 3; ++a)
    for (int b = 0; b < 3; ++b) m[a][b] = 0.0;
  for (int q = 0; q < 3; ++q) {
    double w[3][3];
    for (int e = 0; e < 3; ++e) {
      const int a = te[e][0], b = te[e][1];
      for (int k = 0; k < 3; ++k) w[e][k] = ql[q][a] * g[b][k] - ql[q][b] * g[a][k];
    }
    for (int a = 0; a < 3; ++a)
      for (int b = 0; b < 3; ++b) m[a][b] += w[a][0] * w[b][0] + w[a][1] * w[b][1] + w[a][2] * w[b][2];
  }
  const double sc = (a2 / 2.0) / 3.0;
  for (int a = 0; a < 3; ++a)
    for (int b = 0; b < 3; ++b) m[a][b] *= sc;
}

// position of column c in CSR row r (sorted), -1 if absent
__device__ __forceinline__ int csr_find(const int32_t* __restrict__ rowptr,
                                        const int32_t* __restrict__ cols, int r, int c) {
  int lo = rowptr[r], hi = rowptr[r + 1] - 1;
  while (lo <= hi) {
    const int mid = (lo + hi) >> 1;
    const int v = cols[mid];
    if (v == c) return mid;
    if (v < c) lo = mid + 1; else hi = mid - 1;
  }
  return -1;
}

}  // namespace mdd
