// Batched multifrontal factorisation (block Gauss-Jordan sweeps); the
// forward/backward solves are in solve.cu.  See frontal.h for the algebra.
//
// Replaces linalg.DenseLU (zgetrf, reference linalg.py:73-101) and
// DenseLU.solve (zgetrs, linalg.py:103-107) as used per subdomain and for
// the coarse block in precond.PreconditionerState (precond.py:166-192,
// 347-358).
#include <algorithm>
#include <cmath>
#include <cstring>
#include <atomic>
#include <exception>
#include <mutex>
#include <thread>

#include "frontal.h"
#include "mdd_kernels.cuh"

namespace mdd {

// ------------------------------------------------------------ kernels
// warp per (node,row): F[row][:] = sum_children S_child[g(row)][g(:)], one
// write per element (extend-add in gather form: no atomics)
__global__ void __launch_bounds__(256) k_front_init(const int2* __restrict__ tasks, int64_t ntask,
                                                    const NodeDev* __restrict__ nodes,
                                                    const int32_t* __restrict__ children,
                                                    const int32_t* __restrict__ gmap,
                                                    double2* __restrict__ fronts) {
  const int64_t w = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const int lane = threadIdx.x & 31;
  if (w >= ntask) return;
  const int2 tk = tasks[w];
  const NodeDev nd = nodes[tk.x];
  const int r = tk.y, m = nd.m;
  double2* row = fronts + nd.front_off + (int64_t)r * m;
  constexpr int kMaxCh = 4;
  const double2* S[kMaxCh];
  const int32_t* G[kMaxCh];
  int nsrc = 0;
  for (int ci = 0; ci < nd.nch && nsrc < kMaxCh; ++ci) {
    const int32_t* g = gmap + nd.gmap_off + (int64_t)ci * m;
    const int gr = g[r];
    if (gr < 0) continue;
    const NodeDev ch = nodes[children[nd.child_off + ci]];
    S[nsrc] = fronts + ch.front_off + (int64_t)(ch.np + gr) * ch.m + ch.np;
    G[nsrc] = g;
    ++nsrc;
  }
  for (int q = lane; q < m; q += 32) {
    double2 acc = make_double2(0.0, 0.0);
    for (int k = 0; k < nsrc; ++k) {
      const int gq = G[k][q];
      if (gq >= 0) acc = cadd(acc, S[k][gq]);
    }
    row[q] = acc;
  }
  // children beyond kMaxCh (not produced by bisection; kept for generality)
  for (int ci = kMaxCh; ci < nd.nch; ++ci) {
    const int32_t* g = gmap + nd.gmap_off + (int64_t)ci * m;
    const int gr = g[r];
    if (gr < 0) continue;
    const NodeDev ch = nodes[children[nd.child_off + ci]];
    const double2* Sx = fronts + ch.front_off + (int64_t)(ch.np + gr) * ch.m + ch.np;
    for (int q = lane; q < m; q += 32) {
      const int gq = g[q];
      if (gq >= 0) row[q] = cadd(row[q], Sx[gq]);
    }
  }
}

__global__ void k_front_scatter(int64_t n, const int64_t* __restrict__ pos,
                                const int32_t* __restrict__ src, const double2* __restrict__ vals,
                                double2* __restrict__ fronts) {
  for (int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; e < n;
       e += (int64_t)gridDim.x * blockDim.x) {
    const int64_t p = pos[e];
    fronts[p] = cadd(fronts[p], vals[src[e]]);
  }
}

// Whole pivot-block inverse of a small front (np <= 32 levels) in one CTA,
// the block in shared memory: F_PP <- -F_PP^{-1} by unpivoted in-place
// Gauss-Jordan.  Per pivot, the pivot row and column are copied to shared
// memory, one barrier, then every thread updates its elements (dealt
// round-robin, only the np x np block is touched), one barrier.  It replaces
// the sweep steps where those are latency-bound; it is issue-bound at ~30
// instructions per element update, so larger pivot blocks keep the sweeps.
__global__ void __launch_bounds__(256) k_gj_smem(const NodeDev* __restrict__ nodes, const int32_t* __restrict__ act,
                                                 double2* __restrict__ fronts, double* __restrict__ pivstat) {
  extern __shared__ double2 A[];
  __shared__ double2 colp[96], rowp[96];
  const int node = act[blockIdx.x];
  const NodeDev nd = nodes[node];
  const int np = nd.np, m = nd.m, ne = np * np;
  double2* F = fronts + nd.front_off;
  for (int e = threadIdx.x; e < ne; e += 256) A[e] = F[(int64_t)(e / np) * m + e % np];
  __syncthreads();
  double pmin = INFINITY, pmax = 0.0;
  for (int p = 0; p < np; ++p) {
    const int t = threadIdx.x;
    if (t < np) colp[t] = A[t * np + p];
    else if (t < 2 * np) rowp[t - np] = A[p * np + t - np];
    __syncthreads();
    const double2 piv = colp[p];
    const double2 d = cdiv(make_double2(1.0, 0.0), piv);
    if (t == 0) {
      const double am = hypot(piv.x, piv.y);
      pmin = fmin(pmin, isfinite(am) ? am : 0.0);
      pmax = fmax(pmax, isfinite(am) ? am : INFINITY);
    }
    int r = t / np, c = t - r * np;
    const int dr = 256 / np, dc = 256 - dr * np;  // e += 256 in (r, c)
    for (int e = t; e < ne; e += 256) {
      double2 v;
      if (r == p) v = (c == p) ? d : cmul(rowp[c], d);
      else if (c == p) v = cneg(cmul(colp[r], d));
      else v = csub(A[e], cmul(colp[r], cmul(rowp[c], d)));
      A[e] = v;
      r += dr;
      c += dc;
      if (c >= np) {
        c -= np;
        ++r;
      }
    }
    __syncthreads();
  }
  for (int e = threadIdx.x; e < ne; e += 256) F[(int64_t)(e / np) * m + e % np] = cneg(A[e]);
  if (threadIdx.x == 0) {
    pivstat[2 * node] = fmin(pivstat[2 * node], pmin);
    pivstat[2 * node + 1] = fmax(pivstat[2 * node + 1], pmax);
  }
}

// Inverse of the 32x32 pivot block of one sweep step, one 256-thread CTA
// per active node (replaced the one-warp k_invert of round 1:
// 10 us instead of 59 us
// per step at the cfg1 root level).  The kb x kb diagonal block at
// K0 = step*kPB, padded with the identity, is held in registers (thread
// (ti,tj) of a 16x16 grid owns an NBxNB tile); per pivot the owners of row p
// and column p publish them to shared memory (double-buffered by parity),
// one barrier, then every thread applies the rank-1 update to its tile.
// Output P = inverse (not negated) in pbuf.  (SWEEP = false would invert a
// whole np <= 16*NB pivot block in place as -F_PP^{-1}.)
template <int NB, bool SWEEP = false>
__global__ void __launch_bounds__(256, NB <= 4 ? 2 : 1) k_gj_small(const NodeDev* __restrict__ nodes,
                                                  const int32_t* __restrict__ act, double2* __restrict__ fronts,
                                                  double* __restrict__ pivstat, int step = 0,
                                                  double2* __restrict__ pbuf = nullptr) {
  constexpr int N = 16 * NB;
  __shared__ double2 rowb[2][N], colb[2][N];
  __shared__ double2 pivs[2];
  const int node = act[blockIdx.x];
  const NodeDev nd = nodes[node];
  const int K0 = SWEEP ? step * kPB : 0;
  const int np = SWEEP ? min(kPB, nd.np - K0) : nd.np, m = nd.m;
  double2* F = fronts + nd.front_off + (int64_t)K0 * m + K0;
  const int ti = threadIdx.x >> 4, tj = threadIdx.x & 15;
  const int r0 = NB * ti, c0 = NB * tj;
  double2 a[NB][NB];
#pragma unroll
  for (int i = 0; i < NB; ++i)
#pragma unroll
    for (int j = 0; j < NB; ++j) {
      const int r = r0 + i, c = c0 + j;
      a[i][j] = (r < np && c < np) ? F[(int64_t)r * m + c] : make_double2(r == c ? 1.0 : 0.0, 0.0);
    }
  double pmin = INFINITY, pmax = 0.0;
  for (int p = 0; p < np; ++p) {
    const int b = p & 1;
    const int pi = p / NB, pj = p - NB * (p / NB);  // owner tile row/col and offset
    // owners of column p publish the old column (incl. the pivot)
    // (compile-time indices only, so the tile stays in registers)
    if (tj == pi) {
#pragma unroll
      for (int i = 0; i < NB; ++i)
#pragma unroll
        for (int jj = 0; jj < NB; ++jj)
          if (jj == pj) colb[b][r0 + i] = a[i][jj];
    }
    if (ti == pi) {
#pragma unroll
      for (int ii = 0; ii < NB; ++ii)
        if (ii == pj) {
#pragma unroll
          for (int j = 0; j < NB; ++j) {
            rowb[b][c0 + j] = a[ii][j];
            if (tj == pi && j == pj) {  // the pivot's owner: reciprocal + magnitude
              const double2 piv = a[ii][j];
              pivs[b] = cdiv(make_double2(1.0, 0.0), piv);
              const double am = hypot(piv.x, piv.y);
              pmin = fmin(pmin, isfinite(am) ? am : 0.0);
              pmax = fmax(pmax, isfinite(am) ? am : INFINITY);
            }
          }
        }
    }
    __syncthreads();
    const double2 d = pivs[b];
    double2 cf[NB];
#pragma unroll
    for (int i = 0; i < NB; ++i) cf[i] = colb[b][r0 + i];
    // uniform rank-1 update, then overwrite row p / column p (their owners)
#pragma unroll
    for (int j = 0; j < NB; ++j) {
      const double2 rs = cmul(rowb[b][c0 + j], d);  // scaled pivot row
#pragma unroll
      for (int i = 0; i < NB; ++i) a[i][j] = csub(a[i][j], cmul(cf[i], rs));
      if (ti == pi) {
#pragma unroll
        for (int ii = 0; ii < NB; ++ii)
          if (ii == pj) a[ii][j] = rs;
      }
    }
    if (tj == pi) {
#pragma unroll
      for (int jj = 0; jj < NB; ++jj)
        if (jj == pj) {
#pragma unroll
          for (int i = 0; i < NB; ++i) a[i][jj] = (r0 + i == p) ? d : cneg(cmul(cf[i], d));
        }
    }
  }
#pragma unroll
  for (int i = 0; i < NB; ++i)
#pragma unroll
    for (int j = 0; j < NB; ++j) {
      const int r = r0 + i, c = c0 + j;
      if (SWEEP) pbuf[(int64_t)blockIdx.x * kPB * kPB + r * kPB + c] = a[i][j];
      else if (r < np && c < np) F[(int64_t)r * m + c] = cneg(a[i][j]);
    }
  // pivot magnitudes: each diagonal owner saw its own pivots
  __shared__ double pm[2][16];
  if (ti == tj) {
    pm[0][ti] = pmin;
    pm[1][ti] = pmax;
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    double mn = pm[0][0], mx = pm[1][0];
    for (int k = 1; k < 16; ++k) {
      mn = fmin(mn, pm[0][k]);
      mx = fmax(mx, pm[1][k]);
    }
    pivstat[2 * node] = fmin(pivstat[2 * node], mn);
    pivstat[2 * node + 1] = fmax(pivstat[2 * node + 1], mx);
  }
}

// Row panel F[K][c] <- P F[K][c] (c outside K), F[K][K] <- -P, and the copy
// W[r][:] = old F[r][K] (r outside K) used by the trailing update.
__global__ void __launch_bounds__(kPanelCols) k_panel(const int2* __restrict__ tasks,
                                                      const NodeDev* __restrict__ nodes,
                                                      const int32_t* __restrict__ act,
                                                      const int64_t* __restrict__ woff, int step,
                                                      double2* __restrict__ fronts,
                                                      const double2* __restrict__ pbuf,
                                                      double2* __restrict__ wbuf) {
  __shared__ double2 P[kPB][kPB + 1];
  const int2 tk = tasks[blockIdx.x];
  const int ai = tk.x, chunk = tk.y;
  const NodeDev nd = nodes[act[ai]];
  const int m = nd.m;
  const int K0 = step * kPB;
  const int kb = min(kPB, nd.np - K0);
  for (int t = threadIdx.x; t < kPB * kPB; t += blockDim.x)
    P[t / kPB][t % kPB] = pbuf[(int64_t)ai * kPB * kPB + t];
  __syncthreads();
  double2* T = fronts + nd.front_off;
  const int np = nd.np;
  const int c = chunk * kPanelCols + threadIdx.x;
  if (c < np) {  // the sweeps work on the pivot block only (F_PU, F_UP, F_UU: GEMMs)
    if (c >= K0 && c < K0 + kb) {
      for (int r = 0; r < kb; ++r) T[(int64_t)(K0 + r) * m + c] = cneg(P[r][c - K0]);
    } else {
      double2 x[kPB];
#pragma unroll
      for (int l = 0; l < kPB; ++l)
        x[l] = l < kb ? T[(int64_t)(K0 + l) * m + c] : make_double2(0.0, 0.0);
      for (int r = 0; r < kb; ++r) {
        double2 acc = make_double2(0.0, 0.0);
#pragma unroll
        for (int l = 0; l < kPB; ++l) acc = cfma(P[r][l], x[l], acc);
        T[(int64_t)(K0 + r) * m + c] = acc;
      }
    }
  }
  // W copy: rows [chunk*128, chunk*128+128)
  double2* W = wbuf + woff[ai];
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  for (int rr = wid; rr < kPanelCols; rr += kPanelCols / 32) {
    const int r = chunk * kPanelCols + rr;
    if (r >= np) break;
    const bool inK = r >= K0 && r < K0 + kb;
    W[(int64_t)r * kPB + lane] =
        (inK || lane >= kb) ? make_double2(0.0, 0.0) : T[(int64_t)r * m + K0 + lane];
  }
}

// FP64 tensor-core MMA (DMMA): D(8x8) += A(8x4, row) * B(4x8, col).
// Fragments: a = A[lane/4][lane%4], b = B[lane%4][lane/4],
//            d0,d1 = D[lane/4][2*(lane%4) + {0,1}].
__device__ __forceinline__ void dmma884(double& d0, double& d1, double a, double b) {
  asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};"
               : "+d"(d0), "+d"(d1)
               : "d"(a), "d"(b));
}

// Trailing update of one 64x64 tile on the FP64 tensor cores:
//   F[r][c] = (c in K ? 0 : F[r][c]) - W[r][:] F[K][c]
// Complex product = 4 real DMMA products per 8x8x4 block
//   (re += Ar Br - Ai Bi, im += Ar Bi + Ai Br).
// 8 warps, each owning a 16x32 sub-tile = 2x4 DMMA blocks; W (64 x kPB) and
// the pivot row panel F[K][c0:c0+64] are staged in shared memory.
__global__ void __launch_bounds__(256, 2) k_update(const int4* __restrict__ tasks,
                                                const NodeDev* __restrict__ nodes,
                                                const int32_t* __restrict__ act,
                                                const int64_t* __restrict__ woff, int step,
                                                double2* __restrict__ fronts,
                                                const double2* __restrict__ wbuf) {
  extern __shared__ double2 sm[];
  double2(*Ws)[kPB + 1] = reinterpret_cast<double2(*)[kPB + 1]>(sm);
  double2(*Ks)[kTile + 1] = reinterpret_cast<double2(*)[kTile + 1]>(sm + kTile * (kPB + 1));
  const int4 tk = tasks[blockIdx.x];
  const int ai = tk.x;
  const NodeDev nd = nodes[act[ai]];
  const int m = nd.m;
  const int K0 = step * kPB;
  const int kb = min(kPB, nd.np - K0);
  const int r0 = tk.y * kTile, c0 = tk.z * kTile;
  const double2* W = wbuf + woff[ai];
  double2* T = fronts + nd.front_off;
  for (int t = threadIdx.x; t < kTile * kPB; t += blockDim.x) {
    const int rr = t / kPB, l = t % kPB;
    const int r = r0 + rr;
    Ws[rr][l] = r < m ? W[(int64_t)r * kPB + l] : make_double2(0.0, 0.0);
  }
  for (int t = threadIdx.x; t < kTile * kPB; t += blockDim.x) {
    const int l = t / kTile, cc = t % kTile;
    const int c = c0 + cc;
    Ks[l][cc] = (l < kb && c < m) ? T[(int64_t)(K0 + l) * m + c] : make_double2(0.0, 0.0);
  }
  __syncthreads();
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int gid = lane >> 2, tig = lane & 3;
  const int wr = (warp >> 1) * 16, wc = (warp & 1) * 32;
  double cre[2][4][2], cim[2][4][2];
#pragma unroll
  for (int i = 0; i < 2; ++i)
#pragma unroll
    for (int j = 0; j < 4; ++j) cre[i][j][0] = cre[i][j][1] = cim[i][j][0] = cim[i][j][1] = 0.0;
#pragma unroll 2
  for (int kk = 0; kk < kPB / 4; ++kk) {
    double are[2], aim[2], naim[2], bre[4], bim[4];
#pragma unroll
    for (int i = 0; i < 2; ++i) {
      const double2 v = Ws[wr + 8 * i + gid][4 * kk + tig];
      are[i] = v.x;
      aim[i] = v.y;
      naim[i] = -v.y;
    }
#pragma unroll
    for (int j = 0; j < 4; ++j) {
      const double2 v = Ks[4 * kk + tig][wc + 8 * j + gid];
      bre[j] = v.x;
      bim[j] = v.y;
    }
#pragma unroll
    for (int i = 0; i < 2; ++i)
#pragma unroll
      for (int j = 0; j < 4; ++j) {
        dmma884(cre[i][j][0], cre[i][j][1], are[i], bre[j]);
        dmma884(cre[i][j][0], cre[i][j][1], naim[i], bim[j]);
        dmma884(cim[i][j][0], cim[i][j][1], are[i], bim[j]);
        dmma884(cim[i][j][0], cim[i][j][1], aim[i], bre[j]);
      }
  }
  // epilogue: issue all 16 loads of the old values first (independent), then
  // subtract and store; a lane's two columns are 32 contiguous bytes and the
  // 4 lanes of a row cover 128 contiguous bytes
  double2 old[2][4][2];
#pragma unroll
  for (int i = 0; i < 2; ++i) {
    const int r = r0 + wr + 8 * i + gid;
    const bool rok = r < m && !(r >= K0 && r < K0 + kb);
#pragma unroll
    for (int j = 0; j < 4; ++j)
#pragma unroll
      for (int e = 0; e < 2; ++e) {
        const int c = c0 + wc + 8 * j + 2 * tig + e;
        const bool load = rok && c < nd.np && !(c >= K0 && c < K0 + kb) && r < nd.np;
        old[i][j][e] = load ? T[(int64_t)r * m + c] : make_double2(0.0, 0.0);
      }
  }
#pragma unroll
  for (int i = 0; i < 2; ++i) {
    const int r = r0 + wr + 8 * i + gid;
    if (r >= m || (r >= K0 && r < K0 + kb)) continue;
#pragma unroll
    for (int j = 0; j < 4; ++j)
#pragma unroll
      for (int e = 0; e < 2; ++e) {
        const int c = c0 + wc + 8 * j + 2 * tig + e;
        if (c >= nd.np || r >= nd.np) continue;  // outside the pivot block: k_gemm
        T[(int64_t)r * m + c] =
            make_double2(old[i][j][e].x - cre[i][j][e], old[i][j][e].y - cim[i][j][e]);
      }
  }
}

// Batched complex GEMM tiles on the FP64 tensor cores (DMMA), used for the
// parts of each front the pivot-block sweeps leave out (A = F_PP, with
// -A^{-1} in place after the sweeps; B_orig / C_orig the original F_PU / F_UP):
//   F_PU = A^{-1} B_orig = -(-A^{-1}) B_orig          (mode 0)
//   F_UP = C_orig A^{-1} = -C_orig (-A^{-1})          (mode 0)
//   F_UU -= C_orig F_PU   (deferred Schur complement) (mode 1)
// Each is one GEMM with K = np instead of np/32 rank-32 passes.  One 64x64
// output tile per CTA, 8 warps of 16x32, complex product = 4 real DMMA
// products; K is consumed in chunks of kGemmKC through a 2-stage cp.async
// pipeline; padded shared-memory rows keep the fragment loads conflict-free.
__device__ __forceinline__ void cp_async16(void* dst, const void* src, bool ok) {
  const unsigned d = (unsigned)__cvta_generic_to_shared(dst);
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16, %2;" ::"r"(d), "l"(src), "r"(ok ? 16 : 0) : "memory");
}
__global__ void __launch_bounds__(256, 2) k_gemm(const GemmTask* __restrict__ tasks, double2* __restrict__ fronts,
                                                 const double2* __restrict__ bbuf, const int* __restrict__ gate = nullptr,
                                                 const int* __restrict__ mirror = nullptr) {
  // gated launches are the work a symmetric factorisation does not need: the F_UP GEMM
  // (k_transpose_up does it) and the strictly upper tiles of the Schur complement (mode 2 below)
  if (gate && *gate == 0) return;
  extern __shared__ double2 sm[];
  constexpr int LA = kGemmKC + 4, LB = kTile + 2;  // padded leading dimensions
  const GemmTask tk = tasks[blockIdx.x];
  const int M = tk.M, N = tk.N, K = tk.K, r0 = tk.r0, c0 = tk.c0;
  const double2* Xg = fronts + tk.xo;
  const double2* Wg = (tk.wsel ? bbuf : fronts) + tk.wo;
  double2* Og = fronts + tk.oo;
  const int ldx = tk.ldx, ldw = tk.ldw, ldo = tk.ldo;
  auto As = [&](int st) { return sm + st * (kTile * LA + kGemmKC * LB); };
  auto Bs = [&](int st) { return sm + st * (kTile * LA + kGemmKC * LB) + kTile * LA; };
  auto load = [&](int st, int k0) {
    double2* A = As(st);
    double2* B = Bs(st);
    for (int t = threadIdx.x; t < kTile * kGemmKC; t += 256) {
      const int rr = t / kGemmKC, kk = t % kGemmKC;
      const bool ok = r0 + rr < M && k0 + kk < K;
      cp_async16(A + rr * LA + kk, ok ? Xg + (int64_t)(r0 + rr) * ldx + k0 + kk : Xg, ok);
    }
    for (int t = threadIdx.x; t < kGemmKC * kTile; t += 256) {
      const int kk = t / kTile, cc = t % kTile;
      const bool ok = k0 + kk < K && c0 + cc < N;
      cp_async16(B + kk * LB + cc, ok ? Wg + (int64_t)(k0 + kk) * ldw + c0 + cc : Wg, ok);
    }
    asm volatile("cp.async.commit_group;" ::: "memory");
  };
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int gid = lane >> 2, tig = lane & 3;
  const int wr = (warp >> 1) * 16, wc = (warp & 1) * 32;
  double cre[2][4][2], cim[2][4][2];
#pragma unroll
  for (int i = 0; i < 2; ++i)
#pragma unroll
    for (int j = 0; j < 4; ++j) cre[i][j][0] = cre[i][j][1] = cim[i][j][0] = cim[i][j][1] = 0.0;
  const int nk = (K + kGemmKC - 1) / kGemmKC;
  if (tk.mode >= 1) {
    // accumulate mode: pull the output tile's old values toward L2 now, so the
    // epilogue's read-modify-write does not pay HBM latency after the K loop
    // (each thread covers its 2x4 blocks' 32-byte row segments)
#pragma unroll
    for (int i = 0; i < 2; ++i) {
      const int r = r0 + (warp >> 1) * 16 + 8 * i + gid;
      if (r >= M) continue;
#pragma unroll
      for (int j = 0; j < 4; ++j) {
        const int c = c0 + (warp & 1) * 32 + 8 * j + 2 * tig;
        if (c < N) asm volatile("prefetch.global.L2 [%0];" ::"l"(Og + (int64_t)r * ldo + c));
      }
    }
  }
  load(0, 0);
  for (int kc = 0; kc < nk; ++kc) {
    if (kc + 1 < nk) {
      load((kc + 1) & 1, (kc + 1) * kGemmKC);
      asm volatile("cp.async.wait_group 1;" ::: "memory");
    } else {
      asm volatile("cp.async.wait_group 0;" ::: "memory");
    }
    __syncthreads();
    const double2* A = As(kc & 1);
    const double2* B = Bs(kc & 1);
#pragma unroll
    for (int kk = 0; kk < kGemmKC / 4; ++kk) {
      double are[2], aim[2], naim[2], bre[4], bim[4];
#pragma unroll
      for (int i = 0; i < 2; ++i) {
        const double2 v = A[(wr + 8 * i + gid) * LA + 4 * kk + tig];
        are[i] = v.x;
        aim[i] = v.y;
        naim[i] = -v.y;
      }
#pragma unroll
      for (int j = 0; j < 4; ++j) {
        const double2 v = B[(4 * kk + tig) * LB + wc + 8 * j + gid];
        bre[j] = v.x;
        bim[j] = v.y;
      }
#pragma unroll
      for (int i = 0; i < 2; ++i)
#pragma unroll
        for (int j = 0; j < 4; ++j) {
          dmma884(cre[i][j][0], cre[i][j][1], are[i], bre[j]);
          dmma884(cre[i][j][0], cre[i][j][1], naim[i], bim[j]);
          dmma884(cim[i][j][0], cim[i][j][1], are[i], bim[j]);
          dmma884(cim[i][j][0], cim[i][j][1], aim[i], bre[j]);
        }
    }
    __syncthreads();  // stage kc&1 is refilled by the next iteration's load
  }
  const bool acc = tk.mode >= 1;
  // mode 2: a tile below the diagonal of the Schur complement F_UU -= C F_PU of a complex
  // symmetric front (C = B^T, A^{-1} symmetric, so the product is symmetric): its transpose is
  // the tile above the diagonal, which is then not computed at all (the gated launch).  Per
  // store the 8 lanes of a column write 128 contiguous bytes of the mirrored row.
  const bool mir = tk.mode == 2 && mirror && *mirror == 0;
#pragma unroll
  for (int i = 0; i < 2; ++i) {
    const int r = r0 + wr + 8 * i + gid;
    if (r >= M) continue;
#pragma unroll
    for (int j = 0; j < 4; ++j)
#pragma unroll
      for (int e = 0; e < 2; ++e) {
        const int c = c0 + wc + 8 * j + 2 * tig + e;
        if (c >= N) continue;
        double2* o = Og + (int64_t)r * ldo + c;
        const double2 old = acc ? *o : make_double2(0.0, 0.0);
        const double2 v = make_double2(old.x - cre[i][j][e], old.y - cim[i][j][e]);
        *o = v;
        if (mir) Og[(int64_t)c * ldo + r] = v;
      }
  }
}

// Complex-symmetric fronts: F_UP = C A^{-1} = (A^{-1} B)^T = F_PU^T (A^{-1} is
// symmetric, C = B^T), so the packed F_UP rows of the solve are a transpose
// of F_PU instead of a second GEMM (8 np^2 nu flops).  One 32x32 tile per CTA
// through shared memory, coalesced on both sides.
__global__ void __launch_bounds__(256) k_transpose_up(const int4* __restrict__ tasks,
                                                      const NodeDev* __restrict__ nodes,
                                                      double2* __restrict__ fronts, const int* __restrict__ gate) {
  if (*gate != 0) return;  // not symmetric: the F_UP GEMM ran
  __shared__ double2 t[32][33];
  const int4 tk = tasks[blockIdx.x];
  const NodeDev nd = nodes[tk.x];
  const int r0 = tk.y, c0 = tk.z, np = nd.np, nu = nd.nu, m = nd.m;
  const double2* pu = fronts + nd.front_off + np;  // F_PU: np x nu, ld m
  double2* up = fronts + nd.upk_off;              // packed F_UP: nu x np, ld np
  const int tx = threadIdx.x, ty = threadIdx.y;
  for (int k = ty; k < 32; k += 8) {
    const int c = c0 + k, r = r0 + tx;  // F_PU[c][r]
    if (c < np && r < nu) t[k][tx] = pu[(int64_t)c * m + r];
  }
  __syncthreads();
  for (int k = ty; k < 32; k += 8) {
    const int r = r0 + k, c = c0 + tx;  // F_UP[r][c] = F_PU[c][r]
    if (r < nu && c < np) up[(int64_t)r * np + c] = t[tx][k];
  }
}

// B_orig rows: front row r (< np), columns np..m -> bbuf (np x nu, row-major)
__global__ void __launch_bounds__(256) k_copy_b(const int2* __restrict__ tasks, int64_t ntask,
                                                const NodeDev* __restrict__ nodes,
                                                const double2* __restrict__ fronts, double2* __restrict__ bbuf) {
  const int64_t w = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const int lane = threadIdx.x & 31;
  if (w >= ntask) return;
  const int2 tk = tasks[w];
  const NodeDev nd = nodes[tk.x];
  const double2* src = fronts + nd.front_off + (int64_t)tk.y * nd.m + nd.np;
  double2* dst = bbuf + nd.bb_off + (int64_t)tk.y * nd.nu;
  for (int q = lane; q < nd.nu; q += 32) dst[q] = src[q];
}

__global__ void k_pivinit(double* p, int64_t n) {
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x) {
    p[2 * i] = INFINITY;
    p[2 * i + 1] = 0.0;
  }
}

// ------------------------------------------------------------- host plan
template <typename F>
static void par_for(int64_t n, F&& f) {
  const unsigned nth = std::max(1u, std::min(16u, std::thread::hardware_concurrency()));
  if (n <= 1 || nth == 1) {
    for (int64_t i = 0; i < n; ++i) f(i);
    return;
  }
  std::vector<std::thread> th;
  std::atomic<int64_t> next{0};
  std::exception_ptr err;
  std::mutex mu;
  for (unsigned t = 0; t < std::min<int64_t>(nth, n); ++t)
    th.emplace_back([&] {
      try {
        for (int64_t i = next++; i < n; i = next++) f(i);
      } catch (...) {
        std::lock_guard<std::mutex> g(mu);
        if (!err) err = std::current_exception();
      }
    });
  for (auto& x : th) x.join();
  if (err) std::rethrow_exception(err);
}

void FrontPlan::build(mdd_ctx* c, std::vector<MatrixInput>& mats, int32_t leaf) {
  ctx = c;
  cudaStream_t s = ctx->stream;
  nmat = (int32_t)mats.size();
  std::vector<SymOut> sym(nmat);
  par_for(nmat, [&](int64_t i) {
    SymIn in;
    in.n = mats[i].n;
    in.rowptr = mats[i].rowptr.data();
    in.cols = mats[i].cols.data();
    in.xyz = mats[i].xyz.data();
    in.grid = mats[i].grid;
    nd_analyze(in, leaf, sym[i]);
  });
  mat_n.resize(nmat);
  mat_off.resize(nmat);
  perm.resize(nmat);
  int64_t off = 0;
  std::vector<int32_t> node_base(nmat);
  int64_t nn = 0;
  nlevels = 0;
  for (int i = 0; i < nmat; ++i) {
    mat_n[i] = mats[i].n;
    if (off > INT32_MAX) fail(MDD_EINVAL, "local vector space exceeds 2^31");
    mat_off[i] = (int32_t)off;
    off += mats[i].n;
    node_base[i] = (int32_t)nn;
    nn += (int64_t)sym[i].nodes.size();
    nlevels = std::max(nlevels, sym[i].nlevels);
    perm[i] = sym[i].perm;
  }
  nloc = off;
  nnodes = (int32_t)nn;
  h_nodes.resize(nn);
  std::vector<int32_t> h_children, h_gmap_sizes;
  int64_t gm_total = 0, upd_total = 0;
  front_total = 0;
  uvec_total = 0;
  factor_flops = 0;
  schur_flops = 0;
  lu_flops = exec_flops_full = exec_flops_sym = 0;
  factor_entries = 0;
  max_np = 0;
  max_m = 0;
  std::vector<int32_t> node_level(nn);
  for (int i = 0; i < nmat; ++i)
    for (size_t k = 0; k < sym[i].nodes.size(); ++k) {
      const SymNode& sn = sym[i].nodes[k];
      const int64_t g = node_base[i] + (int64_t)k;
      NodeDev& nd = h_nodes[g];
      nd.np = sn.np;
      nd.nu = (int32_t)sn.upd.size();
      nd.m = nd.np + nd.nu;
      nd.pivb = sn.piv_begin;
      nd.mat_off = mat_off[i];
      nd.mat = i;
      nd.front_off = front_total;
      front_total += (int64_t)nd.m * nd.m;
      nd.uvec_off = uvec_total;
      uvec_total += nd.nu;
      nd.upd_off = upd_total;
      upd_total += nd.nu;
      nd.nch = (int32_t)sn.children.size();
      nd.child_off = (int32_t)h_children.size();
      for (int32_t ch : sn.children) h_children.push_back(node_base[i] + ch);
      nd.gmap_off = gm_total;
      gm_total += (int64_t)nd.nch * nd.m;
      node_level[g] = sn.level;
      max_np = std::max(max_np, nd.np);
      max_m = std::max(max_m, nd.m);
      factor_flops += 8.0 * nd.np * (double)nd.m * nd.m;
      schur_flops += 8.0 * nd.np * (double)nd.nu * nd.nu;
      {
        // (a) what a partial LU of the front needs (zgetrf on the np pivot columns, 8 real
        // flops per complex multiply-add): 8 sum_{k<np} (m-1-k)^2;
        // (b) what the kernels here execute: Gauss-Jordan inverse of the pivot block (8 np^3),
        // F_PU = A^{-1} B (8 np^2 nu), the Schur complement (8 np nu^2: all 64x64 tiles, or the
        // tiles on and below the diagonal when the matrix is symmetric), and the F_UP GEMM
        // (8 np^2 nu) only when it is not symmetric
        auto sq = [](double x) { return x <= 0 ? 0.0 : x * (x + 1) * (2 * x + 1) / 6.0; };
        const double np = nd.np, nu = nd.nu, m = nd.m;
        lu_flops += 8.0 * (sq(m - 1) - sq(m - np - 1));
        const double nt = (nd.nu + kTile - 1) / kTile;
        const double lower = nu > 0 ? (nt * (nt + 1) / 2) / (nt * nt) : 0.0;
        exec_flops_full += 8.0 * np * np * np + 16.0 * np * np * nu + 8.0 * np * nu * nu;
        exec_flops_sym += 8.0 * np * np * np + 8.0 * np * np * nu + 8.0 * np * nu * nu * lower;
      }
      factor_entries += (double)nd.m * nd.m - (double)nd.nu * nd.nu;
    }
  // packed F_UP rows for the solve kernels live after the fronts
  upk_total = 0;
  std::vector<int32_t> h_parent(nn, -1);
  for (int i = 0; i < nmat; ++i)
    for (size_t k = 0; k < sym[i].nodes.size(); ++k) {
      const int64_t g = node_base[i] + (int64_t)k;
      NodeDev& nd = h_nodes[g];
      nd.upk_off = front_total + upk_total;
      upk_total += (int64_t)nd.nu * nd.np;
      if (sym[i].nodes[k].parent >= 0) h_parent[g] = node_base[i] + sym[i].nodes[k].parent;
    }
  std::vector<int32_t> h_upd(upd_total), h_gmap(gm_total, -1);
  // upd lists + gather maps
  par_for(nmat, [&](int64_t i) {
    const SymOut& so = sym[i];
    for (size_t k = 0; k < so.nodes.size(); ++k) {
      const SymNode& sn = so.nodes[k];
      const NodeDev& nd = h_nodes[node_base[i] + k];
      std::copy(sn.upd.begin(), sn.upd.end(), h_upd.begin() + nd.upd_off);
      const int32_t pend = sn.piv_begin + sn.np;
      for (size_t ci = 0; ci < sn.children.size(); ++ci) {
        const SymNode& ch = so.nodes[sn.children[ci]];
        int32_t* g = h_gmap.data() + nd.gmap_off + (int64_t)ci * nd.m;
        for (size_t a = 0; a < ch.upd.size(); ++a) {
          const int32_t j = ch.upd[a];
          int32_t pos;
          if (j < pend) {
            if (j < sn.piv_begin) throw std::runtime_error("multifrontal: child update outside parent");
            pos = j - sn.piv_begin;
          } else {
            auto it = std::lower_bound(sn.upd.begin(), sn.upd.end(), j);
            if (it == sn.upd.end() || *it != j)
              throw std::runtime_error("multifrontal: child update not in parent front");
            pos = sn.np + (int32_t)(it - sn.upd.begin());
          }
          g[pos] = (int32_t)a;
        }
      }
    }
  });
  // original entries -> (level, pos, src)
  std::vector<std::vector<int64_t>> epos(nlevels);
  std::vector<std::vector<int32_t>> esrc(nlevels);
  {
    std::vector<std::vector<std::vector<int64_t>>> tpos(nmat);
    std::vector<std::vector<std::vector<int32_t>>> tsrc(nmat);
    par_for(nmat, [&](int64_t i) {
      const SymOut& so = sym[i];
      const MatrixInput& mi = mats[i];
      tpos[i].assign(nlevels, {});
      tsrc[i].assign(nlevels, {});
      std::vector<int32_t> owner(mi.n);
      for (size_t k = 0; k < so.nodes.size(); ++k)
        for (int32_t q = 0; q < so.nodes[k].np; ++q) owner[so.nodes[k].piv_begin + q] = (int32_t)k;
      auto front_pos = [&](const SymNode& sn, int32_t j) -> int32_t {
        if (j < sn.piv_begin + sn.np) return j - sn.piv_begin;
        auto it = std::lower_bound(sn.upd.begin(), sn.upd.end(), j);
        if (it == sn.upd.end() || *it != j) throw std::runtime_error("multifrontal: entry outside front");
        return sn.np + (int32_t)(it - sn.upd.begin());
      };
      for (int32_t r = 0; r < mi.n; ++r)
        for (int32_t e = mi.rowptr[r]; e < mi.rowptr[r + 1]; ++e) {
          const int32_t a = so.iperm[r], b = so.iperm[mi.cols[e]];
          const int32_t k = owner[std::min(a, b)];
          const SymNode& sn = so.nodes[k];
          const NodeDev& nd = h_nodes[node_base[i] + k];
          const int64_t p = nd.front_off + (int64_t)front_pos(sn, a) * nd.m + front_pos(sn, b);
          tpos[i][sn.level].push_back(p);
          tsrc[i][sn.level].push_back(mi.src[e]);
        }
    });
    for (int L = 0; L < nlevels; ++L)
      for (int i = 0; i < nmat; ++i) {
        epos[L].insert(epos[L].end(), tpos[i][L].begin(), tpos[i][L].end());
        esrc[L].insert(esrc[L].end(), tsrc[i][L].begin(), tsrc[i][L].end());
      }
  }
  // level lists
  std::vector<std::vector<int32_t>> lev(nlevels);
  for (int64_t g = 0; g < nn; ++g) lev[node_level[g]].push_back((int32_t)g);
  std::vector<int64_t> h_epos;
  std::vector<int32_t> h_esrc;
  std::vector<int2> h_init, h_panel;
  std::vector<int4> h_tile;
  std::vector<int2> h_copyb;
  std::vector<GemmTask> h_yz, h_yzup, h_s, h_su;
  std::vector<int4> h_tr;
  std::vector<int32_t> h_act;
  std::vector<int64_t> h_woff;
  lev_ent_off.assign(1, 0);
  lev_init_off.assign(1, 0);
  lev_steps.assign(nlevels, 0);
  lev_step_base.assign(nlevels, 0);
  step_act_off.assign(1, 0);
  step_panel_off.assign(1, 0);
  step_tile_off.assign(1, 0);
  lev_copyb_off.assign(1, 0);
  lev_gjs_off.assign(1, 0);
  lev_gj_nb.clear();
  std::vector<int32_t> h_gjs;
  lev_yz_off.assign(1, 0);
  lev_yzup_off.clear();
  lev_tr_off.assign(1, 0);
  lev_s_off.assign(1, 0);
  lev_sup_off.clear();
  int64_t bb_max = 0;
  w_max = 0;
  max_act = 0;
  int64_t nsteps_total = 0;
  for (int L = 0; L < nlevels; ++L) {
    h_epos.insert(h_epos.end(), epos[L].begin(), epos[L].end());
    h_esrc.insert(h_esrc.end(), esrc[L].begin(), esrc[L].end());
    lev_ent_off.push_back((int64_t)h_epos.size());
    int32_t lnp = 0;
    int64_t bb = 0;  // B_orig workspace of this level
    for (int32_t g : lev[L]) {
      NodeDev& nd = h_nodes[g];
      for (int r = 0; r < nd.m; ++r) h_init.push_back(make_int2(g, r));
      lnp = std::max(lnp, nd.np);
      nd.bb_off = bb;
      if (nd.np > 0 && nd.nu > 0) {
        bb += (int64_t)nd.np * nd.nu;
        // the front's F_UP block keeps C_orig (the sweeps do not touch it); the
        // F_UP GEMM writes the final values straight into the packed solve layout
        for (int r = 0; r < nd.np; ++r) h_copyb.push_back(make_int2((int)g, r));
        const int np = nd.np, nu = nd.nu, m = nd.m;
        const int64_t A = nd.front_off, B = nd.front_off + np, C = nd.front_off + (int64_t)np * m,
                      D = C + np;
        auto tiles = [&](std::vector<GemmTask>& out, int64_t xo, int ldx, int64_t wo, int ldw, int wsel,
                         int64_t oo, int ldo, int M, int N, int mode) {
          for (int r0 = 0; r0 < M; r0 += kTile)
            for (int c0 = 0; c0 < N; c0 += kTile) {
              GemmTask t{};
              t.xo = xo; t.ldx = ldx; t.wo = wo; t.ldw = ldw; t.wsel = wsel; t.oo = oo; t.ldo = ldo;
              t.M = M; t.N = N; t.K = np; t.r0 = r0; t.c0 = c0; t.mode = mode;
              out.push_back(t);
            }
        };
        tiles(h_yz, A, m, nd.bb_off, nu, 1, B, m, np, nu, 0);            // F_PU = -(-A^-1) B_orig
        tiles(h_yzup, C, m, A, m, 0, nd.upk_off, np, nu, np, 0);         // F_UP = -C_orig (-A^-1), packed
        // F_UU -= C_orig F_PU: tiles on and below the diagonal always; the strictly upper tiles
        // only for a non-symmetric matrix (gated), else they are mirrored from below (mode 2)
        for (int r0 = 0; r0 < nu; r0 += kTile)
          for (int c0 = 0; c0 < nu; c0 += kTile) {
            GemmTask t{};
            t.xo = C; t.ldx = m; t.wo = B; t.ldw = m; t.wsel = 0; t.oo = D; t.ldo = m;
            t.M = nu; t.N = nu; t.K = np; t.r0 = r0; t.c0 = c0;
            t.mode = r0 > c0 ? 2 : 1;
            (c0 > r0 ? h_su : h_s).push_back(t);
          }
        // symmetric matrices: packed F_UP = F_PU^T, 32x32 transpose tiles
        for (int r0 = 0; r0 < nu; r0 += 32)
          for (int c0 = 0; c0 < np; c0 += 32) h_tr.push_back(make_int4(g, r0, c0, 0));
      }
    }
    bb_max = std::max(bb_max, bb);
    lev_init_off.push_back((int64_t)h_init.size());
    lev_copyb_off.push_back((int64_t)h_copyb.size());
    lev_yzup_off.push_back((int64_t)h_yz.size());
    h_yz.insert(h_yz.end(), h_yzup.begin(), h_yzup.end());
    h_yzup.clear();
    lev_yz_off.push_back((int64_t)h_yz.size());
    lev_sup_off.push_back((int64_t)h_s.size());  // this level's gated (strictly upper) Schur tiles start here
    h_s.insert(h_s.end(), h_su.begin(), h_su.end());
    h_su.clear();
    lev_s_off.push_back((int64_t)h_s.size());
    lev_tr_off.push_back((int64_t)h_tr.size());
    // small pivot blocks: one k_gj_smem CTA per node instead of the sweeps
    // (k_gj_smem is issue-bound at ~30 instructions per element update; it
    // beats the sweeps for np <= 32 only, measured on the B200)
    lev_gj_nb.push_back(lnp <= 32 ? lnp : 0);
    for (int32_t g : lev[L])
      if (lev_gj_nb.back() && h_nodes[g].np > 0) h_gjs.push_back(g);
    lev_gjs_off.push_back((int64_t)h_gjs.size());
    const int nst = lev_gj_nb.back() ? 0 : (lnp + kPB - 1) / kPB;
    lev_steps[L] = nst;
    lev_step_base[L] = nsteps_total;
    for (int st = 0; st < nst; ++st) {
      int64_t wo = 0;
      int32_t nact = 0;
      for (int32_t g : lev[L]) {
        const NodeDev& nd = h_nodes[g];
        if (nd.np <= st * kPB) continue;
        const int32_t ai = nact++;
        h_act.push_back(g);
        h_woff.push_back(wo);
        wo += (int64_t)nd.m * kPB;
        // sweeps over the pivot block A only (F_PU, F_UP, F_UU: k_gemm)
        for (int ch = 0; ch * kPanelCols < nd.np; ++ch) h_panel.push_back(make_int2(ai, ch));
        const int K0 = st * kPB, kb = std::min(kPB, nd.np - K0);
        const int nt = (nd.np + kTile - 1) / kTile;
        for (int tr = 0; tr < nt; ++tr) {
          const int rb = tr * kTile, re = std::min(nd.np, rb + kTile);
          if (rb >= K0 && re <= K0 + kb) continue;  // tile rows all pivots
          for (int tc = 0; tc < nt; ++tc) h_tile.push_back(make_int4(ai, tr, tc, 0));
        }
      }
      w_max = std::max(w_max, wo);
      max_act = std::max(max_act, nact);
      step_act_off.push_back((int64_t)h_act.size());
      step_panel_off.push_back((int64_t)h_panel.size());
      step_tile_off.push_back((int64_t)h_tile.size());
      ++nsteps_total;
    }
  }
  std::vector<int32_t> h_gabs(h_gmap.size(), -1);
  for (int64_t g = 0; g < nn; ++g) {
    const NodeDev& nd = h_nodes[g];
    for (int ci = 0; ci < nd.nch; ++ci) {
      const NodeDev& ch = h_nodes[h_children[nd.child_off + ci]];
      if (ch.uvec_off + ch.nu > INT32_MAX) fail(MDD_EINVAL, "update-vector space exceeds 2^31");
      for (int q = 0; q < nd.m; ++q) {
        const int32_t r = h_gmap[nd.gmap_off + (int64_t)ci * nd.m + q];
        if (r >= 0) h_gabs[nd.gmap_off + (int64_t)ci * nd.m + q] = (int32_t)(ch.uvec_off + r);
      }
    }
  }
  nodes.upload(h_nodes, s);
  children.upload(h_children, s);
  gmap.upload(h_gmap, s);
  gmap_abs.upload(h_gabs, s);
  upd.upload(h_upd, s);
  ent_pos.upload(h_epos, s);
  ent_src.upload(h_esrc, s);
  init_tasks.upload(h_init, s);
  panel_tasks.upload(h_panel, s);
  tile_tasks.upload(h_tile, s);
  copyb_tasks.upload(h_copyb, s);
  tr_tasks.upload(h_tr.empty() ? std::vector<int4>{make_int4(0, 0, 0, 0)} : h_tr, s);
  // one task list: the YZ tiles of every level, then the Schur tiles of every level
  {
    const int64_t nyz = (int64_t)h_yz.size();
    for (auto& o : lev_s_off) o += nyz;
    for (auto& o : lev_sup_off) o += nyz;
    h_yz.insert(h_yz.end(), h_s.begin(), h_s.end());
    gemm_tasks.upload(h_yz, s);
  }
  bbuf.alloc(std::max<int64_t>(1, bb_max));
  act_node.upload(h_act, s);
  gjs_node.upload(h_gjs.empty() ? std::vector<int32_t>{0} : h_gjs, s);
  act_woff.upload(h_woff, s);
  fronts.alloc(front_total + upk_total);
  uvec.alloc(std::max<int64_t>(1, uvec_total));
  pbuf.alloc(std::max<int64_t>(1, (int64_t)max_act * kPB * kPB));
  wbuf.alloc(std::max<int64_t>(1, w_max));
  pivstat.alloc(std::max<int64_t>(2, 2 * (int64_t)nn));
  bloc.alloc(std::max<int64_t>(1, nloc));
  fpst.alloc(std::max<int64_t>(1, nloc));
  xloc.alloc(std::max<int64_t>(1, nloc));
  static bool attr_set = false;
  if (!attr_set) {
    CK(cudaFuncSetAttribute(k_update, cudaFuncAttributeMaxDynamicSharedMemorySize,
                            (int)(sizeof(double2) * (kTile * (kPB + 1) + kPB * (kTile + 1)))));
    CK(cudaFuncSetAttribute(k_gemm, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)kGemmSmem));
    CK(cudaFuncSetAttribute(k_gj_smem, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)(sizeof(double2) * 96 * 96)));
    attr_set = true;
  }
  build_solve(lev);
  if (getenv("MDD_PLAN_STATS")) {
    // per-level histogram: nodes, sum np, max m, GJ flops, Schur flops
    for (int L = 0; L < nlevels; ++L) {
      double gj = 0, sc = 0, sm = 0;
      int mx = 0;
      for (int32_t g : lev[L]) {
        const NodeDev& nd = h_nodes[g];
        sc += 8.0 * nd.np * (double)nd.nu * nd.nu;
        gj += 8.0 * nd.np * ((double)nd.m * nd.m - (double)nd.nu * nd.nu);
        sm += nd.np;
        mx = std::max(mx, nd.m);
      }
      fprintf(stderr, "[plan] L%d nodes=%zu sum_np=%.0f max_m=%d gj_flops=%.3e schur_flops=%.3e\n", L,
              lev[L].size(), sm, mx, gj, sc);
    }
  }
  CK(cudaStreamSynchronize(s));
}

static unsigned gblocks(int64_t n, int bs, int cap) {
  return (unsigned)std::max<int64_t>(1, std::min<int64_t>((n + bs - 1) / bs, cap));
}


void FrontPlan::factor(const double2* vals, cudaStream_t s, const int* sym_flag) {
  if (nnodes == 0) return;
  k_pivinit<<<gblocks(nnodes, 256, 1024), 256, 0, s>>>(pivstat.p, nnodes);
  CK_LAUNCH(ctx);
  const size_t upd_smem = sizeof(double2) * (kTile * (kPB + 1) + kPB * (kTile + 1));
  for (int L = 0; L < nlevels; ++L) {
    const int64_t ni = lev_init_off[L + 1] - lev_init_off[L];
    if (ni) {
      k_front_init<<<(unsigned)((ni + 7) / 8), 256, 0, s>>>(init_tasks.p + lev_init_off[L], ni,
                                                           nodes.p, children.p, gmap.p, fronts.p);
      CK_LAUNCH(ctx);
    }
    const int64_t ne = lev_ent_off[L + 1] - lev_ent_off[L];
    if (ne) {
      k_front_scatter<<<gblocks(ne, 256, ctx->nsm * 32), 256, 0, s>>>(
          ne, ent_pos.p + lev_ent_off[L], ent_src.p + lev_ent_off[L], vals, fronts.p);
      CK_LAUNCH(ctx);
    }
    const int64_t cb0 = lev_copyb_off[L], ncb = lev_copyb_off[L + 1] - cb0;
    if (ncb) {  // B_orig = F_PU before the sweeps
      k_copy_b<<<(unsigned)((ncb + 7) / 8), 256, 0, s>>>(copyb_tasks.p + cb0, ncb, nodes.p, fronts.p, bbuf.p);
      CK_LAUNCH(ctx);
    }
    if (lev_gj_nb[L]) {
      const int64_t g0 = lev_gjs_off[L], ng = lev_gjs_off[L + 1] - g0;
      if (ng) {
        const int n = lev_gj_nb[L];  // max np of the level
        k_gj_smem<<<(unsigned)ng, 256, sizeof(double2) * n * n, s>>>(nodes.p, gjs_node.p + g0, fronts.p,
                                                                      pivstat.p);
        CK_LAUNCH(ctx);
      }
    }
    for (int st = 0; st < lev_steps[L]; ++st) {
      const int64_t si = lev_step_base[L] + st;
      const int64_t a0 = step_act_off[si], na = step_act_off[si + 1] - a0;
      const int64_t p0 = step_panel_off[si], npn = step_panel_off[si + 1] - p0;
      const int64_t t0 = step_tile_off[si], ntl = step_tile_off[si + 1] - t0;
      if (!na) continue;
      k_gj_small<2, true><<<(unsigned)na, 256, 0, s>>>(nodes.p, act_node.p + a0, fronts.p, pivstat.p, st, pbuf.p);
      CK_LAUNCH(ctx);
      k_panel<<<(unsigned)npn, kPanelCols, 0, s>>>(panel_tasks.p + p0, nodes.p, act_node.p + a0,
                                                   act_woff.p + a0, st, fronts.p, pbuf.p, wbuf.p);
      CK_LAUNCH(ctx);
      if (ntl) {
        k_update<<<(unsigned)ntl, 256, upd_smem, s>>>(tile_tasks.p + t0, nodes.p, act_node.p + a0,
                                                      act_woff.p + a0, st, fronts.p, wbuf.p);
        CK_LAUNCH(ctx);
      }
    }
    // F_PU from -A^{-1}; F_UP by GEMM, or (sym_flag == 0 on the device: the
    // matrices are bitwise symmetric) as F_PU^T -- decided on the device, no sync
    const int64_t y0 = lev_yz_off[L], yup = lev_yzup_off[L], y1 = lev_yz_off[L + 1];
    if (yup > y0) {
      k_gemm<<<(unsigned)(yup - y0), 256, kGemmSmem, s>>>(gemm_tasks.p + y0, fronts.p, bbuf.p);
      CK_LAUNCH(ctx);
    }
    if (y1 > yup) {
      k_gemm<<<(unsigned)(y1 - yup), 256, kGemmSmem, s>>>(gemm_tasks.p + yup, fronts.p, bbuf.p, sym_flag);
      CK_LAUNCH(ctx);
    }
    const int64_t r0t = lev_tr_off[L], nt = lev_tr_off[L + 1] - r0t;
    if (sym_flag && nt) {
      k_transpose_up<<<(unsigned)nt, dim3(32, 8), 0, s>>>(tr_tasks.p + r0t, nodes.p, fronts.p, sym_flag);
      CK_LAUNCH(ctx);
    }
    // deferred Schur complement: lower + diagonal tiles (mirrored upwards when symmetric),
    // then the strictly upper tiles unless the matrices are symmetric (device-side gate)
    const int64_t s0 = lev_s_off[L], sup = lev_sup_off[L], s1 = lev_s_off[L + 1];
    if (sup > s0) {
      k_gemm<<<(unsigned)(sup - s0), 256, kGemmSmem, s>>>(gemm_tasks.p + s0, fronts.p, bbuf.p, nullptr, sym_flag);
      CK_LAUNCH(ctx);
    }
    if (s1 > sup) {
      if (sym_flag) k_gemm<<<(unsigned)(s1 - sup), 256, kGemmSmem, s>>>(gemm_tasks.p + sup, fronts.p, bbuf.p, sym_flag);
      else k_gemm<<<(unsigned)(s1 - sup), 256, kGemmSmem, s>>>(gemm_tasks.p + sup, fronts.p, bbuf.p);
      CK_LAUNCH(ctx);
    }
  }
}

int FrontPlan::check_pivots(std::string& msg, cudaStream_t s) {
  std::vector<double> ps(2 * (size_t)nnodes);
  if (nnodes) pivstat.download(ps.data(), ps.size(), s);
  CK(cudaStreamSynchronize(s));
  std::vector<double> mn(nmat, INFINITY), mx(nmat, 0.0);
  for (int64_t g = 0; g < nnodes; ++g) {
    if (h_nodes[g].np == 0) continue;
    const int i = h_nodes[g].mat;
    mn[i] = std::min(mn[i], ps[2 * g]);
    mx[i] = std::max(mx[i], ps[2 * g + 1]);
  }
  min_pivot_ratio = INFINITY;
  for (int i = 0; i < nmat; ++i)
    if (mat_n[i] != 0 && mx[i] > 0.0) min_pivot_ratio = std::min(min_pivot_ratio, mn[i] / mx[i]);
  for (int i = 0; i < nmat; ++i) {
    if (mat_n[i] == 0) continue;
    const bool bad = !(mx[i] > 0.0) || !std::isfinite(mx[i]) || !(mn[i] > 1e-14 * mx[i]);
    if (bad) {
      char buf[256];
      snprintf(buf, sizeof(buf),
               "pivot ratio %.2e below tolerance, matrix is numerically singular",
               mn[i] / std::max(mx[i], 1e-300));
      msg = buf;
      return i;
    }
  }
  return -1;
}

}  // namespace mdd
