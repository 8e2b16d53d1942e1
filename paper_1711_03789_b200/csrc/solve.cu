// Forward/backward solves over a multifrontal plan (frontal.h).
//
// Replaces DenseLU.solve (zgetrs, reference linalg.py:103-107) as called per
// subdomain in PreconditionerState._one_level (precond.py:217-225) and for the
// coarse block in coarse_solve (precond.py:227-228).
//
// Algebra (frontal.h): forward  r_U -= F_UP r_P   (leaves -> root)
//                      backward x_P  = -(F_PP r_P + F_PU x_U)   (root -> leaves)
// One launch per tree level, one CTA per task; consecutive levels are chained
// with programmatic dependent launch (the next level's CTAs start their factor
// TMA copies during this level's tail and wait in griddepcontrol.wait before
// touching vectors).  A task is a row range of one
// front block holding ~32 KB of factor data: [F_PP F_PU] rows are contiguous
// in the row-major front, and F_UP rows are written row-contiguous by the
// factorisation's F_UP GEMM (frontal.cu), so every task is one contiguous byte range that
// thread 0 moves into shared memory with a single TMA bulk copy
// (cp.async.bulk + mbarrier complete_tx) while the block gathers the task's
// vector; the GEMV then runs out of shared memory.  Thread 0 also issues an
// L2 bulk prefetch for the task kTSolvePrefetch positions later (which near a
// level's end reaches into the next level), so HBM stays busy independently
// of each CTA's gather latency.  The restriction v[I_l] is fused into the
// forward gathers.  Summation order per row is fixed: results are bitwise
// reproducible.
#include <algorithm>
#include <cstdlib>

#include "frontal.h"
#include "mdd_kernels.cuh"

namespace mdd {

// -------------------------------------------------------------- kernels
// GEMV of R rows (row-major, row length len, in shared memory) with the
// vector z (shared memory): a group of tpr threads per row, tpr chosen from
// the row count so all 256 threads work; groups wider than a warp combine
// their warp sums through `red`.  emit(r, sum) is called once per row.
template <typename Emit, typename Sync>
__device__ __forceinline__ void smem_gemv(const double2* __restrict__ D, int R, int len,
                                          const double2* __restrict__ z, int ct, double2* red,
                                          Emit emit, Sync sync) {
  constexpr int T = 256;
  int tpr = R > 0 ? T / R : T;
  tpr = tpr >= 256 ? 256 : tpr >= 128 ? 128 : tpr >= 64 ? 64 : tpr >= 32 ? 32 : tpr >= 16 ? 16 : 8;
  while (tpr > 8 && (tpr >> 1) >= len) tpr >>= 1;
  const int ng = T / tpr, grp = ct / tpr, lig = ct % tpr, lane = ct & 31, cw = ct >> 5;
  const int iters = (R + ng - 1) / ng;
  for (int it = 0; it < iters; ++it) {
    const int r = it * ng + grp;
    double2 a0 = make_double2(0.0, 0.0), a1 = a0, a2 = a0, a3 = a0;
    if (r < R) {
      const double2* row = D + (int64_t)r * len;
      int q = lig;
      for (; q + 3 * tpr < len; q += 4 * tpr) {
        a0 = cfma(row[q], z[q], a0);
        a1 = cfma(row[q + tpr], z[q + tpr], a1);
        a2 = cfma(row[q + 2 * tpr], z[q + 2 * tpr], a2);
        a3 = cfma(row[q + 3 * tpr], z[q + 3 * tpr], a3);
      }
      for (; q < len; q += tpr) a0 = cfma(row[q], z[q], a0);
    }
    double2 acc = cadd(cadd(a0, a1), cadd(a2, a3));
    for (int o = min(tpr, 32) >> 1; o > 0; o >>= 1) {
      acc.x += __shfl_xor_sync(0xffffffffu, acc.x, o);
      acc.y += __shfl_xor_sync(0xffffffffu, acc.y, o);
    }
    if (tpr > 32) {
      if (lane == 0) red[cw] = acc;
      sync();
      if (lig == 0) {
        acc = red[cw];
        for (int k = 1; k < tpr / 32; ++k) acc = cadd(acc, red[cw + k]);
      }
      sync();
    }
    if (lig == 0 && r < R) emit(r, acc);
  }
}

// One CTA per task.  Thread 0 issues the task's TMA bulk copy, then an L2
// bulk prefetch of the task `pf` positions later in the solve order (the
// task list runs forward levels then backward levels, so near the end of a
// level this reaches into the next level's first tasks and also covers the
// launch gap).  HBM is thus kept busy by prefetches independently of how long
// each CTA spends in its vector gathers.
template <bool FWD, int MINB>
__global__ void __launch_bounds__(256, MINB) k_solve_tma(const LvlTask* __restrict__ tasks, int64_t first,
                                                   int64_t total, int pf,
                                                   const int32_t* __restrict__ gabs,
                                                   const int32_t* __restrict__ upd,
                                                   const double2* __restrict__ data,
                                                   const double2* __restrict__ bloc,
                                                   const double2* __restrict__ v,
                                                   const int32_t* __restrict__ gidx,
                                                   double2* __restrict__ fpst, double2* __restrict__ uvec,
                                                   double2* __restrict__ xloc, int dcap,
                                                   const double2* __restrict__ zbuf) {
  extern __shared__ __align__(128) unsigned char smraw[];
  __shared__ __align__(8) uint64_t bar;
  __shared__ double2 red[8];
  double2* D = reinterpret_cast<double2*>(smraw);
  double2* z = D + dcap;
  // programmatic dependent launch: let the next level's grid get resident
  // while this level's last wave runs (its prologue only touches factor data)
  asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
  const int64_t t = first + blockIdx.x;
  const LvlTask tk = tasks[t];
  const int np = tk.np, nrow = tk.nrow, len = tk.len;
  const uint32_t bytes = (uint32_t)nrow * (uint32_t)len * 16u;
  if (threadIdx.x == 0) {
    mbar_init(&bar, 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    if (bytes) {
      mbar_arrive_tx(&bar, bytes);
      bulk_g2s(D, data + tk.off, bytes, &bar);
    }
    if (pf > 0 && t + pf < total) {
      const LvlTask tp = tasks[t + pf];
      const uint32_t pb = (uint32_t)tp.nrow * (uint32_t)tp.len * 16u;
      if (pb)
        asm volatile("cp.async.bulk.prefetch.L2.global [%0], %1;" ::"l"(data + tp.off), "r"(pb) : "memory");
    }
  }
  const int64_t base = tk.base;
  // everything below reads vectors written by the previous level (or the
  // kernels before the solve): wait for the prerequisite grid to complete
  asm volatile("griddepcontrol.wait;" ::: "memory");
  if (tk.zoff >= 0) {
    // the node's vector was assembled once by k_level_gather: a contiguous copy
    const double2* zn = zbuf + tk.zoff;
    if (FWD) {
      for (int q = threadIdx.x; q < np + nrow; q += blockDim.x) z[q] = zn[q < np ? q : tk.r0 + q];
    } else {
      for (int q = threadIdx.x; q < tk.m; q += blockDim.x) z[q] = zn[q];
    }
  } else if (FWD) {
    const int32_t* ga = gabs + tk.aux_off;
    const int m = tk.m;
    for (int q = threadIdx.x; q < np + nrow; q += blockDim.x) {
      const int pos = q < np ? q : np + tk.r0 + (q - np);
      double2 f = make_double2(0.0, 0.0);
      if (q < np) f = v ? v[gidx[base + q]] : bloc[base + q];
      for (int ci = 0; ci < tk.nch; ++ci) {
        const int g = ga[(int64_t)ci * m + pos];
        if (g >= 0) f = cadd(f, uvec[g]);
      }
      z[q] = f;
      if (q < np && tk.r0 == 0) fpst[base + q] = f;
    }
  } else {
    const int32_t* up = upd + tk.aux_off;
    const int64_t moff = tk.mat_off;
    for (int q = threadIdx.x; q < tk.m; q += blockDim.x)
      z[q] = q < np ? fpst[base + q] : xloc[moff + up[q - np]];
  }
  __syncthreads();
  if (!bytes) return;
  mbar_wait(&bar, 0);
  auto sync = [] { __syncthreads(); };
  double2* out = (FWD ? uvec : xloc) + tk.out_off;
  if (FWD) {
    const double2* fu = z + np;
    smem_gemv(D, nrow, len, z, threadIdx.x, red, [&](int r, double2 acc) { out[r] = csub(fu[r], acc); }, sync);
  } else {
    smem_gemv(D, nrow, len, z, threadIdx.x, red, [&](int r, double2 acc) { out[r] = cneg(acc); }, sync);
  }
}

// One CTA per node of a level whose fronts are cut into many tasks: the node's vector z
// (forward: [f_P ; children's updates on the U rows], backward: [f_P ; x_U]) is assembled
// once here instead of once per task (a front with np = 1000 has ~350 forward tasks, each of
// which would repeat the same gathers through the children's maps).
template <bool FWD>
__global__ void __launch_bounds__(256) k_level_gather(const LvlTask* __restrict__ nodes, int64_t first,
                                                      const int32_t* __restrict__ gabs,
                                                      const int32_t* __restrict__ upd,
                                                      const double2* __restrict__ bloc,
                                                      const double2* __restrict__ v,
                                                      const int32_t* __restrict__ gidx, double2* __restrict__ fpst,
                                                      const double2* __restrict__ uvec,
                                                      const double2* __restrict__ xloc, double2* __restrict__ zbuf) {
  asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
  const LvlTask tk = nodes[first + blockIdx.x];
  asm volatile("griddepcontrol.wait;" ::: "memory");
  double2* zn = zbuf + tk.zoff;
  const int np = tk.np, m = tk.m;
  const int64_t base = tk.base;
  if (FWD) {
    const int32_t* ga = gabs + tk.aux_off;
    for (int pos = threadIdx.x; pos < m; pos += blockDim.x) {
      double2 f = make_double2(0.0, 0.0);
      if (pos < np) f = v ? v[gidx[base + pos]] : bloc[base + pos];
      for (int ci = 0; ci < tk.nch; ++ci) {
        const int g = ga[(int64_t)ci * m + pos];
        if (g >= 0) f = cadd(f, uvec[g]);
      }
      zn[pos] = f;
      if (pos < np) fpst[base + pos] = f;
    }
  } else {
    const int32_t* up = upd + tk.aux_off;
    const int64_t moff = tk.mat_off;
    for (int q = threadIdx.x; q < m; q += blockDim.x) zn[q] = q < np ? fpst[base + q] : xloc[moff + up[q - np]];
  }
}

// ------------------------------------------------------------- host side
void FrontPlan::build_solve(const std::vector<std::vector<int32_t>>& lev) {
  const int64_t te = kTSolveTaskElems;
  // backward tasks gather the node's whole z (m entries) per task: a floor on
  // the rows per task bounds that overhead for large fronts
  const int64_t minrows = kTSolveMinRows;
  std::vector<LvlTask> ht, hg;
  gnode_off.assign(1, 0);
  int64_t zmax = 1;
  lvl_off.assign(1, 0);
  lvl_dcap.clear();
  lvl_zcap.clear();
  auto level_tasks = [&](int L, int kind) {
    int64_t dcap = 8, zc = 8;
    const size_t first_task = ht.size();
    int64_t zoff = 0;
    std::vector<LvlTask> nodes_here;
    for (int32_t g : lev[L]) {
      const NodeDev& nd = h_nodes[g];
      const int len = kind == 0 ? nd.np : nd.m;
      const int nrows = kind == 0 ? nd.nu : nd.np;
      int rows = (int)std::max<int64_t>(1, len > 0 ? te / len : te);
      if (kind == 1) rows = (int)std::max<int64_t>(rows, std::min<int64_t>(minrows, (200 * 1024 / 16 - len) / std::max(1, len)));
      int r = 0;
      {
        LvlTask nt{};  // node descriptor for k_level_gather
        nt.base = (int64_t)nd.mat_off + nd.pivb;
        nt.aux_off = kind == 0 ? nd.gmap_off : nd.upd_off;
        nt.mat_off = nd.mat_off;
        nt.np = nd.np;
        nt.m = nd.m;
        nt.nch = nd.nch;
        nt.zoff = zoff;
        nodes_here.push_back(nt);
      }
      do {  // a zero-row forward task still assembles fp (fpst) for its node
        const int r1 = std::min(nrows, r + rows);
        LvlTask t{};
        t.zoff = zoff;
        t.off = (kind == 0 ? nd.upk_off : nd.front_off) + (int64_t)r * len;
        t.base = (int64_t)nd.mat_off + nd.pivb;
        t.out_off = kind == 0 ? nd.uvec_off + r : t.base + r;
        t.aux_off = kind == 0 ? nd.gmap_off : nd.upd_off;
        t.mat_off = nd.mat_off;
        t.r0 = r;
        t.nrow = r1 - r;
        t.len = len;
        t.np = nd.np;
        t.m = nd.m;
        t.nch = nd.nch;
        ht.push_back(t);
        dcap = std::max<int64_t>(dcap, (int64_t)(r1 - r) * len);
        zc = std::max<int64_t>(zc, kind == 0 ? (int64_t)nd.np + (r1 - r) : nd.m);
        r = r1;
      } while (r < nrows);
      zoff += nd.m;
    }
    // gather once per node where the fronts are cut into many tasks; otherwise the tasks keep
    // their fused gathers (one task per small front: nothing is repeated)
    const size_t ntask = ht.size() - first_task;
    // threshold swept on cfg4 (apply per solve: off 2056, 2x 2010, 4x 1983, 8x 1980 ms)
    if (!nodes_here.empty() && ntask >= 6 * nodes_here.size()) {
      hg.insert(hg.end(), nodes_here.begin(), nodes_here.end());
      zmax = std::max(zmax, zoff);
    } else {
      for (size_t k = first_task; k < ht.size(); ++k) ht[k].zoff = -1;
    }
    gnode_off.push_back((int64_t)hg.size());
    lvl_off.push_back((int64_t)ht.size());
    lvl_dcap.push_back((dcap + 7) / 8 * 8);
    lvl_zcap.push_back(zc);
    if (16 * (lvl_dcap.back() + zc) > 220 * 1024) fail(MDD_EINVAL, "front too large for the solve kernels");
  };
  for (int L = 0; L < nlevels; ++L) level_tasks(L, 0);
  for (int L = nlevels - 1; L >= 0; --L) level_tasks(L, 1);
  ltasks.upload(ht, ctx->stream);
  if (!hg.empty()) gnodes.upload(hg, ctx->stream);
  zbuf = DevBuf<double2>(zmax);
  static bool attr = false;  // per-function attribute shared by every plan
  if (!attr) {
    CK(cudaFuncSetAttribute(k_solve_tma<true, 0>, cudaFuncAttributeMaxDynamicSharedMemorySize, 220 * 1024));
    CK(cudaFuncSetAttribute(k_solve_tma<false, 0>, cudaFuncAttributeMaxDynamicSharedMemorySize, 220 * 1024));
    CK(cudaFuncSetAttribute(k_solve_tma<true, 6>, cudaFuncAttributeMaxDynamicSharedMemorySize, 220 * 1024));
    CK(cudaFuncSetAttribute(k_solve_tma<false, 6>, cudaFuncAttributeMaxDynamicSharedMemorySize, 220 * 1024));
    CK(cudaFuncSetAttribute(k_solve_tma<true, 8>, cudaFuncAttributeMaxDynamicSharedMemorySize, 220 * 1024));
    CK(cudaFuncSetAttribute(k_solve_tma<false, 8>, cudaFuncAttributeMaxDynamicSharedMemorySize, 220 * 1024));
    attr = true;
  }
}

void FrontPlan::solve(cudaStream_t s, const double2* v, const int32_t* gidx) {
  if (nnodes == 0) return;
  const int nl = nlevels;
  const int pf = kTSolvePrefetch;
  const bool pdl = true;  // programmatic dependent launch between the level kernels (measured 1.296 -> 1.233 ms per cfg1 apply)
  const int minb = 6;     // register cap: 40 registers, 6 CTAs per SM (swept 0/6/8 in round 1)
  const int64_t total = lvl_off[2 * nl];
  for (int k = 0; k < 2 * nl; ++k) {
    const int64_t n = lvl_off[k + 1] - lvl_off[k];
    if (!n) continue;
    const int64_t ng = gnode_off[k + 1] - gnode_off[k];
    if (ng > 0) {
      cudaLaunchConfig_t gc = {};
      gc.gridDim = dim3((unsigned)ng);
      gc.blockDim = dim3(256);
      gc.stream = s;
      cudaLaunchAttribute ga[1];
      ga[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
      ga[0].val.programmaticStreamSerializationAllowed = 1;
      gc.attrs = ga;
      gc.numAttrs = pdl ? 1 : 0;
      auto gfn = k < nl ? k_level_gather<true> : k_level_gather<false>;
      CK(cudaLaunchKernelEx(&gc, gfn, (const LvlTask*)gnodes.p, gnode_off[k], (const int32_t*)gmap_abs.p,
                            (const int32_t*)upd.p, (const double2*)bloc.p, v, gidx, fpst.p, (const double2*)uvec.p,
                            (const double2*)xloc.p, zbuf.p));
      CK_LAUNCH(ctx);
    }
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3((unsigned)n);
    cfg.blockDim = dim3(256);
    cfg.dynamicSmemBytes = 16 * (size_t)(lvl_dcap[k] + lvl_zcap[k]);
    cfg.stream = s;
    cudaLaunchAttribute attr[1];
    attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    attr[0].val.programmaticStreamSerializationAllowed = 1;
    cfg.attrs = attr;
    cfg.numAttrs = pdl ? 1 : 0;
    auto kfn = k < nl ? (minb == 8 ? k_solve_tma<true, 8> : minb == 6 ? k_solve_tma<true, 6> : k_solve_tma<true, 0>)
                      : (minb == 8 ? k_solve_tma<false, 8> : minb == 6 ? k_solve_tma<false, 6> : k_solve_tma<false, 0>);
    CK(cudaLaunchKernelEx(&cfg, kfn, (const LvlTask*)ltasks.p, lvl_off[k], total, pf, (const int32_t*)gmap_abs.p,
                          (const int32_t*)upd.p, (const double2*)fronts.p, (const double2*)bloc.p, v, gidx, fpst.p,
                          uvec.p, xloc.p, (int)lvl_dcap[k], (const double2*)zbuf.p));
    CK_LAUNCH(ctx);
  }
}

}  // namespace mdd
