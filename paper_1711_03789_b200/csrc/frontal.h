// Batched multifrontal factorisation plan + numeric kernels (device).
//
// A "plan" holds several independent sparse matrices (the overlapping
// subdomain blocks, or the coarse block) after nested-dissection analysis.
// Each tree node owns a dense row-major front  F = [F_PP F_PU; F_UP F_UU]
// (P = its pivots, U = its update rows).  The numeric phase assembles fronts
// level by level (children's Schur complements extend-added in gather form,
// original entries scattered), then applies block Gauss-Jordan sweeps over
// the pivot blocks, leaving
//     F_PP <- -F_PP^{-1},  F_PU <- F_PP^{-1} F_PU,  F_UP <- F_UP F_PP^{-1},
//     F_UU <- F_UU - F_UP F_PP^{-1} F_PU           (Schur complement).
// A solve is then a sequence of batched GEMVs per level:
//     forward   r_U -= F_UP r_P                  (leaves -> root)
//     backward  x_P  = -(F_PP r_P + F_PU x_U)     (root -> leaves)
// No pivoting: the absorptive operators have Im(Theta v*Av) > 0 on every
// principal submatrix; pivot magnitudes are still tracked and
// the reference's ratio test (linalg.py:95-101) is applied per matrix.
#pragma once
#include <stdint.h>

#include <string>
#include <vector>

#include "mdd_internal.h"
#include "symbolic.h"

namespace mdd {

constexpr int kPB = 32;      // pivot block of the sweep
constexpr int kTile = 64;    // update tile
constexpr int kPanelCols = 128;
constexpr int kGemmKC = 16;  // K chunk of the front GEMMs (k_gemm)
constexpr size_t kGemmSmem = 2 * sizeof(double2) * (kTile * (kGemmKC + 4) + kGemmKC * (kTile + 2));

struct NodeDev {
  int64_t front_off;  // complex elements into the front storage
  int64_t upd_off;    // into upd (int32 ND indices)
  int64_t uvec_off;   // into the forward update-vector buffer
  int64_t gmap_off;   // into gmap: nch * m entries
  int32_t m, np, nu, pivb;
  int32_t mat_off;    // offset of the node's matrix in the local vector space
  int32_t nch, child_off, mat;
  int64_t upk_off;    // packed F_UP rows (solve.cu), elements into the front storage
  int64_t bb_off;     // B_orig workspace (np x nu) of the node's level, elements into bbuf
};

// One 64x64 output tile of a batched complex GEMM on the fronts (k_gemm):
//   mode 0: O = -X W     mode 1: O -= X W     mode 2: as 1, and the transposed tile is written too
//   when the factorisation is symmetric (Schur complement tiles below the diagonal)
// X (M x K, ld ldx), W (K x N, ld ldw), O (M x N, ld ldo) as element offsets
// into the front storage (wsel bit 0: W lives in the B_orig workspace).
struct GemmTask {
  int64_t xo, wo, oo;
  int32_t ldx, ldw, ldo, M, N, K, r0, c0, mode, wsel;
};

// one solve task (solve.cu): rows [r0, r0+nrow) of a front block of row length len
struct LvlTask {
  int64_t off;      // factor rows (elements into the front storage)
  int64_t out_off;  // forward: uvec index of row r0; backward: xloc index of row r0
  int64_t aux_off;  // forward: gather map (gmap_abs); backward: update list (upd)
  int64_t base;     // local vector index of the node's first pivot
  int64_t zoff;     // >= 0: the node's vector z was gathered once into zbuf (k_level_gather); -1: gather in the task
  int32_t mat_off, r0, nrow, len, np, m, nch, pad;
};
constexpr int kTSolveTaskElems = 2048;  // factor entries per solve task (32 KB)
constexpr int kTSolvePrefetch = 500;    // L2 prefetch distance (tasks)
constexpr int kTSolveMinRows = 4;       // backward tasks: minimum rows per task (measured: cfg2 apply 4.14 -> 3.85 ms; cfg4 apply per solve 2 / 3 / 4 / 8 rows: 2006 / 1993 / 1962 / 2044 ms)

struct MatrixInput {
  int32_t n = 0;
  std::vector<int32_t> rowptr, cols;  // local pattern (sorted)
  std::vector<int32_t> src;           // per local entry: index into the value array
  std::vector<int32_t> xyz;           // (n,3)
  int32_t grid = 2;                   // xyz units per mesh cell
};

struct FrontPlan {
  mdd_ctx* ctx = nullptr;
  int32_t nmat = 0;
  std::vector<int32_t> mat_n, mat_off;
  std::vector<std::vector<int32_t>> perm;  // per matrix: ND index -> local index
  int64_t nloc = 0;
  double min_pivot_ratio = 0.0;  // smallest min|pivot| / max|pivot| over the matrices (check_pivots)
  int32_t nnodes = 0, nlevels = 0;
  std::vector<NodeDev> h_nodes;
  DevBuf<NodeDev> nodes;
  DevBuf<int32_t> children, gmap, upd;
  // original entries, grouped by level
  DevBuf<int64_t> ent_pos;
  DevBuf<int32_t> ent_src;
  std::vector<int64_t> lev_ent_off;
  // task lists
  DevBuf<int2> init_tasks;
  std::vector<int64_t> lev_init_off;
  std::vector<int32_t> lev_steps;        // sweep steps per level
  std::vector<int64_t> lev_step_base;    // index of (level, step 0) in step arrays
  std::vector<int64_t> step_act_off;     // per (level,step): offset into act arrays
  std::vector<int64_t> step_panel_off;
  std::vector<int64_t> step_tile_off;
  DevBuf<int32_t> act_node;
  // levels whose pivot blocks all have np <= 96: one k_gj_small CTA per node
  std::vector<int32_t> lev_gj_nb;        // 0 (sweeps) or the level's max np (<= 96, k_gj_smem)
  std::vector<int64_t> lev_gjs_off;
  DevBuf<int32_t> gjs_node;
  DevBuf<int64_t> act_woff;
  DevBuf<int2> panel_tasks;
  DevBuf<int4> tile_tasks;
  // per level: B_orig copy tasks, GEMM tiles for F_PU = A^-1 B and
  // F_UP = C A^-1 (one launch) and the Schur update (next launch)
  DevBuf<int2> copyb_tasks;
  DevBuf<GemmTask> gemm_tasks;
  DevBuf<double2> bbuf;
  std::vector<int64_t> lev_copyb_off, lev_yz_off, lev_s_off, lev_sup_off;
  // per level: start of the F_UP tiles inside the YZ range; transpose tiles
  // (symmetric fronts: packed F_UP = F_PU^T, k_transpose_up)
  std::vector<int64_t> lev_yzup_off, lev_tr_off;
  DevBuf<int4> tr_tasks;
  DevBuf<int32_t> gmap_abs;            // gather maps as absolute uvec indices (solve)
  int32_t max_np = 0, max_m = 0, max_act = 0;
  int64_t front_total = 0, uvec_total = 0, w_max = 0;
  double factor_flops = 0, factor_entries = 0, schur_flops = 0;
  double lu_flops = 0, exec_flops_full = 0, exec_flops_sym = 0;  // see FrontPlan::build
  // numeric storage
  DevBuf<double2> fronts, uvec, pbuf, wbuf;
  DevBuf<double> pivstat;  // per node: [min |pivot|, max |pivot|]
  // solve workspace (local vectors)
  DevBuf<double2> bloc, fpst, xloc;
  float factor_ms = 0;
  // solve (solve.cu): per-level task lists over the fronts and the packed F_UP rows
  int64_t upk_total = 0;
  DevBuf<LvlTask> ltasks;
  std::vector<int64_t> lvl_off, lvl_dcap, lvl_zcap;  // forward levels ascending, then backward descending
  // levels whose fronts are cut into many tasks gather each node's vector once (k_level_gather)
  // instead of once per task: node descriptors per level and the shared z buffer
  DevBuf<LvlTask> gnodes;
  std::vector<int64_t> gnode_off;   // per solve level: [gnode_off[k], gnode_off[k+1]) into gnodes (empty: fused gathers)
  DevBuf<double2> zbuf;
  void build_solve(const std::vector<std::vector<int32_t>>& lev);

  // build from analysed matrices
  void build(mdd_ctx* c, std::vector<MatrixInput>& mats, int32_t leaf);
  // numeric factorisation from `vals` (complex, indexed by MatrixInput.src)
  // sym_flag (device, may be null): 0 = the matrices are bitwise complex
  // symmetric, F_UP is transposed from F_PU instead of a second GEMM
  void factor(const double2* vals, cudaStream_t s, const int* sym_flag = nullptr);
  // per-matrix pivot ratio check; returns index of the first failing matrix or -1
  int check_pivots(std::string& msg, cudaStream_t s);
  // solve: bloc (ND-ordered local rhs) -> xloc; with v/gidx the local rhs is
  // gathered as v[gidx[i]] inside the solve (fused restriction)
  void solve(cudaStream_t s, const double2* v = nullptr, const int32_t* gidx = nullptr);
};

}  // namespace mdd
