// Unrestarted GMRES on the device (reference krylov.gmres, krylov.py:64-209).
//
// The whole Arnoldi loop runs on the GPU: one iteration (preconditioner
// kernels, SpMV, optional weight SpMV, Arnoldi kernel) is captured once into
// the body of a CUDA-graph conditional WHILE node; the Arnoldi kernel clears
// the condition on convergence / happy breakdown / maxit, so there is no host
// round trip per iteration.  (A host-driven loop with per-phase CUDA events
// is kept for `ctx->timing` and for Python-callable operators.)
//
// The Arnoldi kernel is a persistent cooperative kernel, one CTA per SM; each
// CTA owns a contiguous slice of the vectors.  It performs, in the reference
// order (krylov.py:134-187):
//   2 passes x m MGS steps  h_j = <V_j, dw>; col[j] += h_j; w -= h_j V_j;
//       dw -= h_j DV_j                                      (krylov.py:137-143)
//   hnorm2 = Re vdot(w, dw), breakdown test, normalisation  (krylov.py:144-151)
//   complex Givens rotations + history clamp                (krylov.py:162-187)
// One grid barrier per MGS step: the axpy of step j and the partial dot of
// step j+1 are one fused sweep, and the slice needed at step j+2 is prefetched
// into L2 with a TMA bulk prefetch while the CTA waits at the barrier.  The
// orthogonality drift of the vector appended by the previous iteration
// (krylov.py:152-160) rides along in the first MGS pass (it needs the same
// V_j reads), so it costs no extra pass over the basis.  Cross-CTA sums use a
// fixed order: reruns are bitwise identical.
#include <cooperative_groups.h>

#include <chrono>
#include <cmath>
#include <cstring>

#include "mdd_internal.h"
#include "mdd_kernels.cuh"

namespace cg = cooperative_groups;

namespace mdd {

void prec_apply_dev(mdd_prec* P, const double2* v, double2* out, cudaStream_t s);
bool prec_is_distributed(const mdd_prec* P);
mdd_comm* prec_comm(const mdd_prec* P);
mdd_halo* prec_halo(const mdd_prec* P);
void prec_apply_dist(mdd_prec* P, const double2* v, double2* out, cudaStream_t s);
void prec_gather_owned(mdd_prec* P, double2* vec, cudaStream_t s);

constexpr int kArnThreads = 256;
constexpr int kMaxArnCTAs = 160;  // grid <= #SMs (148 on B200)

struct ArnoldiArgs {
  int64_t n;
  int64_t slice;   // elements per CTA
  int maxit;
  double2* V;      // (maxit+1) x n
  double2* DV;     // weighted basis or nullptr
  double2* w;      // new direction (input: operator output)
  double2* dw;     // D w (weighted) or nullptr
  double2* vin;    // out: copy of V[m] = next operator input
  double2* partials;  // (2*maxit+1) publications x G slots of `pad` double2 (dot, drift), NaN-filled per launch
  double2* H;      // (maxit+1) x maxit, column j at H + j*(maxit+1)
  double2* cs;
  double2* sn;
  double2* g;
  double* hist;
  double* drift;
  const double* beta;
  double tol;
  int check_drift;
  int* iter;             // device: completed iterations
  int* dstatus;          // device: [done, breakdown, iterations]
  volatile int* hstatus; // host-mapped copy (host loop) or nullptr
  cudaGraphConditionalHandle cond;
  int use_cond;
  int64_t wcap;  // STREAM path: w elements of the slice held in shared memory
  int pad;       // double2 per publication slot (2 or 8)
  int wg;        // 1: warp 0 alone polls the slots (gather_sum)
  int pf;        // REG path: L2 prefetch distance in MGS steps (kArnPf; MDD_ARN_PF)
  int zigzag;        // WIDE path: 1 = odd passes sweep the slice downwards
  int64_t pf_bytes;  // WIDE path: bytes of the next dot operand's slice prefetched into L2 during the exchange
  int pf_trips;      // WIDE path: in-sweep L2 prefetch distance of the dot operand, in trips (0 = off)
};

__device__ __forceinline__ void prefetch_l2(const void* p, int64_t bytes) {
  bytes &= ~(int64_t)15;
  if (bytes <= 0) return;
  asm volatile("cp.async.bulk.prefetch.L2.global [%0], %1;" ::"l"(p), "r"((unsigned)bytes) : "memory");
}

// two complex block sums at once (all threads receive both)
__device__ __forceinline__ void block_sum2x2(double2& a, double2& b, double2* sh) {
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5, nw = blockDim.x >> 5;
  a = warp_sum2(a);
  b = warp_sum2(b);
  __syncthreads();
  if (lane == 0) {
    sh[2 * wid] = a;
    sh[2 * wid + 1] = b;
  }
  __syncthreads();
  if (wid == 0) {
    double2 x = lane < nw ? sh[2 * lane] : make_double2(0.0, 0.0);
    double2 y = lane < nw ? sh[2 * lane + 1] : make_double2(0.0, 0.0);
    x = warp_sum2(x);
    y = warp_sum2(y);
    if (lane == 0) {
      sh[64] = x;
      sh[65] = y;
    }
  }
  __syncthreads();
  a = sh[64];
  b = sh[65];
}

constexpr int kArnE = 12;  // vector elements per thread kept in registers (register path)
constexpr int kArnPf = 4;  // REG path: L2 prefetch distance in MGS steps

__device__ __forceinline__ unsigned ld_acquire_u32(const unsigned* p) {
  unsigned v;
  asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}
__device__ __forceinline__ void st_release_u32(unsigned* p, unsigned v) {
  asm volatile("st.release.gpu.global.u32 [%0], %1;" ::"l"(p), "r"(v) : "memory");
}

// Self-validating all-gather.  Every (step, CTA) pair has its own pair of
// 16-byte slots, filled with 0xFF bytes by a memset before the kernel; a CTA
// publishes by plain stores, and a reader polls a slot until neither 8-byte
// half holds the fill pattern (each half is single-copy atomic).  Reading the
// value *is* the synchronisation: one round trip, no flags, no fences.
// Each CTA's (dot, drift) pair is one slot of `pad` double2 (pad = 8: alone
// on a 128-byte L2 line).  In isolation the flat all-gather runs at 3.3 us per
// step with 16-byte slots and 1.8 us with one slot per line (hot-line
// serialisation of the G*G polls, tools/allgather_bench.cu); inside k_arnoldi
// the padded layout is slower on the REG path and faster on the STREAM path,
// so the host picks the stride per path (measured on the B200).
// "Not yet published" is the exact 0xFF..FF pattern of the memset, not NaN-ness: a
// NaN that the arithmetic produced (operator or preconditioner output with a NaN or
// Inf) is published as the canonical quiet NaN, flows through the sums like in the
// reference (krylov.py:137-151) and ends as a NaN residual history, not as a spin.
__device__ __forceinline__ double canon_nan(double v) {
  return isnan(v) ? __longlong_as_double(0x7ff8000000000000ll) : v;
}
__device__ __forceinline__ void publish(double2* slot_step, int pad, double2 a, double2 b) {
  a = make_double2(canon_nan(a.x), canon_nan(a.y));
  b = make_double2(canon_nan(b.x), canon_nan(b.y));
  __stcg(slot_step + (int64_t)blockIdx.x * pad, a);
  __stcg(slot_step + (int64_t)blockIdx.x * pad + 1, b);
}

__device__ __forceinline__ bool unpublished(double v) { return __double_as_longlong(v) == -1ll; }
__device__ __forceinline__ bool bad2(double2 v) { return unpublished(v.x) || unpublished(v.y); }

// Relaxed gpu-scope load: always served coherently (L2), never hoisted out of
// a polling loop (asm volatile), but NOT ordered like a volatile access, so
// several polls of one thread are in flight together.
__device__ __forceinline__ double2 ld_relaxed2(const double2* p) {
  double2 v;
  asm volatile("ld.relaxed.gpu.global.v2.f64 {%0,%1}, [%2];" : "=d"(v.x), "=d"(v.y) : "l"(p) : "memory");
  return v;
}

// Thread t < G waits for CTA t's slots of this step (the dot slot, and the
// drift slot only when `with_drift`: both loads in flight together); warp 0
// then sums them in CTA order (fixed order -> bitwise reproducible) and
// broadcasts the result.
__device__ __forceinline__ void gather_sum(const double2* slot_step, int G, int pad, bool warp_gather,
                                           double2* sh, double2& dot, double2& dr, bool with_drift = true) {
  if (warp_gather) {
    // warp 0 alone polls: each lane keeps its <= kNPL slots' loads in flight
    // together and re-polls only the missing ones; it sums in the same order
    // as the staged variant below (bitwise-identical results), and the CTA
    // needs one barrier instead of two
    constexpr int kNPL = (kMaxArnCTAs + 31) / 32;
    if (threadIdx.x < 32) {
      double2 u[kNPL], v[kNPL];
#pragma unroll
      for (int i = 0; i < kNPL; ++i) {
        const int k = threadIdx.x + 32 * i;
        const double2* line = slot_step + (int64_t)k * pad;
        u[i] = k < G ? ld_relaxed2(line) : make_double2(0.0, 0.0);
        v[i] = (k < G && with_drift) ? ld_relaxed2(line + 1) : make_double2(0.0, 0.0);
      }
      long long spins = 0;
      for (;;) {
        bool miss = false;
#pragma unroll
        for (int i = 0; i < kNPL; ++i) {
          const int k = threadIdx.x + 32 * i;
          const double2* line = slot_step + (int64_t)k * pad;
          if (bad2(u[i])) { u[i] = ld_relaxed2(line); miss = true; }
          if (bad2(v[i])) { v[i] = ld_relaxed2(line + 1); miss = true; }
        }
        if (!miss) break;
        if (++spins > (1ll << 28)) __trap();  // never hang the device
      }
      double2 x = make_double2(0.0, 0.0), y = make_double2(0.0, 0.0);
#pragma unroll
      for (int i = 0; i < kNPL; ++i) {
        x = cadd(x, u[i]);
        y = cadd(y, v[i]);
      }
      x = warp_sum2(x);
      y = warp_sum2(y);
      if (threadIdx.x == 0) {
        sh[66] = x;
        sh[67] = y;
      }
    }
    __syncthreads();
    dot = sh[66];
    dr = sh[67];
    return;
  }
  double2* stage = sh + 68;  // 2*G slots after the block-reduce scratch
  if ((int)threadIdx.x < G) {
    const int k = threadIdx.x;
    long long spins = 0;
    const double2* line = slot_step + (int64_t)k * pad;
    double2 u = ld_relaxed2(line);
    double2 v = with_drift ? ld_relaxed2(line + 1) : make_double2(0.0, 0.0);
    while (bad2(u) || bad2(v)) {
      if (++spins > (1ll << 28)) __trap();  // never hang the device
      if (bad2(u)) u = ld_relaxed2(line);
      if (bad2(v)) v = ld_relaxed2(line + 1);
    }
    stage[k] = u;
    stage[G + k] = v;
  }
  __syncthreads();
  if (threadIdx.x < 32) {
    double2 x = make_double2(0.0, 0.0), y = make_double2(0.0, 0.0);
    for (int k = threadIdx.x; k < G; k += 32) {
      x = cadd(x, stage[k]);
      y = cadd(y, stage[G + k]);
    }
    x = warp_sum2(x);
    y = warp_sum2(y);
    if (threadIdx.x == 0) {
      sh[66] = x;
      sh[67] = y;
    }
  }
  __syncthreads();
  dot = sh[66];
  dr = sh[67];
}

// Block sum of (a, b) delivered to thread 0 only (it publishes): one block
// barrier.  `sh` is double-buffered by step parity: a buffer is rewritten two
// steps later, after thread 0 has passed the next step's barrier.
__device__ __forceinline__ void block_sum_t0(double2& a, double2& b, double2* sh) {
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5, nw = blockDim.x >> 5;
  a = warp_sum2(a);
  b = warp_sum2(b);
  if (lane == 0) {
    sh[2 * wid] = a;
    sh[2 * wid + 1] = b;
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    a = sh[0];
    b = sh[1];
    for (int k = 1; k < nw; ++k) {
      a = cadd(a, sh[2 * k]);
      b = cadd(b, sh[2 * k + 1]);
    }
  }
}

// max(x, 0.0) as Python evaluates it (krylov.py:145): a NaN stays a NaN
__device__ __forceinline__ double pymax0(double x) { return 0.0 > x ? 0.0 : x; }

__device__ __forceinline__ double2 cdotc_acc(double2 acc, double2 x, double2 y) {  // acc + conj(x) y
  acc.x += x.x * y.x + x.y * y.y;
  acc.y += x.x * y.y - x.y * y.x;
  return acc;
}
__device__ __forceinline__ double2 caxmy(double2 w, double2 h, double2 v) {  // w - h v
  return make_double2(w.x - (h.x * v.x - h.y * v.y), w.y - (h.x * v.y + h.y * v.x));
}

// Complex Givens update of Hessenberg column m-1 (krylov.py:162-187), residual
// history clamp and loop status; one thread.  col[0..m] holds the new column.
// The rotations are a dependent chain; their operands (cs, sn and the
// untouched col[j+1]) are loaded kTailBlk at a time into registers ahead of
// the chain, because col may alias the global arrays as far as the compiler
// knows and a load per step would otherwise wait out a full memory latency
// (m x ~0.5 us at m = 200).  Same operations in the same order as the
// straight loop: bitwise identical.
constexpr int kTailBlk = 16;
__device__ __forceinline__ void tail_rotate(const double2* cs, const double2* snv, double2* col, int m) {
  double2 cur = col[0];
  for (int j0 = 0; j0 < m - 1; j0 += kTailBlk) {
    const int nb = min(kTailBlk, m - 1 - j0);
    double2 c[kTailBlk], sn[kTailBlk], nx[kTailBlk];
#pragma unroll
    for (int q = 0; q < kTailBlk; ++q) {
      if (q < nb) {
        c[q] = cs[j0 + q];
        sn[q] = snv[j0 + q];
        nx[q] = col[j0 + q + 1];
      }
    }
#pragma unroll
    for (int q = 0; q < kTailBlk; ++q) {
      if (q < nb) {
        const double2 t = cadd(cmul(c[q], cur), cmul(sn[q], nx[q]));
        cur = cadd(cmul(cneg(cconj(sn[q])), cur), cmul(c[q], nx[q]));
        col[j0 + q] = t;
      }
    }
  }
  if (m >= 2) col[m - 1] = cur;
}

// New rotation m-1, rhs g, history clamp and loop status, after the stored
// rotations were applied to col; returns the final H(m-1, m-1).
__device__ double2 tail_finish(const ArnoldiArgs& a, const double2* col, int m, bool breakdown) {
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
  const double2 hmm = cadd(cmul(csm, col[m - 1]), cmul(snm, col[m]));
  const double2 gm1 = a.g[m - 1];
  a.g[m] = cmul(cneg(cconj(snm)), gm1);
  a.g[m - 1] = cmul(csm, gm1);
  // min(x, prev) as Python evaluates it (krylov.py:180): prev only if prev < x, so a
  // NaN residual is recorded as NaN instead of being clamped away
  const double relx = hypot(a.g[m].x, a.g[m].y) / *a.beta, relp = a.hist[m - 1];
  const double rel = relp < relx ? relp : relx;
  a.hist[m] = rel;
  const int done = (breakdown || rel <= a.tol) ? 1 : 0;
  *a.iter = m;
  a.dstatus[0] = done;
  a.dstatus[1] = breakdown ? 1 : 0;
  a.dstatus[2] = m;
  if (a.hstatus) {
    // host-mapped; [0] = the iteration that finished the solve (0 while running), one
    // 4-byte store, so a host loop that reads it while a later iteration runs still
    // sees a consistent value (gmres_cgs breaks on iterations it knows are complete)
    a.hstatus[1] = breakdown ? 1 : 0;
    a.hstatus[2] = m;
    a.hstatus[0] = done ? m : 0;
  }
  if (a.use_cond) cudaGraphSetConditional(a.cond, (done || m >= a.maxit) ? 0u : 1u);
  return hmm;
}

__device__ void arnoldi_tail(const ArnoldiArgs& a, double2* col, int m, bool breakdown) {
  tail_rotate(a.cs, a.sn, col, m);
  double2* Hc = a.H + (int64_t)(m - 1) * (a.maxit + 1);
  for (int j0 = 0; j0 <= m; j0 += kTailBlk) {
    double2 t[kTailBlk];
#pragma unroll
    for (int q = 0; q < kTailBlk; ++q)
      if (j0 + q <= m) t[q] = col[j0 + q];
#pragma unroll
    for (int q = 0; q < kTailBlk; ++q)
      if (j0 + q <= m) Hc[j0 + q] = t[q];
  }
  Hc[m - 1] = tail_finish(a, col, m, breakdown);
  Hc[m] = make_double2(0.0, 0.0);
}

// out-of-line copy for k_arnoldi_stream, whose hot loop needs the registers that the
// inlined rotation blocks (3 x kTailBlk complex) would otherwise claim
__device__ __noinline__ void arnoldi_tail_call(const ArnoldiArgs& a, double2* col, int m, bool breakdown) {
  arnoldi_tail(a, col, m, breakdown);
}

// MODE 1 (REG): unweighted, every CTA slice fits in registers (slice <=
// kArnThreads*kArnE): w stays in registers for the whole kernel and the basis
// slice of step s+2 is loaded into registers right after publishing step s,
// so its latency overlaps the barrier wait.
// Larger unweighted slices (cfg3/cfg4 on one GPU) use k_arnoldi_wide below.
// MODE 0: the general (weighted) path, w and D w streamed from memory.
template <int MODE>
__global__ void __launch_bounds__(kArnThreads, 1) k_arnoldi(ArnoldiArgs a) {
  constexpr bool REG = MODE == 1;
  extern __shared__ double2 col[];  // m+1, identical in every CTA
  __shared__ double2 red[68 + 2 * kMaxArnCTAs + 32];
  const int G = gridDim.x;
  const int m = *a.iter + 1;
  const int64_t n = a.n;
  const int64_t lo = (int64_t)blockIdx.x * a.slice;
  const int64_t hi = min(n, lo + a.slice);
  const int64_t len = hi > lo ? hi - lo : 0;
  const bool weighted = MODE == 0 && a.DV != nullptr;
  double2* w = a.w;
  double2* dw = weighted ? a.dw : a.w;
  const bool do_drift = a.check_drift && m >= 2;  // drift of V_{m-1} vs V_j, j < m-1
  const double2* dvm1 = (weighted ? a.DV : a.V) + (int64_t)(m - 1) * n;
  const int nsteps = 2 * m;
  // slots of publication k (k = s+1 for step s; k = 0 for the initial dot)
  auto slots = [&](int k) { return a.partials + (int64_t)k * G * a.pad; };
  for (int j = threadIdx.x; j <= m; j += blockDim.x) col[j] = make_double2(0.0, 0.0);
  // X_t = V_{t mod m} for t < nsteps; X_nsteps = w (the norm)
  auto xvec = [&](int t) { return a.V + (int64_t)(t % m) * n; };

  double2 W[kArnE], XN[kArnE], XNN[kArnE];
  double2* DM = col + (a.maxit + 1);  // drift vector slice in shared memory (REG path)
  if constexpr (REG) {
    if (threadIdx.x == 0)
      for (int t = 2; t < a.pf && t < nsteps; ++t) prefetch_l2(xvec(t) + lo, len * 16);
#pragma unroll
    for (int k = 0; k < kArnE; ++k) {
      const int64_t i = lo + threadIdx.x + (int64_t)k * kArnThreads;
      const bool ok = i < hi;
      W[k] = ok ? w[i] : make_double2(0.0, 0.0);
      XN[k] = ok ? a.V[i] : make_double2(0.0, 0.0);
      DM[threadIdx.x + k * kArnThreads] = (ok && do_drift) ? dvm1[i] : make_double2(0.0, 0.0);
    }
  } else if (threadIdx.x == 0) {
    prefetch_l2(xvec(1) + lo, len * 16);
  }
  // iteration -1: dot with X_0 (+ drift of X_0 if 0 < m-1)
  {
    double2 acc = make_double2(0.0, 0.0), dacc = make_double2(0.0, 0.0);
    if constexpr (REG) {
#pragma unroll
      for (int k = 0; k < kArnE; ++k) {
        acc = cdotc_acc(acc, XN[k], W[k]);
        if (do_drift) dacc = cdotc_acc(dacc, XN[k], DM[threadIdx.x + k * kArnThreads]);
      }
    } else {
      for (int64_t i = lo + threadIdx.x; i < hi; i += blockDim.x) {
        const double2 x = a.V[i];
        acc = cdotc_acc(acc, x, dw[i]);
        if (do_drift) dacc = cdotc_acc(dacc, x, dvm1[i]);
      }
    }
    block_sum_t0(acc, dacc, red + 68 + 2 * kMaxArnCTAs + 16);
    if (threadIdx.x == 0) publish(slots(0), a.pad, acc, dacc);
    if constexpr (REG) {
      const double2* x1 = xvec(1);
#pragma unroll
      for (int k = 0; k < kArnE; ++k) {
        const int64_t i = lo + threadIdx.x + (int64_t)k * kArnThreads;
        XNN[k] = i < hi ? x1[i] : make_double2(0.0, 0.0);
      }
    }
  }
  double dmax = 0.0;
  for (int s = 0; s < nsteps; ++s) {
    const int j = s % m;
    double2 h, d;
    // the drift slot carries data only in the first pass (s <= m-2)
    gather_sum(slots(s), G, a.pad, a.wg, red, h, d, do_drift && s < m - 1);
    if (do_drift && s < m - 1) dmax = fmax(dmax, hypot(d.x, d.y));  // drift term of X_s = V_s
    if (threadIdx.x == 0) {
      col[j] = cadd(col[j], h);
      if (!REG && s + 2 < nsteps) prefetch_l2(xvec(s + 2) + lo, len * 16);
      // REG: the register preload of X_{s+2} happens after this step's publish;
      // an L2 bulk prefetch kArnPf steps ahead makes that preload an L2 hit
      if (REG && s + a.pf < nsteps) prefetch_l2(xvec(s + a.pf) + lo, len * 16);
    }
    const bool last = (s + 1 == nsteps);
    const bool drift_next = do_drift && s + 1 < m - 1;
    double2 acc = make_double2(0.0, 0.0), dacc = make_double2(0.0, 0.0);
    if constexpr (REG) {
      // axpy with X_s (= XN), dot with X_{s+1} (= XNN, or w itself at the end)
#pragma unroll
      for (int k = 0; k < kArnE; ++k) {
        W[k] = caxmy(W[k], h, XN[k]);
        const double2 x = last ? W[k] : XNN[k];
        acc = cdotc_acc(acc, x, W[k]);
        if (drift_next) dacc = cdotc_acc(dacc, x, DM[threadIdx.x + k * kArnThreads]);
        XN[k] = XNN[k];
      }
    } else {
      const double2* vj = a.V + (int64_t)j * n;
      const double2* dvj = weighted ? a.DV + (int64_t)j * n : nullptr;
      const double2* vn = last ? w : xvec(s + 1);
      for (int64_t i = lo + threadIdx.x; i < hi; i += blockDim.x) {
        const double2 v = vj[i];
        const double2 wi = caxmy(w[i], h, v);
        w[i] = wi;
        double2 dwi = wi;
        if (weighted) {
          dwi = caxmy(dw[i], h, dvj[i]);
          dw[i] = dwi;
        }
        const double2 x = last ? wi : vn[i];
        acc = cdotc_acc(acc, x, dwi);
        if (drift_next) dacc = cdotc_acc(dacc, x, dvm1[i]);
      }
    }
    block_sum_t0(acc, dacc, red + 68 + 2 * kMaxArnCTAs + 16 * (s & 1));
    if (threadIdx.x == 0) publish(slots(s + 1), a.pad, acc, dacc);
    if constexpr (REG) {
      if (s + 2 < nsteps) {  // preload X_{s+2} while the other CTAs arrive
        const double2* x2 = xvec(s + 2);
#pragma unroll
        for (int k = 0; k < kArnE; ++k) {
          const int64_t i = lo + threadIdx.x + (int64_t)k * kArnThreads;
          XNN[k] = i < hi ? x2[i] : make_double2(0.0, 0.0);
        }
      }
    }
  }
  double2 hn2, dummy;
  gather_sum(slots(nsteps), G, a.pad, a.wg, red, hn2, dummy, false);
  const double hlast = sqrt(pymax0(hn2.x));
  __syncthreads();
  if (threadIdx.x == 0) col[m] = make_double2(hlast, 0.0);
  __syncthreads();
  // max |col_j| (breakdown test): strided over the CTA, then warp and CTA max
  // (exact, order-free; every CTA needs it to decide whether to write V_m)
  __shared__ double cmax_w[kArnThreads / 32];
  double cmax = 0.0;
  for (int j = threadIdx.x; j <= m; j += blockDim.x) cmax = fmax(cmax, hypot(col[j].x, col[j].y));
  cmax = warp_max(cmax);
  if ((threadIdx.x & 31) == 0) cmax_w[threadIdx.x >> 5] = cmax;
  __syncthreads();
#pragma unroll
  for (int k = 0; k < kArnThreads / 32; ++k) cmax = fmax(cmax, cmax_w[k]);
  const bool breakdown = hlast <= 1e-13 * cmax;
  if (!breakdown) {
    double2* vm = a.V + (int64_t)m * n;
    if constexpr (REG) {
#pragma unroll
      for (int k = 0; k < kArnE; ++k) {
        const int64_t i = lo + threadIdx.x + (int64_t)k * kArnThreads;
        if (i < hi) {
          const double2 q = make_double2(W[k].x / hlast, W[k].y / hlast);
          vm[i] = q;
          a.vin[i] = q;
        }
      }
    } else {
      double2* dvm = weighted ? a.DV + (int64_t)m * n : nullptr;
      for (int64_t i = lo + threadIdx.x; i < hi; i += blockDim.x) {
        const double2 wi = w[i];
        const double2 q = make_double2(wi.x / hlast, wi.y / hlast);
        vm[i] = q;
        a.vin[i] = q;
        if (weighted) {
          const double2 dd = dw[i];
          dvm[i] = make_double2(dd.x / hlast, dd.y / hlast);
        }
      }
    }
  }
  if (blockIdx.x != 0 || threadIdx.x != 0) return;
  if (do_drift) a.drift[m - 1] = dmax;
  arnoldi_tail(a, col, m, breakdown);
}

// Block sum of (a, b) over 32 warps delivered to thread 0: warp 0 reduces the 32 warp
// partials (fixed tree -> bitwise reproducible); one block barrier.  `sh` (64 double2) is
// double-buffered by the caller.
__device__ __forceinline__ void block_sum_t0_wide(double2& a, double2& b, double2* sh) {
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5, nw = blockDim.x >> 5;
  a = warp_sum2(a);
  b = warp_sum2(b);
  if (lane == 0) {
    sh[2 * wid] = a;
    sh[2 * wid + 1] = b;
  }
  __syncthreads();
  if (wid == 0) {
    const double2 zero = make_double2(0.0, 0.0);
    a = warp_sum2(lane < nw ? sh[2 * lane] : zero);
    b = warp_sum2(lane < nw ? sh[2 * lane + 1] : zero);
  }
}

// ------------------------------------------------------------------ WIDE
// Unweighted MGS2 for large slices with many warps per CTA: the streaming passes are issue- and latency-bound with 8 warps (ncu on the
// 8-warp kernels: 0.15 instructions per cycle per scheduler, ~13 cycles per dependent
// instruction), so the parallelism comes from warps, not from per-thread unrolling.
// w lives in shared memory as far as it fits (a.wcap elements), the rest in L2 with an
// evict_last policy; the axpy operand (second and last use of a basis chunk) is loaded
// with evict_first so the incoming vector replaces it and not the vector needed next.
#ifdef MDD_ARN_TRACE
// tools build only (tools/arn_trace.py): per-CTA timeline of one k_arnoldi_wide launch
__device__ unsigned long long g_arn_trace[(2 * 512 + 1) * kMaxArnCTAs * 2];
__device__ __forceinline__ unsigned long long gtimer() {
  unsigned long long t;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
  return t;
}
extern "C" int mdd_debug_arn_trace(unsigned long long* out, size_t count) {
  return (int)cudaMemcpyFromSymbol(out, g_arn_trace, count * sizeof(unsigned long long));
}
#define ARN_TRACE(step, which)                                                                  \
  if (threadIdx.x == 0 && (step) < 2 * 512 + 1)                                                  \
    g_arn_trace[((size_t)(step) * kMaxArnCTAs + blockIdx.x) * 2 + (which)] = gtimer();
#else
#define ARN_TRACE(step, which)
#endif
constexpr int kWideThreads = 1024;  // 32 warps x 64 registers
constexpr int kWideU = 2;          // elements per thread with their loads in flight together (1024 threads)
// loads in flight per thread: 1024 threads x 2 under the 64-register cap, 512 threads x 6 with 128
constexpr int wide_unroll(int threads) { return threads >= 1024 ? kWideU : 6; }

__device__ __forceinline__ double2 ld_hint(const double2* p, uint64_t policy) {
  double2 v;
  asm volatile("ld.global.L2::cache_hint.v2.f64 {%0, %1}, [%2], %3;" : "=d"(v.x), "=d"(v.y) : "l"(p), "l"(policy));
  return v;
}
__device__ __forceinline__ void st_hint2(double2* p, double2 v, uint64_t policy) {
  asm volatile("st.global.L2::cache_hint.v2.f64 [%0], {%1, %2}, %3;" ::"l"(p), "d"(v.x), "d"(v.y), "l"(policy)
               : "memory");
}
__device__ __forceinline__ uint64_t policy_evict_first() {
  uint64_t p;
  asm volatile("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(p));
  return p;
}
__device__ __forceinline__ uint64_t policy_evict_last() {
  uint64_t p;
  asm volatile("createpolicy.fractional.L2::evict_last.b64 %0, 1.0;" : "=l"(p));
  return p;
}

// Tensor memory as a scratchpad for the tail of w (E < 0).  The 256 KB of TMEM per SM are idle
// in this kernel (no tcgen05.mma), and together with the shared-memory head they hold cfg4's
// whole 381 KB w slice on the SM, which registers could not (the 512-thread register-tail
// variant spilled).  Layout: a double2 is four 32-bit columns; with the 32x32b access shape
// thread l of warp q reaches lane 32*(q%4)+l only, so the eight warps that share a lane
// quarter take 64 columns each: 16 elements per thread, 16,384 per CTA.  Every thread only
// ever reads back what it stored itself, so tcgen05.wait::st at the end of a sweep is the only
// ordering needed.
constexpr int kTmemElems = 16;  // double2 per thread
__device__ __forceinline__ void tmem_ld4(uint32_t taddr, uint32_t (&r)[4]) {
  asm volatile("tcgen05.ld.sync.aligned.32x32b.x4.b32 {%0, %1, %2, %3}, [%4];"
               : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3])
               : "r"(taddr));
}
// the loaded registers pass through the wait, so no use of them can be scheduled above it
__device__ __forceinline__ void tmem_wait_ld(uint32_t (&r)[4]) {
  asm volatile("tcgen05.wait::ld.sync.aligned;" : "+r"(r[0]), "+r"(r[1]), "+r"(r[2]), "+r"(r[3])::"memory");
}
__device__ __forceinline__ double2 tmem_unpack(const uint32_t (&r)[4]) {
  return make_double2(__hiloint2double((int)r[1], (int)r[0]), __hiloint2double((int)r[3], (int)r[2]));
}
__device__ __forceinline__ void tmem_st4(uint32_t taddr, double2 v) {
  asm volatile("tcgen05.st.sync.aligned.32x32b.x4.b32 [%0], {%1, %2, %3, %4};" ::"r"(taddr),
               "r"((uint32_t)__double2loint(v.x)), "r"((uint32_t)__double2hiint(v.x)),
               "r"((uint32_t)__double2loint(v.y)), "r"((uint32_t)__double2hiint(v.y))
               : "memory");
}
__device__ __forceinline__ void tmem_wait_st() { asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory"); }

// One sweep of the CTA's slice: w <- w - h A (axpy with X_t), acc = <B, w> (dot with X_{t+1}),
// dacc = <B, D> (drift partner, first pass only).  Flags are compile-time so the loop body is a
// handful of loads and DFMAs (the generic loop ran at ~150 instructions per element under the
// 64-register cap of a 1024-thread CTA and was issue-bound, ncu r02 profile); the slice is
// walked in two pieces, w in shared memory and w in L2, so there is no per-element tier test.
// Template parameters: T threads per CTA; E > 0: the tail of w (beyond shared memory) lives in
// registers, E elements per thread (T x E must cover it: cfg4's 23.8k-element slices = 13.6k in
// shared memory + 512 x 20 in registers), so w never touches the L2 and the L2 is left to the
// basis; E = 0: the tail stays in L2 under an evict_last policy (any slice length); E < 0: the
// tail lives in tensor memory (tm_ne trips of T elements, at most kTmemElems).
template <int T, int E, bool HASB, bool HASD, bool DOWN>
__device__ __forceinline__ void wide_sweep(const double2* __restrict__ A, const double2* __restrict__ B,
                                           const double2* __restrict__ D, double2* __restrict__ WS,
                                           double2* __restrict__ wg, double2 (&W)[E > 0 ? E : 1], int ws, int len,
                                           double2 h, uint64_t pol_first, uint64_t pol_last, double2& acc,
                                           double2& dacc, uint32_t tm_addr, int tm_ne, int pft) {
  constexpr int KU = wide_unroll(T);
  // in-sweep L2 prefetch of the dot operand (its first touch: DRAM latency), pft trips ahead of
  // the loads.  The sweep is a monotone walk over [0, len), upwards or downwards, in trips of
  // KU*T elements; thread 0 issues one bulk prefetch per trip.
  auto pf_at = [&](int x) {  // x: start (UP) or exclusive upper end (DOWN) of the current trip
    if (!HASB || pft <= 0 || threadIdx.x != 0) return;
    constexpr int c = KU * T;
    if (DOWN) {
      const int hi = x - pft * c;
      if (hi > 0) {
        const int lo = max(0, hi - c);
        prefetch_l2(B + lo, (int64_t)(hi - lo) * 16);
      }
    } else {
      const int lo = x + pft * c;
      if (lo < len) prefetch_l2(B + lo, (int64_t)min(c, len - lo) * 16);
    }
  };
  // piece 1: w in shared memory.  KU elements per thread are loaded before any is used: the
  // un-unrolled loop had one element's loads in flight per thread and ran at DRAM/L2 latency
  // per trip (ncu, profiles/r02_prof_wide_final_cfg4.ncu-rep: long scoreboard 36 warps per issue)
  auto piece1 = [&]() {
    for (int i0 = threadIdx.x; i0 < ws; i0 += KU * T) {
      pf_at(DOWN ? ws - (i0 - (int)threadIdx.x) : i0 - (int)threadIdx.x);
      double2 av[KU], bv[KU], dv[KU];
#pragma unroll
      for (int u = 0; u < KU; ++u) {
        // out-of-range lanes load a clamped (valid) element and are masked below: no branch
        // around the loads, so all KU go out back to back
        const int iu = min(i0 + u * T, ws - 1);
        const int i = DOWN ? ws - 1 - iu : iu;
        av[u] = ld_hint(A + i, pol_first);
        if (HASB) bv[u] = __ldcg(B + i);
        if (HASD) dv[u] = __ldcg(D + i);
      }
#pragma unroll
      for (int u = 0; u < KU; ++u) {
        const int iu = i0 + u * T;
        if (iu < ws) {
          const int i = DOWN ? ws - 1 - iu : iu;
          const double2 wi = caxmy(WS[i], h, av[u]);
          WS[i] = wi;
          const double2 x = HASB ? bv[u] : wi;
          acc = cdotc_acc(acc, x, wi);
          if (HASD) dacc = cdotc_acc(dacc, x, dv[u]);
        }
      }
    }
  };
  // piece 2: the tail of w
  auto piece2 = [&]() {
    if constexpr (E < 0) {
      // trip counts and the branches around tcgen05 instructions are CTA-uniform (.sync.aligned)
      for (int k0 = 0; k0 < tm_ne; k0 += KU) {
        pf_at(DOWN ? min(len, ws + (tm_ne - k0) * T) : ws + k0 * T);
        double2 av[KU], bv[KU], dv[KU];
        uint32_t r[KU][4];
#pragma unroll
        for (int u = 0; u < KU; ++u) {
          const int k = min(k0 + u, tm_ne - 1);
          const int e = DOWN ? tm_ne - 1 - k : k;
          const int i = min(ws + e * T + (int)threadIdx.x, len - 1);
          av[u] = ld_hint(A + i, pol_first);
          if (HASB) bv[u] = __ldcg(B + i);
          if (HASD) dv[u] = __ldcg(D + i);
          tmem_ld4(tm_addr + 4 * e, r[u]);
        }
#pragma unroll
        for (int u = 0; u < KU; ++u) tmem_wait_ld(r[u]);
#pragma unroll
        for (int u = 0; u < KU; ++u) {
          if (k0 + u < tm_ne) {
            const int e = DOWN ? tm_ne - 1 - (k0 + u) : k0 + u;
            const int i = ws + e * T + (int)threadIdx.x;
            const double2 wi = caxmy(tmem_unpack(r[u]), h, av[u]);
            tmem_st4(tm_addr + 4 * e, wi);
            if (i < len) {
              const double2 x = HASB ? bv[u] : wi;
              acc = cdotc_acc(acc, x, wi);
              if (HASD) dacc = cdotc_acc(dacc, x, dv[u]);
            }
          }
        }
      }
      tmem_wait_st();
    } else if constexpr (E > 0) {
#pragma unroll
      for (int e = 0; e < E; ++e) {
        const int i = ws + (int)threadIdx.x + e * T;
        if (i < len) {
          const double2 av = ld_hint(A + i, pol_first);
          double2 bv, dv;
          if (HASB) bv = __ldcg(B + i);
          if (HASD) dv = __ldcg(D + i);
          const double2 wi = caxmy(W[e], h, av);
          W[e] = wi;
          const double2 x = HASB ? bv : wi;
          acc = cdotc_acc(acc, x, wi);
          if (HASD) dacc = cdotc_acc(dacc, x, dv);
        }
      }
    } else {
      for (int i0 = ws + threadIdx.x; i0 < len; i0 += KU * T) {
        double2 av[KU], bv[KU], dv[KU], wv[KU];
#pragma unroll
        for (int u = 0; u < KU; ++u) {
          const int iu = min(i0 + u * T, len - 1);
          const int i = DOWN ? len - 1 - (iu - ws) : iu;
          av[u] = ld_hint(A + i, pol_first);
          wv[u] = ld_hint(wg + i, pol_last);
          if (HASB) bv[u] = __ldcg(B + i);
          if (HASD) dv[u] = __ldcg(D + i);
        }
#pragma unroll
        for (int u = 0; u < KU; ++u) {
          const int iu = i0 + u * T;
          if (iu < len) {
            const int i = DOWN ? len - 1 - (iu - ws) : iu;
            const double2 wi = caxmy(wv[u], h, av[u]);
            st_hint2(wg + i, wi, pol_last);
            const double2 x = HASB ? bv[u] : wi;
            acc = cdotc_acc(acc, x, wi);
            if (HASD) dacc = cdotc_acc(dacc, x, dv[u]);
          }
        }
      }
    }
  };
  if (DOWN) {  // the top of the slice (fetched last by the upward pass before) first
    piece2();
    piece1();
  } else {
    piece1();
    piece2();
  }
}

template <int T, int E>
__global__ void __launch_bounds__(T, 1) k_arnoldi_wide(ArnoldiArgs a) {
  extern __shared__ double2 col[];  // m+1, identical in every CTA; then the w head
  __shared__ double2 red[68 + 2 * kMaxArnCTAs + 2 * 64];
  __shared__ double cmax_w[T / 32];
  const int G = gridDim.x;
  const int m = *a.iter + 1;
  const int64_t n = a.n;
  const int64_t lo = (int64_t)blockIdx.x * a.slice;
  const int64_t hi = min(n, lo + a.slice);
  const int len = hi > lo ? (int)(hi - lo) : 0;
  const bool do_drift = a.check_drift && m >= 2;
  const double2* dvm1 = a.V + (int64_t)(m - 1) * n + lo;
  const int nsteps = 2 * m;
  auto slots = [&](int k) { return a.partials + (int64_t)k * G * a.pad; };
  auto xvec = [&](int t) { return a.V + (int64_t)(t % m) * n + lo; };
  double2* WS = col + (a.maxit + 1);
  const int ws = (int)min((int64_t)len, a.wcap);
  double2* wg = a.w + lo;
  double2 W[E > 0 ? E : 1];
  // E < 0: the tail of w in tensor memory (all 512 columns; one CTA per SM, nobody else uses TMEM)
  __shared__ uint32_t tm_base_s;
  uint32_t tm_addr = 0;
  int tm_ne = 0;
  if constexpr (E < 0) {
    if (threadIdx.x < 32) {
      asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(
                       (uint32_t)__cvta_generic_to_shared(&tm_base_s)),
                   "r"(512u)
                   : "memory");
      asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;" ::: "memory");
    }
    asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
    __syncthreads();
    asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
    const uint32_t wq = threadIdx.x >> 5;
    tm_addr = tm_base_s + (((wq & 3u) * 32u) << 16) + (wq >> 2) * (4u * kTmemElems * (1024 / T));
    tm_ne = len > ws ? (len - ws + T - 1) / T : 0;  // <= kTmemElems (checked by the host)
  }
  const uint64_t pol_first = policy_evict_first(), pol_last = policy_evict_last();  // (evict_normal for the w tail: cfg4 Arnoldi 1265 -> 1290 ms)
  for (int j = threadIdx.x; j <= m; j += T) col[j] = make_double2(0.0, 0.0);
  const double2 zero = make_double2(0.0, 0.0);
  double dmax = 0.0;
#ifdef MDD_ARN_TRACE
  if (threadIdx.x == 0) {
    unsigned smid;
    asm volatile("mov.u32 %0, %%smid;" : "=r"(smid));
    g_arn_trace[((size_t)(2 * 512) * kMaxArnCTAs + blockIdx.x) * 2] = smid;
    g_arn_trace[((size_t)(2 * 512) * kMaxArnCTAs + blockIdx.x) * 2 + 1] = gtimer();
  }
#endif
  // pass -1: load w into its tiers, dot with X_0 (+ drift partner)
  {
    const double2* B = xvec(0);
    double2 acc = zero, dacc = zero;
    for (int i = threadIdx.x; i < ws; i += T) {
      const double2 wi = __ldcg(wg + i);
      WS[i] = wi;
      const double2 x = __ldcg(B + i);
      acc = cdotc_acc(acc, x, wi);
      if (do_drift) dacc = cdotc_acc(dacc, x, __ldcg(dvm1 + i));
    }
    if constexpr (E < 0) {
      for (int e = 0; e < tm_ne; ++e) {
        const int i = ws + (int)threadIdx.x + e * T;
        double2 wi = zero;
        if (i < len) {
          wi = __ldcg(wg + i);
          const double2 x = __ldcg(B + i);
          acc = cdotc_acc(acc, x, wi);
          if (do_drift) dacc = cdotc_acc(dacc, x, __ldcg(dvm1 + i));
        }
        tmem_st4(tm_addr + 4 * e, wi);
      }
      tmem_wait_st();
    } else if constexpr (E > 0) {
#pragma unroll
      for (int e = 0; e < E; ++e) {
        const int i = ws + (int)threadIdx.x + e * T;
        W[e] = zero;
        if (i < len) {
          const double2 wi = __ldcg(wg + i);
          W[e] = wi;
          const double2 x = __ldcg(B + i);
          acc = cdotc_acc(acc, x, wi);
          if (do_drift) dacc = cdotc_acc(dacc, x, __ldcg(dvm1 + i));
        }
      }
    } else {
      for (int i = ws + threadIdx.x; i < len; i += T) {
        const double2 wi = __ldcg(wg + i);
        const double2 x = __ldcg(B + i);
        acc = cdotc_acc(acc, x, wi);
        if (do_drift) dacc = cdotc_acc(dacc, x, __ldcg(dvm1 + i));
      }
    }
    block_sum_t0_wide(acc, dacc, red + 68 + 2 * kMaxArnCTAs + 64);
    if (threadIdx.x == 0) publish(slots(0), a.pad, acc, dacc);
  }
  for (int t = 0; t < nsteps; ++t) {
    const bool hasB = t + 1 < nsteps, hasD = do_drift && t + 1 < m - 1;
    double2 h, d;
    gather_sum(slots(t), G, a.pad, false, red, h, d, do_drift && t < m - 1);
    ARN_TRACE(t, 0)
    if (do_drift && t < m - 1) dmax = fmax(dmax, hypot(d.x, d.y));
    if (threadIdx.x == 0) col[t % m] = cadd(col[t % m], h);
    const double2* A = xvec(t);
    const double2* B = hasB ? xvec(t + 1) : nullptr;
    double2 acc = zero, dacc = zero;
    // odd passes sweep the slice downwards when the vectors exceed what the L2 retains: the
    // chunks of X_{t+1} fetched last in pass t are then the first ones pass t+1 needs again
    const bool down = a.zigzag && (t & 1);
#define MDD_SWEEP(HB, HD, DN) \
  wide_sweep<T, E, HB, HD, DN>(A, B, dvm1, WS, wg, W, ws, len, h, pol_first, pol_last, acc, dacc, tm_addr, tm_ne, a.pf_trips)
    if (!hasB) MDD_SWEEP(false, false, false);
    else if (hasD) {
      if (down) MDD_SWEEP(true, true, true);
      else MDD_SWEEP(true, true, false);
    } else {
      if (down) MDD_SWEEP(true, false, true);
      else MDD_SWEEP(true, false, false);
    }
#undef MDD_SWEEP
    block_sum_t0_wide(acc, dacc, red + 68 + 2 * kMaxArnCTAs + 64 * (t & 1));
    ARN_TRACE(t, 1)
    if (threadIdx.x == 0) {
      publish(slots(t + 1), a.pad, acc, dacc);
      // DRAM idles while the CTAs exchange their partial sums: pull the head of the slice the
      // next sweep dots with (X_{t+2}, its first touch in this iteration) into L2 meanwhile.
      // a.pf_bytes caps it, so that at cfg4 (56 MB vectors) the prefetch does not evict X_{t+1}
      // before its second use
      if (t + 2 < nsteps) {
        const int64_t pb = min((int64_t)len * 16, a.pf_bytes);
        // pass t+1 starts at the top of the slice if it sweeps downwards
        const int64_t start = (a.zigzag && ((t + 1) & 1)) ? (int64_t)len - pb / 16 : 0;
        prefetch_l2(xvec(t + 2) + start, pb);
      }
    }
  }
  double2 hn2, dummy;
  gather_sum(slots(nsteps), G, a.pad, false, red, hn2, dummy, false);
  const double hlast = sqrt(pymax0(hn2.x));
  __syncthreads();
  if (threadIdx.x == 0) col[m] = make_double2(hlast, 0.0);
  __syncthreads();
  double cmax = 0.0;
  for (int j = threadIdx.x; j <= m; j += T) cmax = fmax(cmax, hypot(col[j].x, col[j].y));
  cmax = warp_max(cmax);
  if ((threadIdx.x & 31) == 0) cmax_w[threadIdx.x >> 5] = cmax;
  __syncthreads();
#pragma unroll
  for (int k = 0; k < T / 32; ++k) cmax = fmax(cmax, cmax_w[k]);
  const bool breakdown = hlast <= 1e-13 * cmax;
  if (!breakdown) {
    double2* vm = a.V + (int64_t)m * n + lo;
    double2* vin = a.vin + lo;
    for (int i = threadIdx.x; i < (E != 0 ? ws : len); i += T) {
      // the tail's last read demotes its L2 lines (evict_first): left as evict_last they sit in
      // the L2 through the next preconditioner apply (measured: 65 ms per cfg4 solve)
      const double2 wi = i < ws ? WS[i] : ld_hint(wg + i, pol_first);
      const double2 q = make_double2(wi.x / hlast, wi.y / hlast);
      vm[i] = q;
      vin[i] = q;
    }
    if constexpr (E < 0) {
      for (int e = 0; e < tm_ne; ++e) {
        const int i = ws + (int)threadIdx.x + e * T;
        uint32_t r[4];
        tmem_ld4(tm_addr + 4 * e, r);
        tmem_wait_ld(r);
        if (i < len) {
          const double2 wi = tmem_unpack(r);
          const double2 q = make_double2(wi.x / hlast, wi.y / hlast);
          vm[i] = q;
          vin[i] = q;
        }
      }
    } else if constexpr (E > 0) {
#pragma unroll
      for (int e = 0; e < E; ++e) {
        const int i = ws + (int)threadIdx.x + e * T;
        if (i < len) {
          const double2 q = make_double2(W[e].x / hlast, W[e].y / hlast);
          vm[i] = q;
          vin[i] = q;
        }
      }
    }
  }
  if constexpr (E < 0) {
    asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
    __syncthreads();
    if (threadIdx.x < 32)
      asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tm_base_s), "r"(512u) : "memory");
  }
  if (blockIdx.x != 0 || threadIdx.x != 0) return;
  if (do_drift) a.drift[m - 1] = dmax;
  arnoldi_tail_call(a, col, m, breakdown);
}

// ------------------------------------------------------------ drift panels
// Orthogonality drift (krylov.py:152-160: max_j |<V_j, V_k>| for every accepted V_k) for the
// large-slice path.  Riding along in the MGS sweeps costs one extra n-vector of DRAM traffic
// per first-pass step there (V_{m-1} is re-read for every dot, and the L2 cannot keep it:
// cfg4 1415 vs 1163 ms per solve).  Instead the drift of kDriftP consecutive new vectors is
// computed together, GEMM-style: every CTA walks its row slab in tiles of kDriftR rows, stages
// the tile of ALL older vectors in shared memory once and accumulates the kDriftP x J Gram
// block in registers (thread j owns column j), so the basis is read once per kDriftP
// iterations instead of once per iteration.  Partial blocks are summed over the CTAs in fixed
// order by k_drift_finish.
constexpr int kDriftP = 8;
constexpr int kDriftR = 16;  // rows per tile, two tiles in shared memory
constexpr int kDriftThreads = 256;  // >= maxit: one thread per older vector

struct DriftArgs {
  int64_t n;
  const double2* V;
  const int* iter;      // in-loop: panel [m-P+1, m] when m % P == 0 and no breakdown; nullptr: explicit range
  const int* dstatus;
  int k0, k1;           // explicit range (iter == nullptr), inclusive
  double2* partial;     // gridDim.x x kDriftP x kDriftThreads
  double* drift;        // out: drift[k]
  int ncta;
  int stage_elems;      // double2 per pipeline stage of k_drift_panel (two stages in shared memory)
};

__device__ __forceinline__ bool drift_range(const DriftArgs& a, int& k0, int& k1) {
  if (a.iter) {
    const int m = *a.iter;
    if (m < 1 || m % kDriftP != 0 || a.dstatus[1]) return false;
    k0 = m - kDriftP + 1;
    k1 = m;
  } else {
    k0 = a.k0;
    k1 = a.k1;
  }
  return k1 >= k0 && k1 >= 1;
}

__device__ __forceinline__ void drift_cp16(double2* dst, const double2* src, bool valid) {
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16, %2;" ::"r"((unsigned)__cvta_generic_to_shared(dst)), "l"(src),
               "r"(valid ? 16 : 0)
               : "memory");
}

// Row tiles go through a two-stage cp.async ring: the next tile's loads are in flight while
// thread j accumulates its column of the current one.  The tile height adapts to the panel:
// a stage holds R x (J + P) elements, so early panels (few older vectors) take hundreds of rows
// per tile and late ones kDriftR.  (Round 2's single-buffered 32-row tiles paid a DRAM round
// trip and two barriers per tile whatever J was: 2.1 ms for the first panel of cfg4, which reads
// 0.5 GB, 105 ms per solve.)  Rows are accumulated in the same order as before: the drift values
// are bitwise unchanged.
__global__ void __launch_bounds__(kDriftThreads) k_drift_panel(DriftArgs a) {
  int k0, k1;
  if (!drift_range(a, k0, k1)) return;
  k0 = max(k0, 1);
  const int J = k1;                 // older vectors V_0 .. V_{k1-1}
  const int np = k1 - k0 + 1;       // new vectors V_{k0} .. V_{k1}
  const int Jp = J | 1;             // odd row stride: conflict-free transposed stores
  extern __shared__ double2 sm[];
  const size_t stage_elems = (size_t)a.stage_elems;
  const int R = max(kDriftR, min(512, (a.stage_elems / (Jp + kDriftP)) & ~15));  // rows per tile
  const int64_t slab = (a.n + gridDim.x - 1) / gridDim.x;
  const int64_t lo = (int64_t)blockIdx.x * slab, hi = min(a.n, lo + slab);
  double2 acc[kDriftP];
#pragma unroll
  for (int k = 0; k < kDriftP; ++k) acc[k] = make_double2(0.0, 0.0);
  // stage: element e = (vector j, row r), r fastest (coalesced along the rows of one vector);
  // rows beyond the slab are zero-filled
  auto stage = [&](int st, int64_t r0) {
    double2* As = sm + st * stage_elems;        // R x Jp
    double2* Bs = As + (size_t)R * Jp;          // R x kDriftP
    const int nr = (int)min((int64_t)R, hi - r0);
    for (int e = threadIdx.x; e < (J + np) * R; e += kDriftThreads) {
      const int j = e / R, r = e % R;
      const bool ok = r < nr;
      const double2* src = a.V + (int64_t)(j < J ? j : k0 + (j - J)) * a.n + r0 + (ok ? r : 0);
      double2* dst = j < J ? As + (size_t)r * Jp + j : Bs + r * kDriftP + (j - J);
      drift_cp16(dst, src, ok);
    }
    asm volatile("cp.async.commit_group;" ::: "memory");
  };
  if (lo < hi) stage(0, lo);
  int it = 0;
  for (int64_t r0 = lo; r0 < hi; r0 += R, ++it) {
    if (r0 + R < hi) {
      stage((it + 1) & 1, r0 + R);
      asm volatile("cp.async.wait_group 1;" ::: "memory");
    } else {
      asm volatile("cp.async.wait_group 0;" ::: "memory");
    }
    __syncthreads();
    const double2* As = sm + (it & 1) * stage_elems;
    const double2* Bs = As + (size_t)R * Jp;
    if ((int)threadIdx.x < J) {
#pragma unroll 4
      for (int r = 0; r < R; ++r) {
        const double2 x = As[(size_t)r * Jp + threadIdx.x];
#pragma unroll
        for (int k = 0; k < kDriftP; ++k) acc[k] = cdotc_acc(acc[k], x, Bs[r * kDriftP + k]);
      }
    }
    __syncthreads();  // the stage is refilled by the next iteration's loads
  }
  double2* out = a.partial + (size_t)blockIdx.x * kDriftP * kDriftThreads;
#pragma unroll
  for (int k = 0; k < kDriftP; ++k) out[k * kDriftThreads + threadIdx.x] = acc[k];
}

// drift[k] = max_{j < k} | sum over CTAs (fixed order) of the partial <V_j, V_k> |
__global__ void __launch_bounds__(kDriftThreads) k_drift_finish(DriftArgs a) {
  int k0, k1;
  if (!drift_range(a, k0, k1)) return;
  k0 = max(k0, 1);
  __shared__ double wmax[kDriftThreads / 32];
  const int k = k0 + blockIdx.x;
  if (k > k1) return;
  const int j = threadIdx.x;
  double v = 0.0;
  if (j < k) {
    double2 sacc = make_double2(0.0, 0.0);
    for (int c = 0; c < a.ncta; ++c)
      sacc = cadd(sacc, a.partial[((size_t)c * kDriftP + (k - k0)) * kDriftThreads + j]);
    v = hypot(sacc.x, sacc.y);
  }
  v = warp_max(v);
  if ((threadIdx.x & 31) == 0) wmax[threadIdx.x >> 5] = v;
  __syncthreads();
  if (threadIdx.x == 0) {
    for (int w = 1; w < kDriftThreads / 32; ++w) v = fmax(v, wmax[w]);
    a.drift[k] = v;
  }
}

// drift of the final basis vector V_m: |vdot(V_j, DV_m)| for j < m (one CTA per j)
__global__ void k_final_drift(int64_t n, int m, const double2* V, const double2* DVm, double* out) {
  __shared__ double2 red[32];
  const int j = blockIdx.x;
  const double2* vj = V + (int64_t)j * n;
  double2 acc = make_double2(0.0, 0.0);
  for (int64_t i = threadIdx.x; i < n; i += blockDim.x) {
    const double2 x = vj[i], y = DVm[i];
    acc.x += x.x * y.x + x.y * y.y;
    acc.y += x.x * y.y - x.y * y.x;
  }
  acc = block_sum2(acc, red);
  if (threadIdx.x == 0) out[j] = hypot(acc.x, acc.y);
}

__global__ void k_max_into(const double* v, int m, double* out) {
  if (threadIdx.x || blockIdx.x) return;
  double d = 0.0;
  for (int j = 0; j < m; ++j) d = fmax(d, v[j]);
  *out = d;
}

// phase 0: beta = sqrt(Re vdot(r, dr)), g[0]=beta, hist[0]=1 ; phase 1: V0 = r/beta (+DV0, vin)
__global__ void k_init_basis(int64_t n, const double2* r, const double2* dr, double2* V0,
                             double2* DV0, double2* vin, double* beta_out, double2* g, double* hist,
                             int phase) {
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
    const double2 q = make_double2(x.x / beta, x.y / beta);
    V0[i] = q;
    vin[i] = q;
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
// one warp: each row's dot is split over the lanes (fixed lane-strided order +
// shuffle tree), y kept in shared memory; m sequential rows of one L2 round trip
// each instead of m^2/2 dependent single-thread loads (2.7 ms -> ~0.1 ms at m = 200)
__global__ void k_backsub(int m, int maxit, const double2* H, const double2* g, double2* y) {
  extern __shared__ double2 ys[];
  if (blockIdx.x != 0 || threadIdx.x >= 32) return;
  const int ld = maxit + 1, lane = threadIdx.x;
  for (int i = m - 1; i >= 0; --i) {
    double2 s = make_double2(0.0, 0.0);
    for (int j = i + 1 + lane; j < m; j += 32) s = cadd(s, cmul(H[(int64_t)j * ld + i], ys[j]));
    s = warp_sum2(s);
    if (lane == 0) ys[i] = cdiv(csub(g[i], s), H[(int64_t)i * ld + i]);
    __syncwarp();
  }
  for (int i = lane; i < m; i += 32) y[i] = ys[i];
}

// y in dynamic shared memory: 16 B per iteration, beyond 48 KB needs the opt-in attribute
static void launch_backsub(mdd_ctx* ctx, int m, int maxit, const double2* H, const double2* g, double2* y,
                           cudaStream_t s) {
  const size_t bytes = sizeof(double2) * (size_t)std::max(1, m);
  if (bytes > 227 * 1024) fail(MDD_EINVAL, "gmres: more than 14528 iterations are not supported");
  if (bytes > 48 * 1024)
    CK(cudaFuncSetAttribute(k_backsub, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)bytes));
  k_backsub<<<1, 32, bytes, s>>>(m, maxit, H, g, y);
  CK_LAUNCH(ctx);
}

__global__ void k_axpy_out(int64_t n, const double2* x0, const double2* u, double2* x) {
  for (int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; e < n;
       e += (int64_t)gridDim.x * blockDim.x)
    x[e] = x0 ? cadd(x0[e], u[e]) : u[e];
}

// ------------------------------------------------------------ CGS2 path
// Classical Gram-Schmidt with one reorthogonalisation pass: per iteration two
// block projections h = V^H w, w -= V h (each one sweep over the basis) and a
// norm, i.e. three reductions whatever m is.  This is the Krylov loop of the
// sharded multi-GPU solve (vectors split in row blocks, each reduction one
// small ncclAllReduce); on one GPU it is available through
// KrylovConfig.orthogonalization = "cgs2".  The default stays MGS2 as in the
// reference (krylov.py:137-143).  Partial sums are combined in a fixed order.

// partial[k*G + cta] = sum over the CTA's chunk of conj(X_k) y_k, where job k < nv
// is (V_k, y) and job nv + j (j < nd) is (V_j, d); one warp per job at a time
__global__ void __launch_bounds__(256) k_mdot(int64_t nl, int64_t ldv, const double2* __restrict__ V, int nv,
                                              const double2* __restrict__ y, const double2* __restrict__ d,
                                              int nd, double2* __restrict__ partial) {
  const int G = gridDim.x;
  const int64_t chunk = (nl + G - 1) / G;
  const int64_t i0 = (int64_t)blockIdx.x * chunk, i1 = min(nl, i0 + chunk);
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  for (int k = warp; k < nv + nd; k += blockDim.x >> 5) {
    const double2* x = V + (int64_t)(k < nv ? k : k - nv) * ldv;
    const double2* yy = k < nv ? y : d;
    double2 a0 = make_double2(0.0, 0.0), a1 = a0, a2 = a0, a3 = a0;
    int64_t i = i0 + lane;
    for (; i + 96 < i1; i += 128) {
      a0 = cdotc_acc(a0, __ldcs(x + i), __ldg(yy + i));
      a1 = cdotc_acc(a1, __ldcs(x + i + 32), __ldg(yy + i + 32));
      a2 = cdotc_acc(a2, __ldcs(x + i + 64), __ldg(yy + i + 64));
      a3 = cdotc_acc(a3, __ldcs(x + i + 96), __ldg(yy + i + 96));
    }
    for (; i < i1; i += 32) a0 = cdotc_acc(a0, __ldcs(x + i), __ldg(yy + i));
    double2 acc = warp_sum2(cadd(cadd(a0, a1), cadd(a2, a3)));
    if (lane == 0) partial[(int64_t)k * G + blockIdx.x] = acc;
  }
}

// out[k] = sum_c partial[k*G + c] in CTA order; one warp per k
__global__ void k_colsum(const double2* __restrict__ partial, int G, int nk, double2* __restrict__ out) {
  const int k = blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5), lane = threadIdx.x & 31;
  if (k >= nk) return;
  double2 acc = make_double2(0.0, 0.0);
  for (int c = lane; c < G; c += 32) acc = cadd(acc, partial[(int64_t)k * G + c]);
  acc = warp_sum2(acc);
  if (lane == 0) out[k] = acc;
}

// w[i] -= sum_{j < nv} h[j] V_j[i]
__global__ void __launch_bounds__(256) k_maxpy(int64_t nl, int64_t ldv, const double2* __restrict__ V, int nv,
                                               const double2* __restrict__ h, double2* __restrict__ w) {
  extern __shared__ double2 hs[];
  for (int j = threadIdx.x; j < nv; j += blockDim.x) hs[j] = h[j];
  __syncthreads();
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < nl; i += (int64_t)gridDim.x * blockDim.x) {
    double2 wi = w[i];
    int j = 0;
    for (; j + 3 < nv; j += 4) {
      const double2 v0 = __ldcs(V + (int64_t)j * ldv + i), v1 = __ldcs(V + (int64_t)(j + 1) * ldv + i);
      const double2 v2 = __ldcs(V + (int64_t)(j + 2) * ldv + i), v3 = __ldcs(V + (int64_t)(j + 3) * ldv + i);
      wi = caxmy(wi, hs[j], v0);
      wi = caxmy(wi, hs[j + 1], v1);
      wi = caxmy(wi, hs[j + 2], v2);
      wi = caxmy(wi, hs[j + 3], v3);
    }
    for (; j < nv; ++j) wi = caxmy(wi, hs[j], __ldcs(V + (int64_t)j * ldv + i));
    w[i] = wi;
  }
}

// Row-tiled CGS2 passes: three sweeps over the basis per iteration instead of
// four.  A CTA stages a tile of kCgsRows rows of all nv basis vectors (and of
// w) in shared memory with cp.async, two tiles in flight, so each basis
// element is read from HBM once per pass:
//   kProj    : partial h_j = conj(V_j) . w      (+ drift conj(V_j) . V_{nv-1}, j < nd)
//   kSubProj : w -= V h;  partial h_j = conj(V_j) . w   (the update and the
//              reorthogonalisation dots share one read of the tile)
//   kSubNorm : w -= V h;  partial |w|^2
// Partials land in partial[k*G + cta] (k-major, CTA order) for k_colsum; the
// per-row and per-CTA summation orders are fixed, so reruns are bitwise
// identical.  Rows of the tail tile beyond nl are zero-filled.
constexpr int kCgsThreads = 256;
constexpr int kCgsMaxNv = 2 * kCgsThreads;  // dots: thread t owns basis vectors t and t + 256
enum CgsMode { kProj = 0, kSubProj = 1, kSubNorm = 2 };

// tile of R rows: nv vectors at a padded pitch of R+1 double2 (conflict-free column reads) + w
__host__ __device__ constexpr size_t cgs_tile_elems(int nv, int R) { return (size_t)nv * (R + 1) + R; }
static size_t cgs_smem_bytes(int nv, int R, int ns) {
  return sizeof(double2) * (ns * cgs_tile_elems(nv, R) + (size_t)kCgsThreads + 64);
}

__device__ __forceinline__ uint32_t smem_u32_g(const void* p) {
  return (uint32_t)__cvta_generic_to_shared(p);
}
__device__ __forceinline__ void cp_async16(void* dst, const void* src, bool valid) {
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16, %2;" ::"r"(smem_u32_g(dst)), "l"(src),
               "r"(valid ? 16 : 0)
               : "memory");
}

template <int MODE, int R>
__global__ void __launch_bounds__(kCgsThreads) k_cgs_tile(int64_t nl, int64_t ldv, const double2* __restrict__ V,
                                                          int nv, const double2* __restrict__ h,
                                                          double2* __restrict__ w, int nd,
                                                          double2* __restrict__ partial, int ns) {
  extern __shared__ double2 sm[];
  const int tid = threadIdx.x, G = gridDim.x;
  const size_t TE = cgs_tile_elems(nv, R);
  constexpr int kCgsRows = R, kCgsPitch = R + 1;
  double2* red = sm + ns * TE;  // [kCgsThreads/kCgsRows][kCgsRows]
  const int64_t ntiles = (nl + kCgsRows - 1) / kCgsRows;
  auto issue = [&](int64_t tile, int buf) {
    double2* Vs = sm + buf * TE;
    double2* ws = Vs + (size_t)nv * kCgsPitch;
    const int64_t row0 = tile * kCgsRows;
    const int total = nv * kCgsRows;
    for (int e = tid; e < total; e += kCgsThreads) {
      const int j = e / kCgsRows, r = e % kCgsRows;
      const int64_t i = row0 + r;
      const bool ok = i < nl;
      cp_async16(Vs + j * kCgsPitch + r, V + (int64_t)j * ldv + (ok ? i : 0), ok);
    }
    if (tid < kCgsRows) {
      const int64_t i = row0 + tid;
      cp_async16(ws + tid, w + (i < nl ? i : 0), i < nl);
    }
    asm volatile("cp.async.commit_group;" ::: "memory");
  };
  double2 acc0 = make_double2(0.0, 0.0), acc1 = acc0, dacc0 = acc0, dacc1 = acc0, nacc = acc0;
  const int r = tid % kCgsRows, grp = tid / kCgsRows;
  constexpr int NG = kCgsThreads / kCgsRows;
  // ns-stage ring (ns = 2 or 3): one commit group per tile slot, empty past the end
  int64_t tile = blockIdx.x;
  for (int q = 0; q < ns - 1; ++q) {
    if (tile + (int64_t)q * G < ntiles) issue(tile + (int64_t)q * G, q);
    else asm volatile("cp.async.commit_group;" ::: "memory");
  }
  for (int it = 0; tile < ntiles; ++it, tile += G) {
    const int buf = it % ns;
    const int64_t tn = tile + (int64_t)(ns - 1) * G;
    if (tn < ntiles) issue(tn, (it + ns - 1) % ns);
    else asm volatile("cp.async.commit_group;" ::: "memory");
    if (ns == 3) asm volatile("cp.async.wait_group 2;" ::: "memory");
    else asm volatile("cp.async.wait_group 1;" ::: "memory");
    __syncthreads();
    double2* Vs = sm + buf * TE;
    double2* ws = Vs + (size_t)nv * kCgsPitch;
    if (MODE != kProj) {
      // w_r -= sum_j h_j V_j[r]: NG groups of kCgsRows threads, combined in group order
      double2 s = make_double2(0.0, 0.0);
      for (int j = grp; j < nv; j += NG) s = cfma(__ldg(h + j), Vs[j * kCgsPitch + r], s);
      red[grp * kCgsRows + r] = s;
      __syncthreads();
      if (tid < kCgsRows) {
        double2 t = red[tid];
#pragma unroll
        for (int g = 1; g < NG; ++g) t = cadd(t, red[g * kCgsRows + tid]);
        const double2 wn = csub(ws[tid], t);
        ws[tid] = wn;
        const int64_t i = tile * kCgsRows + tid;
        if (i < nl) w[i] = wn;
        if (MODE == kSubNorm) nacc.x += wn.x * wn.x + wn.y * wn.y;
      }
      __syncthreads();
    }
    if (MODE != kSubNorm) {
      // h_j partials over the tile's rows in row order; thread t owns j = t, t + 256
      for (int q = 0; q < 2; ++q) {
        const int j = tid + q * kCgsThreads;
        if (j >= nv) break;
        const double2* vj = Vs + j * kCgsPitch;
        double2 a = q ? acc1 : acc0;
#pragma unroll
        for (int rr = 0; rr < kCgsRows; ++rr) a = cdotc_acc(a, vj[rr], ws[rr]);
        if (q) acc1 = a; else acc0 = a;
        if (MODE == kProj && j < nd) {
          const double2* vm = Vs + (nv - 1) * kCgsPitch;
          double2 d = q ? dacc1 : dacc0;
#pragma unroll
          for (int rr = 0; rr < kCgsRows; ++rr) d = cdotc_acc(d, vj[rr], vm[rr]);
          if (q) dacc1 = d; else dacc0 = d;
        }
      }
    }
    __syncthreads();  // buffer `buf` is refilled by the next iteration's issue
  }
  if constexpr (MODE == kSubNorm) {
    const double2 t = block_sum2(nacc, red);
    if (tid == 0) partial[blockIdx.x] = t;
  } else {
    for (int q = 0; q < 2; ++q) {
      const int j = tid + q * kCgsThreads;
      if (j < nv) partial[(int64_t)j * G + blockIdx.x] = q ? acc1 : acc0;
      if (MODE == kProj && j < nd) partial[(int64_t)(nv + j) * G + blockIdx.x] = q ? dacc1 : dacc0;
    }
  }
}

// Column m-1 of H from the two projections and the norm, drift of V_{m-1},
// breakdown test, Givens update.  scal[0] = hlast, scal[1] = 1 on breakdown
// (k_vscale then leaves V_m alone).
constexpr int kTailThreads = 256;
__device__ __forceinline__ double block_max(double v, double* sh) {
  v = warp_max(v);
  if ((threadIdx.x & 31) == 0) sh[threadIdx.x >> 5] = v;
  __syncthreads();
  if (threadIdx.x < 32) {
    double r = threadIdx.x < (blockDim.x >> 5) ? sh[threadIdx.x] : 0.0;
    r = warp_max(r);
    if (threadIdx.x == 0) sh[32] = r;
  }
  __syncthreads();
  return sh[32];
}
// One CTA of kTailThreads: the column sums and maxima in parallel; col, cs
// and sn staged in shared memory (cap = entries that fit, else global), so
// thread 0 runs the Givens chain off shared memory; H column copied by all.
__global__ void __launch_bounds__(kTailThreads) k_cgs_tail(ArnoldiArgs a, const double2* h1, const double2* h2,
                                                           const double2* nrm, const double2* dr, int do_drift,
                                                           double2* colg, double* scal, int cap) {
  extern __shared__ double2 tsm[];
  __shared__ double shm[40];
  __shared__ double2 hmm_s;
  if (blockIdx.x) return;
  // the host loop runs one iteration ahead of its convergence check: an
  // iteration enqueued after convergence must leave the converged state alone
  if (a.dstatus[0]) return;
  const int m = *a.iter + 1;
  const bool staged = m + 1 <= cap;
  double2* col = staged ? tsm : colg;
  double2* css = staged ? tsm + cap : a.cs;
  double2* sns = staged ? tsm + 2 * cap : a.sn;
  const double hlast = sqrt(pymax0(nrm[0].x));
  double cm = 0.0, dm = 0.0;
  for (int j = threadIdx.x; j <= m; j += blockDim.x) {
    const double2 c = j < m ? cadd(h1[j], h2[j]) : make_double2(hlast, 0.0);
    col[j] = c;
    if (staged && j < m - 1) {
      css[j] = a.cs[j];
      sns[j] = a.sn[j];
    }
    cm = fmax(cm, hypot(c.x, c.y));
    if (do_drift && j < m - 1) dm = fmax(dm, hypot(dr[j].x, dr[j].y));
  }
  const double cmax = block_max(cm, shm);
  const double dmax = block_max(dm, shm);
  __syncthreads();  // col, cs, sn visible to thread 0
  const bool breakdown = hlast <= 1e-13 * cmax;
  if (threadIdx.x == 0) {
    if (do_drift && m >= 2) a.drift[m - 1] = dmax;
    scal[0] = hlast;
    scal[1] = breakdown ? 1.0 : 0.0;
    tail_rotate(css, sns, col, m);
    hmm_s = tail_finish(a, col, m, breakdown);
  }
  __syncthreads();
  double2* Hc = a.H + (int64_t)(m - 1) * (a.maxit + 1);
  for (int j = threadIdx.x; j <= m; j += blockDim.x)
    Hc[j] = j == m ? make_double2(0.0, 0.0) : j == m - 1 ? hmm_s : col[j];
}

__global__ void k_vscale(int64_t nl, const double2* __restrict__ w, const double* __restrict__ scal,
                         double2* __restrict__ vm) {
  if (scal[1] != 0.0) return;
  const double hl = scal[0];
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < nl; i += (int64_t)gridDim.x * blockDim.x) {
    const double2 x = w[i];
    vm[i] = make_double2(x.x / hl, x.y / hl);
  }
}

// y = x[off .. off+n) ; zero-filled beyond `valid`
__global__ void k_slice(int64_t n, int64_t valid, const double2* __restrict__ x, double2* __restrict__ y) {
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
    y[i] = i < valid ? x[i] : make_double2(0.0, 0.0);
}

struct OpRunner {
  mdd_ctx* ctx;
  const mdd_gmres_ops* ops;
  int64_t n;
  cudaStream_t s;
  mdd_complex* hin = nullptr;
  mdd_complex* hout = nullptr;
  bool host_ops() const { return ops->a_fn || ops->m_fn; }
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

static unsigned gs_grid(int64_t n) {
  return std::max<unsigned>(1, (unsigned)std::min<int64_t>((n + 255) / 256, 8192));
}

// CGS2 GMRES over row-block-sharded Krylov vectors (one block when the
// preconditioner is not sharded).  Same recurrences and outputs as the MGS
// path: breakdown test, Givens, history clamp, drift (arnoldi_tail).
static void gmres_cgs(mdd_ctx* ctx, const mdd_gmres_ops* ops, int64_t n, const mdd_complex* b,
                      const mdd_complex* x0, const mdd_gmres_cfg* cfg, mdd_complex* x, double* history,
                      double* drift, int32_t* iterations, int32_t* converged) {
  cudaStream_t s = ctx->stream;
  if (!ops->A) fail(MDD_EINVAL, "CGS2 GMRES needs the operator as a matrix");
  if (ops->a_fn || ops->m_fn) fail(MDD_EINVAL, "CGS2 GMRES does not take host callables");
  if (ops->D) fail(MDD_EINVAL, "CGS2 GMRES: weighted inner products are not supported");
  if (cfg->keep_basis) fail(MDD_EINVAL, "CGS2 GMRES: keep_basis is not supported");
  mdd_comm* comm = ops->P ? prec_comm(ops->P) : nullptr;
  const bool dist = comm_active(comm);
  const int N = dist ? comm->nranks : 1, rank = dist ? comm->rank : 0;
  const int64_t chunk = (n + N - 1) / N;
  const int64_t lo = std::min<int64_t>(n, (int64_t)rank * chunk);
  const int64_t nl = std::min<int64_t>(chunk, n - lo);
  const int maxit = cfg->maxit;
  const bool right = cfg->side == 0, dio = cfg->device_io != 0;
  const bool hasM = ops->P || ops->Mcsr;
  auto allreduce = [&](double2* buf, int64_t k) {
    if (dist) comm_allreduce_z(comm, buf, k, s);
  };
  DevBuf<double2> V((size_t)(maxit + 1) * chunk), w(chunk), t(chunk), full((size_t)N * chunk), z(n), bfull,
      x0full, u(chunk);
  const int G = (int)std::max<int64_t>(1, std::min<int64_t>(2 * ctx->nsm, (nl + 511) / 512));
  // row-tiled passes (k_cgs_tile): 3 sweeps over the basis per iteration; MDD_CGS_FUSED=0 keeps
  // the 4-sweep k_mdot/k_maxpy sequence
  const bool fused_env = !getenv("MDD_CGS_FUSED") || atoi(getenv("MDD_CGS_FUSED")) != 0;
  constexpr size_t kCgsSmemMax = 227 * 1024;
  // 16-row tiles (256 B per basis vector per tile); MDD_CGS_ROWS=8 halves the tile (measured slower:
  // cfg1 411 vs 393 ms/step)
  // two tiles in flight (2 CTAs per SM at cfg1's basis sizes); MDD_CGS_STAGES=3 triples the ring
  // where it fits (measured slower: 1 CTA per SM, cfg1 414 vs 397 ms/step)
  static const int cgs_stages = 2;
  static const int cgs_rows = 16;
  const int64_t ntiles = (nl + cgs_rows - 1) / cgs_rows;
  const int Gt_max = (int)std::max<int64_t>(1, std::min<int64_t>((int64_t)ctx->nsm * 8, ntiles));
  if (fused_env) {
    CK(cudaFuncSetAttribute(k_cgs_tile<kProj, 8>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)kCgsSmemMax));
    CK(cudaFuncSetAttribute(k_cgs_tile<kSubProj, 8>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)kCgsSmemMax));
    CK(cudaFuncSetAttribute(k_cgs_tile<kSubNorm, 8>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)kCgsSmemMax));
    CK(cudaFuncSetAttribute(k_cgs_tile<kProj, 16>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)kCgsSmemMax));
    CK(cudaFuncSetAttribute(k_cgs_tile<kSubProj, 16>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)kCgsSmemMax));
    CK(cudaFuncSetAttribute(k_cgs_tile<kSubNorm, 16>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)kCgsSmemMax));
  }
  DevBuf<double2> partial((size_t)(2 * maxit + 2) * std::max(G, Gt_max)), hb(2 * maxit + 2), h2(maxit + 1), nrm(1),
      col(maxit + 2);
  DevBuf<double2> H((size_t)(maxit + 1) * maxit), cs(maxit), sn(maxit), g(maxit + 1), y(maxit);
  DevBuf<double> hist(maxit + 1), dbeta(1), ddrift(maxit + 1), scal(2);
  DevBuf<int> diter(1), dstat(4);
  H.zero(s);
  cs.zero(s);
  sn.zero(s);
  g.zero(s);
  diter.zero(s);
  dstat.zero(s);
  V.zero(s);  // padding rows of the last block stay zero
  full.zero(s);
  {
    std::vector<double> nanv(maxit + 1, NAN);
    ddrift.upload(nanv, s);
  }
  const double2* bdev;
  if (dio) {
    bdev = reinterpret_cast<const double2*>(b);
  } else {
    bfull.upload(reinterpret_cast<const double2*>(b), n, s);
    bdev = bfull.p;
  }
  const double2* x0dev = nullptr;
  if (x0) {
    if (dio) {
      x0dev = reinterpret_cast<const double2*>(x0);
    } else {
      x0full.upload(reinterpret_cast<const double2*>(x0), n, s);
      x0dev = x0full.p;
    }
  }
  auto slice = [&](const double2* src_full, double2* dst) {
    k_slice<<<gs_grid(chunk), 256, 0, s>>>(chunk, nl, src_full + lo, dst);
    CK_LAUNCH(ctx);
  };
  mdd_halo* halo = dist ? prec_halo(ops->P) : nullptr;
  if (dist && !halo) fail(MDD_EINVAL, "sharded GMRES: the preconditioner has no row ranges (mdd_prec_set_halo)");
  // Sharded vectors: `full`, `z` are full-length arrays of which a rank fills its owned rows and,
  // after a halo gather, its needed rows (the unknowns of its subdomains and the columns of its
  // rows of A).  No collective moves a whole vector inside the loop.
  auto spread = [&](const double2* local, double2* vec) {  // owned rows in, needed rows valid
    if (dist) {
      if (nl > 0) CK(cudaMemcpyAsync(vec + lo, local, sizeof(double2) * nl, cudaMemcpyDeviceToDevice, s));
      comm_halo_gather(comm, halo, vec, s);
    } else {
      CK(cudaMemcpyAsync(vec, local, sizeof(double2) * nl, cudaMemcpyDeviceToDevice, s));
    }
  };
  // M: needed-valid in -> owned-valid out (sharded); whole vectors otherwise
  auto applyM = [&](const double2* in_full, double2* out_full) {
    if (dist) prec_apply_dist(ops->P, in_full, out_full, s);
    else if (ops->P) prec_apply_dev(ops->P, in_full, out_full, s);
    else spmv_dev(ctx, ops->Mcsr, in_full, out_full, s);
  };
  // local rows of the (preconditioned) operator applied to a needed-valid vector
  auto op = [&](const double2* vfull, double2* wl) {
    if (right) {
      const double2* in = vfull;
      if (hasM) {
        applyM(vfull, z.p);
        if (dist) comm_halo_gather(comm, halo, z.p, s);  // the columns of my rows of A
        in = z.p;
      }
      spmv_rows_dev(ctx, ops->A, lo, nl, in, wl, s);
    } else {
      spmv_rows_dev(ctx, ops->A, lo, nl, vfull, t.p, s);
      if (hasM) {
        spread(t.p, full.p);
        applyM(full.p, z.p);
        slice(z.p, wl);
      } else {
        CK(cudaMemcpyAsync(wl, t.p, sizeof(double2) * chunk, cudaMemcpyDeviceToDevice, s));
      }
    }
  };
  auto dots = [&](const double2* Vb, int nv, const double2* yv, const double2* d, int nd, double2* out) {
    k_mdot<<<G, 256, 0, s>>>(nl, chunk, Vb, nv, yv, d, nd, partial.p);
    CK_LAUNCH(ctx);
    k_colsum<<<(unsigned)((nv + nd + 7) / 8), 256, 0, s>>>(partial.p, G, nv + nd, out);
    CK_LAUNCH(ctx);
    allreduce(out, nv + nd);
  };
  // r0 (krylov.py:94-106), local rows
  double2* r = w.p;
  slice(bdev, r);
  if (x0dev) {
    spmv_rows_dev(ctx, ops->A, lo, nl, x0dev, t.p, s);
    vec_sub(ctx, r, t.p, r, chunk, s);
  }
  if (!right && hasM) {
    spread(r, full.p);
    applyM(full.p, z.p);
    slice(z.p, r);
  }
  dots(r, 1, r, nullptr, 0, nrm.p);
  std::vector<double2> hn(1);
  nrm.download(hn.data(), 1, s);
  CK(cudaStreamSynchronize(s));
  const double beta = std::sqrt(std::max(hn[0].x, 0.0));
  double2* xout_dev = nullptr;
  DevBuf<double2> xo(dio ? 0 : n);
  xout_dev = dio ? reinterpret_cast<double2*>(x) : xo.p;
  if (beta == 0.0) {  // zero residual: 0 iterations (krylov.py:110-118)
    if (x0dev) CK(cudaMemcpyAsync(xout_dev, x0dev, sizeof(double2) * n, cudaMemcpyDeviceToDevice, s));
    else CK(cudaMemsetAsync(xout_dev, 0, sizeof(double2) * n, s));
    if (!dio) xo.download(reinterpret_cast<double2*>(x), n, s);
    CK(cudaStreamSynchronize(s));
    history[0] = 0.0;
    *iterations = 0;
    *converged = 1;
    return;
  }
  {
    const double h0[2] = {beta, 0.0};
    scal.upload(h0, 2, s);
    const double one = 1.0;
    hist.upload(&one, 1, s);
    const double2 g0 = make_double2(beta, 0.0);
    g.upload(&g0, 1, s);
    dbeta.upload(&beta, 1, s);
  }
  k_vscale<<<gs_grid(chunk), 256, 0, s>>>(chunk, r, scal.p, V.p);
  CK_LAUNCH(ctx);
  ArnoldiArgs aa{};
  aa.maxit = maxit;
  aa.H = H.p;
  aa.cs = cs.p;
  aa.sn = sn.p;
  aa.g = g.p;
  aa.hist = hist.p;
  aa.drift = ddrift.p;
  aa.beta = dbeta.p;
  aa.tol = cfg->tol;
  aa.check_drift = cfg->check_drift;
  aa.iter = diter.p;
  aa.dstatus = dstat.p;
  // convergence is checked one iteration behind (host-mapped status written by
  // the tail kernel), so the host enqueues iteration it+1 while the device
  // still runs iteration it instead of idling through every enqueue
  if (!ctx->mapped_status) CK(cudaHostAlloc(&ctx->mapped_status, sizeof(int) * 4, cudaHostAllocMapped));
  volatile int* hst = ctx->mapped_status;
  int* hst_dev = nullptr;
  CK(cudaHostGetDevicePointer(&hst_dev, (void*)ctx->mapped_status, 0));
  hst[0] = 0;
  aa.hstatus = hst_dev;
  cudaEvent_t itev[2];
  CK(cudaEventCreateWithFlags(&itev[0], cudaEventDisableTiming));
  CK(cudaEventCreateWithFlags(&itev[1], cudaEventDisableTiming));
  int st[4] = {0, 0, 0, 0};
  for (int it = 1; it <= maxit; ++it) {
    const int m = it - 1;  // newest basis vector
    double2* vm = V.p + (int64_t)m * chunk;
    spread(vm, full.p);
    op(full.p, w.p);
    const int nd = (cfg->check_drift && m >= 1) ? m : 0;
    const int nv = m + 1;
    if (fused_env && nv <= kCgsMaxNv && cgs_smem_bytes(nv, cgs_rows, 2) <= kCgsSmemMax) {
      const int ns = cgs_stages >= 3 && cgs_smem_bytes(nv, cgs_rows, 3) <= kCgsSmemMax ? 3 : 2;
      const size_t sm = cgs_smem_bytes(nv, cgs_rows, ns);
      const int per_sm = std::max(1, std::min(8, (int)((228 * 1024) / (sm + 1024))));
      const int Gt = (int)std::max<int64_t>(1, std::min<int64_t>((int64_t)ctx->nsm * per_sm, ntiles));
      auto colsum = [&](int nk, double2* out) {
        k_colsum<<<(unsigned)((nk + 7) / 8), 256, 0, s>>>(partial.p, Gt, nk, out);
        CK_LAUNCH(ctx);
        allreduce(out, nk);
      };
      auto pass = [&](auto kern, const double2* hh, int ndd) {
        kern<<<Gt, kCgsThreads, sm, s>>>(nl, chunk, V.p, nv, hh, w.p, ndd, partial.p, ns);
        CK_LAUNCH(ctx);
      };
      if (cgs_rows == 16) pass(k_cgs_tile<kProj, 16>, nullptr, nd);
      else pass(k_cgs_tile<kProj, 8>, nullptr, nd);
      colsum(nv + nd, hb.p);  // pass 1 (+ drift of V_m)
      if (cgs_rows == 16) pass(k_cgs_tile<kSubProj, 16>, hb.p, 0);
      else pass(k_cgs_tile<kSubProj, 8>, hb.p, 0);
      colsum(nv, h2.p);  // pass 2 projections, after the pass-1 update
      if (cgs_rows == 16) pass(k_cgs_tile<kSubNorm, 16>, h2.p, 0);
      else pass(k_cgs_tile<kSubNorm, 8>, h2.p, 0);
      colsum(1, nrm.p);
    } else {
    dots(V.p, m + 1, w.p, vm, nd, hb.p);  // pass 1 (+ drift of V_m)
    k_maxpy<<<gs_grid(chunk), 256, sizeof(double2) * (m + 1), s>>>(nl, chunk, V.p, m + 1, hb.p, w.p);
    CK_LAUNCH(ctx);
    dots(V.p, m + 1, w.p, nullptr, 0, h2.p);  // pass 2
    k_maxpy<<<gs_grid(chunk), 256, sizeof(double2) * (m + 1), s>>>(nl, chunk, V.p, m + 1, h2.p, w.p);
    CK_LAUNCH(ctx);
    dots(w.p, 1, w.p, nullptr, 0, nrm.p);
    }
    const int tcap = (it + 1) * 3 * (int)sizeof(double2) <= 48 * 1024 ? it + 1 : 0;
    k_cgs_tail<<<1, kTailThreads, sizeof(double2) * 3 * tcap, s>>>(aa, hb.p, h2.p, nrm.p, hb.p + m + 1,
                                                                  nd > 0 ? 1 : 0, col.p, scal.p, tcap);
    CK_LAUNCH(ctx);
    k_vscale<<<gs_grid(chunk), 256, 0, s>>>(chunk, w.p, scal.p, V.p + (int64_t)(m + 1) * chunk);
    CK_LAUNCH(ctx);
    CK(cudaEventRecord(itev[it & 1], s));
    if (it >= 2) {  // iteration it-1 finished: its tail has published the status
      CK(cudaEventSynchronize(itev[(it - 1) & 1]));
      // break only on a solve finished by iteration it-1 (complete on every rank): the
      // status word may already show iteration it, which one rank can observe and
      // another not yet, and every rank must leave the loop after the same collectives
      const int fin = hst[0];
      if (fin != 0 && fin <= it - 1) break;
    }
  }
  cudaEventDestroy(itev[0]);
  cudaEventDestroy(itev[1]);
  dstat.download(st, 4, s);
  CK(cudaStreamSynchronize(s));
  const int m = st[2];
  const bool done = st[0] != 0;
  const bool breakdown = done && st[1];
  if (m < 1) fail(MDD_ECUDA, "gmres: no iteration completed");
  double final_drift = NAN;
  if (cfg->check_drift && !breakdown) {  // drift of the final vector V_m (krylov.py:152-160)
    dots(V.p, m, V.p + (int64_t)m * chunk, nullptr, 0, hb.p);
    std::vector<double2> hv(m);
    hb.download(hv.data(), m, s);
    CK(cudaStreamSynchronize(s));
    final_drift = 0.0;
    for (int j = 0; j < m; ++j) final_drift = std::max(final_drift, std::hypot(hv[j].x, hv[j].y));
  }
  // solution (krylov.py:189-198): x = x0 + M (V y) (right) or x0 + V y (left)
  launch_backsub(ctx, m, maxit, H.p, g.p, y.p, s);
  k_combine_basis<<<gs_grid(chunk), 256, 0, s>>>(chunk, m, V.p, y.p, u.p);
  CK_LAUNCH(ctx);
  spread(u.p, full.p);
  double2* upd = full.p;
  if (right && hasM) {
    applyM(full.p, z.p);
    upd = z.p;
  }
  if (dist) prec_gather_owned(ops->P, upd, s);  // once per solve: the caller gets the whole solution
  k_axpy_out<<<gs_grid(n), 256, 0, s>>>(n, x0dev, upd, xout_dev);
  CK_LAUNCH(ctx);
  if (!dio) xo.download(reinterpret_cast<double2*>(x), n, s);
  hist.download(history, m + 1, s);
  if (drift) ddrift.download(drift, m + 1, s);
  CK(cudaStreamSynchronize(s));
  if (drift && !std::isnan(final_drift)) drift[m] = final_drift;
  *iterations = m;
  *converged = done ? (breakdown ? 2 : 1) : 0;
}

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
  if (cfg->ortho == 1) {
    gmres_cgs(ctx, ops, n, b, x0, cfg, x, history, drift, iterations, converged);
    *seconds = std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
    return MDD_OK;
  }
  if (cfg->ortho != 0) fail(MDD_EINVAL, "gmres: unknown orthogonalisation");
  OpRunner op{ctx, ops, n, s};
  if (op.host_ops()) {
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
  const bool dio = cfg->device_io != 0;
  DevBuf<double2> V((size_t)(maxit + 1) * n), DV, db(n), dx0, r(n), dr, z(n), t(n), w(n), dw, vin(n);
  if (weighted) {
    DV.alloc((size_t)(maxit + 1) * n);
    dr.alloc(n);
    dw.alloc(n);
  }
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
  DevBuf<double> hist(maxit + 1), dbeta(1), ddrift(maxit + 1), dtmp(maxit + 1);
  DevBuf<int> diter(1), dstat(4);
  H.zero(s);
  cs.zero(s);
  sn.zero(s);
  g.zero(s);
  diter.zero(s);
  dstat.zero(s);
  {
    std::vector<double> nanv(maxit + 1, NAN);
    ddrift.upload(nanv, s);
  }
  k_init_basis<<<1, 1024, 0, s>>>(n, r.p, weighted ? dr.p : r.p, V.p, nullptr, vin.p, dbeta.p,
                                  g.p, hist.p, 0);
  CK_LAUNCH(ctx);
  double beta = 0.0;
  dbeta.download(&beta, 1, s);
  CK(cudaStreamSynchronize(s));
  if (beta == 0.0) {  // zero residual: 0 iterations (krylov.py:110-118)
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
  k_init_basis<<<gs_grid(n), 256, 0, s>>>(n, r.p, weighted ? dr.p : r.p, V.p,
                                          weighted ? DV.p : nullptr, vin.p, dbeta.p, g.p, hist.p,
                                          1);
  CK_LAUNCH(ctx);

  // ---- Arnoldi launch configuration: one CTA per SM
  int G = (int)std::max<int64_t>(1, std::min<int64_t>(ctx->nsm, (n + 255) / 256));
  if (const char* e = getenv("MDD_ARN_GRID")) G = std::max(1, std::min(G, atoi(e)));  // test hook: long slices on small n
  const int64_t slice = (n + G - 1) / G;
  G = (int)((n + slice - 1) / slice);
  const bool reg_path = !weighted && slice <= (int64_t)kArnThreads * kArnE;
  int mode = weighted ? 0 : reg_path ? 1 : 2;
  // test hook: force the STREAM path (2) or the general path (0) of an
  // unweighted solve; MDD_ARNOLDI_WCAP shrinks the shared-memory w head
  if (const char* e = getenv("MDD_ARNOLDI_MODE"))
    if (!weighted && (atoi(e) == 0 || atoi(e) == 2)) mode = atoi(e);
  // WIDE (mode 2): col + as much of the w slice as fits in the 227 KB per CTA
  const int64_t static_sm = 16 * (68 + 2 * kMaxArnCTAs + 128) + 1024;
  int64_t wcap = std::max<int64_t>(0, (int64_t)(227 * 1024 - static_sm) / 16 - (maxit + 1));
  if (const char* e = getenv("MDD_ARNOLDI_WCAP")) wcap = std::min<int64_t>(wcap, std::max(0, atoi(e)));
  const size_t shmem = sizeof(double2) * ((size_t)maxit + 1 +
                                          (mode == 1 ? (size_t)kArnThreads * kArnE
                                                     : mode == 2 ? (size_t)std::min<int64_t>(slice, wcap) : 0));
  using ArnFn = void (*)(ArnoldiArgs);
  // (a 512-thread variant holding the tail of w in 20 registers per thread instead of L2 was
  // measured on cfg4: Arnoldi 1291 -> 1358 ms, spills and half the warps; not kept)
  // the tail of w beyond shared memory goes to tensor memory when it fits its 16 elements per
  // thread (cfg4: 10.2k of 16.4k), to L2 otherwise; MDD_ARN_TMEM=0 forces the L2 tail (tests, A/B)
  const int64_t wtail = mode == 2 ? std::max<int64_t>(0, slice - wcap) : 0;
  const bool tm_tail = wtail > 0 && wtail <= (int64_t)kTmemElems * kWideThreads &&
                       !(getenv("MDD_ARN_TMEM") && atoi(getenv("MDD_ARN_TMEM")) == 0);
  // (512 threads x 6 loads in flight with the tensor-memory tail: cfg4 Arnoldi 901 -> 967 ms; not kept)
  ArnFn kfn = mode == 1 ? k_arnoldi<1>
              : mode == 2 ? (tm_tail ? k_arnoldi_wide<kWideThreads, -1> : k_arnoldi_wide<kWideThreads, 0>)
                          : k_arnoldi<0>;
  const int arn_threads = mode == 2 ? kWideThreads : kArnThreads;
  CK(cudaFuncSetAttribute(kfn, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)shmem));
  int per_sm = 0;
  CK(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kfn, arn_threads, shmem));
  if (per_sm < 1) fail(MDD_ECUDA, "arnoldi kernel cannot be resident");
  if (G > per_sm * ctx->nsm || G > kMaxArnCTAs) fail(MDD_ECUDA, "arnoldi grid exceeds co-resident CTAs");
  const int pad = mode == 1 ? 2 : 8;  // measured per path (allgather_bench + in-kernel, round 1)
  const size_t part_elems = (size_t)(2 * maxit + 1) * G * pad;
  DevBuf<double2> partials(part_elems);
  // host-mapped status word, allocated once per context (cudaHostAlloc and
  // cudaFreeHost are slow and cudaFreeHost synchronises the device)
  if (!ctx->mapped_status) CK(cudaHostAlloc(&ctx->mapped_status, sizeof(int) * 4, cudaHostAllocMapped));
  int* hstatus = ctx->mapped_status;
  int* hstatus_dev = nullptr;
  CK(cudaHostGetDevicePointer(&hstatus_dev, hstatus, 0));

  ArnoldiArgs aa{};
  aa.n = n;
  aa.slice = slice;
  aa.maxit = maxit;
  aa.V = V.p;
  aa.DV = weighted ? DV.p : nullptr;
  aa.w = w.p;
  aa.dw = weighted ? dw.p : nullptr;
  aa.vin = vin.p;
  aa.partials = partials.p;
  aa.H = H.p;
  aa.cs = cs.p;
  aa.sn = sn.p;
  aa.g = g.p;
  aa.hist = hist.p;
  aa.drift = ddrift.p;
  aa.beta = dbeta.p;
  aa.tol = cfg->tol;
  // large slices: the drift is computed in panels of kDriftP vectors (k_drift_panel) instead of
  // riding along in the sweeps
  const bool panel_drift = mode == 2 && cfg->check_drift && maxit < kDriftThreads;
  aa.check_drift = panel_drift ? 0 : cfg->check_drift;
  aa.iter = diter.p;
  aa.dstatus = dstat.p;
  aa.wcap = wcap;
  aa.pad = pad;
  // measured per path: warp-0 polling helps the REG path (cfg1 123.9 -> 119.5 ms), hurts STREAM
  aa.wg = mode == 1 ? 1 : 0;
  aa.pf = kArnPf;
  {
    // what DRAM delivers during one exchange (~4 us at ~6 TB/s), spread over the CTAs
    aa.pf_bytes = (int64_t)(24e6 / G) & ~(int64_t)127;
    // (measured on cfg4 with the tensor-memory tail, Arnoldi ms per solve: no head prefetch 979,
    // 162 KB per CTA 901, the whole 381 KB slice 952)
    // in-sweep prefetch distance: off 901, 2 trips 921, 4 trips 876; MDD_ARN_PF_TRIPS overrides
    aa.pf_trips = getenv("MDD_ARN_PF_TRIPS") ? atoi(getenv("MDD_ARN_PF_TRIPS")) : (tm_tail ? 4 : 0);
    // vectors that the L2 cannot keep whole between their two uses are swept in alternating
    // directions (cfg4: 56 MB; measured 1508 -> 1350 ms per solve; cfg3's 24 MB vectors lose 10%)
    aa.zigzag = n * 16 > 40000000ll ? 1 : 0;
    if (const char* e = getenv("MDD_ARN_ZIGZAG")) aa.zigzag = atoi(e) != 0;  // test hook / A-B runs
  }

  auto launch_arnoldi = [&](const ArnoldiArgs& args) {
    // NaN-fill the publication slots (0xFF bytes are a NaN pattern)
    CK(cudaMemsetAsync(partials.p, 0xFF, part_elems * sizeof(double2), s));
    cudaLaunchConfig_t lc = {};
    lc.gridDim = dim3(G);
    lc.blockDim = dim3(arn_threads);
    lc.dynamicSmemBytes = shmem;
    lc.stream = s;
    cudaLaunchAttribute at[1];
    at[0].id = cudaLaunchAttributeCooperative;
    at[0].val.cooperative = 1;
    lc.attrs = at;
    lc.numAttrs = 1;
    CK(cudaLaunchKernelEx(&lc, kfn, args));
    CK_LAUNCH(ctx);
  };
  const int drift_ctas = 2 * ctx->nsm;
  DevBuf<double2> drift_partial(panel_drift ? (size_t)drift_ctas * kDriftP * kDriftThreads : 1);
  const size_t drift_smem = 2 * sizeof(double2) * ((size_t)kDriftR * (maxit | 1) + (size_t)kDriftR * kDriftP);
  if (panel_drift)
    CK(cudaFuncSetAttribute(k_drift_panel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)drift_smem));
  // in_loop: the kernels decide from the device iteration counter whether a panel is complete
  auto launch_drift = [&](bool in_loop, int k0, int k1) {
    DriftArgs da{};
    da.n = n;
    da.V = V.p;
    da.iter = in_loop ? diter.p : nullptr;
    da.dstatus = dstat.p;
    da.k0 = k0;
    da.k1 = k1;
    da.partial = drift_partial.p;
    da.drift = ddrift.p;
    da.ncta = drift_ctas;
    da.stage_elems = (int)(drift_smem / (2 * sizeof(double2)));
    k_drift_panel<<<drift_ctas, kDriftThreads, drift_smem, s>>>(da);
    CK_LAUNCH(ctx);
    k_drift_finish<<<kDriftP, kDriftThreads, 0, s>>>(da);
    CK_LAUNCH(ctx);
  };
  // one iteration's operator part: w = A M vin (right) or M A vin (left)
  auto op_part = [&]() {
    if (right) {
      if (op.has_M()) {
        op.M(vin.p, z.p);
        op.A(z.p, w.p);
      } else {
        op.A(vin.p, w.p);
      }
    } else {
      if (op.has_M()) {
        op.A(vin.p, t.p);
        op.M(t.p, w.p);
      } else {
        op.A(vin.p, w.p);
      }
    }
    if (weighted) spmv_dev(ctx, ops->D, w.p, dw.p, s);
  };

  double t_op = 0, t_prec = 0, t_arn = 0;
  CK(cudaStreamSynchronize(s));
  auto t_loop0 = std::chrono::steady_clock::now();
  // MDD_NO_GRAPH=1: host-driven loop (profilers cannot see kernels inside
  // conditional graph nodes)
  static const bool no_graph = getenv("MDD_NO_GRAPH") != nullptr;
  // sharded preconditioners issue an NCCL allreduce per apply: host-driven loop
  // (NCCL kernels inside a conditional-node body are not relied upon)
  const bool use_graph = !ctx->timing && !op.host_ops() && !no_graph && !prec_is_distributed(ops->P);
  int64_t body_launches = 0;
  if (use_graph) {
    const int64_t l0 = ctx->launches;
    // device-side while loop: no host round trip per iteration
    const auto tg0 = std::chrono::steady_clock::now();
    cudaGraph_t graph;
    CK(cudaGraphCreate(&graph, 0));
    cudaGraphConditionalHandle cond;
    CK(cudaGraphConditionalHandleCreate(&cond, graph, 1, cudaGraphCondAssignDefault));
    cudaGraphNodeParams cp = {};
    cp.type = cudaGraphNodeTypeConditional;
    cp.conditional.handle = cond;
    cp.conditional.type = cudaGraphCondTypeWhile;
    cp.conditional.size = 1;
    cudaGraphNode_t cnode;
    CK(cudaGraphAddNode(&cnode, graph, nullptr, 0, &cp));
    cudaGraph_t body = cp.conditional.phGraph_out[0];
    CK(cudaStreamBeginCaptureToGraph(s, body, nullptr, nullptr, 0, cudaStreamCaptureModeRelaxed));
    op_part();
    ArnoldiArgs ga = aa;
    ga.hstatus = nullptr;
    ga.cond = cond;
    ga.use_cond = 1;
    launch_arnoldi(ga);
    if (panel_drift) launch_drift(true, 0, 0);
    cudaGraph_t captured = nullptr;
    CK(cudaStreamEndCapture(s, &captured));
    body_launches = ctx->launches - l0;
    cudaGraphExec_t exec;
    CK(cudaGraphInstantiate(&exec, graph, 0));
    ctx->timers[6] = std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now() - tg0).count();
    CK(cudaGraphLaunch(exec, s));
    CK(cudaStreamSynchronize(s));
    cudaGraphExecDestroy(exec);
    cudaGraphDestroy(graph);
  } else {
    cudaEvent_t ev[4];
    for (auto& e : ev) CK(cudaEventCreate(&e));
    ArnoldiArgs ha = aa;
    ha.hstatus = hstatus_dev;
    ha.use_cond = 0;
    for (int it = 1; it <= maxit; ++it) {
      if (ctx->timing) CK(cudaEventRecord(ev[0], s));
      if (right) {
        if (op.has_M()) {
          op.M(vin.p, z.p);
          if (ctx->timing) CK(cudaEventRecord(ev[1], s));
          op.A(z.p, w.p);
        } else {
          if (ctx->timing) CK(cudaEventRecord(ev[1], s));
          op.A(vin.p, w.p);
        }
      } else {
        if (op.has_M()) {
          op.A(vin.p, t.p);
          if (ctx->timing) CK(cudaEventRecord(ev[1], s));
          op.M(t.p, w.p);
        } else {
          if (ctx->timing) CK(cudaEventRecord(ev[1], s));
          op.A(vin.p, w.p);
        }
      }
      if (weighted) spmv_dev(ctx, ops->D, w.p, dw.p, s);
      if (ctx->timing) CK(cudaEventRecord(ev[2], s));
      hstatus[0] = 0;
      launch_arnoldi(ha);
      if (panel_drift) launch_drift(true, 0, 0);
      if (ctx->timing) CK(cudaEventRecord(ev[3], s));
      CK(cudaStreamSynchronize(s));
      if (ctx->timing) {
        float a1 = 0, b1 = 0, c1 = 0;
        CK(cudaEventElapsedTime(&a1, ev[0], ev[1]));
        CK(cudaEventElapsedTime(&b1, ev[1], ev[2]));
        CK(cudaEventElapsedTime(&c1, ev[2], ev[3]));
        if (right) { t_prec += a1; t_op += b1; } else { t_op += a1; t_prec += b1; }
        t_arn += c1;
      }
      if (((volatile int*)hstatus)[0]) break;
    }
    for (auto& e : ev) cudaEventDestroy(e);
  }
  auto t_loop1 = std::chrono::steady_clock::now();
  int st[4] = {0, 0, 0, 0};
  dstat.download(st, 4, s);
  CK(cudaStreamSynchronize(s));
  const int m = st[2];
  const bool done = st[0] != 0;
  const bool breakdown = done && st[1];
  if (m < 1) fail(MDD_ECUDA, "gmres: no iteration completed");
  if (use_graph) ctx->launches += body_launches * (m - 1);  // graph replays of the loop body
  // drift of the final appended vector (krylov.py:152-160)
  if (panel_drift) {
    // the vectors after the last complete panel (a panel ending in a breakdown iteration was skipped)
    const int done_upto = (breakdown && m % kDriftP == 0) ? m - kDriftP : (m / kDriftP) * kDriftP;
    const int hi_k = breakdown ? m - 1 : m;
    if (hi_k > done_upto) launch_drift(false, done_upto + 1, hi_k);
  } else if (cfg->check_drift && !breakdown) {
    k_final_drift<<<m, 256, 0, s>>>(n, m, V.p, (weighted ? DV.p : V.p) + (int64_t)m * n, dtmp.p);
    CK_LAUNCH(ctx);
    k_max_into<<<1, 32, 0, s>>>(dtmp.p, m, ddrift.p + m);
    CK_LAUNCH(ctx);
  }
  // solution (krylov.py:189-198)
  launch_backsub(ctx, m, maxit, H.p, g.p, y.p, s);
  k_combine_basis<<<gs_grid(n), 256, 0, s>>>(n, m, V.p, y.p, t.p);
  CK_LAUNCH(ctx);
  double2* upd = t.p;
  if (right && op.has_M()) {
    op.M(t.p, z.p);
    upd = z.p;
  }
  DevBuf<double2> dxo(dio ? 0 : n);
  double2* xout = dio ? reinterpret_cast<double2*>(x) : dxo.p;
  k_axpy_out<<<gs_grid(n), 256, 0, s>>>(n, x0 ? dx0.p : nullptr, upd, xout);
  CK_LAUNCH(ctx);
  if (!dio) dxo.download(reinterpret_cast<double2*>(x), n, s);
  hist.download(history, m + 1, s);
  if (drift) ddrift.download(drift, m + 1, s);
  if (basis) {
    const int nb = breakdown ? m : m + 1;
    V.download(reinterpret_cast<double2*>(basis), (size_t)nb * n, s);
  }
  CK(cudaStreamSynchronize(s));
  auto t_end = std::chrono::steady_clock::now();
  if (ctx->timing) {
    ctx->timers[0] = t_op;
    ctx->timers[1] = t_prec;
    ctx->timers[2] = t_arn;
  }
  // host wall split: setup (allocation, r0, basis), loop, finalisation (ms)
  ctx->timers[3] = std::chrono::duration<double, std::milli>(t_loop0 - t0).count();
  ctx->timers[4] = std::chrono::duration<double, std::milli>(t_loop1 - t_loop0).count();
  ctx->timers[5] = std::chrono::duration<double, std::milli>(t_end - t_loop1).count();
  *iterations = m;
  *converged = done ? (breakdown ? 2 : 1) : 0;
  *seconds = std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
  MDD_API_END
}
