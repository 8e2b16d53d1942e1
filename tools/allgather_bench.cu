// Microbenchmark: latency of one deterministic grid-wide reduction step in a
// persistent kernel (the MGS step of k_arnoldi), three schemes:
//   0  flat all-gather (current k_arnoldi): every CTA polls all G NaN-filled slots
//   1  last arriver reduces: publish + atomic ticket; the last CTA sums the G
//      slots in fixed order and publishes one result; everyone polls it
//   2  cluster pairs: partner CTAs combine through DSMEM, G/2 publishers,
//      every CTA polls the G/2 pair slots
// Each step also does a small amount of per-CTA work (a 256-thread block sum).
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o /tmp/agb tools/allgather_bench.cu
#include <cooperative_groups.h>
#include <cstdio>
#include <cstdlib>
#include <vector>
namespace cg = cooperative_groups;

__device__ __forceinline__ double2 ld_relaxed2(const double2* p) {
  double2 v;
  asm volatile("ld.relaxed.gpu.global.v2.f64 {%0,%1}, [%2];" : "=d"(v.x), "=d"(v.y) : "l"(p) : "memory");
  return v;
}
__device__ __forceinline__ bool bad2(double2 v) { return isnan(v.x) || isnan(v.y); }
__device__ __forceinline__ double2 wsum(double2 v) {
  for (int o = 16; o; o >>= 1) {
    v.x += __shfl_xor_sync(~0u, v.x, o);
    v.y += __shfl_xor_sync(~0u, v.y, o);
  }
  return v;
}

template <int MODE>
__global__ void __launch_bounds__(256, 1) k_steps(int nsteps, double2* slots, double2* res, unsigned* cnt,
                                                  double* out) {
  __shared__ double2 sh[64 + 2 * 160];
  __shared__ double2 pairbuf[2];
  const int G = gridDim.x;
  double2 mine = make_double2(1.0 + blockIdx.x * 1e-3 + threadIdx.x * 1e-6, 0.5);
  double acc = 0;
  for (int s = 0; s < nsteps; ++s) {
    // per-CTA work: block sum of `mine`
    double2 v = wsum(mine);
    if ((threadIdx.x & 31) == 0) sh[threadIdx.x >> 5] = v;
    __syncthreads();
    double2 part = make_double2(0, 0);
    if (threadIdx.x == 0)
      for (int k = 0; k < 8; ++k) part.x += sh[k].x, part.y += sh[k].y;
    double2 tot;
    if (MODE == 0) {
      if (threadIdx.x == 0) __stcg(slots + (size_t)s * G + blockIdx.x, part);
      double2* st = sh + 64;
      if ((int)threadIdx.x < G) {
        double2 u = ld_relaxed2(slots + (size_t)s * G + threadIdx.x);
        { long long sp = 0; while (bad2(u)) { if (++sp > (1ll << 26)) __trap(); u = ld_relaxed2(slots + (size_t)s * G + threadIdx.x); } }
        st[threadIdx.x] = u;
      }
      __syncthreads();
      if (threadIdx.x < 32) {
        double2 x = make_double2(0, 0);
        for (int k = threadIdx.x; k < G; k += 32) x.x += st[k].x, x.y += st[k].y;
        x = wsum(x);
        if (threadIdx.x == 0) sh[62] = x;
      }
      __syncthreads();
      tot = sh[62];
    } else if (MODE == 3) {
      // flat all-gather with every slot on its own 128-byte L2 line
      constexpr int PAD = 8;
      if (threadIdx.x == 0) __stcg(slots + ((size_t)s * G + blockIdx.x) * PAD, part);
      double2* st = sh + 64;
      if ((int)threadIdx.x < G) {
        double2 u = ld_relaxed2(slots + ((size_t)s * G + threadIdx.x) * PAD);
        { long long sp = 0; while (bad2(u)) { if (++sp > (1ll << 26)) __trap(); u = ld_relaxed2(slots + ((size_t)s * G + threadIdx.x) * PAD); } }
        st[threadIdx.x] = u;
      }
      __syncthreads();
      if (threadIdx.x < 32) {
        double2 x = make_double2(0, 0);
        for (int k = threadIdx.x; k < G; k += 32) x.x += st[k].x, x.y += st[k].y;
        x = wsum(x);
        if (threadIdx.x == 0) sh[62] = x;
      }
      __syncthreads();
      tot = sh[62];
    } else if (MODE == 1) {
      if (threadIdx.x < 32) {
        unsigned old = 0;
        if (threadIdx.x == 0) {
          __stcg(slots + (size_t)s * G + blockIdx.x, part);
          __threadfence();
          old = atomicAdd(cnt + s, 1u);
        }
        old = __shfl_sync(~0u, old, 0);
        if (old == (unsigned)G - 1) {
          __threadfence();
          double2 x = make_double2(0, 0);
          for (int k = threadIdx.x; k < G; k += 32) {
            const double2 u = __ldcg(slots + (size_t)s * G + k);
            x.x += u.x, x.y += u.y;
          }
          x = wsum(x);
          if (threadIdx.x == 0) __stcg(res + s, x);
        }
        if (threadIdx.x == 0) {
          double2 u = ld_relaxed2(res + s);
          { long long sp = 0; while (bad2(u)) { if (++sp > (1ll << 26)) __trap(); u = ld_relaxed2(res + s); } }
          sh[62] = u;
        }
      }
      __syncthreads();
      tot = sh[62];
    } else {
      cg::cluster_group cl = cg::this_cluster();
      const unsigned rank = cl.block_rank();
      const int P = G / 2;
      if (threadIdx.x == 0) {
        double2* dst = cl.map_shared_rank(pairbuf, 0);
        dst[rank] = part;
      }
      cl.sync();
      if (rank == 0 && threadIdx.x == 0) {
        double2 q = make_double2(pairbuf[0].x + pairbuf[1].x, pairbuf[0].y + pairbuf[1].y);
        __stcg(slots + (size_t)s * G + blockIdx.x / 2, q);
      }
      double2* st = sh + 64;
      if ((int)threadIdx.x < P) {
        double2 u = ld_relaxed2(slots + (size_t)s * G + threadIdx.x);
        { long long sp = 0; while (bad2(u)) { if (++sp > (1ll << 26)) __trap(); u = ld_relaxed2(slots + (size_t)s * G + threadIdx.x); } }
        st[threadIdx.x] = u;
      }
      __syncthreads();
      if (threadIdx.x < 32) {
        double2 x = make_double2(0, 0);
        for (int k = threadIdx.x; k < P; k += 32) x.x += st[k].x, x.y += st[k].y;
        x = wsum(x);
        if (threadIdx.x == 0) sh[62] = x;
      }
      __syncthreads();
      tot = sh[62];
    }
    acc += tot.x;
    mine.x += 1e-9 * tot.y;
  }
  if (threadIdx.x == 0) out[blockIdx.x] = acc;
}

int main(int argc, char** argv) {
  const int steps = argc > 1 ? atoi(argv[1]) : 20000;
  int nsm = 0;
  cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, 0);
  const int G = nsm;  // 148 (even)
  double2* slots;
  double2* res;
  unsigned* cnt;
  double* out;
  cudaMalloc(&slots, sizeof(double2) * (size_t)steps * G * 8);
  cudaMalloc(&res, sizeof(double2) * steps);
  cudaMalloc(&cnt, sizeof(unsigned) * steps);
  cudaMalloc(&out, sizeof(double) * G);
  cudaEvent_t a, b;
  cudaEventCreate(&a);
  cudaEventCreate(&b);
  for (int mode = 0; mode < 4; ++mode)
    for (int rep = 0; rep < 3; ++rep) {
      cudaMemset(slots, 0xff, sizeof(double2) * (size_t)steps * G * 8);  // NaN
      cudaMemset(res, 0xff, sizeof(double2) * steps);
      cudaMemset(cnt, 0, sizeof(unsigned) * steps);
      cudaEventRecord(a);
      if (mode == 0) k_steps<0><<<G, 256>>>(steps, slots, res, cnt, out);
      if (mode == 1) k_steps<1><<<G, 256>>>(steps, slots, res, cnt, out);
      if (mode == 3) k_steps<3><<<G, 256>>>(steps, slots, res, cnt, out);
      if (mode == 2) {
        cudaLaunchConfig_t cfg = {};
        cfg.gridDim = dim3(G);
        cfg.blockDim = dim3(256);
        cudaLaunchAttribute at[1];
        at[0].id = cudaLaunchAttributeClusterDimension;
        at[0].val.clusterDim.x = 2;
        at[0].val.clusterDim.y = 1;
        at[0].val.clusterDim.z = 1;
        cfg.attrs = at;
        cfg.numAttrs = 1;
        cudaLaunchKernelEx(&cfg, k_steps<2>, steps, slots, res, cnt, out);
      }
      cudaEventRecord(b);
      cudaError_t e = cudaEventSynchronize(b);
      float ms = 0;
      cudaEventElapsedTime(&ms, a, b);
      printf("mode %d rep %d: %s  %.3f us/step\n", mode, rep, cudaGetErrorString(e), 1e3 * ms / steps);
    }
  return 0;
}
