// FP64 peak microbenchmark on the B200: DMMA (mma.sync m8n8k4 f64) vs DFMA.
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 tools/fp64_peak.cu -o probe_bin/fp64_peak
#include <cstdio>
#include <cuda_runtime.h>

__global__ void dmma_kernel(double* out, int iters) {
  double a = threadIdx.x * 1e-3, b = blockIdx.x * 1e-3;
  double c[8][2];
#pragma unroll
  for (int k = 0; k < 8; ++k) c[k][0] = c[k][1] = 0.0;
  for (int i = 0; i < iters; ++i) {
#pragma unroll
    for (int k = 0; k < 8; ++k)
      asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};"
                   : "+d"(c[k][0]), "+d"(c[k][1]) : "d"(a), "d"(b));
  }
  double s = 0;
#pragma unroll
  for (int k = 0; k < 8; ++k) s += c[k][0] + c[k][1];
  if (s == 123.456) out[0] = s;
}

__global__ void dfma_kernel(double* out, int iters) {
  double a = threadIdx.x * 1e-3, b = blockIdx.x * 1e-3;
  double c[16];
#pragma unroll
  for (int k = 0; k < 16; ++k) c[k] = k;
  for (int i = 0; i < iters; ++i) {
#pragma unroll
    for (int k = 0; k < 16; ++k) c[k] = fma(a, c[k], b);
  }
  double s = 0;
#pragma unroll
  for (int k = 0; k < 16; ++k) s += c[k];
  if (s == 123.456) out[0] = s;
}

int main() {
  double* d;
  cudaMalloc(&d, 8);
  int nsm;
  cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, 0);
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  const int iters = 4096;
  for (int rep = 0; rep < 2; ++rep) {
    for (int bpsm : {1, 2, 4}) {
      const int blocks = nsm * bpsm, threads = 256;
      dmma_kernel<<<blocks, threads>>>(d, 16);
      cudaEventRecord(e0);
      dmma_kernel<<<blocks, threads>>>(d, iters);
      cudaEventRecord(e1);
      cudaEventSynchronize(e1);
      float ms;
      cudaEventElapsedTime(&ms, e0, e1);
      const double flops = 2.0 * 256.0 * 8 * iters * (blocks * threads / 32);
      printf("DMMA blocks/SM=%d: %.2f TFLOP/s\n", bpsm, flops / ms / 1e9);
      dfma_kernel<<<blocks, threads>>>(d, 16);
      cudaEventRecord(e0);
      dfma_kernel<<<blocks, threads>>>(d, iters);
      cudaEventRecord(e1);
      cudaEventSynchronize(e1);
      cudaEventElapsedTime(&ms, e0, e1);
      const double f2 = 2.0 * 16 * iters * (double)blocks * threads;
      printf("DFMA blocks/SM=%d: %.2f TFLOP/s\n", bpsm, f2 / ms / 1e9);
    }
  }
  return 0;
}
