// DFMA throughput microbenchmark: measures the FP64 FMA peak of this B200
// (MEASURED_PEAKS.json has no FP64 figure). Each thread runs 8 independent
// DFMA chains; the grid is a multiple of the SM count.
#include <cstdio>
#include <cuda_runtime.h>
__global__ void dfma_loop(double* out, int iters, double a, double b) {
  double x0 = threadIdx.x, x1 = x0 + 1, x2 = x0 + 2, x3 = x0 + 3, x4 = x0 + 4, x5 = x0 + 5, x6 = x0 + 6, x7 = x0 + 7;
  for (int i = 0; i < iters; ++i) {
#pragma unroll
    for (int u = 0; u < 16; ++u) {
      x0 = fma(x0, a, b); x1 = fma(x1, a, b); x2 = fma(x2, a, b); x3 = fma(x3, a, b);
      x4 = fma(x4, a, b); x5 = fma(x5, a, b); x6 = fma(x6, a, b); x7 = fma(x7, a, b);
    }
  }
  out[blockIdx.x * blockDim.x + threadIdx.x] = x0 + x1 + x2 + x3 + x4 + x5 + x6 + x7;
}
int main() {
  int dev = 0; cudaDeviceProp p; cudaGetDeviceProperties(&p, dev);
  int sms = p.multiProcessorCount;
  printf("gpu %s sms %d cc %d.%d l2 %d MB mem %.1f GB\n", p.name, sms, p.major, p.minor, p.l2CacheSize >> 20, p.totalGlobalMem / 1e9);
  double* out; int threads = 256;
  for (int bps : {1, 2, 4, 8}) {
    int blocks = sms * bps; cudaMalloc(&out, (size_t)blocks * threads * 8);
    int iters = 4096;
    dfma_loop<<<blocks, threads>>>(out, 16, 0.999999, 1e-7);
    cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
    float best = 1e30f;
    for (int rep = 0; rep < 5; ++rep) {
      cudaEventRecord(e0); dfma_loop<<<blocks, threads>>>(out, iters, 0.999999, 1e-7); cudaEventRecord(e1);
      cudaEventSynchronize(e1); float ms; cudaEventElapsedTime(&ms, e0, e1); if (ms < best) best = ms;
    }
    double flops = 2.0 * 8 * 16 * (double)iters * blocks * threads;
    printf("blocks/SM %d: %.3f ms  %.2f TFLOP/s fp64 (FMA=2)\n", bps, best, flops / best / 1e9);
    cudaFree(out);
  }
  return 0;
}
