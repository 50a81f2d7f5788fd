// Microbenchmark: FP64 / FP32 SIMT issue throughput on this B200 (roofline denominators
// the driver does not measure). Separate DMUL+DADD chains (the no-FMA pyramid mix) and DFMA.
#include <cstdio>
#include <cuda_runtime.h>
template <int MODE>
__global__ void k(double* out, double a, double b, int iters) {
  double x0 = threadIdx.x * 1e-3, x1 = x0 + 1, x2 = x0 + 2, x3 = x0 + 3, x4 = x0 + 4, x5 = x0 + 5, x6 = x0 + 6, x7 = x0 + 7;
  for (int i = 0; i < iters; ++i) {
#pragma unroll
    for (int u = 0; u < 8; ++u) {
      if (MODE == 0) { x0 = __fma_rn(x0, a, b); x1 = __fma_rn(x1, a, b); x2 = __fma_rn(x2, a, b); x3 = __fma_rn(x3, a, b);
                       x4 = __fma_rn(x4, a, b); x5 = __fma_rn(x5, a, b); x6 = __fma_rn(x6, a, b); x7 = __fma_rn(x7, a, b); }
      else if (MODE == 1) { x0 = __dmul_rn(x0, a); x1 = __dadd_rn(x1, b); x2 = __dmul_rn(x2, a); x3 = __dadd_rn(x3, b);
                            x4 = __dmul_rn(x4, a); x5 = __dadd_rn(x5, b); x6 = __dmul_rn(x6, a); x7 = __dadd_rn(x7, b); }
    }
  }
  out[blockIdx.x * blockDim.x + threadIdx.x] = x0 + x1 + x2 + x3 + x4 + x5 + x6 + x7;
}
__global__ void kf(float* out, float a, float b, int iters) {
  float x[8];
  for (int u = 0; u < 8; ++u) x[u] = threadIdx.x * 1e-3f + u;
  for (int i = 0; i < iters; ++i)
#pragma unroll
    for (int r = 0; r < 8; ++r)
#pragma unroll
      for (int u = 0; u < 8; ++u) x[u] = __fmaf_rn(x[u], a, b);
  float s = 0; for (int u = 0; u < 8; ++u) s += x[u];
  out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}
int main() {
  cudaDeviceProp p; cudaGetDeviceProperties(&p, 0);
  int clk = 0; cudaDeviceGetAttribute(&clk, cudaDevAttrClockRate, 0);
  printf("device %s sms %d clock_khz %d l2 %d smem/blk optin %zu\n", p.name, p.multiProcessorCount, clk, p.l2CacheSize, p.sharedMemPerBlockOptin);
  double* d; cudaMalloc(&d, 148 * 64 * 1024 * sizeof(double));
  int blocks = p.multiProcessorCount * 8, threads = 256, iters = 4096;
  cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
  for (int mode = 0; mode < 3; ++mode) {
    float best = 1e30f;
    for (int rep = 0; rep < 5; ++rep) {
      cudaEventRecord(e0);
      if (mode == 0) k<0><<<blocks, threads>>>(d, 0.999, 1e-3, iters);
      else if (mode == 1) k<1><<<blocks, threads>>>(d, 0.999, 1e-3, iters);
      else kf<<<blocks, threads>>>((float*)d, 0.999f, 1e-3f, iters);
      cudaEventRecord(e1); cudaEventSynchronize(e1);
      float ms; cudaEventElapsedTime(&ms, e0, e1); if (ms < best) best = ms;
    }
    double ops = (double)blocks * threads * iters * 64;
    printf("%s: %.3f ms  %.2f Tops/s (%s)\n", mode == 0 ? "DFMA" : mode == 1 ? "DMUL/DADD" : "FFMA", best, ops / best / 1e9,
           mode == 1 ? "1 op each" : "x2 for flops");
  }
  printf("err %s\n", cudaGetErrorString(cudaGetLastError()));
  return 0;
}
