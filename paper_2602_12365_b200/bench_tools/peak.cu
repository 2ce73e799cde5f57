// peak.cu — FP64 FMA throughput microbenchmark (the "alu" roofline denominator of
// DESIGN.md §5).  Each thread runs 8 independent DFMA chains; the kernel is launched
// with enough warps to saturate every SM's FP64 pipe.  Not part of the hot path.
#include <cuda_runtime.h>
#include <stdint.h>

__global__ void k_dfma(double *out, int iters, double a, double b) {
  double x0 = threadIdx.x, x1 = x0 + 1, x2 = x0 + 2, x3 = x0 + 3;
  double x4 = x0 + 4, x5 = x0 + 5, x6 = x0 + 6, x7 = x0 + 7;
  for (int i = 0; i < iters; ++i) {
#pragma unroll
    for (int k = 0; k < 16; ++k) {
      x0 = fma(x0, a, b); x1 = fma(x1, a, b); x2 = fma(x2, a, b); x3 = fma(x3, a, b);
      x4 = fma(x4, a, b); x5 = fma(x5, a, b); x6 = fma(x6, a, b); x7 = fma(x7, a, b);
    }
  }
  if (x0 + x1 + x2 + x3 + x4 + x5 + x6 + x7 == 12345.678) out[0] = x0;
}

extern "C" double fem_peak_fp64_tflops(int n_sm) {
  double *d = nullptr;
  cudaMalloc(&d, 8);
  const int threads = 512, blocks = n_sm * 4, iters = 4096;
  k_dfma<<<blocks, threads>>>(d, 64, 0.999999, 1e-9);  // warm-up
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  float best = 1e30f;
  for (int r = 0; r < 5; ++r) {
    cudaEventRecord(e0);
    k_dfma<<<blocks, threads>>>(d, iters, 0.999999, 1e-9);
    cudaEventRecord(e1);
    cudaEventSynchronize(e1);
    float ms = 0;
    cudaEventElapsedTime(&ms, e0, e1);
    if (ms < best) best = ms;
  }
  cudaFree(d);
  const double flops = 2.0 * 8 * 16 * (double)iters * threads * blocks;
  return flops / (best * 1e-3) / 1e12;
}
