// Shared-memory wavefronts of 64-bit warp loads for chosen address patterns (ncu metric
// l1tex__data_pipe_lsu_wavefronts_mem_shared_op_ld.sum per kernel / loads issued).
#include <cstdio>
__global__ void k(const int *pat, double *out, int reps) {
  __shared__ double sh[1024];
  for (int i = threadIdx.x; i < 1024; i += blockDim.x) sh[i] = i;
  __syncthreads();
  const int idx = pat[threadIdx.x & 31];
  double s = 0;
  for (int r = 0; r < reps; ++r) {
    s += *(volatile double *)&sh[idx];
  }
  out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}
int main() {
  int h[4][32];
  for (int l = 0; l < 32; ++l) {
    h[0][l] = l;                                   // P0: 32 consecutive doubles
    h[1][l] = l < 16 ? l : 16 + (l - 16);          // P1: halves 0..15 / 16..31 (same as P0)
    h[2][l] = l < 8 ? l : l < 16 ? 16 + (l - 8) : l < 24 ? 8 + (l - 16) : 24 + (l - 24);  // P2
    h[3][l] = (l % 16) * 16 + (l / 16);            // P3: 16 lanes per double-bank pair... stride 16
  }
  int *d; double *o; cudaMalloc(&d, sizeof(h)); cudaMalloc(&o, 32 * 1024 * 8);
  cudaMemcpy(d, h, sizeof(h), cudaMemcpyHostToDevice);
  for (int p = 0; p < 4; ++p) k<<<1, 32>>>(d + 32 * p, o, 1000);
  cudaDeviceSynchronize();
  printf("done\n");
}
