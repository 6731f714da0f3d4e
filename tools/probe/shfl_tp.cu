// SHFL throughput probe: independent __shfl_down_sync chains, all SMs.
#include <cstdio>
#include <cuda_runtime.h>

__global__ void __launch_bounds__(256) k(float* out, int iters) {
  float v[8];
#pragma unroll
  for (int i = 0; i < 8; ++i) v[i] = threadIdx.x + i;
  for (int it = 0; it < iters; ++it)
#pragma unroll
    for (int i = 0; i < 8; ++i) v[i] = __shfl_down_sync(0xffffffffu, v[i], 1) + 1.0f;
  float s = 0;
#pragma unroll
  for (int i = 0; i < 8; ++i) s += v[i];
  out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}

int main() {
  float* d;
  cudaMalloc(&d, 148 * 8 * 256 * 4);
  cudaEvent_t a, b;
  cudaEventCreate(&a);
  cudaEventCreate(&b);
  const int iters = 4096;
  float best = 1e9;
  for (int r = 0; r < 4; ++r) {
    cudaEventRecord(a);
    k<<<148 * 8, 256>>>(d, iters);
    cudaEventRecord(b);
    cudaEventSynchronize(b);
    float ms;
    cudaEventElapsedTime(&ms, a, b);
    if (r && ms < best) best = ms;
  }
  int clk = 0;
  cudaDeviceGetAttribute(&clk, cudaDevAttrClockRate, 0);
  const double warp_shfl = 148.0 * 8 * 8 * iters * 8;  // warps x shuffles
  const double cycles = best * 1e-3 * clk * 1e3;
  printf("SHFL: %.3f ms, %.2f warp-shuffles per SM per cycle (at %d MHz)\n", best, warp_shfl / 148 / cycles,
         clk / 1000);
  return 0;
}
