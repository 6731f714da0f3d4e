// Throughput of the legacy warp-level tensor MMA (mma.sync m16n8k8, TF32
// inputs, FP32 accumulate) on sm_100a: independent accumulator chains on
// every warp of every SM.  Feasibility probe for moving NBody's
// accumulation onto tensor cores.
// Build: nvcc -O3 -gencode arch=compute_100a,code=sm_100a mma_tf32.cu -o mma_tf32
#include <cstdio>
#include <cuda_runtime.h>

__global__ void __launch_bounds__(256) k(float* out, int iters) {
  unsigned a0 = __float_as_uint(1.0f + threadIdx.x), a1 = a0 ^ 7, a2 = a0 ^ 13, a3 = a0 ^ 29;
  unsigned b0 = __float_as_uint(0.5f), b1 = __float_as_uint(0.25f);
  float c[4][4] = {};
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int j = 0; j < 4; ++j)
      asm volatile(
          "mma.sync.aligned.m16n8k8.row.col.f32.tf32.tf32.f32 {%0,%1,%2,%3}, {%4,%5,%6,%7}, {%8,%9}, "
          "{%0,%1,%2,%3};"
          : "+f"(c[j][0]), "+f"(c[j][1]), "+f"(c[j][2]), "+f"(c[j][3])
          : "r"(a0), "r"(a1), "r"(a2), "r"(a3), "r"(b0), "r"(b1));
  }
  float s = 0;
#pragma unroll
  for (int j = 0; j < 4; ++j) s += c[j][0] + c[j][1] + c[j][2] + c[j][3];
  out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}

int main() {
  float* d;
  cudaMalloc(&d, 148 * 8 * 256 * 4);
  cudaEvent_t a, b;
  cudaEventCreate(&a);
  cudaEventCreate(&b);
  const int iters = 20000;
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
  const double flops = 2.0 * 16 * 8 * 8 * 4.0 * iters * (148.0 * 8 * 256 / 32);
  printf("mma.sync m16n8k8 tf32: %.3f ms, %.1f TFLOP/s\n", best, flops / best / 1e9);
  return 0;
}
