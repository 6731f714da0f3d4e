// Packed FP32 probe: FFMA vs FFMA2 (__ffma2_rn, sm_100a) throughput, and
// FFMA2 mixed with independent integer/ALU work (does halving FP32 issue
// slots free issue bandwidth for the rest of the instruction mix?).
#include <cstdio>
#include <cuda_runtime.h>

template <int MODE>
__global__ void __launch_bounds__(256) k(float* out, int iters, float b0) {
  float2 acc[8], v[8];
  unsigned ia[8];
#pragma unroll
  for (int i = 0; i < 8; ++i) {
    acc[i] = make_float2(0.f, 0.f);
    v[i] = make_float2(threadIdx.x * 1e-3f + i, threadIdx.x * 2e-3f + i);
    ia[i] = threadIdx.x + i;
  }
  const float2 bb = make_float2(b0, b0 * 0.5f);
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int j = 0; j < 8; ++j)
#pragma unroll
      for (int i = 0; i < 8; ++i) {
        if (MODE == 0) {  // scalar: two FFMA per element pair
          acc[i].x = fmaf(v[i].x, bb.x, acc[i].x);
          acc[i].y = fmaf(v[i].y, bb.y, acc[i].y);
        } else if (MODE == 1) {  // packed
          acc[i] = __ffma2_rn(v[i], bb, acc[i]);
        } else {  // packed + one independent integer op per FFMA2
          acc[i] = __ffma2_rn(v[i], bb, acc[i]);
          ia[i] = ia[i] * 3u + static_cast<unsigned>(j);
        }
      }
#pragma unroll
    for (int i = 0; i < 8; ++i) v[i].x += 1e-7f;
  }
  float s = 0;
#pragma unroll
  for (int i = 0; i < 8; ++i) s += acc[i].x + acc[i].y + static_cast<float>(ia[i] & 1u);
  out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}

template <int M>
void run(const char* name, float* d) {
  cudaEvent_t a, b;
  cudaEventCreate(&a);
  cudaEventCreate(&b);
  float best = 1e9;
  for (int r = 0; r < 5; ++r) {
    cudaEventRecord(a);
    k<M><<<148 * 8, 256>>>(d, 2048, 1.0001f);
    cudaEventRecord(b);
    cudaEventSynchronize(b);
    float ms;
    cudaEventElapsedTime(&ms, a, b);
    if (r && ms < best) best = ms;
  }
  const double flops = 2.0 * 2 * 148 * 8 * 256 * 2048.0 * 64;  // 2 lanes of FMA per element pair
  printf("%-16s %.3f ms  %.1f TFLOP/s (fp32)\n", name, best, flops / best / 1e9);
}

int main() {
  float* d;
  cudaMalloc(&d, 148 * 8 * 256 * 4);
  run<0>("ffma", d);
  run<1>("ffma2", d);
  run<2>("ffma2+int", d);
  return 0;
}
