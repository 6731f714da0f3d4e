// FFMA operand-form throughput probe (register / immediate / constant bank).
#include <cstdio>
#include <cuda_runtime.h>
struct W { float w[64]; };
__constant__ float cw[64];
template <int MODE>
__global__ void __launch_bounds__(256) k(float* out, int iters, W wp, const float* gw) {
  float acc[8], v[8], r[8];
#pragma unroll
  for (int i = 0; i < 8; ++i) { acc[i] = 0; v[i] = threadIdx.x * 1e-3f + i; r[i] = gw[i]; }
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int j = 0; j < 8; ++j)
#pragma unroll
      for (int i = 0; i < 8; ++i) {
        if (MODE == 0) acc[i] = fmaf(v[i], r[j], acc[i]);          // 3 registers
        else if (MODE == 1) acc[i] = fmaf(v[i], 1.0001f + j, acc[i]);  // immediate
        else if (MODE == 2) acc[i] = fmaf(v[i], wp.w[j], acc[i]);  // kernel param (c[0])
        else acc[i] = fmaf(v[i], cw[j], acc[i]);                   // __constant__
      }
#pragma unroll
    for (int i = 0; i < 8; ++i) v[i] += 1e-7f;
  }
  float s = 0;
#pragma unroll
  for (int i = 0; i < 8; ++i) s += acc[i];
  out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}
template <int M> void run(const char* name, float* d, W w, float* gw) {
  cudaEvent_t a, b; cudaEventCreate(&a); cudaEventCreate(&b);
  float best = 1e9;
  for (int r = 0; r < 4; ++r) {
    cudaEventRecord(a); k<M><<<148 * 8, 256>>>(d, 4096, w, gw); cudaEventRecord(b); cudaEventSynchronize(b);
    float ms; cudaEventElapsedTime(&ms, a, b); if (r && ms < best) best = ms;
  }
  double flops = 2.0 * 148 * 8 * 256 * 4096.0 * 64;
  printf("%-10s %.3f ms  %.1f TFLOP/s\n", name, best, flops / best / 1e9);
}
int main() {
  float* d; cudaMalloc(&d, 148 * 8 * 256 * 4); float* gw; cudaMalloc(&gw, 256); cudaMemset(gw, 0, 256);
  W w; for (int i = 0; i < 64; ++i) w.w[i] = 1.0f + i * 1e-4f;
  cudaMemcpyToSymbol(cw, w.w, sizeof(w.w));
  run<0>("reg", d, w, gw); run<1>("imm", d, w, gw); run<2>("param", d, w, gw); run<3>("constant", d, w, gw);
  return 0;
}
