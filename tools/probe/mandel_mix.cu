// Achievable FP64 instruction rate for the Mandelbrot iteration's mix and
// dependency structure (3 DMUL, 1 DFMA, 2 DADD + 1 LOP3 per iteration), with
// no control flow: the ceiling the kernel's bookkeeping is measured against.
#include <cstdio>
#include <cuda_runtime.h>

template <int ILP>
__global__ void __launch_bounds__(256) mix(double* out, unsigned* flag, int iters, double cx0, double cy0) {
  double zx[ILP], zy[ILP], cx[ILP], cy[ILP];
  unsigned acc = 0;
#pragma unroll
  for (int k = 0; k < ILP; ++k) {
    cx[k] = cx0 + 1e-9 * (threadIdx.x + k);
    cy[k] = cy0;
    zx[k] = 0;
    zy[k] = 0;
  }
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int r = 0; r < 16; ++r) {
#pragma unroll
      for (int k = 0; k < ILP; ++k) {
        const double xx = __dmul_rn(zx[k], zx[k]);
        const double yy = __dmul_rn(zy[k], zy[k]);
        acc |= __double2hiint(xx) | __double2hiint(yy);
        const double t = __dmul_rn(zx[k], zy[k]);
        zy[k] = __fma_rn(t, 2.0, cy[k]);
        zx[k] = __dadd_rn(__dsub_rn(xx, yy), cx[k]);
      }
    }
  }
  double s = 0;
#pragma unroll
  for (int k = 0; k < ILP; ++k) s += zx[k] + zy[k];
  out[blockIdx.x * blockDim.x + threadIdx.x] = s;
  if (acc == 0x12345) *flag = acc;
}

template <int ILP>
void run(int blocks_per_sm, double* d, unsigned* f) {
  cudaEvent_t a, b;
  cudaEventCreate(&a);
  cudaEventCreate(&b);
  const int blocks = 148 * blocks_per_sm, iters = 512;
  float best = 1e9;
  for (int r = 0; r < 4; ++r) {
    cudaEventRecord(a);
    mix<ILP><<<blocks, 256>>>(d, f, iters, -0.1, 0.1);
    cudaEventRecord(b);
    cudaEventSynchronize(b);
    float ms;
    cudaEventElapsedTime(&ms, a, b);
    if (r && ms < best) best = ms;
  }
  const double instr = 6.0 * 16 * iters * ILP * double(blocks) * 256;
  const double flops = 8.0 * 16 * iters * ILP * double(blocks) * 256;
  printf("ILP %d, %d CTAs/SM: %.3f ms  %.2f T FP64-instr/s  %.2f TFLOP/s (8 flop/iter)\n", ILP, blocks_per_sm, best,
         instr / best / 1e9, flops / best / 1e9);
}

int main() {
  double* d;
  unsigned* f;
  cudaMalloc(&d, 148 * 8 * 256 * 8);
  cudaMalloc(&f, 4);
  for (int bps : {2, 4, 8}) run<1>(bps, d, f);
  for (int bps : {2, 4}) run<2>(bps, d, f);
  return 0;
}
