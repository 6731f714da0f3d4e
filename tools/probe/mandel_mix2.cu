// Mandelbrot FP64 iteration mixes: DMUL/DADD forms vs all-DFMA forms (each
// exact: squares and products as fma(x, y, +0), subtraction as
// fma(yy, -1, xx), addition as fma(d, 1, cx)), with and without the
// speculation's LOP3.
#include <cstdio>
#include <cuda_runtime.h>

template <int MODE>
__global__ void __launch_bounds__(256) mix(double* out, unsigned* flag, int iters) {
  double zx[2] = {0, 0}, zy[2] = {0, 0}, cx[2], cy[2];
  double pxx[2] = {0, 0}, pyy[2] = {0, 0};
  unsigned acc = 0;
#pragma unroll
  for (int k = 0; k < 2; ++k) {
    cx[k] = -0.1 + 1e-9 * (threadIdx.x + k);
    cy[k] = 0.1;
  }
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int r = 0; r < 16; ++r) {
#pragma unroll
      for (int k = 0; k < 2; ++k) {
        double xx, yy, t;
        if (MODE == 1 || MODE == 3) {
          xx = __fma_rn(zx[k], zx[k], 0.0);
          yy = __fma_rn(zy[k], zy[k], 0.0);
          t = __fma_rn(zx[k], zy[k], 0.0);
        } else {
          xx = __dmul_rn(zx[k], zx[k]);
          yy = __dmul_rn(zy[k], zy[k]);
          t = __dmul_rn(zx[k], zy[k]);
        }
        if (MODE < 2) acc |= static_cast<unsigned>(__double2hiint(xx)) | static_cast<unsigned>(__double2hiint(yy));
        if (MODE == 4) acc |= static_cast<unsigned>(__double2hiint(xx));
        if (MODE == 5 && (r & 1)) acc |= static_cast<unsigned>(__double2hiint(xx)) | static_cast<unsigned>(__double2hiint(yy));
        if (MODE == 6) acc = max(acc, static_cast<unsigned>(__double2hiint(xx)) | static_cast<unsigned>(__double2hiint(yy)));
        if (MODE == 7) acc += static_cast<unsigned>(__double2hiint(xx)) + static_cast<unsigned>(__double2hiint(yy));
        if (MODE == 8) {  // previous iteration's squares: no wait on this iteration's DMULs
          acc |= static_cast<unsigned>(__double2hiint(pxx[k])) | static_cast<unsigned>(__double2hiint(pyy[k]));
          pxx[k] = xx;
          pyy[k] = yy;
        }
        zy[k] = __fma_rn(t, 2.0, cy[k]);
        if (MODE == 1 || MODE == 3) zx[k] = __fma_rn(__fma_rn(yy, -1.0, xx), 1.0, cx[k]);
        else zx[k] = __dadd_rn(__dsub_rn(xx, yy), cx[k]);
      }
    }
  }
  out[blockIdx.x * blockDim.x + threadIdx.x] = zx[0] + zx[1] + zy[0] + zy[1] + pxx[0] + pyy[1];
  if (acc == 0x12345u) *flag = acc;
}

template <int M>
void run(const char* name, double* d, unsigned* f) {
  cudaEvent_t a, b;
  cudaEventCreate(&a);
  cudaEventCreate(&b);
  const int blocks = 148 * 4, iters = 512;
  float best = 1e9;
  for (int r = 0; r < 4; ++r) {
    cudaEventRecord(a);
    mix<M><<<blocks, 256>>>(d, f, iters);
    cudaEventRecord(b);
    cudaEventSynchronize(b);
    float ms;
    cudaEventElapsedTime(&ms, a, b);
    if (r && ms < best) best = ms;
  }
  const double it = 16.0 * iters * 2 * blocks * 256;
  printf("%-22s %.3f ms  %.2f T FP64-instr/s  %.2f algorithmic TFLOP/s\n", name, best, 6 * it / best / 1e9,
         8 * it / best / 1e9);
}

int main() {
  double* d;
  unsigned* f;
  cudaMalloc(&d, 148 * 4 * 256 * 8);
  cudaMalloc(&f, 4);
  run<0>("dmul/dadd + lop3", d, f);
  run<1>("all-dfma + lop3", d, f);
  run<2>("dmul/dadd, no lop3", d, f);
  run<3>("all-dfma, no lop3", d, f);
  run<4>("hi(xx) only", d, f);
  run<5>("lop3 every 2nd iter", d, f);
  run<6>("max(acc, xx|yy)", d, f);
  run<7>("iadd3 acc+xx+yy", d, f);
  run<8>("lop3 on previous iter", d, f);
  return 0;
}
