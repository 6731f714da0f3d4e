// FP64 dependent-chain latency probe (one warp): DADD, DMUL, DFMA cycles.
#include <cstdio>
#include <cuda_runtime.h>

template <int OP>
__global__ void chain(double* out, long long* cyc, double a, double b, int n) {
  double x = a + threadIdx.x;
  const long long t0 = clock64();
  for (int i = 0; i < n; ++i) {
#pragma unroll
    for (int k = 0; k < 16; ++k) {
      if (OP == 0) x = __dadd_rn(x, b);
      else if (OP == 1) x = __dmul_rn(x, b);
      else x = __fma_rn(x, b, a);
    }
  }
  const long long t1 = clock64();
  out[threadIdx.x] = x;
  if (threadIdx.x == 0) *cyc = t1 - t0;
}

int main() {
  double* d; long long* c; cudaMalloc(&d, 256); cudaMalloc(&c, 8);
  const char* names[3] = {"DADD", "DMUL", "DFMA"};
  for (int op = 0; op < 3; ++op) {
    const int n = 4096;
    for (int rep = 0; rep < 2; ++rep) {
      if (op == 0) chain<0><<<1, 32>>>(d, c, 1.0, 1e-9, n);
      else if (op == 1) chain<1><<<1, 32>>>(d, c, 1.0, 1.0000001, n);
      else chain<2><<<1, 32>>>(d, c, 1.0, 0.9999999, n);
      long long h; cudaMemcpy(&h, c, 8, cudaMemcpyDeviceToHost);
      if (rep) printf("%s latency %.2f cycles\n", names[op], double(h) / (n * 16.0));
    }
  }
  return 0;
}
