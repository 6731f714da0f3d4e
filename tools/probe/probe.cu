// Hardware probe: FP64/FP32 pipe throughput and pinned PCIe bandwidth on the B200 box.
#include <cstdio>
#include <cuda_runtime.h>
#define CK(x) do{cudaError_t e=(x); if(e!=cudaSuccess){printf("ERR %s %s\n",#x,cudaGetErrorString(e)); return 1;}}while(0)

template<int MODE>
__global__ void fp64_loop(double* out, int iters, double a, double b) {
  double x0 = threadIdx.x * 1e-9, x1 = x0 + 1, x2 = x0 + 2, x3 = x0 + 3, x4 = x0+4, x5=x0+5, x6=x0+6, x7=x0+7;
  for (int i = 0; i < iters; ++i) {
#pragma unroll
    for (int k = 0; k < 8; ++k) {
      if (MODE == 0) { x0 = fma(x0, a, b); x1 = fma(x1, a, b); x2 = fma(x2, a, b); x3 = fma(x3, a, b);
                       x4 = fma(x4, a, b); x5 = fma(x5, a, b); x6 = fma(x6, a, b); x7 = fma(x7, a, b); }
      else { x0 = __dadd_rn(x0, b); x1 = __dadd_rn(x1, b); x2 = __dadd_rn(x2, b); x3 = __dadd_rn(x3, b);
             x4 = __dadd_rn(x4, b); x5 = __dadd_rn(x5, b); x6 = __dadd_rn(x6, b); x7 = __dadd_rn(x7, b); }
    }
  }
  out[blockIdx.x * blockDim.x + threadIdx.x] = x0 + x1 + x2 + x3 + x4 + x5 + x6 + x7;
}
__global__ void fp32_loop(float* out, int iters, float a, float b) {
  float x[8]; for (int k=0;k<8;++k) x[k]=threadIdx.x*1e-6f+k;
  for (int i = 0; i < iters; ++i) {
#pragma unroll
    for (int k = 0; k < 8; ++k) {
#pragma unroll
      for (int j=0;j<8;++j) x[j] = fmaf(x[j], a, b);
    }
  }
  float s=0; for (int k=0;k<8;++k) s+=x[k];
  out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}
int main() {
  int dev = 0; cudaDeviceProp p; CK(cudaGetDeviceProperties(&p, dev));
  int clk=0; cudaDeviceGetAttribute(&clk, cudaDevAttrClockRate, dev);
  printf("name=%s sms=%d clock_khz=%d\n", p.name, p.multiProcessorCount, clk);
  int blocks = p.multiProcessorCount * 8, threads = 256, iters = 4096;
  double* d; CK(cudaMalloc(&d, blocks * threads * 8));
  cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
  for (int mode = 0; mode < 2; ++mode) {
    for (int rep = 0; rep < 3; ++rep) {
      cudaEventRecord(e0);
      if (mode == 0) fp64_loop<0><<<blocks, threads>>>(d, iters, 0.999999, 1e-7);
      else fp64_loop<1><<<blocks, threads>>>(d, iters, 0.999999, 1e-7);
      cudaEventRecord(e1); CK(cudaEventSynchronize(e1));
      float ms; cudaEventElapsedTime(&ms, e0, e1);
      double ops = (double)blocks * threads * iters * 64;
      printf("%s: %.3f ms  %.2f Tinstr/s  (%.2f TFLOP/s if fma)\n", mode ? "DADD" : "DFMA", ms, ops / ms / 1e9, (mode?1:2)*ops/ms/1e9);
    }
  }
  for (int rep = 0; rep < 3; ++rep) {
    cudaEventRecord(e0);
    fp32_loop<<<blocks, threads>>>((float*)d, iters, 0.999999f, 1e-7f);
    cudaEventRecord(e1); CK(cudaEventSynchronize(e1));
    float ms; cudaEventElapsedTime(&ms, e0, e1);
    double ops = (double)blocks * threads * iters * 64;
    printf("FFMA: %.3f ms %.2f TFLOP/s\n", ms, 2 * ops / ms / 1e9);
  }
  // PCIe pinned bandwidth
  size_t bytes = 1ull << 30; void* h; CK(cudaHostAlloc(&h, bytes, 0)); void* dd; CK(cudaMalloc(&dd, bytes));
  cudaMemset(dd, 1, bytes);
  for (int rep = 0; rep < 3; ++rep) {
    cudaEventRecord(e0); cudaMemcpyAsync(h, dd, bytes, cudaMemcpyDeviceToHost); cudaEventRecord(e1); cudaEventSynchronize(e1);
    float ms; cudaEventElapsedTime(&ms, e0, e1); printf("D2H 1GiB pinned: %.2f GB/s\n", bytes / ms / 1e6);
    cudaEventRecord(e0); cudaMemcpyAsync(dd, h, bytes, cudaMemcpyHostToDevice); cudaEventRecord(e1); cudaEventSynchronize(e1);
    cudaEventElapsedTime(&ms, e0, e1); printf("H2D 1GiB pinned: %.2f GB/s\n", bytes / ms / 1e6);
  }
  // pageable
  void* hp = malloc(bytes); memset(hp, 0, bytes);
  for (int rep = 0; rep < 2; ++rep) {
    cudaEventRecord(e0); cudaMemcpy(hp, dd, bytes, cudaMemcpyDeviceToHost); cudaEventRecord(e1); cudaEventSynchronize(e1);
    float ms; cudaEventElapsedTime(&ms, e0, e1); printf("D2H 1GiB pageable: %.2f GB/s\n", bytes / ms / 1e6);
  }
  return 0;
}
