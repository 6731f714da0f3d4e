// Host cost of cudaLaunchKernel on this box: an empty kernel with a small
// parameter, with a ~400 B and a ~8 KB __grid_constant__ parameter, and with
// 63 KB of opted-in dynamic shared memory.  Mean host time per launch over
// 2000 asynchronous launches on one stream.
#include <chrono>
#include <cstdio>
#include <cuda_runtime.h>

struct P400 { float v[100]; };
struct P8K { float v[2000]; };
__global__ void k_small(int x) { if (x == -1) asm volatile("trap;"); }
__global__ void k_400(const __grid_constant__ P400 p) { if (p.v[0] == -1.f) asm volatile("trap;"); }
__global__ void k_8k(const __grid_constant__ P8K p) { if (p.v[0] == -1.f) asm volatile("trap;"); }
__global__ void k_smem(int x) { extern __shared__ float s[]; if (x == -1) s[threadIdx.x] = 0; }

template <typename F>
double per_launch_us(F launch) {
  cudaStream_t st;
  cudaStreamCreateWithFlags(&st, cudaStreamNonBlocking);
  for (int i = 0; i < 100; ++i) launch(st);
  cudaStreamSynchronize(st);
  const int n = 2000;
  const auto t0 = std::chrono::steady_clock::now();
  for (int i = 0; i < n; ++i) launch(st);
  const auto t1 = std::chrono::steady_clock::now();
  cudaStreamSynchronize(st);
  cudaStreamDestroy(st);
  return std::chrono::duration<double, std::micro>(t1 - t0).count() / n;
}

int main() {
  P400 p4{};
  P8K p8{};
  cudaFuncSetAttribute(k_smem, cudaFuncAttributeMaxDynamicSharedMemorySize, 63 * 1024);
  printf("small param       %.2f us\n", per_launch_us([](cudaStream_t s) { k_small<<<128, 256, 0, s>>>(1); }));
  printf("400 B param       %.2f us\n", per_launch_us([&](cudaStream_t s) { k_400<<<128, 256, 0, s>>>(p4); }));
  printf("8 KB param        %.2f us\n", per_launch_us([&](cudaStream_t s) { k_8k<<<128, 256, 0, s>>>(p8); }));
  printf("63 KB dyn smem    %.2f us\n", per_launch_us([](cudaStream_t s) { k_smem<<<128, 256, 63 * 1024, s>>>(1); }));
  return 0;
}
