// What bounds the Binomial lattice?  The packed two-option lattice of
// binomial.cu (8 nodes per lane, one shuffle per level, phases of 32 levels
// with a shared-memory repack) timed alone on constants, against variants
// that each remove one ingredient:
//   full     — as binomial.cu (254 levels, repack to NL-1 every 32 levels)
//   noshfl   — the neighbour is the lane's own c[0] (wrong values, no SHFL)
//   smemx    — the neighbour exchanged through shared memory instead
//   dual     — two option pairs per warp advanced in lockstep (twice the
//              independent work between exchanges)
//   halo4    — like flat, but each lane also carries a 4-node halo (the
//              neighbour's first 4 nodes, updated redundantly) and exchanges
//              it every 4 levels: a quarter of the exchange events, the same
//              shuffled words, +25 % FFMA2
//   flat     — no repack: all 254 levels at 8 nodes per lane
//   u4 / u16 — unroll 4 / 16 instead of 8
//   half     — two pairs per warp, 16 nodes per lane, phases of 16 levels
//              (binomial.cu's binomial_half: half the shuffles per node)
//   g4       — four lanes per pair, 64 nodes per lane (8 pairs per warp, one
//              shuffle pair per level serves all 8), repacked down a menu of
//              node counts (64, 56, ..., 1) through shared memory
// Grid: one warp per option pair, 4.19M pairs (the 8M-option config).
// Measured (B200): full 14.9 ms, noshfl 9.9, smemx 19.7, dual 14.9, flat 19.2, halo4 20.4 (vs flat), u4 15.6, u16 14.7,
// half 17.3-18.1 (12.3 without shuffles), g4 21.2 (16.3 without shuffles,
// 163 registers: one CTA per SM).  Removing the shuffles saves ~5 ms in every
// layout, also in g4 where they are 8x rarer per option: the cost is not the
// shuffle unit's throughput.
// Build: nvcc -O3 -std=c++17 -gencode arch=compute_100a,code=sm_100a binomial_lattice.cu -o binomial_lattice
#include <cuda_runtime.h>

#include <cstdint>
#include <cstdio>

constexpr int kThreads = 256;

template <bool Shfl, int U>
__device__ __forceinline__ int backward8(float2 (&c)[8], int j, int stop, float2 r) {
#pragma unroll U
  for (; j > stop; --j) {
    float2 right;
    if (Shfl)
      right = make_float2(__shfl_down_sync(0xffffffffu, c[0].x, 1), __shfl_down_sync(0xffffffffu, c[0].y, 1));
    else
      right = c[0];
#pragma unroll
    for (int k = 0; k < 7; ++k) c[k] = __ffma2_rn(r, c[k + 1], c[k]);
    c[7] = __ffma2_rn(r, right, c[7]);
  }
  return j;
}

template <int NL, bool Shfl, int U, int G = 32, bool Smem = false>
__device__ __forceinline__ float2 phases(float2 (&c)[NL], int j, float2 r, float2 s, float2* buf, unsigned lane) {
  const int stop = NL > 1 ? G * (NL - 1) - 1 : 0;
  if (j > stop) {
#pragma unroll U
    for (; j > stop; --j) {
      float2 right;
      if (Smem) {
        float2* x = buf + 256 - 64 + 32 * (j & 1);  // double-buffered exchange slots
        x[lane] = c[0];
        __syncwarp();
        right = x[(lane + 1) & 31];
      } else if (Shfl)
        right = make_float2(__shfl_down_sync(0xffffffffu, c[0].x, 1, G), __shfl_down_sync(0xffffffffu, c[0].y, 1, G));
      else
        right = c[0];
#pragma unroll
      for (int k = 0; k < NL - 1; ++k) c[k] = __ffma2_rn(r, c[k + 1], c[k]);
      c[NL - 1] = __ffma2_rn(r, right, c[NL - 1]);
    }
    if constexpr (NL > 1) {
#pragma unroll
      for (int k = 0; k < NL; ++k) c[k] = __fmul2_rn(c[k], s);
    }
  }
  if constexpr (NL == 1) {
    return c[0];
  } else {
#pragma unroll
    for (int k = 0; k < NL; ++k) buf[NL * lane + k] = c[k];
    __syncwarp();
    float2 h[NL - 1];
#pragma unroll
    for (int k = 0; k < NL - 1; ++k) h[k] = buf[(NL - 1) * lane + k];
    __syncwarp();
    return phases<NL - 1, Shfl, U, G, Smem>(h, j, r, s, buf, lane);
  }
}

template <int NL>
__device__ __forceinline__ float2 phases2(float2 (&c)[NL], float2 (&e)[NL], int j, float2 r, float2 s, float2* buf,
                                          unsigned lane, float2* out_e) {
  const int stop = NL > 1 ? 32 * (NL - 1) - 1 : 0;
  if (j > stop) {
#pragma unroll 4
    for (; j > stop; --j) {
      const float2 rc = make_float2(__shfl_down_sync(0xffffffffu, c[0].x, 1), __shfl_down_sync(0xffffffffu, c[0].y, 1));
      const float2 re = make_float2(__shfl_down_sync(0xffffffffu, e[0].x, 1), __shfl_down_sync(0xffffffffu, e[0].y, 1));
#pragma unroll
      for (int k = 0; k < NL - 1; ++k) {
        c[k] = __ffma2_rn(r, c[k + 1], c[k]);
        e[k] = __ffma2_rn(r, e[k + 1], e[k]);
      }
      c[NL - 1] = __ffma2_rn(r, rc, c[NL - 1]);
      e[NL - 1] = __ffma2_rn(r, re, e[NL - 1]);
    }
  }
  if constexpr (NL == 1) {
    *out_e = e[0];
    return c[0];
  } else {
#pragma unroll
    for (int k = 0; k < NL; ++k) {
      buf[NL * lane + k] = __fmul2_rn(c[k], s);
      buf[256 + NL * lane + k] = __fmul2_rn(e[k], s);
    }
    __syncwarp();
    float2 h[NL - 1], g[NL - 1];
#pragma unroll
    for (int k = 0; k < NL - 1; ++k) {
      h[k] = buf[(NL - 1) * lane + k];
      g[k] = buf[256 + (NL - 1) * lane + k];
    }
    __syncwarp();
    return phases2<NL - 1>(h, g, j, r, s, buf, lane, out_e);
  }
}

template <int MB>
__global__ void __launch_bounds__(kThreads, MB) lattice_dual(float* out, uint64_t pairs, int steps) {
  __shared__ float2 buf_all[kThreads / 32][512];
  const unsigned lane = threadIdx.x & 31u;
  float2* buf = buf_all[threadIdx.x >> 5];
  const uint64_t warps = static_cast<uint64_t>(gridDim.x) * (kThreads / 32);
  for (uint64_t w = blockIdx.x * static_cast<uint64_t>(kThreads / 32) + (threadIdx.x >> 5); 2 * w < pairs;
       w += warps) {
    float2 c[8], e[8];
#pragma unroll
    for (int k = 0; k < 8; ++k) {
      c[k] = make_float2(1.0f + 1e-3f * (lane * 8 + k) + 1e-9f * w, 2.0f - 1e-3f * k);
      e[k] = make_float2(1.5f + 1e-3f * (lane * 8 + k) + 1e-9f * w, 2.5f - 1e-3f * k);
    }
    const float2 r = make_float2(0.999f, 0.998f), s = make_float2(0.97f, 0.96f);
    float2 ve;
    const float2 v = phases2<8>(c, e, steps, r, s, buf, lane, &ve);
    if (lane == 0) out[w] = v.x + v.y + ve.x + ve.y;
  }
}

template <int MB>
void run_dual(const char* name, float* d, uint64_t pairs) {
  cudaEvent_t a, b;
  cudaEventCreate(&a);
  cudaEventCreate(&b);
  const unsigned blocks = 148 * 8 * 16;
  float best = 1e9f;
  for (int rep = 0; rep < 4; ++rep) {
    cudaEventRecord(a);
    lattice_dual<MB><<<blocks, kThreads>>>(d, pairs, 254);
    cudaEventRecord(b);
    cudaEventSynchronize(b);
    float ms;
    cudaEventElapsedTime(&ms, a, b);
    if (rep && ms < best) best = ms;
  }
  printf("%-8s MB=%d %.3f ms  %s\n", name, MB, best, cudaGetErrorString(cudaGetLastError()));
}

__device__ __forceinline__ void halo4_steps(float2 (&c)[8], int j, int stop, float2 r) {
  float2 h[4];
  for (; j > stop;) {
#pragma unroll
    for (int k = 0; k < 4; ++k)
      h[k] = make_float2(__shfl_down_sync(0xffffffffu, c[k].x, 1), __shfl_down_sync(0xffffffffu, c[k].y, 1));
#pragma unroll
    for (int s = 0; s < 4; ++s) {  // 4 levels on own + halo nodes (halo shrinks by one per level)
#pragma unroll
      for (int k = 0; k < 7; ++k) c[k] = __ffma2_rn(r, c[k + 1], c[k]);
      c[7] = __ffma2_rn(r, h[0], c[7]);
#pragma unroll
      for (int k = 0; k < 3 - s; ++k) h[k] = __ffma2_rn(r, h[k + 1], h[k]);
    }
    j -= 4;
  }
}

template <int Mode, int U>
__global__ void __launch_bounds__(kThreads, 4) lattice(float* out, uint64_t pairs, int steps) {
  __shared__ float2 buf_all[kThreads / 32][256];
  const unsigned lane = threadIdx.x & 31u;
  float2* buf = buf_all[threadIdx.x >> 5];
  const uint64_t warps = static_cast<uint64_t>(gridDim.x) * (kThreads / 32);
  for (uint64_t w = blockIdx.x * static_cast<uint64_t>(kThreads / 32) + (threadIdx.x >> 5); w < pairs; w += warps) {
    float2 c[8];
#pragma unroll
    for (int k = 0; k < 8; ++k) c[k] = make_float2(1.0f + 1e-3f * (lane * 8 + k) + 1e-9f * w, 2.0f - 1e-3f * k);
    const float2 r = make_float2(0.999f, 0.998f), s = make_float2(0.97f, 0.96f);
    float2 v;
    if (Mode == 0) v = phases<8, true, U>(c, steps, r, s, buf, lane);
    else if (Mode == 3) v = phases<8, false, U, 32, true>(c, steps, r, s, buf, lane);
    else if (Mode == 4) {
      halo4_steps(c, steps, 0, r);
      v = c[0];
    }
    else if (Mode == 1) v = phases<8, false, U>(c, steps, r, s, buf, lane);
    else {
      backward8<true, U>(c, steps, 0, r);
      v = c[0];
    }
    if (lane == 0) out[w] = v.x + v.y;
  }
}

template <bool Shfl, int MB>
__global__ void __launch_bounds__(kThreads, MB) lattice_half(float* out, uint64_t pairs, int steps) {
  __shared__ float2 buf_all[kThreads / 16][256];
  const unsigned lane = threadIdx.x & 15u;
  float2* buf = buf_all[threadIdx.x >> 4];
  const uint64_t halves = static_cast<uint64_t>(gridDim.x) * (kThreads / 16);
  for (uint64_t w = blockIdx.x * static_cast<uint64_t>(kThreads / 16) + (threadIdx.x >> 4); w < pairs;
       w += halves) {
    float2 c[16];
#pragma unroll
    for (int k = 0; k < 16; ++k) c[k] = make_float2(1.0f + 1e-3f * (lane * 16 + k) + 1e-9f * w, 2.0f - 1e-3f * k);
    const float2 r = make_float2(0.999f, 0.998f), s = make_float2(0.97f, 0.96f);
    const float2 v = phases<16, Shfl, 8, 16>(c, steps, r, s, buf, lane);
    if (lane == 0) out[w] = v.x + v.y;
  }
}

template <bool Shfl, int MB>
void run_half(const char* name, float* d, uint64_t pairs) {
  cudaEvent_t a, b;
  cudaEventCreate(&a);
  cudaEventCreate(&b);
  const unsigned blocks = 148 * 8 * 16;
  float best = 1e9f;
  for (int rep = 0; rep < 4; ++rep) {
    cudaEventRecord(a);
    lattice_half<Shfl, MB><<<blocks, kThreads>>>(d, pairs, 254);
    cudaEventRecord(b);
    cudaEventSynchronize(b);
    float ms;
    cudaEventElapsedTime(&ms, a, b);
    if (rep && ms < best) best = ms;
  }
  printf("%-8s MB=%d %.3f ms\n", name, MB, best);
}

// Next node count of the G=4 menu.
__host__ __device__ constexpr int next_nl(int nl) {
  return nl > 32 ? nl - 8 : nl > 16 ? nl - 4 : nl > 8 ? nl - 2 : nl - 1;
}

template <int NL, bool Shfl>
__device__ __forceinline__ float2 phases4(float2 (&c)[NL], int j, float2 r, float2 s, float2* buf, unsigned lane) {
  constexpr int NN = NL > 1 ? next_nl(NL) : 0;
  const int stop = NL > 1 ? 4 * NN - 1 : 0;
  if (j > stop) {
#pragma unroll 2
    for (; j > stop; --j) {
      float2 right;
      if (Shfl)
        right = make_float2(__shfl_down_sync(0xffffffffu, c[0].x, 1, 4), __shfl_down_sync(0xffffffffu, c[0].y, 1, 4));
      else
        right = c[0];
#pragma unroll
      for (int k = 0; k < NL - 1; ++k) c[k] = __ffma2_rn(r, c[k + 1], c[k]);
      c[NL - 1] = __ffma2_rn(r, right, c[NL - 1]);
    }
  }
  if constexpr (NL == 1) {
    return c[0];
  } else {
#pragma unroll
    for (int k = 0; k < NL; ++k) buf[NL * lane + k] = __fmul2_rn(c[k], s);
    __syncwarp();
    float2 h[NN];
#pragma unroll
    for (int k = 0; k < NN; ++k) h[k] = buf[NN * lane + k];
    __syncwarp();
    return phases4<NN, Shfl>(h, j, r, s, buf, lane);
  }
}

template <bool Shfl, int MB>
__global__ void __launch_bounds__(kThreads, MB) lattice_g4(float* out, uint64_t pairs, int steps) {
  extern __shared__ float2 dyn[];
  const unsigned lane = threadIdx.x & 3u;
  float2* buf = dyn + (threadIdx.x >> 2) * 256;
  const uint64_t groups = static_cast<uint64_t>(gridDim.x) * (kThreads / 4);
  for (uint64_t w = blockIdx.x * static_cast<uint64_t>(kThreads / 4) + (threadIdx.x >> 2); w < pairs; w += groups) {
    float2 c[64];
#pragma unroll
    for (int k = 0; k < 64; ++k) c[k] = make_float2(1.0f + 1e-3f * (lane * 64 + k) + 1e-9f * w, 2.0f - 1e-3f * k);
    const float2 r = make_float2(0.999f, 0.998f), s = make_float2(0.97f, 0.96f);
    const float2 v = phases4<64, Shfl>(c, steps, r, s, buf, lane);
    if (lane == 0) out[w] = v.x + v.y;
  }
}

template <bool Shfl, int MB>
void run_g4(const char* name, float* d, uint64_t pairs) {
  cudaEvent_t a, b;
  cudaEventCreate(&a);
  cudaEventCreate(&b);
  const size_t smem = (kThreads / 4) * 256 * sizeof(float2);
  cudaFuncSetAttribute(lattice_g4<Shfl, MB>, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(smem));
  int occ = 0;
  cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, lattice_g4<Shfl, MB>, kThreads, smem);
  const unsigned blocks = 148 * occ;
  float best = 1e9f;
  for (int rep = 0; rep < 4; ++rep) {
    cudaEventRecord(a);
    lattice_g4<Shfl, MB><<<blocks, kThreads, smem>>>(d, pairs, 254);
    cudaEventRecord(b);
    cudaEventSynchronize(b);
    float ms;
    cudaEventElapsedTime(&ms, a, b);
    if (rep && ms < best) best = ms;
  }
  printf("%-8s MB=%d occ=%d %.3f ms  %s\n", name, MB, occ, best, cudaGetErrorString(cudaGetLastError()));
}

template <int Mode, int U>
void run(const char* name, float* d, uint64_t pairs) {
  cudaEvent_t a, b;
  cudaEventCreate(&a);
  cudaEventCreate(&b);
  const unsigned blocks = 148 * 8 * 16;
  float best = 1e9f;
  for (int rep = 0; rep < 4; ++rep) {
    cudaEventRecord(a);
    lattice<Mode, U><<<blocks, kThreads>>>(d, pairs, 254);
    cudaEventRecord(b);
    cudaEventSynchronize(b);
    float ms;
    cudaEventElapsedTime(&ms, a, b);
    if (rep && ms < best) best = ms;
  }
  printf("%-8s %.3f ms\n", name, best);
}

int main() {
  const uint64_t pairs = 1ull << 22;
  float* d;
  cudaMalloc(&d, pairs * 4);
  run<0, 8>("full", d, pairs);
  run<1, 8>("noshfl", d, pairs);
  run<2, 8>("flat", d, pairs);
  run<3, 8>("smemx", d, pairs);
  run<4, 8>("halo4", d, pairs);
  run<0, 4>("u4", d, pairs);
  run<0, 16>("u16", d, pairs);
  run_half<true, 2>("half", d, pairs);
  run_half<true, 3>("half", d, pairs);
  run_half<true, 4>("half", d, pairs);
  run_half<false, 3>("halfnosh", d, pairs);
  run_dual<2>("dual", d, pairs);
  run_dual<3>("dual", d, pairs);
  run_g4<true, 1>("g4", d, pairs);
  run_g4<false, 1>("g4nosh", d, pairs);
  const cudaError_t e = cudaDeviceSynchronize();
  printf("%s\n", cudaGetErrorString(e));
  return 0;
}
