// nbody.cu — one all-pairs N-body step (the paper's NBody benchmark,
// Listing 2; absent from the reference, definition in
// SURVEY.md Appendix B / oracle.c:orc_nbody_step).
//
//   acc_i = sum_j m_j * r_ij / (|r_ij|^2 + eps2)^(3/2),  r_ij = p_j - p_i
//   p_i' = p_i + v_i dt + acc_i dt^2 / 2,   v_i' = v_i + acc_i dt
//
// Mapping: a thread integrates kBodies consecutive bodies of the package
// (independent accumulator chains for ILP); the CTA walks the whole body
// array in 256-body tiles staged in shared memory as float4 (xyz + mass), so
// each source body is read from HBM/L2 once per CTA and from shared memory
// (broadcast, conflict-free) by every thread.  Per interaction: 3 FADD,
// 3 FFMA (|r|^2 + eps2), one MUFU.RSQ, 3 FMUL (m/r^3), 3 FFMA (acc):
// FP32-pipe bound (the "20 flops/interaction" convention).
#include <cuda_runtime.h>

#include "kernels.cuh"

namespace ecl {
namespace {

constexpr int kThreads = 256;
constexpr int kBodies = 2;  // bodies per thread

__global__ void __launch_bounds__(kThreads)
    nbody_step(const float4* __restrict__ pos, const float4* __restrict__ vel, uint64_t n, float dt, float eps2,
               float4* __restrict__ npos, float4* __restrict__ nvel, uint64_t first, uint64_t count) {
  __shared__ float4 tile[kThreads];
  const uint64_t base = first + (static_cast<uint64_t>(blockIdx.x) * kThreads * kBodies) + threadIdx.x;
  float4 p[kBodies];
  float ax[kBodies], ay[kBodies], az[kBodies];
#pragma unroll
  for (int b = 0; b < kBodies; ++b) {
    const uint64_t i = base + static_cast<uint64_t>(b) * kThreads;
    p[b] = i < first + count ? pos[i] : make_float4(0.f, 0.f, 0.f, 0.f);
    ax[b] = ay[b] = az[b] = 0.0f;
  }
  for (uint64_t t0 = 0; t0 < n; t0 += kThreads) {
    const uint64_t j = t0 + threadIdx.x;
    tile[threadIdx.x] = j < n ? pos[j] : make_float4(0.f, 0.f, 0.f, 0.f);  // mass 0: no force
    __syncthreads();
    const int lim = n - t0 < static_cast<uint64_t>(kThreads) ? static_cast<int>(n - t0) : kThreads;
#pragma unroll 8
    for (int k = 0; k < lim; ++k) {
      const float4 q = tile[k];
#pragma unroll
      for (int b = 0; b < kBodies; ++b) {
        const float rx = q.x - p[b].x, ry = q.y - p[b].y, rz = q.z - p[b].z;
        const float d2 = fmaf(rx, rx, fmaf(ry, ry, fmaf(rz, rz, eps2)));
        const float inv = rsqrtf(d2);
        const float s = q.w * (inv * inv * inv);
        ax[b] = fmaf(s, rx, ax[b]);
        ay[b] = fmaf(s, ry, ay[b]);
        az[b] = fmaf(s, rz, az[b]);
      }
    }
    __syncthreads();
  }
  const float hdt2 = 0.5f * dt * dt;
#pragma unroll
  for (int b = 0; b < kBodies; ++b) {
    const uint64_t i = base + static_cast<uint64_t>(b) * kThreads;
    if (i >= first + count) continue;
    const float4 v = vel[i];
    npos[i] = make_float4(p[b].x + v.x * dt + ax[b] * hdt2, p[b].y + v.y * dt + ay[b] * hdt2,
                          p[b].z + v.z * dt + az[b] * hdt2, p[b].w);
    nvel[i] = make_float4(v.x + ax[b] * dt, v.y + ay[b] * dt, v.z + az[b] * dt, v.w);
  }
}

}  // namespace

cudaError_t launch_nbody(const KernelSpec& spec, const LaunchEnv& env, uint64_t first, uint64_t count) {
  if (count == 0) return cudaSuccess;
  const uint64_t per_block = static_cast<uint64_t>(kThreads) * kBodies;
  const uint64_t blocks = (count + per_block - 1) / per_block;
  nbody_step<<<static_cast<unsigned>(blocks), kThreads, 0, env.stream>>>(
      static_cast<const float4*>(env.in[0]), static_cast<const float4*>(env.in[1]), spec.nbody.bodies,
      spec.nbody.dt, spec.nbody.eps2, static_cast<float4*>(env.out[0]), static_cast<float4*>(env.out[1]), first,
      count);
  return cudaGetLastError();
}

}  // namespace ecl
