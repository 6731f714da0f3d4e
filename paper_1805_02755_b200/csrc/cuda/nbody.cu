// nbody.cu — one all-pairs N-body step (the paper's NBody benchmark,
// Listing 2; absent from the reference, definition in
// SURVEY.md Appendix B / oracle.c:orc_nbody_step).
//
//   acc_i = sum_j m_j * r_ij / (|r_ij|^2 + eps2)^(3/2),  r_ij = p_j - p_i
//   p_i' = p_i + v_i dt + acc_i dt^2 / 2,   v_i' = v_i + acc_i dt
//
// Mapping: a thread integrates B consecutive-in-block bodies of the package
// (independent accumulator chains); the CTA walks the whole body array in
// T-body tiles staged in shared memory as float4 (xyz + mass), so each
// source body is read from L2 once per CTA and from shared memory
// (broadcast) by every thread.  Per interaction: 3 FADD, 3 FFMA
// (|r|^2 + eps2), one MUFU.RSQ, 3 FMUL (m/r^3), 3 FFMA (acc): FP32-pipe
// bound (the "20 flops/interaction" convention).  The grid is
// sized so a package of 1M/8 bodies gives every SM several CTAs (the first
// profile showed < 2 CTAs/SM and 21 % warp occupancy with 512-body CTAs).
#include <cuda_runtime.h>

#include <cstdlib>

#include "kernels.cuh"

namespace ecl {
namespace {

template <int T, int B>
__global__ void __launch_bounds__(T)
    nbody_step(const float4* __restrict__ pos, const float4* __restrict__ vel, uint64_t n, float dt, float eps2,
               float4* __restrict__ npos, float4* __restrict__ nvel, uint64_t first, uint64_t count) {
  __shared__ float4 tile[T];
  const uint64_t base = first + (static_cast<uint64_t>(blockIdx.x) * T * B) + threadIdx.x;
  float4 p[B];
  float ax[B], ay[B], az[B];
#pragma unroll
  for (int b = 0; b < B; ++b) {
    const uint64_t i = base + static_cast<uint64_t>(b) * T;
    p[b] = i < first + count ? pos[i] : make_float4(0.f, 0.f, 0.f, 0.f);
    ax[b] = ay[b] = az[b] = 0.0f;
  }
  for (uint64_t t0 = 0; t0 < n; t0 += T) {
    const uint64_t j = t0 + threadIdx.x;
    tile[threadIdx.x] = j < n ? pos[j] : make_float4(0.f, 0.f, 0.f, 0.f);  // mass 0: no force
    __syncthreads();
    const int lim = n - t0 < static_cast<uint64_t>(T) ? static_cast<int>(n - t0) : T;
#pragma unroll 8
    for (int k = 0; k < lim; ++k) {
      const float4 q = tile[k];
#pragma unroll
      for (int b = 0; b < B; ++b) {
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
  for (int b = 0; b < B; ++b) {
    const uint64_t i = base + static_cast<uint64_t>(b) * T;
    if (i >= first + count) continue;
    const float4 v = vel[i];
    npos[i] = make_float4(p[b].x + v.x * dt + ax[b] * hdt2, p[b].y + v.y * dt + ay[b] * hdt2,
                          p[b].z + v.z * dt + az[b] * hdt2, p[b].w);
    nvel[i] = make_float4(v.x + ax[b] * dt, v.y + ay[b] * dt, v.z + az[b] * dt, v.w);
  }
}

template <int T, int B>
cudaError_t launch(const KernelSpec& spec, const LaunchEnv& env, uint64_t first, uint64_t count) {
  const uint64_t per_block = static_cast<uint64_t>(T) * B;
  const uint64_t blocks = (count + per_block - 1) / per_block;
  nbody_step<T, B><<<static_cast<unsigned>(blocks), T, 0, env.stream>>>(
      static_cast<const float4*>(env.in[0]), static_cast<const float4*>(env.in[1]), spec.nbody.bodies,
      spec.nbody.dt, spec.nbody.eps2, static_cast<float4*>(env.out[0]), static_cast<float4*>(env.out[1]), first,
      count);
  return cudaGetLastError();
}

}  // namespace

cudaError_t launch_nbody(const KernelSpec& spec, const LaunchEnv& env, uint64_t first, uint64_t count) {
  if (count == 0) return cudaSuccess;
  // Tuning hook (ECL_NBODY_VARIANT): CTA size x bodies per thread.
  static const int variant = [] {
    const char* v = std::getenv("ECL_NBODY_VARIANT");
    return v ? std::atoi(v) : 0;
  }();
  switch (variant) {
    case 1: return launch<256, 2>(spec, env, first, count);  // the first version
    case 2: return launch<256, 1>(spec, env, first, count);
    case 3: return launch<64, 2>(spec, env, first, count);
    case 4: return launch<128, 4>(spec, env, first, count);
    default: return launch<128, 2>(spec, env, first, count);
  }
}

}  // namespace ecl
