// nbody.cu — one all-pairs N-body step (the paper's NBody benchmark,
// Listing 2; absent from the reference, definition in
// SURVEY.md Appendix B / oracle.c:orc_nbody_step).
//
//   acc_i = sum_j m_j * r_ij / (|r_ij|^2 + eps2)^(3/2),  r_ij = p_j - p_i
//   p_i' = p_i + v_i dt + acc_i dt^2 / 2,   v_i' = v_i + acc_i dt
//
// Mapping: a thread integrates B = 4 bodies of the package (two packed
// float2 pairs per coordinate, FFMA2/FADD2/FMUL2) against a contiguous share of every 1024-body source
// tile staged in shared memory as float4 (xyz + mass): each source body is
// read from L2 once per CTA and from shared memory (broadcast) by every
// thread.  Per interaction: 3 FADD, 3 FFMA (|r|^2 + eps2), one MUFU.RSQ,
// 3 FMUL (m/r^3), 3 FFMA (acc) — 12 FP32 operations for the "20
// flops/interaction" convention, issued as 6 packed
// instructions per target, so the attainable ceiling is 20/24 of the FFMA
// peak without the issue slots binding first.  The source split S is chosen per launch so even a
// small package fills every SM (the first profile: 21 % warp occupancy).
#include <cuda_runtime.h>

#include <cstdlib>

#include "kernels.cuh"

namespace ecl {
namespace {

// CTA = kThreads threads = T target slots x S source splits; thread
// (s, t) = threadIdx.x / T, % T integrates B targets (t, t+T, ...) against
// the s-th contiguous quarter/eighth/... of every source tile, so all lanes
// of a warp (same s) read the same shared-memory word (broadcast).  Partial
// accelerations of the S splits are summed in split order at the end.  S > 1
// multiplies the CTAs of a package — small packages (Dynamic at 8 GPUs is
// 32768 bodies) otherwise leave most of the 148 SMs idle.
constexpr int kThreads = 256;
constexpr int kTile = 4 * kThreads;  // sources staged per __syncthreads pair

// 1/sqrt on the MUFU without the denormal-input fixup rsqrtf carries
// (FSETP + 2 predicated FMUL per call): d2 >= eps2 > 0 is never denormal.
__device__ __forceinline__ float rsqrt_ftz(float x) {
  float y;
  asm("rsqrt.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x));
  return y;
}

// One thread integrates 2*B2 targets held as B2 packed pairs (float2 per
// coordinate): every interaction step is an FADD2/FFMA2/FMUL2 on the pair
// (the source body is a broadcast .F32 operand), halving the FP32 issue
// slots; only the two MUFU.RSQ stay scalar.
// Fused exchange: the other devices' output buffers of this step (pos, vel
// per peer); the new state of every body this launch integrates is stored
// there too — the per-step allgather rides on the kernel's own stores over
// NVLink instead of following it as a copy.
struct PeerOut {
  float4* pos[kMaxPeerWrites];
  float4* vel[kMaxPeerWrites];
  uint32_t n;
};

template <int S, int B2, int MB>
__global__ void __launch_bounds__(kThreads, MB)
    nbody_step(const float4* __restrict__ pos, const float4* __restrict__ vel, uint64_t n, float dt, float eps2,
               float4* __restrict__ npos, float4* __restrict__ nvel, uint64_t first, uint64_t count,
               const __grid_constant__ PeerOut peers) {
  constexpr int T = kThreads / S, B = 2 * B2;
  __shared__ float4 tile[kTile];
  __shared__ float3 part[S > 1 ? (S - 1) * B * T : 1];
  const int t = threadIdx.x % T, split = threadIdx.x / T;
  const uint64_t base = first + static_cast<uint64_t>(blockIdx.x) * T * B + t;
  float4 p[B];
#pragma unroll
  for (int b = 0; b < B; ++b) {
    const uint64_t i = base + static_cast<uint64_t>(b) * T;
    p[b] = i < first + count ? pos[i] : make_float4(0.f, 0.f, 0.f, 0.f);
  }
  float2 px[B2], py[B2], pz[B2], ax[B2], ay[B2], az[B2];
#pragma unroll
  for (int h = 0; h < B2; ++h) {
    px[h] = make_float2(p[2 * h].x, p[2 * h + 1].x);
    py[h] = make_float2(p[2 * h].y, p[2 * h + 1].y);
    pz[h] = make_float2(p[2 * h].z, p[2 * h + 1].z);
    ax[h] = ay[h] = az[h] = make_float2(0.f, 0.f);
  }
  const float2 e2 = make_float2(eps2, eps2);
  for (uint64_t t0 = 0; t0 < n; t0 += kTile) {
#pragma unroll
    for (int r = 0; r < kTile / kThreads; ++r) {
      const uint64_t j = t0 + r * kThreads + threadIdx.x;
      tile[r * kThreads + threadIdx.x] = j < n ? pos[j] : make_float4(0.f, 0.f, 0.f, 0.f);  // mass 0: no force
    }
    __syncthreads();
    const float4* src = tile + split * (kTile / S);
#pragma unroll 4
    for (int k = 0; k < kTile / S; ++k) {
      const float4 q = src[k];
#pragma unroll
      for (int h = 0; h < B2; ++h) {
        const float2 rx = __fadd2_rn(make_float2(q.x, q.x), make_float2(-px[h].x, -px[h].y));
        const float2 ry = __fadd2_rn(make_float2(q.y, q.y), make_float2(-py[h].x, -py[h].y));
        const float2 rz = __fadd2_rn(make_float2(q.z, q.z), make_float2(-pz[h].x, -pz[h].y));
        const float2 d2 = __ffma2_rn(rx, rx, __ffma2_rn(ry, ry, __ffma2_rn(rz, rz, e2)));
        const float2 inv = make_float2(rsqrt_ftz(d2.x), rsqrt_ftz(d2.y));
        const float2 s = __fmul2_rn(__fmul2_rn(make_float2(q.w, q.w), inv), __fmul2_rn(inv, inv));
        ax[h] = __ffma2_rn(s, rx, ax[h]);
        ay[h] = __ffma2_rn(s, ry, ay[h]);
        az[h] = __ffma2_rn(s, rz, az[h]);
      }
    }
    __syncthreads();
  }
  float3 acc[B];
#pragma unroll
  for (int h = 0; h < B2; ++h) {
    acc[2 * h] = make_float3(ax[h].x, ay[h].x, az[h].x);
    acc[2 * h + 1] = make_float3(ax[h].y, ay[h].y, az[h].y);
  }
  if constexpr (S > 1) {
    if (split > 0) {
#pragma unroll
      for (int b = 0; b < B; ++b) part[((split - 1) * B + b) * T + t] = acc[b];
    }
    __syncthreads();
    if (split > 0) return;
#pragma unroll
    for (int b = 0; b < B; ++b)
      for (int s2 = 1; s2 < S; ++s2) {
        const float3 q = part[((s2 - 1) * B + b) * T + t];
        acc[b].x += q.x;
        acc[b].y += q.y;
        acc[b].z += q.z;
      }
  }
  const float hdt2 = 0.5f * dt * dt;
#pragma unroll
  for (int b = 0; b < B; ++b) {
    const uint64_t i = base + static_cast<uint64_t>(b) * T;
    if (i >= first + count) continue;
    const float4 v = vel[i];
    const float4 np = make_float4(p[b].x + v.x * dt + acc[b].x * hdt2, p[b].y + v.y * dt + acc[b].y * hdt2,
                                  p[b].z + v.z * dt + acc[b].z * hdt2, p[b].w);
    const float4 nv = make_float4(v.x + acc[b].x * dt, v.y + acc[b].y * dt, v.z + acc[b].z * dt, v.w);
    npos[i] = np;
    nvel[i] = nv;
    for (uint32_t q = 0; q < peers.n; ++q) {
      if (peers.pos[q]) peers.pos[q][i] = np;
      if (peers.vel[q]) peers.vel[q][i] = nv;
    }
  }
}

template <int S, int B2, int MB = 1>
cudaError_t launch(const KernelSpec& spec, const LaunchEnv& env, uint64_t first, uint64_t count) {
  const uint64_t per_block = static_cast<uint64_t>(kThreads / S) * 2 * B2;
  const uint64_t blocks = (count + per_block - 1) / per_block;
  PeerOut peers{};
  peers.n = env.n_peers < kMaxPeerWrites ? env.n_peers : kMaxPeerWrites;
  for (uint32_t q = 0; q < peers.n; ++q) {
    peers.pos[q] = static_cast<float4*>(env.peer_out[2 * q]);
    peers.vel[q] = static_cast<float4*>(env.peer_out[2 * q + 1]);
  }
  nbody_step<S, B2, MB><<<static_cast<unsigned>(blocks), kThreads, 0, env.stream>>>(
      static_cast<const float4*>(env.in[0]), static_cast<const float4*>(env.in[1]), spec.nbody.bodies,
      spec.nbody.dt, spec.nbody.eps2, static_cast<float4*>(env.out[0]), static_cast<float4*>(env.out[1]), first,
      count, peers);
  return cudaGetLastError();
}

}  // namespace

cudaError_t launch_nbody(const KernelSpec& spec, const LaunchEnv& env, uint64_t first, uint64_t count) {
  if (count == 0) return cudaSuccess;
  // Source splits: the fewest that still give ~4 CTAs per SM for this
  // package (ECL_NBODY_SPLIT forces 1/2/4/8).
  static const int forced = [] {
    const char* v = std::getenv("ECL_NBODY_SPLIT");
    return v ? std::atoi(v) : 0;
  }();
  // ECL_NBODY_PAIRS: target pairs per thread (2 measured 4.6 % faster than 1;
  // 3 pairs — six targets, 78 registers, 3 CTAs/SM — 435 vs 428 ms per step)
  static const int env_pairs = [] {
    const char* v = std::getenv("ECL_NBODY_PAIRS");
    return v && std::atoi(v) == 1 ? 1 : 2;
  }();
  const int pairs = spec.variant == 1 ? 1 : spec.variant == 0 ? 2 : env_pairs;  // nbody@1: one pair
  const int B = 2 * pairs;
  const uint64_t want = 4ull * static_cast<uint64_t>(env.sms > 0 ? env.sms : 148);
  int split = forced;
  if (split <= 0) {
    split = 1;
    while (split < 8 && (count + (kThreads / split) * B - 1) / ((kThreads / split) * B) < want) split *= 2;
  }
  // ECL_NBODY_MB: resident CTAs per SM the registers are sized for.  Measured
  // per 1M-body step: 2 (108 regs) 426.0 ms, 4 (64) 427.7, 5 435.2, 6 451.6.
  static const int mb = [] {
    const char* v = std::getenv("ECL_NBODY_MB");
    return v ? std::atoi(v) : 0;
  }();
  if (pairs == 2 && mb == 5) {
    switch (split) {
      case 1: return launch<1, 2, 5>(spec, env, first, count);
      case 2: return launch<2, 2, 5>(spec, env, first, count);
      case 4: return launch<4, 2, 5>(spec, env, first, count);
      default: return launch<8, 2, 5>(spec, env, first, count);
    }
  }
  if (pairs == 2 && mb == 6) {
    switch (split) {
      case 1: return launch<1, 2, 6>(spec, env, first, count);
      case 2: return launch<2, 2, 6>(spec, env, first, count);
      case 4: return launch<4, 2, 6>(spec, env, first, count);
      default: return launch<8, 2, 6>(spec, env, first, count);
    }
  }
  if (pairs == 2 && mb == 2) {
    switch (split) {
      case 1: return launch<1, 2, 2>(spec, env, first, count);
      case 2: return launch<2, 2, 2>(spec, env, first, count);
      case 4: return launch<4, 2, 2>(spec, env, first, count);
      default: return launch<8, 2, 2>(spec, env, first, count);
    }
  }
  if (pairs == 2) {
    switch (split) {
      case 1: return launch<1, 2, 4>(spec, env, first, count);
      case 2: return launch<2, 2, 4>(spec, env, first, count);
      case 4: return launch<4, 2, 4>(spec, env, first, count);
      default: return launch<8, 2, 4>(spec, env, first, count);
    }
  }
  switch (split) {
    case 1: return launch<1, 1>(spec, env, first, count);
    case 2: return launch<2, 1>(spec, env, first, count);
    case 4: return launch<4, 1>(spec, env, first, count);
    default: return launch<8, 1>(spec, env, first, count);
  }
}

}  // namespace ecl
