// binomial.cu — European call on a Cox-Ross-Rubinstein lattice (the paper's
// Binomial Options benchmark, Listing 1; absent from the
// reference, definition in SURVEY.md Appendix B / oracle.c:orc_binomial).
//
// Program shape (Table 2): lws = steps + 1 work-items per work-group, one
// float4 (four options) per work-group, out pattern 1:lws.  A package of
// work-groups [o, o+n) is options [4o, 4(o+n)).
//
// Mapping: one warp per option.  Lane l holds lattice nodes
// t = 8l .. 8l+7 in registers (255 nodes for 254 steps); a backward step
//   c[t] <- puByr * c[t+1] + pdByr * c[t]      (t < j)
// is 8 register updates per lane plus one warp shuffle for the neighbour
// node c[8l+8] held by lane l+1 — the OpenCL kernel's local-memory lattice
// and barriers become registers and __shfl_down_sync.  Per-option
// parameters (dt, u, d, pu/a, pd/a) are formed in FP64 so the subtraction
// a - d does not lose the 1e-5 relative budget; the lattice itself is FP32.
#include <cuda_runtime.h>

#include "kernels.cuh"

namespace ecl {
namespace {

constexpr int kThreads = 256;
constexpr int kNodesPerLane = 8;  // 32 x 8 = 256 >= steps + 1 for steps <= 255

// Backward steps j, j-1, ... while j > stop, with NL nodes per lane (lane l
// holds nodes NL*l .. NL*l+NL-1): c[t] <- c[t] + pu*(c[t+1] - c[t]).  The
// neighbour of a lane's last node is the next lane's first (one shuffle).
// Returns the next j.  After it, only nodes t < stop are live.
template <int NL>
__device__ __forceinline__ int backward(float (&c)[NL], int j, int stop, float pu) {
  for (; j > stop; --j) {
    const float right = __shfl_down_sync(0xffffffffu, c[0], 1);
#pragma unroll
    for (int k = 0; k < NL - 1; ++k) c[k] = fmaf(pu, c[k + 1] - c[k], c[k]);
    c[NL - 1] = fmaf(pu, right - c[NL - 1], c[NL - 1]);
  }
  return j;
}

// NL -> NL/2 nodes per lane: lane l's new nodes (NL/2)*l + k live in lane
// l/2 at register (l%2)*NL/2 + k.
template <int NL>
__device__ __forceinline__ void repack(const float (&c)[NL], float (&h)[NL / 2], unsigned lane) {
#pragma unroll
  for (int k = 0; k < NL / 2; ++k) {
    const float lo = __shfl_sync(0xffffffffu, c[k], lane >> 1);
    const float hi = __shfl_sync(0xffffffffu, c[NL / 2 + k], lane >> 1);
    h[k] = (lane & 1u) ? hi : lo;
  }
}

__global__ void __launch_bounds__(kThreads, 4)
    binomial_warp(const float* __restrict__ rand, float* __restrict__ out, int steps, uint64_t first_opt,
                  uint64_t n_opt) {
  const unsigned lane = threadIdx.x & 31u;
  const uint64_t warps = static_cast<uint64_t>(gridDim.x) * (kThreads / 32);
  for (uint64_t w = blockIdx.x * static_cast<uint64_t>(kThreads / 32) + (threadIdx.x >> 5); w < n_opt; w += warps) {
    const uint64_t o = first_opt + w;
    const double r = rand[o];
    const double S = 5.0 * (1.0 - r) + 30.0 * r;
    const double K = 1.0 * (1.0 - r) + 100.0 * r;
    const double T = 0.25 * (1.0 - r) + 10.0 * r;
    const double dt = T / steps;
    const double vsdt = 0.30 * sqrt(dt);
    const double a = exp(0.02 * dt);
    const double u = exp(vsdt);
    const double d = 1.0 / u;
    const double pu = (a - d) / (u - d);
    const float fpu = static_cast<float>(pu);

    // Leaves in FP64, then the lattice in FP32 with the per-step discount
    // 1/a factored out: c <- c0 + pu*(c1 - c0) is the reference's
    // puByr*c1 + pdByr*c0 times a, and the a^-steps = exp(-R T) is applied
    // once at the end, so rounding 1/a to f32 does not compound 254 times.
    // S*exp(vsdt*(2t - steps)) for the lane's 8 nodes: one exp per lane, then
    // successive factors u^2 = exp(2 vsdt) (FP64, ~1e-16 relative drift).
    float c[kNodesPerLane];
    double st = S * exp(vsdt * static_cast<double>(2 * static_cast<int>(lane) * kNodesPerLane - steps));
    const double u2 = u * u;
#pragma unroll
    for (int k = 0; k < kNodesPerLane; ++k) {
      const int t = static_cast<int>(lane) * kNodesPerLane + k;
      const double leaf = st - K;
      c[k] = (t <= steps && leaf > 0.0) ? static_cast<float>(leaf) : 0.0f;
      st *= u2;
    }
    // The live part of the lattice shrinks by one node per step: once it fits
    // in 128 / 64 / 32 nodes the warp repacks to 4 / 2 / 1 nodes per lane
    // (one shuffle per register), so later steps cost proportionally less.
    int j = steps;
    j = backward<8>(c, j, 128, fpu);
    float c4[4];
    repack<8>(c, c4, lane);
    j = backward<4>(c4, j, 64, fpu);
    float c2[2];
    repack<4>(c4, c2, lane);
    j = backward<2>(c2, j, 32, fpu);
    float c1[1];
    repack<2>(c2, c1, lane);
    backward<1>(c1, j, 0, fpu);
    if (lane == 0) out[o] = static_cast<float>(static_cast<double>(c1[0]) * exp(-0.02 * T));
  }
}

}  // namespace

cudaError_t launch_binomial(const KernelSpec& spec, const LaunchEnv& env, uint64_t first, uint64_t count) {
  if (count == 0) return cudaSuccess;
  if (spec.binom.steps + 1 > 32 * kNodesPerLane) return cudaErrorInvalidValue;
  // work-items -> work-groups -> scalar options (4 per float4 work-group)
  const uint64_t first_opt = first / spec.lws * 4, n_opt = count / spec.lws * 4;
  const uint64_t warps_per_block = kThreads / 32;
  uint64_t blocks = (n_opt + warps_per_block - 1) / warps_per_block;
  const uint64_t cap = static_cast<uint64_t>(env.sms) * 8 * 16;
  if (blocks > cap) blocks = cap;
  binomial_warp<<<static_cast<unsigned>(blocks), kThreads, 0, env.stream>>>(
      static_cast<const float*>(env.in[0]), static_cast<float*>(env.out[0]), static_cast<int>(spec.binom.steps),
      first_opt, n_opt);
  return cudaGetLastError();
}

}  // namespace ecl
