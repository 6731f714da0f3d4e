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

__global__ void __launch_bounds__(kThreads)
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
    float c[kNodesPerLane];
#pragma unroll
    for (int k = 0; k < kNodesPerLane; ++k) {
      const int t = static_cast<int>(lane) * kNodesPerLane + k;
      const double leaf = S * exp(vsdt * static_cast<double>(2 * t - steps)) - K;
      c[k] = (t <= steps && leaf > 0.0) ? static_cast<float>(leaf) : 0.0f;
    }
    for (int j = steps; j > 0; --j) {
      const float right = __shfl_down_sync(0xffffffffu, c[0], 1);  // node 8(l+1)
#pragma unroll
      for (int k = 0; k < kNodesPerLane - 1; ++k) c[k] = fmaf(fpu, c[k + 1] - c[k], c[k]);
      c[kNodesPerLane - 1] = fmaf(fpu, right - c[kNodesPerLane - 1], c[kNodesPerLane - 1]);
    }
    if (lane == 0) out[o] = static_cast<float>(static_cast<double>(c[0]) * exp(-0.02 * T));
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
