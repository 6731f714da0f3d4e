// binomial.cu — European call on a Cox-Ross-Rubinstein lattice (the paper's
// Binomial Options benchmark, Listing 1; absent from the
// reference, definition in SURVEY.md Appendix B / oracle.c:orc_binomial).
//
// Program shape (Table 2): lws = steps + 1 work-items per work-group, one
// float4 (four options) per work-group, out pattern 1:lws.  A package of
// work-groups [o, o+n) is options [4o, 4(o+n)).
//
// Mapping: one warp per option pair.  Lane l holds lattice nodes
// t = 8l .. 8l+7 in registers (255 nodes for 254 steps); a backward step
//   c[t] <- puByr * c[t+1] + pdByr * c[t]      (t < j)
// is 8 register FMAs per lane (scaled form, below) plus one warp shuffle for the neighbour
// node c[8l+8] held by lane l+1 — the OpenCL kernel's local-memory lattice
// and barriers become registers and __shfl_down_sync.  The two options of a
// warp travel packed in float2 registers through FFMA2/FADD2 (half the
// issue slots of the scalar lattice, same per-component rounding).  Per-option
// parameters (dt, u, d, pu/a, pd/a) are formed in FP64 so the subtraction
// a - d does not lose the 1e-5 relative budget; the lattice itself is FP32.
#include <cuda_runtime.h>

#include <cstdlib>
#include <type_traits>

#include "kernels.cuh"

namespace ecl {
namespace {

constexpr int kThreads = 256;
constexpr int kNodesPerLane = 8;  // 32 x 8 = 256 >= steps + 1 for steps <= 255

// Lattice arithmetic on one option (float) or two options packed in a float2
// (FFMA2/FADD2, sm_100a).  __ffma2_rn / __fadd2_rn round each component
// exactly like __fmaf_rn / __fadd_rn, so the packed kernel's prices are
// bit-identical to the scalar kernel's; it issues half the FP32
// instructions, which is what bounds this kernel (ncu: issue-bound).
// One FMA per node: the lattice is carried scaled, w = c / pd^m (m = steps
// since the last rescale), so pd*c + pu*c1 becomes w + (pu/pd)*w1.
__device__ __forceinline__ float lattice_step(float w, float w1, float r) { return fmaf(r, w1, w); }
__device__ __forceinline__ float2 lattice_step(float2 w, float2 w1, float2 r) { return __ffma2_rn(r, w1, w); }
__device__ __forceinline__ float rescale(float w, float s) { return w * s; }
__device__ __forceinline__ float2 rescale(float2 w, float2 s) { return __fmul2_rn(w, s); }
// Next lane's value within lane groups of G (a warp, or a half-warp).
template <int G>
__device__ __forceinline__ float shfl_down1(float v) {
  return __shfl_down_sync(0xffffffffu, v, 1, G);
}
template <int G>
__device__ __forceinline__ float2 shfl_down1(float2 v) {
  return make_float2(__shfl_down_sync(0xffffffffu, v.x, 1, G), __shfl_down_sync(0xffffffffu, v.y, 1, G));
}
__device__ __forceinline__ float shfl_from(float v, unsigned src) { return __shfl_sync(0xffffffffu, v, src); }
__device__ __forceinline__ float2 shfl_from(float2 v, unsigned src) {
  return make_float2(__shfl_sync(0xffffffffu, v.x, src), __shfl_sync(0xffffffffu, v.y, src));
}

// Backward steps j, j-1, ... while j > stop, with NL nodes per lane (lane l
// holds nodes NL*l .. NL*l+NL-1): w[t] <- w[t] + r*w[t+1].  The neighbour of
// a lane's last node is the next lane's first (one shuffle).  Returns the
// next j.
template <int G, int NL, typename V>
__device__ __forceinline__ int backward(V (&c)[NL], int j, int stop, V r) {
#pragma unroll 8
  for (; j > stop; --j) {
    const V right = shfl_down1<G>(c[0]);
#pragma unroll
    for (int k = 0; k < NL - 1; ++k) c[k] = lattice_step(c[k], c[k + 1], r);
    c[NL - 1] = lattice_step(c[NL - 1], right, r);
  }
  return j;
}

// The live lattice (nodes 0..j at level j) shrinks by one node per step, so
// the levels run in phases of G (the lane-group width): phase NL keeps NL
// nodes per lane until the live nodes fit in G*(NL-1), then the lattice is
// rescaled by pd^G (w stays within pd^-G of the true value: no f32
// overflow) and repacked to NL-1 nodes per lane through the group's private
// shared-memory buffer.  Phases above ceil((steps+1)/G) run no steps and
// neither rescale nor repack anything that matters.  Slots beyond the live
// nodes carry don't-care values.  `lane` is the lane within its group.
template <int G, int NL, typename V>
__device__ __forceinline__ V phases(V (&c)[NL], int j, V r, V s, V* buf, unsigned lane) {
  const int stop = NL > 1 ? G * (NL - 1) - 1 : 0;
  if (j > stop) {
    j = backward<G, NL>(c, j, stop, r);
    if constexpr (NL > 1) {
#pragma unroll
      for (int k = 0; k < NL; ++k) c[k] = rescale(c[k], s);
    }
  }
  if constexpr (NL == 1) {
    return c[0];
  } else {
#pragma unroll
    for (int k = 0; k < NL; ++k) buf[NL * lane + k] = c[k];
    __syncwarp();
    V h[NL - 1];
#pragma unroll
    for (int k = 0; k < NL - 1; ++k) h[k] = buf[(NL - 1) * lane + k];
    __syncwarp();
    return phases<G, NL - 1>(h, j, r, s, buf, lane);
  }
}

// x^e for a warp-uniform e >= 0 (square and multiply).
__device__ __forceinline__ double upow(double x, int e) {
  double p = 1.0;
  for (; e > 0; e >>= 1, x *= x)
    if (e & 1) p *= x;
  return p;
}

// Per-option quantities in FP64 (CRR parameters: S, K, T
// from the uniform r, dt = T/steps, u = exp(sigma sqrt(dt)),
// pu = (a - d)/(u - d)), reduced to what the leaves and the lattice need.
struct Option {
  double K, base, f, u2;  // leaf of node t = NL l + k: base * f^l * u2^k - K  (f = u^(2 NL))
  float r, s;             // pu/pd and pd^G (the scaled lattice's step and rescale factors)
  double tail;            // pd^(steps - G R) * exp(-R T) / q^R: undoes the remaining scale, discounts
};

// G = lane-group width (phase length in levels), NL = nodes per lane at the leaves.
template <int G, int NL>
__device__ __forceinline__ Option option_params(double rv, int steps) {
  Option o;
  const double S = 5.0 * (1.0 - rv) + 30.0 * rv;
  o.K = 1.0 * (1.0 - rv) + 100.0 * rv;
  const double T = 0.25 * (1.0 - rv) + 10.0 * rv;
  const double dt = T / steps;
  const double vsdt = 0.30 * sqrt(dt);
  const double a = exp(0.02 * dt);
  const double u = exp(vsdt);
  const double d = 1.0 / u;
  const double pu = (a - d) / (u - d), pd = 1.0 - pu;
  o.r = static_cast<float>(pu / pd);
  const double pg = upow(pd, G);
  o.s = static_cast<float>(pg);
  // R rescales by the f32-rounded pd^G; q is that rounding's factor.
  const int rescales = steps / G;  // = ceil((steps + 1) / G) - 1 phase boundaries
  const double q = static_cast<double>(o.s) / pg;
  o.tail = upow(pd, steps - G * rescales) * exp(-0.02 * T) / upow(q, rescales);
  // S*exp(vsdt*(2t - steps)) = S*exp(-vsdt*steps) * (u^(2 NL))^l * (u^2)^k:
  // one exp per option instead of one per lane.
  o.base = S * exp(-vsdt * static_cast<double>(steps));
  o.u2 = u * u;
  o.f = upow(o.u2, NL);
  return o;
}

// Leaves in FP64, then the lattice in FP32.  The per-step discount 1/a is
// factored out (applied once as exp(-R T) at the end, so rounding it to f32
// does not compound 254 times) and the lattice is carried scaled by
// pd^-m: pd*c + pu*c1 becomes one FMA w + (pu/pd)*w1, rescaled by pd^32 at
// every level that is a multiple of 32; `tail` undoes the rest.  The lane's
// first leaf price is base * f16^lane (lane-divergent square-and-multiply
// with selects), then successive factors u^2 (~1e-15 relative drift).
template <int NL>
__device__ __forceinline__ void leaves(const Option& o, int steps, unsigned lane, float (&c)[NL]) {
  double st = o.base, f = o.f;
#pragma unroll
  for (int bit = 0; bit < 5; ++bit, f *= f) {
    const double m = st * f;
    st = ((lane >> bit) & 1u) ? m : st;
  }
#pragma unroll
  for (int k = 0; k < NL; ++k) {
    const int t = static_cast<int>(lane) * NL + k;
    const double leaf = st - o.K;
    c[k] = (t <= steps && leaf > 0.0) ? static_cast<float>(leaf) : 0.0f;
    st *= o.u2;
  }
}

// Broadcast of an Option computed on lane `src` to the whole warp.
__device__ __forceinline__ Option shfl_option(const Option& x, int src) {
  Option o;
  o.K = __shfl_sync(0xffffffffu, x.K, src);
  o.base = __shfl_sync(0xffffffffu, x.base, src);
  o.f = __shfl_sync(0xffffffffu, x.f, src);
  o.u2 = __shfl_sync(0xffffffffu, x.u2, src);
  o.r = __shfl_sync(0xffffffffu, x.r, src);
  o.s = __shfl_sync(0xffffffffu, x.s, src);
  o.tail = __shfl_sync(0xffffffffu, x.tail, src);
  return o;
}

template <typename V>
__device__ __forceinline__ V lattice(V (&c)[kNodesPerLane], int steps, V r, V s32, V* buf, unsigned lane) {
  return phases<32, kNodesPerLane>(c, steps, r, s32, buf, lane);
}

// P = options per warp (1: scalar lattice, 2: two options packed per lane).
template <int P, int MB>
__global__ void __launch_bounds__(kThreads, MB)
    binomial_warp(const float* __restrict__ rand, float* __restrict__ out, int steps, uint64_t first_opt,
                  uint64_t n_opt) {
  using V = std::conditional_t<P == 2, float2, float>;
  __shared__ V repack_buf[kThreads / 32][32 * kNodesPerLane];
  const unsigned lane = threadIdx.x & 31u;
  V* const buf = repack_buf[threadIdx.x >> 5];
  const uint64_t warps = static_cast<uint64_t>(gridDim.x) * (kThreads / 32);
  const uint64_t groups = (n_opt + P - 1) / P;
  for (uint64_t w = blockIdx.x * static_cast<uint64_t>(kThreads / 32) + (threadIdx.x >> 5); w < groups;
       w += warps) {
    const uint64_t o = first_opt + w * P;
    if constexpr (P == 1) {
      const Option a = option_params<32, kNodesPerLane>(rand[o], steps);
      float c[kNodesPerLane];
      leaves<kNodesPerLane>(a, steps, lane, c);
      const float v = lattice(c, steps, a.r, a.s, buf, lane);
      if (lane == 0) out[o] = static_cast<float>(static_cast<double>(v) * a.tail);
    } else {
      const bool has_b = w * P + 1 < n_opt;
      float2 c[kNodesPerLane], r, s32;
      double tail_a, tail_b;
      // Lanes 0-15 set up option A, lanes 16-31 option B (one pass of the
      // FP64 setup for both), then each half's result is broadcast.
      const Option mine = option_params<32, kNodesPerLane>(rand[o + ((lane >> 4) != 0u && has_b ? 1 : 0)], steps);
      {
        const Option a = shfl_option(mine, 0);
        float ca[kNodesPerLane];
        leaves<kNodesPerLane>(a, steps, lane, ca);
#pragma unroll
        for (int k = 0; k < kNodesPerLane; ++k) c[k].x = ca[k];
        r.x = a.r;
        s32.x = a.s;
        tail_a = a.tail;
      }
      {
        const Option b = shfl_option(mine, 16);
        float cb[kNodesPerLane];
        leaves<kNodesPerLane>(b, steps, lane, cb);
#pragma unroll
        for (int k = 0; k < kNodesPerLane; ++k) c[k].y = cb[k];
        r.y = b.r;
        s32.y = b.s;
        tail_b = b.tail;
      }
      const float2 v = lattice(c, steps, r, s32, buf, lane);
      if (lane == 0) {
        out[o] = static_cast<float>(static_cast<double>(v.x) * tail_a);
        if (has_b) out[o + 1] = static_cast<float>(static_cast<double>(v.y) * tail_b);
      }
    }
  }
}

// Four options per warp: each half-warp carries an option pair packed in
// float2, 16 nodes per lane (16 x 16 = 256 >= steps + 1).  Per lattice level
// a warp issues 16 FFMA2 (for 4 options) and 2 shuffles: shuffles per option
// halve against binomial_warp<2>, whose 2 shuffles per 8 FFMA2 co-limit
// with the FMA pipe (SHFL runs at one warp instruction per cycle per SM,
// tools/probe/shfl_tp.cu).  Phases are 16 levels long (rescale by pd^16).
// Measured 18.3 ms vs 17.2 ms for binomial_warp<2> at the config, so it is
// the "binomial@2" variant, not the default: shuffles were not the binding
// limit.
constexpr int kHalf = 16, kHalfNodes = 16;

template <int MB>
__global__ void __launch_bounds__(kThreads, MB)
    binomial_half(const float* __restrict__ rand, float* __restrict__ out, int steps, uint64_t first_opt,
                  uint64_t n_opt) {
  __shared__ float2 repack_buf[kThreads / kHalf][kHalf * kHalfNodes];
  const unsigned lane = threadIdx.x & 31u, half = lane >> 4, lh = lane & 15u;
  float2* const buf = repack_buf[threadIdx.x >> 4];
  const uint64_t warps = static_cast<uint64_t>(gridDim.x) * (kThreads / 32);
  const uint64_t groups = (n_opt + 3) / 4;
  for (uint64_t w = blockIdx.x * static_cast<uint64_t>(kThreads / 32) + (threadIdx.x >> 5); w < groups;
       w += warps) {
    const uint64_t o = first_opt + w * 4;
    const uint64_t left = first_opt + n_opt - o;  // options of this group that exist (>= 1)
    // Lanes 8q..8q+7 set up option o+q; half h then takes options 2h, 2h+1.
    const unsigned q = lane >> 3;
    const Option mine = option_params<kHalf, kHalfNodes>(rand[o + (q < left ? q : 0)], steps);
    const Option a = shfl_option(mine, static_cast<int>(16 * half));
    const Option b = shfl_option(mine, static_cast<int>(16 * half + 8));
    float ca[kHalfNodes], cb[kHalfNodes];
    leaves<kHalfNodes>(a, steps, lh, ca);
    leaves<kHalfNodes>(b, steps, lh, cb);
    float2 c[kHalfNodes];
#pragma unroll
    for (int k = 0; k < kHalfNodes; ++k) c[k] = make_float2(ca[k], cb[k]);
    const float2 v = phases<kHalf, kHalfNodes>(c, steps, make_float2(a.r, b.r), make_float2(a.s, b.s), buf, lh);
    if (lh == 0) {
      const uint64_t i = 2 * half;
      if (i < left) out[o + i] = static_cast<float>(static_cast<double>(v.x) * a.tail);
      if (i + 1 < left) out[o + i + 1] = static_cast<float>(static_cast<double>(v.y) * b.tail);
    }
  }
}

template <int MB>
cudaError_t launch_half(const KernelSpec& spec, const LaunchEnv& env, uint64_t first_opt, uint64_t n_opt) {
  const uint64_t warps_per_block = kThreads / 32;
  const uint64_t groups = (n_opt + 3) / 4;
  uint64_t blocks = (groups + warps_per_block - 1) / warps_per_block;
  const uint64_t cap = static_cast<uint64_t>(env.sms) * 8 * 16;
  if (blocks > cap) blocks = cap;
  binomial_half<MB><<<static_cast<unsigned>(blocks), kThreads, 0, env.stream>>>(
      static_cast<const float*>(env.in[0]), static_cast<float*>(env.out[0]), static_cast<int>(spec.binom.steps),
      first_opt, n_opt);
  return cudaGetLastError();
}

template <int P, int MB>
cudaError_t launch(const KernelSpec& spec, const LaunchEnv& env, uint64_t first_opt, uint64_t n_opt) {
  const uint64_t warps_per_block = kThreads / 32;
  const uint64_t groups = (n_opt + P - 1) / P;
  uint64_t blocks = (groups + warps_per_block - 1) / warps_per_block;
  const uint64_t cap = static_cast<uint64_t>(env.sms) * 8 * 16;
  if (blocks > cap) blocks = cap;
  binomial_warp<P, MB><<<static_cast<unsigned>(blocks), kThreads, 0, env.stream>>>(
      static_cast<const float*>(env.in[0]), static_cast<float*>(env.out[0]), static_cast<int>(spec.binom.steps),
      first_opt, n_opt);
  return cudaGetLastError();
}

}  // namespace

cudaError_t launch_binomial(const KernelSpec& spec, const LaunchEnv& env, uint64_t first, uint64_t count) {
  if (count == 0) return cudaSuccess;
  if (spec.binom.steps + 1 > 32 * kNodesPerLane) return cudaErrorInvalidValue;
  // work-items -> work-groups -> scalar options (4 per float4 work-group)
  const uint64_t first_opt = first / spec.lws * 4, n_opt = count / spec.lws * 4;
  static const int env_variant = [] {  // ECL_BINOMIAL_VARIANT=1: scalar lattice
    const char* v = std::getenv("ECL_BINOMIAL_VARIANT");
    return v ? std::atoi(v) : 0;
  }();
  const int variant = spec.variant >= 0 ? spec.variant : env_variant;
  static const int mb = [] {  // ECL_BINOMIAL_MB: resident CTAs per SM the registers are sized for
    const char* v = std::getenv("ECL_BINOMIAL_MB");
    return v ? std::atoi(v) : 0;
  }();
  if (variant == 1) return launch<1, 4>(spec, env, first_opt, n_opt);
  if (variant == 2) {
    switch (mb) {
      case 2: return launch_half<2>(spec, env, first_opt, n_opt);
      case 4: return launch_half<4>(spec, env, first_opt, n_opt);
      default: return launch_half<3>(spec, env, first_opt, n_opt);
    }
  }
  switch (mb) {  // measured: 4 (52 registers) 18.8 ms, 5 19.1 ms, 6 19.2 ms
    case 5: return launch<2, 5>(spec, env, first_opt, n_opt);
    case 6: return launch<2, 6>(spec, env, first_opt, n_opt);
    default: return launch<2, 4>(spec, env, first_opt, n_opt);
  }
}

}  // namespace ecl
