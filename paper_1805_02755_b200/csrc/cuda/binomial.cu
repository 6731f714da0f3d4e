// binomial.cu — European call on a Cox-Ross-Rubinstein lattice (the paper's
// Binomial Options benchmark, Listing 1; absent from the
// reference, definition in SURVEY.md Appendix B / oracle.c:orc_binomial).
//
// Program shape (Table 2): lws = steps + 1 work-items per work-group, one
// float4 (four options) per work-group, out pattern 1:lws.  A package of
// work-groups [o, o+n) is options [4o, 4(o+n)).
//
// Mapping (default kernel, binomial_hw): one warp per four options, one
// half-warp per option pair.  The two options of a pair travel packed in
// float2 registers through FFMA2 (half the issue slots of the scalar
// lattice, same per-component rounding).  Nodes below the strike are exactly
// zero and stay zero until the level where their whole subtree has been
// reached, so a pair's live lattice is a window of W = steps - tw + 1 nodes
// (tw = the lowest first-positive leaf of the four options) that slides down
// one node per level, then shrinks by one node per level; at the config W is
// ~116 of 255 nodes and fits 16 lanes x 8 nodes in registers.  A backward
// step is 8 register FMAs per lane (scaled form, below) plus one warp
// shuffle per packed component that serves both pairs of the warp — the
// OpenCL kernel's local-memory lattice and barriers become registers and
// shuffles.  Per-option parameters (dt, u, d, pu/a, pd/a) are formed in FP64
// so the subtraction a - d does not lose the 1e-5 relative budget; the
// lattice itself is FP32.  Every variant (binomial@1..4) computes the same
// node values with the same FMAs, so all prices are bit-identical to the
// scalar full lattice (binomial@1).
#include <cuda_runtime.h>

#include <algorithm>
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

// Backward steps j, j-1, ... while j > stop, with NL nodes per lane (lane l
// holds nodes NL*l .. NL*l+NL-1): w[t] <- w[t] + r*w[t+1].  The neighbour of
// a lane's last node is the next lane's first (one shuffle).  Returns the
// next j.
template <int G, int NL, typename V, int U = 8>
__device__ __forceinline__ int backward(V (&c)[NL], int j, int stop, V r) {
#pragma unroll U
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
// RS: the rescale period in levels (a multiple of G): the lattice is rescaled
// by s = pd^RS at the phase boundaries that are multiples of RS.
template <int G, int NL, typename V, int RS = G, int U = 8>
__device__ __forceinline__ V phases(V (&c)[NL], int j, V r, V s, V* buf, unsigned lane) {
  const int stop = NL > 1 ? G * (NL - 1) - 1 : 0;
  if (j > stop) {
    j = backward<G, NL, V, U>(c, j, stop, r);
    if constexpr (NL > 1 && (G * (NL - 1)) % RS == 0) {
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
    return phases<G, NL - 1, V, RS, U>(h, j, r, s, buf, lane);
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
  int t0;                 // every leaf below node t0 is exactly zero (conservative by 2 nodes)
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
  // leaf(t) = S u^(2t - steps) - K > 0  <=>  t > (steps + ln(K/S)/vsdt) / 2
  const double x = 0.5 * (steps + log(o.K / S) / vsdt);
  const double t0 = floor(x) - 1.0;
  o.t0 = t0 <= 0.0 ? 0 : (t0 >= steps ? steps : static_cast<int>(t0));
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

// ---- Zero window -----------------------------------------------------------
// Leaves below the strike are exactly 0, and node t of level j is a
// combination of leaves t .. t + (steps - j) only, so at level j every node
// below b_j = max(0, tw - (steps - j)) is exactly 0 (tw <= the first
// positive leaf of both options of the pair).  While b_j > 0 the warp keeps
// only nodes b_j .. j: a window of constant width W = steps - tw + 1 whose
// base moves down one node per level.  In window slots (slot s = node
// b_j + s) a backward step reads the slot below:
//   w'[s] = w[s-1] + (pu/pd) w[s]          (w[-1] = node b_j - 1 = 0)
// — the same FMA on the same operands as the full lattice, so every price is
// bit-identical to it; exact zeros are skipped, not approximated.  After tw
// levels the base reaches node 0 with W live nodes in NL = ceil(W/32) nodes
// per lane, which is exactly the layout phases<32, NL> continues from.  At
// the config (rv ~ U[0,1)) tw ~ 139 of 254, W ~ 116: NL = 4 instead of 8
// for half the levels, ~27 % fewer FFMA2s and shuffles.
// Previous lane's value within lane groups of G.
template <int G>
__device__ __forceinline__ float shfl_up1(float v) {
  return __shfl_up_sync(0xffffffffu, v, 1, G);
}
template <int G>
__device__ __forceinline__ float2 shfl_up1(float2 v) {
  return make_float2(__shfl_up_sync(0xffffffffu, v.x, 1, G), __shfl_up_sync(0xffffffffu, v.y, 1, G));
}

// Window steps from level j down to jend in lane groups of G (`lane` = lane
// within the group), rescaling at the levels 32m - 1 as phases() does.
// Returns jend.
template <int G, int NL, typename V, int U = 8>
__device__ __forceinline__ int window_steps(V (&c)[NL], int j, int jend, V r, V s, unsigned lane) {
  while (j > jend) {
    const int nb = (j >> 5) * 32 - 1;  // next rescale level below j (-1: none)
    const int stop = nb > jend ? nb : jend;
#pragma unroll U
    for (; j > stop; --j) {
      V left = shfl_up1<G>(c[NL - 1]);
      if (lane == 0) left = V{};  // node b_j - 1 is zero
#pragma unroll
      for (int k = NL - 1; k > 0; --k) c[k] = lattice_step(c[k - 1], c[k], r);
      c[0] = lattice_step(left, c[0], r);
    }
    if (j == nb) {
#pragma unroll
      for (int k = 0; k < NL; ++k) c[k] = rescale(c[k], s);
    }
  }
  return j;
}

// Leaves (8 per lane, full layout, in buf) -> window slots tw + NL*lane + k,
// window steps, then the shrinking phases from NL nodes per lane.
template <int NL, typename V>
__device__ __forceinline__ V from_window(int steps, int tw, V r, V s, V* buf, unsigned lane) {
  V h[NL];
#pragma unroll
  for (int k = 0; k < NL; ++k) {
    const int i = tw + NL * static_cast<int>(lane) + k;
    h[k] = i < 32 * kNodesPerLane ? buf[i] : V{};
  }
  __syncwarp();  // phases() reuses buf
  const int j = window_steps<32, NL>(h, steps, steps - tw, r, s, lane);
  return phases<32, NL>(h, j, r, s, buf, lane);
}

template <typename V>
__device__ __forceinline__ V lattice_window(V (&c)[kNodesPerLane], int steps, int tw, V r, V s, V* buf,
                                            unsigned lane) {
  if (tw <= 0) return lattice(c, steps, r, s, buf, lane);
#pragma unroll
  for (int k = 0; k < kNodesPerLane; ++k) buf[kNodesPerLane * lane + k] = c[k];
  __syncwarp();
  switch ((steps - tw + 32) >> 5) {  // ceil(W / 32), W = steps - tw + 1
    case 1: return from_window<1>(steps, tw, r, s, buf, lane);
    case 2: return from_window<2>(steps, tw, r, s, buf, lane);
    case 3: return from_window<3>(steps, tw, r, s, buf, lane);
    case 4: return from_window<4>(steps, tw, r, s, buf, lane);
    case 5: return from_window<5>(steps, tw, r, s, buf, lane);
    case 6: return from_window<6>(steps, tw, r, s, buf, lane);
    case 7: return from_window<7>(steps, tw, r, s, buf, lane);
    default: return from_window<8>(steps, tw, r, s, buf, lane);
  }
}

// P = options per warp (1: scalar lattice, 2: two options packed per lane);
// Window: skip the exact-zero nodes below the strike (lattice_window).
template <int P, int MB, bool Window = true>
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
      const int tw = min(__shfl_sync(0xffffffffu, mine.t0, 0), __shfl_sync(0xffffffffu, mine.t0, 16));
      const float2 v = Window ? lattice_window(c, steps, tw, r, s32, buf, lane) : lattice(c, steps, r, s32, buf, lane);
      if (lane == 0) {
        out[o] = static_cast<float>(static_cast<double>(v.x) * tail_a);
        if (has_b) out[o + 1] = static_cast<float>(static_cast<double>(v.y) * tail_b);
      }
    }
  }
}

// ---- Default kernel: half-warp lattices with the zero window -------------
// The lattice's cost is per level, not per node: every level needs the
// neighbour exchange (one SHFL per packed component), and the exchange, not
// the FFMA2 count, paces the warp (skipping a quarter of the FFMA2s with the
// zero window alone left the time unchanged; ncu: SHFLs and their selects,
// branches and scoreboard waits stayed per level).  The zero window makes a
// pair's live lattice W = steps - tw + 1 <= 128 nodes at the config, which
// fits 16 lanes x 8 nodes, so each half-warp runs one option pair: one warp
// SHFL serves two pairs and the per-level overhead halves, with the
// registers of the 8-node warp lattice.  Phases are 16 levels (repack to
// NL-1 nodes per lane every 16 levels, less dead work than 32) while the
// rescale stays at the levels 32m - 1 by pd^32, so the prices are
// bit-identical to the full scalar lattice.  Warps whose four options need
// W > 128 (deep in the money) run their two pairs one after the other as
// 32-lane window lattices instead.
// One code path for every window width (W <= 128): the window steps run at
// 8 nodes per lane whatever W is.  Width-specialised entries (NL = ceil(W/16)
// per pair) cut FFMA2s further but multiplied the kernel's code eightfold:
// ncu's top stall became "no instruction" (instruction-cache misses) and the
// kernel got slower.
template <int U>
__device__ __forceinline__ float2 half_lattice(int steps, int tw, float2 r, float2 s, float2* buf, unsigned lh) {
  float2 h[kNodesPerLane];
#pragma unroll
  for (int k = 0; k < kNodesPerLane; ++k) {
    const int i = tw + kNodesPerLane * static_cast<int>(lh) + k;
    h[k] = i < 32 * kNodesPerLane ? buf[i] : float2{};
  }
  __syncwarp();  // phases() reuses buf
  const int j = window_steps<16, kNodesPerLane, float2, U>(h, steps, steps - tw, r, s, lh);
  return phases<16, kNodesPerLane, float2, 32, U>(h, j, r, s, buf, lh);
}

// Deep in-the-money groups (W > 128): each pair on the whole warp, full
// 32-lane lattice (rare).
template <int U>
__device__ __forceinline__ float2 warp_lattice(const float2* leaves_buf, int steps, float2 r, float2 s, float2* buf,
                                            unsigned lane) {
  float2 c[kNodesPerLane];
#pragma unroll
  for (int k = 0; k < kNodesPerLane; ++k) c[k] = leaves_buf[kNodesPerLane * lane + k];
  __syncwarp();
  return phases<32, kNodesPerLane, float2, 32, U>(c, steps, r, s, buf, lane);
}

// Option records computed ahead (default; binomial@5 keeps the setup inside
// the lattice kernel): one thread per option runs
// option_params once, instead of eight lanes per option inside the lattice
// kernel (its FP64 setup was ~7 % of the lattice kernel's instructions,
// each FP64 instruction holding an issue slot two cycles).  Same function,
// same arguments: the records are bit-identical to the in-kernel ones.
// 12.69 -> 11.71 ms at 8M x 254 including the setup launch (64 B per option
// through HBM, 0.5 GB written and read back).  Two earlier attempts at one
// setup per option *inside* the lattice kernel (32-option chunks, records in
// shared memory) lost to register pressure (12.79, 13.50 ms); here the
// lattice kernel only loads finished records.
struct __align__(16) OptionRec {
  double K, base, f, u2, tail;
  float r, s;
  int t0, pad;
};

__global__ void __launch_bounds__(256)
    binomial_setup(const float* __restrict__ rand, OptionRec* __restrict__ recs, int steps, uint64_t first_opt,
                   uint64_t n_opt) {
  const uint64_t stride = static_cast<uint64_t>(gridDim.x) * blockDim.x;
  for (uint64_t i = blockIdx.x * static_cast<uint64_t>(blockDim.x) + threadIdx.x; i < n_opt; i += stride) {
    const Option o = option_params<32, kNodesPerLane>(rand[first_opt + i], steps);
    OptionRec rec;
    rec.K = o.K;
    rec.base = o.base;
    rec.f = o.f;
    rec.u2 = o.u2;
    rec.tail = o.tail;
    rec.r = o.r;
    rec.s = o.s;
    rec.t0 = o.t0;
    rec.pad = 0;
    recs[first_opt + i] = rec;
  }
}

__device__ __forceinline__ Option load_option(const OptionRec* __restrict__ recs, uint64_t i) {
  const OptionRec rec = recs[i];
  Option o;
  o.K = rec.K;
  o.base = rec.base;
  o.f = rec.f;
  o.u2 = rec.u2;
  o.tail = rec.tail;
  o.r = rec.r;
  o.s = rec.s;
  o.t0 = rec.t0;
  return o;
}

// U: unroll of the level loops (code size: the kernel is instruction-fetch
// sensitive, see half_lattice).
template <int MB, int U, bool PRE = false>
__global__ void __launch_bounds__(kThreads, MB)
    binomial_hw(const float* __restrict__ rand, float* __restrict__ out, int steps, uint64_t first_opt,
                uint64_t n_opt, const OptionRec* __restrict__ recs) {
  // per warp: the leaves of its two pairs (full 32 x 8 layout), then each
  // pair's window / repack buffer
  __shared__ float2 pair_buf[kThreads / 32][2][32 * kNodesPerLane];
  __shared__ double tail_buf[kThreads / 32][4];
  const unsigned lane = threadIdx.x & 31u, half = lane >> 4, lh = lane & 15u;
  float2 (*const bufs)[32 * kNodesPerLane] = pair_buf[threadIdx.x >> 5];
  double* const tails = tail_buf[threadIdx.x >> 5];
  const uint64_t warps = static_cast<uint64_t>(gridDim.x) * (kThreads / 32);
  const uint64_t groups = (n_opt + 3) / 4;
  for (uint64_t w = blockIdx.x * static_cast<uint64_t>(kThreads / 32) + (threadIdx.x >> 5); w < groups;
       w += warps) {
    const uint64_t o = first_opt + w * 4;
    const uint64_t left = first_opt + n_opt - o;  // options of this group that exist (>= 1)
    // Lanes 8q..8q+7 set up option o+q (missing options repeat option o).
    const unsigned q = lane >> 3;
    const Option mine = PRE ? load_option(recs, o + (q < left ? q : 0))
                            : option_params<32, kNodesPerLane>(rand[o + (q < left ? q : 0)], steps);
    const int tw = static_cast<int>(__reduce_min_sync(0xffffffffu, static_cast<unsigned>(mine.t0)));
    // Only the lattice's inputs stay in registers across it: the tails wait
    // in shared memory, each pair's (pu/pd, pd^32) is re-read from its lanes.
    if ((lane & 7u) == 0) tails[q] = mine.tail;
#pragma unroll
    for (int p = 0; p < 2; ++p) {
      const Option a = shfl_option(mine, 16 * p), b = shfl_option(mine, 16 * p + 8);
      float ca[kNodesPerLane], cb[kNodesPerLane];
      leaves<kNodesPerLane>(a, steps, lane, ca);
      leaves<kNodesPerLane>(b, steps, lane, cb);
#pragma unroll
      for (int k = 0; k < kNodesPerLane; ++k) bufs[p][kNodesPerLane * lane + k] = make_float2(ca[k], cb[k]);
    }
    const float mr = mine.r, ms = mine.s;
    __syncwarp();
    if (steps - tw + 1 <= 16 * kNodesPerLane) {
      const unsigned src = 16 * half;
      const float2 r = make_float2(__shfl_sync(0xffffffffu, mr, src), __shfl_sync(0xffffffffu, mr, src + 8));
      const float2 sc = make_float2(__shfl_sync(0xffffffffu, ms, src), __shfl_sync(0xffffffffu, ms, src + 8));
      const float2 v = half_lattice<U>(steps, tw, r, sc, bufs[half], lh);
      if (lh == 0) {
        const uint64_t i = 2 * half;
        if (i < left) out[o + i] = static_cast<float>(static_cast<double>(v.x) * tails[i]);
        if (i + 1 < left) out[o + i + 1] = static_cast<float>(static_cast<double>(v.y) * tails[i + 1]);
      }
    } else {
#pragma unroll 1
      for (int p = 0; p < 2; ++p) {
        const float2 r = make_float2(__shfl_sync(0xffffffffu, mr, 16 * p), __shfl_sync(0xffffffffu, mr, 16 * p + 8));
        const float2 sc = make_float2(__shfl_sync(0xffffffffu, ms, 16 * p), __shfl_sync(0xffffffffu, ms, 16 * p + 8));
        const float2 v = warp_lattice<U>(bufs[p], steps, r, sc, bufs[p], lane);
        if (lane == 0) {
          const uint64_t i = 2 * p;
          if (i < left) out[o + i] = static_cast<float>(static_cast<double>(v.x) * tails[i]);
          if (i + 1 < left) out[o + i + 1] = static_cast<float>(static_cast<double>(v.y) * tails[i + 1]);
        }
      }
    }
    __syncwarp();  // the next group rewrites the buffers
  }
}

template <int MB, int U, bool PRE = false>
cudaError_t launch_hw(const KernelSpec& spec, const LaunchEnv& env, uint64_t first_opt, uint64_t n_opt) {
  const uint64_t warps_per_block = kThreads / 32;
  const uint64_t groups = (n_opt + 3) / 4;
  uint64_t blocks = (groups + warps_per_block - 1) / warps_per_block;
  const uint64_t cap = static_cast<uint64_t>(env.sms) * 8 * 16;  // measured: a persistent grid (1 wave) 13.3 ms vs 12.7
  if (blocks > cap) blocks = cap;
  OptionRec* recs = nullptr;
  if (PRE) {
    recs = static_cast<OptionRec*>(env.scratch);
    if (!recs) return cudaErrorInvalidValue;
    const uint64_t sb = std::min<uint64_t>((n_opt + 255) / 256, static_cast<uint64_t>(env.sms) * 16);
    binomial_setup<<<static_cast<unsigned>(sb), 256, 0, env.stream>>>(static_cast<const float*>(env.in[0]), recs,
                                                                      static_cast<int>(spec.binom.steps), first_opt,
                                                                      n_opt);
    if (env.extra_launches) ++*env.extra_launches;
  }
  binomial_hw<MB, U, PRE><<<static_cast<unsigned>(blocks), kThreads, 0, env.stream>>>(
      static_cast<const float*>(env.in[0]), static_cast<float*>(env.out[0]), static_cast<int>(spec.binom.steps),
      first_opt, n_opt, recs);
  return cudaGetLastError();
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

template <int P, int MB, bool Window = true>
cudaError_t launch(const KernelSpec& spec, const LaunchEnv& env, uint64_t first_opt, uint64_t n_opt) {
  const uint64_t warps_per_block = kThreads / 32;
  const uint64_t groups = (n_opt + P - 1) / P;
  uint64_t blocks = (groups + warps_per_block - 1) / warps_per_block;
  const uint64_t cap = static_cast<uint64_t>(env.sms) * 8 * 16;
  if (blocks > cap) blocks = cap;
  binomial_warp<P, MB, Window><<<static_cast<unsigned>(blocks), kThreads, 0, env.stream>>>(
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
  static const int env_variant = [] {  // ECL_BINOMIAL_VARIANT: variant when the kernel id has no @n
    const char* v = std::getenv("ECL_BINOMIAL_VARIANT");
    return v ? std::atoi(v) : 0;
  }();
  const int variant = spec.variant >= 0 ? spec.variant : env_variant;
  static const int mb = [] {  // ECL_BINOMIAL_MB: resident CTAs per SM the registers are sized for
    const char* v = std::getenv("ECL_BINOMIAL_MB");
    return v ? std::atoi(v) : 0;
  }();
  // Variants (all bit-identical; times at the 8M x 254 config, one launch):
  //   0  binomial_setup + binomial_hw: option records     11.71 ms
  //      computed ahead, one thread per option; half-warp pairs + zero window
  //   5  binomial_hw with the option setup inside it      12.69 ms (MB 6, unroll 4)
  //   1  scalar full lattice, one option per warp         20.2 ms
  //   2  half-warp pairs, 16 nodes per lane, full lattice 18.8 ms
  //   3  packed pair per warp, full lattice (round 1)     17.5 ms
  //   4  packed pair per warp + zero window (32 lanes)    17.6 ms: 26 % fewer
  //      FFMA2s, same time — the per-level exchange paced it, hence variant 0
  // Measured and dropped: 32-option chunks sorted by t0 (fewer > 128-node
  // windows, FP64 setup once per option) 12.79 ms — the saved FP64 work
  // came back as register pressure at 6 CTAs/SM; a persistent grid 13.3 ms.
  static const int hw_unroll = [] {  // ECL_BINOMIAL_UNROLL: level-loop unroll of the default kernel
    const char* v = std::getenv("ECL_BINOMIAL_UNROLL");
    return v ? std::atoi(v) : 4;
  }();
  switch (variant) {
    case 1: return launch<1, 4>(spec, env, first_opt, n_opt);
    case 2:
      switch (mb) {
        case 2: return launch_half<2>(spec, env, first_opt, n_opt);
        case 4: return launch_half<4>(spec, env, first_opt, n_opt);
        default: return launch_half<3>(spec, env, first_opt, n_opt);
      }
    case 3: return launch<2, 4, false>(spec, env, first_opt, n_opt);
    case 4: return launch<2, 4>(spec, env, first_opt, n_opt);
    case 5: return launch_hw<6, 4, false>(spec, env, first_opt, n_opt);  // option setup inside the lattice kernel
    default:
      // measured with the setup inside the lattice kernel (MB, unroll):
      // (4,2) 13.57, (4,4) 12.93, (5,2) 12.97, (5,4) 12.84, (6,2) 12.69,
      // (6,4) 12.69 ms; with the records computed ahead (default): (6,4)
      // 11.70, (5,4) 11.82, (4,4) 12.47, (6,2) 12.70, (6,3) 12.83, (6,8) 12.63
      switch ((mb ? mb : 6) * 10 + hw_unroll) {
        case 42: return launch_hw<4, 2, true>(spec, env, first_opt, n_opt);
        case 44: return launch_hw<4, 4, true>(spec, env, first_opt, n_opt);
        case 52: return launch_hw<5, 2, true>(spec, env, first_opt, n_opt);
        case 54: return launch_hw<5, 4, true>(spec, env, first_opt, n_opt);
        case 62: return launch_hw<6, 2, true>(spec, env, first_opt, n_opt);
        default: return launch_hw<6, 4, true>(spec, env, first_opt, n_opt);
      }
  }
}

uint64_t binomial_scratch_bytes(const KernelSpec& spec) { return spec.binom.options * sizeof(OptionRec); }

}  // namespace ecl
