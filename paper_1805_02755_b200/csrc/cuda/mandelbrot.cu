// mandelbrot.cu — escape-time Mandelbrot for sm_100a, bit-exact with the
// reference kernel (workloads.hpp:78-100, lambda :215-223).
//
// Parity contract.  Every floating-point operation is an explicit _rn
// intrinsic in the reference's order, so no FMA contraction can happen
// whatever -fmad says:
//   cx = x0 + ((px * (x1 - x0)) / W)          workloads.hpp:97
//   xx = zx*zx; yy = zy*zy; escape if xx+yy > 4   :82-84
//   zy = (2*zx)*zy + cy;  zx = (xx - yy) + cx      :85-86
// Exact rewrites (same bits, fewer FP64-pipe instructions):
//  * (2*zx)*zy rounds to exactly 2*round(zx*zy) (scaling by two is exact
//    away from overflow/subnormals) and round(2*t + cy) is one
//    fma(t, 2, cy) because 2*t is exact.
//  * xx + yy is a sum of squares, so it is >= +0 and its IEEE bit pattern
//    orders like an unsigned integer: "xx + yy > 4.0" is one 64-bit integer
//    compare on the ALU pipe instead of a DSETP on the FP64 pipe.
//  * cx/cy depend on the column/row only: they are computed once per image
//    by coord_tables with the reference formula and looked up per pixel, so
//    the refill path has no IEEE double division.
//  * speculative blocks: 16 iterations run without the escape add while the
//    high words of xx and yy are OR-accumulated; if neither reached 2.0 the
//    sum stayed < 4 and no escape test could have fired, otherwise the lane
//    replays the block exactly (see the loop below).
// 6 FP64-pipe instructions per iteration on the fast path (3 DMUL, 2 DADD,
// 1 DFMA), 7 on the exact replay.
//
// Layout.  One persistent grid per package; each warp claims chunks of
// consecutive pixels from a device-wide counter (256-pixel chunks for the
// first 7/8 of the package, 32-pixel chunks for the tail so a launch drains
// evenly) and keeps all 32 lanes busy by refilling a lane with the next pixel
// of the chunk as soon as its pixel finishes (checked every R iterations):
// the divergence of the irregular set costs at most R-1 idle iterations per
// pixel instead of the warp-wide maximum.  Results are one uint4 per pixel:
// the four identical counts of the reference's 4:1 pattern (:217-222).
#include <atomic>
#include <cstdlib>

#include "kernels.cuh"

namespace ecl {
namespace {

constexpr unsigned kFull = 0xffffffffu;
constexpr uint64_t kBigChunk = 256;   // pixels per claim, bulk of the package
constexpr uint64_t kTailChunk = 32;   // pixels per claim, last 1/8
constexpr int kThreads = 256;
// Resident CTAs per SM: FP64 6 (<= 40 registers, no spills), FP32 8 (64 warps).
template <typename Real>
constexpr int kMinBlocks = sizeof(Real) == 8 ? 6 : 8;

template <typename Real>
struct Arith;

template <>
struct Arith<double> {
  using Bits = unsigned long long;
  static __device__ __forceinline__ double mul(double a, double b) { return __dmul_rn(a, b); }
  static __device__ __forceinline__ double add(double a, double b) { return __dadd_rn(a, b); }
  static __device__ __forceinline__ double sub(double a, double b) { return __dsub_rn(a, b); }
  static __device__ __forceinline__ double div(double a, double b) { return __ddiv_rn(a, b); }
  static __device__ __forceinline__ double twice_plus(double t, double c) { return __fma_rn(t, 2.0, c); }
  static __device__ __forceinline__ double from_u64(uint64_t v) { return __ull2double_rn(v); }
  static __device__ __forceinline__ Bits bits(double v) { return static_cast<Bits>(__double_as_longlong(v)); }
  static __device__ __forceinline__ uint32_t high(double v) { return static_cast<uint32_t>(__double2hiint(v)); }
  static constexpr Bits kFourBits = 0x4010000000000000ull;  // 4.0
};

template <>
struct Arith<float> {
  using Bits = unsigned;
  static __device__ __forceinline__ float mul(float a, float b) { return __fmul_rn(a, b); }
  static __device__ __forceinline__ float add(float a, float b) { return __fadd_rn(a, b); }
  static __device__ __forceinline__ float sub(float a, float b) { return __fsub_rn(a, b); }
  static __device__ __forceinline__ float div(float a, float b) { return __fdiv_rn(a, b); }
  static __device__ __forceinline__ float twice_plus(float t, float c) { return __fmaf_rn(t, 2.0f, c); }
  static __device__ __forceinline__ float from_u64(uint64_t v) { return __ull2float_rn(v); }
  static __device__ __forceinline__ Bits bits(float v) { return __float_as_uint(v); }
  static __device__ __forceinline__ uint32_t high(float v) { return __float_as_uint(v); }
  static constexpr Bits kFourBits = 0x40800000u;  // 4.0f
};

template <typename Real>
struct Viewport {
  uint64_t width, height;
  uint32_t max_iterations;
  Real x0, y0, span_x, span_y, fw, fh;  // span = x1 - x0 rounded in Real
};

// cx[px] for px < W, then cy[py] for py < H: the reference's coordinate map.
template <typename Real>
__global__ void coord_tables(const Viewport<Real> vp, Real* __restrict__ tab) {
  using A = Arith<Real>;
  const uint64_t n = vp.width + vp.height;
  for (uint64_t i = blockIdx.x * static_cast<uint64_t>(blockDim.x) + threadIdx.x; i < n;
       i += static_cast<uint64_t>(gridDim.x) * blockDim.x) {
    tab[i] = i < vp.width ? A::add(vp.x0, A::div(A::mul(A::from_u64(i), vp.span_x), vp.fw))
                          : A::add(vp.y0, A::div(A::mul(A::from_u64(i - vp.width), vp.span_y), vp.fh));
  }
}

// One speculative block of RB iterations for this lane, replayed exactly
// when its flag is raised (see the comment at the call site).  Warp-uniform
// control: every lane of the warp calls it with the same RB.
//
// Loop = true (settled warps): end-checked blocks repeat in a tight loop
// until a live lane raises its flag or the next block could reach max_it,
// so the outer loop's refill ballot, block-length vote and store check run
// once per pixel event instead of once per block (ncu, 16384^2 x 2048: 57
// control instructions per 32-iteration block against 192 FP64 ones, each
// FP64 instruction holding the issue port two cycles).  The block that
// raised a flag ends exactly like a single block: unflagged lanes commit,
// flagged lanes replay it from its saved state.
template <typename Real, int RB, bool Loop = false>
__device__ __forceinline__ void spec_block(Real& zx, Real& zy, uint32_t& n, bool& alive, bool far, Real cx, Real cy,
                                           uint32_t max_it) {
  using A = Arith<Real>;
  using Bits = typename A::Bits;
  Real zx0 = zx, zy0 = zy;
  uint32_t n0 = n;
  bool fast;
  if (__all_sync(kFull, far || !alive)) {
    bool done = false;
    if constexpr (Loop) {
      // Blocks every live lane can take before max_it; the loop runs all but
      // the last, which the regular block below handles with its max_it rule.
      uint32_t room = alive ? (max_it - n) / RB : 0xffffffffu;
      room = __reduce_min_sync(kFull, room);
      uint32_t k = 0;
      for (; k + 1 < room; ++k) {
        zx0 = zx;
        zy0 = zy;
#pragma unroll
        for (int r = 0; r < RB - 1; ++r) {
          const Real xx = A::mul(zx, zx);
          const Real yy = A::mul(zy, zy);
          const Real t = A::mul(zx, zy);
          zy = A::twice_plus(t, cy);
          zx = A::add(A::sub(xx, yy), cx);
        }
        const Real xx = A::mul(zx, zx);
        const Real yy = A::mul(zy, zy);
        const uint32_t acc = A::high(xx) | A::high(yy);
        const Real t = A::mul(zx, zy);
        zy = A::twice_plus(t, cy);
        zx = A::add(A::sub(xx, yy), cx);
        // acc >= 2^30 <=> bit 30 of a square's high word (a square's sign
        // bit is clear unless it is NaN, whose exponent sets bit 30 too):
        // one compare instead of shift, mask and compare.
        const bool flag = alive && acc >= 0x40000000u;
        if (__any_sync(kFull, flag)) {  // this block ends like a regular one
          n += k * RB;
          n0 = n;
          fast = alive && !flag;
          if (fast) n = n0 + RB;  // n0 + RB <= max_it: k + 1 < room
          done = true;
          break;
        }
      }
      if (!done) {
        n += k * RB;
        n0 = n;
        zx0 = zx;
        zy0 = zy;
      }
    }
    if (!done) {
#pragma unroll
      for (int r = 0; r < RB - 1; ++r) {
        const Real xx = A::mul(zx, zx);
        const Real yy = A::mul(zy, zy);
        const Real t = A::mul(zx, zy);
        zy = A::twice_plus(t, cy);
        zx = A::add(A::sub(xx, yy), cx);
      }
      const Real xx = A::mul(zx, zx);
      const Real yy = A::mul(zy, zy);
      const uint32_t acc = A::high(xx) | A::high(yy);
      const Real t = A::mul(zx, zy);
      zy = A::twice_plus(t, cy);
      zx = A::add(A::sub(xx, yy), cx);
      fast = alive && n0 + RB <= max_it && acc < 0x40000000u;
      if (fast) {
        n = n0 + RB;
        alive = n < max_it;
      }
    }
  } else {
    uint32_t acc = 0;
#pragma unroll
    for (int r = 0; r < RB; ++r) {
      const Real xx = A::mul(zx, zx);
      const Real yy = A::mul(zy, zy);
      acc |= A::high(xx) | A::high(yy);
      const Real t = A::mul(zx, zy);
      zy = A::twice_plus(t, cy);
      zx = A::add(A::sub(xx, yy), cx);
    }
    fast = alive && n0 + RB <= max_it && acc < 0x40000000u;
    if (fast) {
      n = n0 + RB;
      alive = n < max_it;
    }
  }
  bool live = alive && !fast;  // lanes replaying the block exactly
  if (__any_sync(kFull, live)) {
    if (live) {
      zx = zx0;
      zy = zy0;
      n = n0;
    }
#pragma unroll
    for (int r = 0; r < RB; ++r) {
      const Real xx = A::mul(zx, zx);
      const Real yy = A::mul(zy, zy);
      const Bits s = A::bits(A::add(xx, yy));  // >= +0: integer order == FP order
      live = live && s <= A::kFourBits;
      const Real t = A::mul(zx, zy);
      const Real nzy = A::twice_plus(t, cy);
      const Real nzx = A::add(A::sub(xx, yy), cx);
      if (live) {
        zx = nzx;
        zy = nzy;
        n += 1u;
      }
      live = live && n < max_it;
      // every replaying lane has escaped (or hit max_it): the rest of the
      // block would change nothing
      if ((r & 1) == 1 && r + 1 < RB && !__any_sync(kFull, live)) break;
    }
    if (alive && !fast) alive = live;
  }
}

// Periodic = true (variant mandelbrot@14): exact early exit for orbits that
// became periodic in floating point.  At block ends the state (zx, zy) is
// compared bit for bit with a checkpoint taken at an earlier block end
// (Brent: re-taken whenever n passes 32, 64, 128, ...).  Equal bits mean the
// deterministic FP64 map repeats the same cycle forever, and the blocks in
// between raised no escape, so the reference's loop would run to max_iter
// without escaping: the count is max_iter, identical to iterating on.  Most
// of the set's interior converges to an exact fixed point or short cycle in
// a few hundred iterations (a 400k-pixel sample of the config: 89 % of the
// interior pixels detected, at 561 iterations on average instead of 2048).
// Off by default: the bench's headline runs every reference iteration.
template <typename Real, int R, int MB = kMinBlocks<Real>, int RL = R, uint32_t kSettle = 32, bool Periodic = false,
          bool Tight = true>
__global__ void __launch_bounds__(kThreads, MB)
    mandel_persistent(const Viewport<Real> vp, const Real* __restrict__ tab, uint64_t first, uint64_t count,
                      uint4* __restrict__ out, const CompactOut compact, unsigned* __restrict__ ctrl) {
  using A = Arith<Real>;
  using Bits = typename A::Bits;
  const unsigned lane = threadIdx.x & 31u;
  const unsigned below = (1u << lane) - 1u;
  const uint64_t big = (count - count / 8) / kBigChunk;  // claims 0..big-1 are 256-pixel chunks
  const uint64_t tail_start = big * kBigChunk;
  const uint64_t nclaims = big + (count - tail_start + kTailChunk - 1) / kTailChunk;
  const Real* __restrict__ cxs = tab;
  const Real* __restrict__ cys = tab + vp.width;

  // Warp-uniform cursor over the claimed chunk: [next, end) relative to
  // first, with (px0, py0) the column/row of `next`.
  uint64_t next = 0, end = 0, px0 = 0, py0 = 0;
  bool more = true;
  auto claim = [&]() {
    unsigned c = 0;
    if (lane == 0) c = atomicAdd(ctrl, 1u);
    c = __shfl_sync(kFull, c, 0);
    if (c >= nclaims) {
      more = false;
      next = end = 0;
      return;
    }
    next = c < big ? c * kBigChunk : tail_start + (c - big) * kTailChunk;
    const uint64_t size = c < big ? kBigChunk : kTailChunk;
    end = next + size < count ? next + size : count;
    const uint64_t g = first + next;
    py0 = g / vp.width;
    px0 = g - py0 * vp.width;
  };
  claim();

  bool valid = false, alive = false, far = true;
  uint64_t idx = 0;
  Real cx = 0, cy = 0, zx = 0, zy = 0;
  uint32_t n = 0;
  const uint32_t max_it = vp.max_iterations;
  Real rx = 0, ry = 0;     // Periodic: checkpoint state
  uint32_t ckpt = 0;       // Periodic: n at which the next checkpoint is taken
  bool have_ckpt = false;

  for (;;) {
    // Refill idle lanes in lane order with the next pixels of the chunk.
    unsigned need = __ballot_sync(kFull, !valid);
    while (need && more) {
      const unsigned rank = __popc(need & below);
      const uint64_t avail = end - next;
      if (!valid && rank < avail) {
        idx = first + next + rank;
        uint64_t px = px0 + rank, py = py0;
        while (px >= vp.width) {  // at most once when W >= chunk size
          px -= vp.width;
          ++py;
        }
        cx = cxs[px];
        cy = cys[py];
        zx = 0;
        zy = 0;
        n = 0;
        valid = true;
        alive = true;
        far = cx * cx + cy * cy < Real(3.6);  // |c| < 1.9 (see end_checked_block)
        if constexpr (Periodic) {
          ckpt = 32;
          have_ckpt = false;
        }
      }
      const uint64_t take = __popc(need) < avail ? __popc(need) : avail;
      next += take;
      px0 += take;
      while (px0 >= vp.width) {
        px0 -= vp.width;
        ++py0;
      }
      if (next >= end) claim();
      need = __ballot_sync(kFull, !valid);
    }
    if (!__any_sync(kFull, valid)) break;

    // Speculative block: R iterations without the escape add.  If neither
    // zx^2 nor zy^2 reached 2.0 anywhere in the block (bit 30 of the IEEE
    // high word, OR-accumulated), xx + yy < 4 held at every step, so the
    // reference's test "xx + yy > 4" was false at every step: the block is
    // exactly R reference iterations.  Otherwise the lane replays the block
    // from the saved state with the per-iteration test.
    //
    // End-checked blocks: when every live pixel of the warp has |c| < 1.9,
    // only the block's last iteration is checked.  Sound: an escape at step
    // e means |z_e|^2 > 4 - O(ulp), so |z_e+1| >= |z_e|^2 - |c| - O(ulp)
    // >= 2.09, and from |z| >= 2.09 on, |z|^2 - |c| >= |z| + 0.37: the orbit
    // grows monotonically, every later square pair has max >= 2.18 (bit 30
    // set; inf and NaN after overflow set it too), so the last iteration of
    // the block raises the flag.  Saves the per-iteration OR — FP64
    // instructions hold the issue port two cycles each, so it cost ~8 %
    // (tools/probe/mandel_mix2.cu) — and skips replays for orbits that only
    // pass |z| > sqrt(2) mid-block.
    // Block length: every live pixel of the warp past its first kSettle
    // iterations (long orbits, mostly the set's interior) -> RL-iteration
    // blocks, amortizing the block control; otherwise R, so pixels that
    // escape early waste fewer speculative iterations.
    if (__all_sync(kFull, !alive || n >= kSettle))
      spec_block<Real, RL, Tight && !Periodic>(zx, zy, n, alive, far, cx, cy, max_it);
    else spec_block<Real, R>(zx, zy, n, alive, far, cx, cy, max_it);
    if constexpr (Periodic) {
      if (valid && alive) {
        if (have_ckpt && A::bits(zx) == A::bits(rx) && A::bits(zy) == A::bits(ry)) {
          n = max_it;  // periodic orbit: never escapes
          alive = false;
        } else if (n >= ckpt) {
          rx = zx;
          ry = zy;
          have_ckpt = true;
          ckpt = 2 * ckpt;
        }
      }
    }
    if (valid && !alive) {
      out[idx] = make_uint4(n, n, n, n);
      if (compact) compact.put(idx, n);  // host-bound copy: one count per pixel
      valid = false;
    }
  }

  // The last block out resets the claim counter for the next package.
  __syncthreads();
  if (threadIdx.x == 0) {
    __threadfence();
    const unsigned done = atomicAdd(ctrl + 1, 1u);
    if (done == gridDim.x - 1) {
      atomicExch(ctrl, 0u);
      atomicExch(ctrl + 1, 0u);
    }
  }
}

// ---- FP32 variant, two pixels per lane ------------------------------------
// The FP32 kernel above is issue-bound (6 FP32 + 1 integer instruction per
// pixel-iteration, ncu: 94 % issue, 58 % FMA pipe).  Here every lane carries
// two pixels ("slots" A and B) in float2 registers and iterates them with
// packed FFMA2/FADD2: per pixel-iteration 3 FP32 + 1 integer instruction.
// Parity: packed ops round each component like the scalar _rn ops.  Products
// are formed as fma(x, y, +0) because ptxas contracts a packed multiply into
// a following packed add (FFMA2) even with -fmad=false; x*y + 0 equals the
// rounded product except that a -0 product becomes +0, and the only -0
// product here (zx*zy) feeds 2t + cy with cy != -0 (a sum y0 + k*span never
// rounds to -0), so the counts stay bit-identical to the FP32 restatement.
// Pair arithmetic: float pairs are packed (FFMA2/FADD2, products as
// fma(x, y, +0)); double pairs are two scalar _rn ops (no packed FP64) —
// there the second pixel only adds independent work per warp (ILP).
template <typename Real>
struct Pair;

template <>
struct Pair<float> {
  using V = float2;
  static __device__ __forceinline__ V mk(float a, float b) { return make_float2(a, b); }
  static __device__ __forceinline__ V mul0(V a, V b) { return __ffma2_rn(a, b, make_float2(0.0f, 0.0f)); }
  static __device__ __forceinline__ V twice_plus(V t, V c) { return __ffma2_rn(t, make_float2(2.0f, 2.0f), c); }
  static __device__ __forceinline__ V add(V a, V b) { return __fadd2_rn(a, b); }
  static __device__ __forceinline__ V sub(V a, V b) { return __fadd2_rn(a, make_float2(-b.x, -b.y)); }
  static __device__ __forceinline__ uint32_t hi(float v) { return __float_as_uint(v); }
  static __device__ __forceinline__ bool le4(float v) { return __float_as_uint(v) <= 0x40800000u; }
};

template <>
struct Pair<double> {
  using V = double2;
  static __device__ __forceinline__ V mk(double a, double b) { return make_double2(a, b); }
  static __device__ __forceinline__ V mul0(V a, V b) { return make_double2(__dmul_rn(a.x, b.x), __dmul_rn(a.y, b.y)); }
  static __device__ __forceinline__ V twice_plus(V t, V c) {
    return make_double2(__fma_rn(t.x, 2.0, c.x), __fma_rn(t.y, 2.0, c.y));
  }
  static __device__ __forceinline__ V add(V a, V b) { return make_double2(__dadd_rn(a.x, b.x), __dadd_rn(a.y, b.y)); }
  static __device__ __forceinline__ V sub(V a, V b) { return make_double2(__dsub_rn(a.x, b.x), __dsub_rn(a.y, b.y)); }
  static __device__ __forceinline__ uint32_t hi(double v) { return static_cast<uint32_t>(__double2hiint(v)); }
  static __device__ __forceinline__ bool le4(double v) {
    return static_cast<unsigned long long>(__double_as_longlong(v)) <= 0x4010000000000000ull;
  }
};

struct Slot2 {
  uint64_t idx = 0;
  uint32_t n = 0;
  bool valid = false, alive = false, far = true;  // far: |c| < 1.9 (end-checked blocks allowed)
};

// One speculative block of RB iterations on both slots of a lane (see
// spec_block); warp-uniform RB.  Loop = true: the tight settled loop of
// spec_block, on both slots.
template <typename Real, int RB, bool Loop = false>
__device__ __forceinline__ void spec_block2(typename Pair<Real>::V& zx, typename Pair<Real>::V& zy, Slot2& sa,
                                            Slot2& sb, typename Pair<Real>::V cx, typename Pair<Real>::V cy,
                                            uint32_t max_it) {
  using A = Pair<Real>;
  using V = typename A::V;
  V zx0 = zx, zy0 = zy;
  uint32_t na0 = sa.n, nb0 = sb.n;
  bool fast_a, fast_b;
  if (__all_sync(kFull, (sa.far || !sa.alive) && (sb.far || !sb.alive))) {  // end-checked block
    bool done = false;
    if constexpr (Loop) {
      const uint32_t ra = sa.alive ? (max_it - sa.n) / RB : 0xffffffffu;
      const uint32_t rb = sb.alive ? (max_it - sb.n) / RB : 0xffffffffu;
      const uint32_t room = __reduce_min_sync(kFull, ra < rb ? ra : rb);
      uint32_t k = 0;
      for (; k + 1 < room; ++k) {
        zx0 = zx;
        zy0 = zy;
#pragma unroll
        for (int r = 0; r < RB - 1; ++r) {
          const V xx = A::mul0(zx, zx);
          const V yy = A::mul0(zy, zy);
          const V t = A::mul0(zx, zy);
          zy = A::twice_plus(t, cy);
          zx = A::add(A::sub(xx, yy), cx);
        }
        const V xx = A::mul0(zx, zx);
        const V yy = A::mul0(zy, zy);
        const uint32_t acc_a = A::hi(xx.x) | A::hi(yy.x);
        const uint32_t acc_b = A::hi(xx.y) | A::hi(yy.y);
        const V t = A::mul0(zx, zy);
        zy = A::twice_plus(t, cy);
        zx = A::add(A::sub(xx, yy), cx);
        // acc >= 2^30 <=> bit 30 of a square (see spec_block)
        const bool flag_a = sa.alive && acc_a >= 0x40000000u;
        const bool flag_b = sb.alive && acc_b >= 0x40000000u;
        if (__any_sync(kFull, flag_a || flag_b)) {  // this block ends like a regular one
          sa.n += k * RB;
          sb.n += k * RB;
          na0 = sa.n;
          nb0 = sb.n;
          fast_a = sa.alive && !flag_a;
          fast_b = sb.alive && !flag_b;
          if (fast_a) sa.n = na0 + RB;  // < max_it: k + 1 < room
          if (fast_b) sb.n = nb0 + RB;
          done = true;
          break;
        }
      }
      if (!done) {
        sa.n += k * RB;
        sb.n += k * RB;
        na0 = sa.n;
        nb0 = sb.n;
        zx0 = zx;
        zy0 = zy;
      }
    }
    if (!done) {
#pragma unroll
      for (int r = 0; r < RB - 1; ++r) {
        const V xx = A::mul0(zx, zx);
        const V yy = A::mul0(zy, zy);
        const V t = A::mul0(zx, zy);
        zy = A::twice_plus(t, cy);
        zx = A::add(A::sub(xx, yy), cx);
      }
      const V xx = A::mul0(zx, zx);
      const V yy = A::mul0(zy, zy);
      const uint32_t acc_a = A::hi(xx.x) | A::hi(yy.x);
      const uint32_t acc_b = A::hi(xx.y) | A::hi(yy.y);
      const V t = A::mul0(zx, zy);
      zy = A::twice_plus(t, cy);
      zx = A::add(A::sub(xx, yy), cx);
      fast_a = sa.alive && na0 + RB <= max_it && acc_a < 0x40000000u;
      fast_b = sb.alive && nb0 + RB <= max_it && acc_b < 0x40000000u;
      if (fast_a) {
        sa.n = na0 + RB;
        sa.alive = sa.n < max_it;
      }
      if (fast_b) {
        sb.n = nb0 + RB;
        sb.alive = sb.n < max_it;
      }
    }
  } else {
    uint32_t acc_a = 0, acc_b = 0;
#pragma unroll
    for (int r = 0; r < RB; ++r) {
      const V xx = A::mul0(zx, zx);
      const V yy = A::mul0(zy, zy);
      acc_a |= A::hi(xx.x) | A::hi(yy.x);
      acc_b |= A::hi(xx.y) | A::hi(yy.y);
      const V t = A::mul0(zx, zy);
      zy = A::twice_plus(t, cy);
      zx = A::add(A::sub(xx, yy), cx);
    }
    fast_a = sa.alive && na0 + RB <= max_it && acc_a < 0x40000000u;
    fast_b = sb.alive && nb0 + RB <= max_it && acc_b < 0x40000000u;
    if (fast_a) {
      sa.n = na0 + RB;
      sa.alive = sa.n < max_it;
    }
    if (fast_b) {
      sb.n = nb0 + RB;
      sb.alive = sb.n < max_it;
    }
  }
  bool live_a = sa.alive && !fast_a, live_b = sb.alive && !fast_b;
  if (__any_sync(kFull, live_a || live_b)) {
    if (live_a) {
      zx.x = zx0.x;
      zy.x = zy0.x;
      sa.n = na0;
    }
    if (live_b) {
      zx.y = zx0.y;
      zy.y = zy0.y;
      sb.n = nb0;
    }
#pragma unroll
    for (int r = 0; r < RB; ++r) {
      const V xx = A::mul0(zx, zx);
      const V yy = A::mul0(zy, zy);
      const V s = A::add(xx, yy);  // >= +0: integer order == FP order
      live_a = live_a && A::le4(s.x);
      live_b = live_b && A::le4(s.y);
      const V t = A::mul0(zx, zy);
      const V nzy = A::twice_plus(t, cy);
      const V nzx = A::add(A::sub(xx, yy), cx);
      if (live_a) {
        zx.x = nzx.x;
        zy.x = nzy.x;
        sa.n += 1u;
      }
      if (live_b) {
        zx.y = nzx.y;
        zy.y = nzy.y;
        sb.n += 1u;
      }
      live_a = live_a && sa.n < max_it;
      live_b = live_b && sb.n < max_it;
    }
    if (sa.alive && !fast_a) sa.alive = live_a;
    if (sb.alive && !fast_b) sb.alive = live_b;
  }
}

constexpr uint32_t kSettle2 = 32;

template <typename Real, int R, int MB, int RL = R, bool Tight = true>
__global__ void __launch_bounds__(kThreads, MB)
    mandel_x2(const Viewport<Real> vp, const Real* __restrict__ tab, uint64_t first, uint64_t count,
              uint4* __restrict__ out, const CompactOut compact, unsigned* __restrict__ ctrl) {
  using A = Pair<Real>;
  using V = typename A::V;
  const unsigned lane = threadIdx.x & 31u;
  const unsigned below = (1u << lane) - 1u;
  const uint64_t big = (count - count / 8) / kBigChunk;
  const uint64_t tail_start = big * kBigChunk;
  const uint64_t nclaims = big + (count - tail_start + kTailChunk - 1) / kTailChunk;
  const Real* __restrict__ cxs = tab;
  const Real* __restrict__ cys = tab + vp.width;

  uint64_t next = 0, end = 0, px0 = 0, py0 = 0;
  bool more = true;
  auto claim = [&]() {
    unsigned c = 0;
    if (lane == 0) c = atomicAdd(ctrl, 1u);
    c = __shfl_sync(kFull, c, 0);
    if (c >= nclaims) {
      more = false;
      next = end = 0;
      return;
    }
    next = c < big ? c * kBigChunk : tail_start + (c - big) * kTailChunk;
    const uint64_t size = c < big ? kBigChunk : kTailChunk;
    end = next + size < count ? next + size : count;
    const uint64_t g = first + next;
    py0 = g / vp.width;
    px0 = g - py0 * vp.width;
  };
  claim();

  Slot2 sa, sb;
  V cx = A::mk(0, 0), cy = cx, zx = cx, zy = cx;
  const uint32_t max_it = vp.max_iterations;

  // Gives pixel `rank` of the chunk's remaining range to a slot.
  auto assign = [&](Slot2& s, Real& scx, Real& scy, Real& szx, Real& szy, unsigned rank) {
    s.idx = first + next + rank;
    uint64_t px = px0 + rank, py = py0;
    while (px >= vp.width) {
      px -= vp.width;
      ++py;
    }
    scx = cxs[px];
    scy = cys[py];
    szx = 0;
    szy = 0;
    s.n = 0;
    s.valid = true;
    s.alive = true;
    s.far = scx * scx + scy * scy < Real(3.6);
  };

  for (;;) {
    // Refill idle slots: the 64 slots of the warp in order A0..A31, B0..B31.
    unsigned need_a = __ballot_sync(kFull, !sa.valid), need_b = __ballot_sync(kFull, !sb.valid);
    while ((need_a | need_b) && more) {
      const uint64_t avail = end - next;
      const unsigned na = __popc(need_a);
      const unsigned ra = __popc(need_a & below), rb = na + __popc(need_b & below);
      if (!sa.valid && ra < avail) assign(sa, cx.x, cy.x, zx.x, zy.x, ra);
      if (!sb.valid && rb < avail) assign(sb, cx.y, cy.y, zx.y, zy.y, rb);
      const uint64_t want = na + __popc(need_b);
      const uint64_t take = want < avail ? want : avail;
      next += take;
      px0 += take;
      while (px0 >= vp.width) {
        px0 -= vp.width;
        ++py0;
      }
      if (next >= end) claim();
      need_a = __ballot_sync(kFull, !sa.valid);
      need_b = __ballot_sync(kFull, !sb.valid);
    }
    if (!__any_sync(kFull, sa.valid || sb.valid)) break;

    // Speculative block on both slots (see mandel_persistent); long blocks
    // once every live pixel of the warp has settled.
    if (__all_sync(kFull, (!sa.alive || sa.n >= kSettle2) && (!sb.alive || sb.n >= kSettle2)))
      spec_block2<Real, RL, Tight>(zx, zy, sa, sb, cx, cy, max_it);
    else
      spec_block2<Real, R>(zx, zy, sa, sb, cx, cy, max_it);
    if (sa.valid && !sa.alive) {
      out[sa.idx] = make_uint4(sa.n, sa.n, sa.n, sa.n);
      if (compact) compact.put(sa.idx, sa.n);
      sa.valid = false;
    }
    if (sb.valid && !sb.alive) {
      out[sb.idx] = make_uint4(sb.n, sb.n, sb.n, sb.n);
      if (compact) compact.put(sb.idx, sb.n);
      sb.valid = false;
    }
  }

  __syncthreads();
  if (threadIdx.x == 0) {
    __threadfence();
    const unsigned done = atomicAdd(ctrl + 1, 1u);
    if (done == gridDim.x - 1) {
      atomicExch(ctrl, 0u);
      atomicExch(ctrl + 1, 0u);
    }
  }
}

template <typename Real>
Viewport<Real> make_viewport(const MandelParams& p) {
  Viewport<Real> vp;
  vp.width = p.width;
  vp.height = p.height;
  vp.max_iterations = p.max_iterations;
  const Real x0 = static_cast<Real>(p.x0), y0 = static_cast<Real>(p.y0);
  const Real x1 = static_cast<Real>(p.x1), y1 = static_cast<Real>(p.y1);
  vp.x0 = x0;
  vp.y0 = y0;
  // x1 - x0 rounded once in Real: the value the reference recomputes per
  // pixel (host subtraction is IEEE round-to-nearest, no contraction).
  volatile Real sx = x1 - x0, sy = y1 - y0;
  vp.span_x = sx;
  vp.span_y = sy;
  vp.fw = static_cast<Real>(p.width);
  vp.fh = static_cast<Real>(p.height);
  return vp;
}

template <typename Real, int R, int MB = kMinBlocks<Real>, int RL = R, uint32_t kSettle = 32, bool Periodic = false,
          bool Tight = true>
cudaError_t launch_real(const MandelParams& p, const LaunchEnv& env, uint64_t first, uint64_t count) {
  // resident CTAs per SM: a property of the instantiation (device threads
  // may race to fill it with the same value)
  static std::atomic<int> occ{0};
  int blocks_per_sm = occ.load(std::memory_order_relaxed);
  if (blocks_per_sm == 0) {
    cudaError_t e = cudaOccupancyMaxActiveBlocksPerMultiprocessor(
        &blocks_per_sm, mandel_persistent<Real, R, MB, RL, kSettle, Periodic, Tight>, kThreads, 0);
    if (e != cudaSuccess) return e;
    if (blocks_per_sm < 1) blocks_per_sm = 1;
    occ.store(blocks_per_sm, std::memory_order_relaxed);
  }
  const Viewport<Real> vp = make_viewport<Real>(p);
  const Real* tab = static_cast<const Real*>(env.scratch);
  const uint64_t claims = (count + kTailChunk - 1) / kTailChunk;
  const uint64_t blocks_needed = (claims + kThreads / 32 - 1) / (kThreads / 32);
  uint64_t grid = static_cast<uint64_t>(env.sms) * static_cast<uint64_t>(blocks_per_sm);
  if (blocks_needed < grid) grid = blocks_needed;
  if (grid == 0) return cudaSuccess;
  mandel_persistent<Real, R, MB, RL, kSettle, Periodic, Tight><<<static_cast<unsigned>(grid), kThreads, 0, env.stream>>>(
      vp, tab, first, count, static_cast<uint4*>(env.out[0]), compact_of(env), env.ctrl);
  return cudaGetLastError();
}

template <typename Real, int R, int MB, int RL = R, bool Tight = true>
cudaError_t launch_x2(const MandelParams& p, const LaunchEnv& env, uint64_t first, uint64_t count) {
  static std::atomic<int> occ{0};
  int blocks_per_sm = occ.load(std::memory_order_relaxed);
  if (blocks_per_sm == 0) {
    cudaError_t e = cudaOccupancyMaxActiveBlocksPerMultiprocessor(&blocks_per_sm, mandel_x2<Real, R, MB, RL, Tight>, kThreads, 0);
    if (e != cudaSuccess) return e;
    if (blocks_per_sm < 1) blocks_per_sm = 1;
    occ.store(blocks_per_sm, std::memory_order_relaxed);
  }
  const Viewport<Real> vp = make_viewport<Real>(p);
  const uint64_t claims = (count + kTailChunk - 1) / kTailChunk;
  const uint64_t blocks_needed = (claims + kThreads / 32 - 1) / (kThreads / 32);
  uint64_t grid = static_cast<uint64_t>(env.sms) * static_cast<uint64_t>(blocks_per_sm);
  if (blocks_needed < grid) grid = blocks_needed;
  if (grid == 0) return cudaSuccess;
  mandel_x2<Real, R, MB, RL, Tight><<<static_cast<unsigned>(grid), kThreads, 0, env.stream>>>(
      vp, static_cast<const Real*>(env.scratch), first, count, static_cast<uint4*>(env.out[0]), compact_of(env),
      env.ctrl);
  return cudaGetLastError();
}

template <typename Real>
cudaError_t tables(const MandelParams& p, const LaunchEnv& env) {
  const uint64_t n = p.width + p.height;
  const unsigned grid = static_cast<unsigned>((n + 255) / 256 < 4096 ? (n + 255) / 256 : 4096);
  coord_tables<Real><<<grid, 256, 0, env.stream>>>(make_viewport<Real>(p), static_cast<Real*>(env.scratch));
  return cudaGetLastError();
}

}  // namespace

uint64_t mandelbrot_scratch_bytes(const KernelSpec& spec) {
  return (spec.mandel.width + spec.mandel.height) * sizeof(double);
}

cudaError_t prepare_mandelbrot(const KernelSpec& spec, const LaunchEnv& env) {
  return spec.kind == KernelKind::MandelbrotF32 ? tables<float>(spec.mandel, env) : tables<double>(spec.mandel, env);
}

cudaError_t launch_mandelbrot(const KernelSpec& spec, const LaunchEnv& env, uint64_t first, uint64_t count) {
  if (count == 0) return cudaSuccess;
  if (spec.kind == KernelKind::MandelbrotF32) {
    static const bool scalar_env = [] {  // ECL_MANDEL_F32_SCALAR=1: one pixel per lane
      const char* v = std::getenv("ECL_MANDEL_F32_SCALAR");
      return v && std::atoi(v) == 1;
    }();
    const bool scalar = spec.variant >= 0 ? spec.variant == 1 : scalar_env;
    // mandelbrot_f32@2: the default without the tight settled loop
    if (spec.variant == 2) return launch_x2<float, 16, 4, 32, false>(spec.mandel, env, first, count);
    static const int mb = [] {  // ECL_MANDEL_F32_MB: resident CTAs per SM
      const char* v = std::getenv("ECL_MANDEL_F32_MB");
      return v ? std::atoi(v) : 0;
    }();
    if (scalar) return launch_real<float, 16>(spec.mandel, env, first, count);
    switch (mb) {
      // measured: adaptive (16 -> 32 after 32 iterations, 4 CTAs) 23.7 ms, (8 -> 32) 23.8,
      // (16 -> 64) 24.0, fixed 16 25.3, fixed 32 (5 CTAs) 25.0
      case 5: return launch_x2<float, 16, 5>(spec.mandel, env, first, count);
      case 6: return launch_x2<float, 16, 6>(spec.mandel, env, first, count);
      case 32: return launch_x2<float, 32, 5>(spec.mandel, env, first, count);
      case 16: return launch_x2<float, 16, 4>(spec.mandel, env, first, count);
      case 7: return launch_x2<float, 8, 4, 32>(spec.mandel, env, first, count);
      case 8: return launch_x2<float, 16, 4, 64>(spec.mandel, env, first, count);
      default: return launch_x2<float, 16, 4, 32>(spec.mandel, env, first, count);
    }
  }
  // Tuning hook (ECL_MANDEL_VARIANT): block length R and resident CTAs per SM.
  static const int env_variant = [] {
    const char* v = std::getenv("ECL_MANDEL_VARIANT");
    return v ? std::atoi(v) : 0;
  }();
  switch (spec.variant >= 0 ? spec.variant : env_variant) {
    case 1: return launch_real<double, 16, 6>(spec.mandel, env, first, count);
    case 2: return launch_real<double, 32, 4>(spec.mandel, env, first, count);
    case 3: return launch_real<double, 8, 4>(spec.mandel, env, first, count);
    case 4: return launch_real<double, 16, 3>(spec.mandel, env, first, count);
    // two pixels per lane: bit-exact but measured slower (46.8 vs 44.3 ms at
    // the config): the FP64 kernel is not short of independent work
    case 5: return launch_x2<double, 16, 2>(spec.mandel, env, first, count);
    case 6: return launch_x2<double, 16, 3>(spec.mandel, env, first, count);
    case 7: return launch_real<double, 16, 4, 32>(spec.mandel, env, first, count);
    case 8: return launch_real<double, 8, 4, 32>(spec.mandel, env, first, count);
    case 9: return launch_real<double, 16, 4, 64>(spec.mandel, env, first, count);
    case 10: return launch_real<double, 8, 4, 64>(spec.mandel, env, first, count);
    case 11: return launch_real<double, 8, 4, 32, 16>(spec.mandel, env, first, count);
    case 12: return launch_real<double, 8, 4, 32, 64>(spec.mandel, env, first, count);
    case 13: return launch_real<double, 8, 4, 24>(spec.mandel, env, first, count);
    // exact early exit for periodic orbits (see mandel_persistent): same
    // counts, a fraction of the interior's iterations
    case 14: return launch_real<double, 8, 4, 32, 32, true>(spec.mandel, env, first, count);
    // the default without the tight settled loop (one outer-loop pass per block)
    case 15: return launch_real<double, 8, 4, 32, 32, false, false>(spec.mandel, env, first, count);
    // measured (16384^2 x 2048): (8, 32 after 32 iterations) 38.85 ms; fixed 16: 41.2 ms;
    // (16, 32) 39.2; (8, 64) 39.1; (16, 64) 39.3; settle after 16 / 64: 39.2; (8, 24) 39.8.
    // With the tight settled loop (kernel only): (8, 32) 36.5 ms; 5 CTAs/SM 36.7;
    // settle after 16: 37.0; (16, 32) 36.9; (8, 64) 38.0; (4, 32) 37.8; settle after
    // 24 / 48: 36.9 / 37.1; (12, 36) 39.3.
    default: return launch_real<double, 8, 4, 32>(spec.mandel, env, first, count);
  }
}

}  // namespace ecl
