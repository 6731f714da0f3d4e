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

template <typename Real, int R, int MB = kMinBlocks<Real>>
__global__ void __launch_bounds__(kThreads, MB)
    mandel_persistent(const Viewport<Real> vp, const Real* __restrict__ tab, uint64_t first, uint64_t count,
                      uint4* __restrict__ out, uint32_t* __restrict__ compact, unsigned* __restrict__ ctrl) {
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

  bool valid = false, alive = false;
  uint64_t idx = 0;
  Real cx = 0, cy = 0, zx = 0, zy = 0;
  uint32_t n = 0;
  const uint32_t max_it = vp.max_iterations;

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
    const Real zx0 = zx, zy0 = zy;
    const uint32_t n0 = n;
    uint32_t acc = 0;
#pragma unroll
    for (int r = 0; r < R; ++r) {
      const Real xx = A::mul(zx, zx);
      const Real yy = A::mul(zy, zy);
      acc |= A::high(xx) | A::high(yy);
      const Real t = A::mul(zx, zy);
      zy = A::twice_plus(t, cy);
      zx = A::add(A::sub(xx, yy), cx);
    }
    const bool fast = alive && n0 + R <= max_it && (acc & 0x40000000u) == 0u;
    if (fast) {
      n = n0 + R;
      alive = n < max_it;
    }
    bool live = alive && !fast;  // lanes replaying the block exactly
    if (__any_sync(kFull, live)) {
      if (live) {
        zx = zx0;
        zy = zy0;
        n = n0;
      }
#pragma unroll
      for (int r = 0; r < R; ++r) {
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
      }
      if (alive && !fast) alive = live;
    }
    if (valid && !alive) {
      out[idx] = make_uint4(n, n, n, n);
      if (compact) compact[idx] = n;  // host-bound copy: one count per pixel
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

template <typename Real, int R, int MB = kMinBlocks<Real>>
cudaError_t launch_real(const MandelParams& p, const LaunchEnv& env, uint64_t first, uint64_t count) {
  static int blocks_per_sm = 0;
  if (blocks_per_sm == 0) {
    cudaError_t e = cudaOccupancyMaxActiveBlocksPerMultiprocessor(&blocks_per_sm, mandel_persistent<Real, R, MB>,
                                                                  kThreads, 0);
    if (e != cudaSuccess) return e;
    if (blocks_per_sm < 1) blocks_per_sm = 1;
  }
  const Viewport<Real> vp = make_viewport<Real>(p);
  const Real* tab = static_cast<const Real*>(env.scratch);
  const uint64_t claims = (count + kTailChunk - 1) / kTailChunk;
  const uint64_t blocks_needed = (claims + kThreads / 32 - 1) / (kThreads / 32);
  uint64_t grid = static_cast<uint64_t>(env.sms) * static_cast<uint64_t>(blocks_per_sm);
  if (blocks_needed < grid) grid = blocks_needed;
  if (grid == 0) return cudaSuccess;
  mandel_persistent<Real, R, MB><<<static_cast<unsigned>(grid), kThreads, 0, env.stream>>>(
      vp, tab, first, count, static_cast<uint4*>(env.out[0]), env.compact, env.ctrl);
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
  if (spec.kind == KernelKind::MandelbrotF32) return launch_real<float, 16>(spec.mandel, env, first, count);
  // Tuning hook (ECL_MANDEL_VARIANT): block length R and resident CTAs per SM.
  static const int variant = [] {
    const char* v = std::getenv("ECL_MANDEL_VARIANT");
    return v ? std::atoi(v) : 0;
  }();
  switch (variant) {
    case 1: return launch_real<double, 16, 6>(spec.mandel, env, first, count);
    case 2: return launch_real<double, 32, 4>(spec.mandel, env, first, count);
    case 3: return launch_real<double, 8, 4>(spec.mandel, env, first, count);
    case 4: return launch_real<double, 16, 3>(spec.mandel, env, first, count);
    default: return launch_real<double, 16, 4>(spec.mandel, env, first, count);  // measured best
  }
}

}  // namespace ecl
