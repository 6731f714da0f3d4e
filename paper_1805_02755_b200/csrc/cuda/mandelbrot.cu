// mandelbrot.cu — escape-time Mandelbrot for sm_100a, bit-exact with the
// reference kernel (workloads.hpp:78-100, lambda :215-223).
//
// Parity contract.  Every floating-point operation is an explicit _rn
// intrinsic in the reference's order, so no FMA contraction can happen
// whatever -fmad says:
//   cx = x0 + ((px * (x1 - x0)) / W)          workloads.hpp:97
//   xx = zx*zx; yy = zy*zy; escape if xx+yy > 4   :82-84
//   zy = (2*zx)*zy + cy;  zx = (xx - yy) + cx      :85-86
// One exact rewrite is used: (2*zx)*zy rounds to exactly 2*round(zx*zy)
// (scaling by two is exact away from overflow/subnormals), and
// round(2*t + cy) is one fma(t, 2, cy) because 2*t is exact — 7 FP64 pipe
// ops per iteration instead of 8, same bits.
//
// Layout.  One persistent grid per package; each warp claims chunks of
// kChunk consecutive pixels from a device-wide counter and keeps all 32
// lanes busy by refilling a lane with the next pixel of the chunk as soon as
// its pixel escapes (checked every R iterations), so the divergence of the
// irregular set costs at most R-1 idle iterations per pixel instead of the
// warp-wide max.  Results are written as one uint4 per pixel: the four
// identical counts of the reference's 4:1 out pattern (workloads.hpp:217-222).
#include "kernels.cuh"

namespace ecl {
namespace {

constexpr unsigned kFull = 0xffffffffu;
constexpr uint64_t kChunk = 256;  // pixels per warp claim
constexpr int kThreads = 256;

template <typename Real>
struct Arith;

template <>
struct Arith<double> {
  static __device__ __forceinline__ double mul(double a, double b) { return __dmul_rn(a, b); }
  static __device__ __forceinline__ double add(double a, double b) { return __dadd_rn(a, b); }
  static __device__ __forceinline__ double sub(double a, double b) { return __dsub_rn(a, b); }
  static __device__ __forceinline__ double div(double a, double b) { return __ddiv_rn(a, b); }
  static __device__ __forceinline__ double twice_plus(double t, double c) { return __fma_rn(t, 2.0, c); }
  static __device__ __forceinline__ double from_u64(uint64_t v) { return __ull2double_rn(v); }
};

template <>
struct Arith<float> {
  static __device__ __forceinline__ float mul(float a, float b) { return __fmul_rn(a, b); }
  static __device__ __forceinline__ float add(float a, float b) { return __fadd_rn(a, b); }
  static __device__ __forceinline__ float sub(float a, float b) { return __fsub_rn(a, b); }
  static __device__ __forceinline__ float div(float a, float b) { return __fdiv_rn(a, b); }
  static __device__ __forceinline__ float twice_plus(float t, float c) { return __fmaf_rn(t, 2.0f, c); }
  static __device__ __forceinline__ float from_u64(uint64_t v) { return __ull2float_rn(v); }
};

template <typename Real>
struct Viewport {
  uint64_t width, height;
  uint32_t max_iterations;
  Real x0, y0, span_x, span_y, fw, fh;  // span = x1 - x0 rounded in Real
};

template <typename Real, int R>
__global__ void __launch_bounds__(kThreads)
    mandel_persistent(const Viewport<Real> vp, uint64_t first, uint64_t count, uint4* __restrict__ out,
                      unsigned* __restrict__ ctrl) {
  using A = Arith<Real>;
  const unsigned lane = threadIdx.x & 31u;
  const unsigned below = (1u << lane) - 1u;
  const uint64_t nchunks = (count + kChunk - 1) / kChunk;

  // Warp-uniform cursor over the claimed chunk: [next, end) relative to first.
  uint64_t next = 0, end = 0;
  bool more = true;
  auto claim = [&]() {
    unsigned c = 0;
    if (lane == 0) c = atomicAdd(ctrl, 1u);
    c = __shfl_sync(kFull, c, 0);
    if (c >= nchunks) {
      more = false;
      next = end = 0;
    } else {
      next = static_cast<uint64_t>(c) * kChunk;
      end = next + kChunk < count ? next + kChunk : count;
    }
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
        const uint64_t px = idx % vp.width, py = idx / vp.width;
        cx = A::add(vp.x0, A::div(A::mul(A::from_u64(px), vp.span_x), vp.fw));
        cy = A::add(vp.y0, A::div(A::mul(A::from_u64(py), vp.span_y), vp.fh));
        zx = 0;
        zy = 0;
        n = 0;
        valid = true;
        alive = true;
      }
      const uint64_t want = __popc(need);
      next += want < avail ? want : avail;
      if (next >= end) claim();
      need = __ballot_sync(kFull, !valid);
    }
    if (!__any_sync(kFull, valid)) break;

#pragma unroll
    for (int r = 0; r < R; ++r) {
      const Real xx = A::mul(zx, zx);
      const Real yy = A::mul(zy, zy);
      alive = alive && !(A::add(xx, yy) > Real(4));
      const Real t = A::mul(zx, zy);
      zy = A::twice_plus(t, cy);
      zx = A::add(A::sub(xx, yy), cx);
      n += alive ? 1u : 0u;
      alive = alive && n < max_it;
    }
    if (valid && !alive) {
      out[idx] = make_uint4(n, n, n, n);
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
  // x1 - x0 rounded once in Real, the same value the reference recomputes
  // per pixel (host subtraction is IEEE round-to-nearest, no contraction).
  volatile Real sx = x1 - x0, sy = y1 - y0;
  vp.span_x = sx;
  vp.span_y = sy;
  vp.fw = static_cast<Real>(p.width);
  vp.fh = static_cast<Real>(p.height);
  return vp;
}

template <typename Real, int R>
cudaError_t launch_real(const MandelParams& p, const LaunchEnv& env, uint64_t first, uint64_t count) {
  static int blocks_per_sm = 0;
  if (blocks_per_sm == 0) {
    cudaError_t e = cudaOccupancyMaxActiveBlocksPerMultiprocessor(&blocks_per_sm, mandel_persistent<Real, R>,
                                                                  kThreads, 0);
    if (e != cudaSuccess) return e;
    if (blocks_per_sm < 1) blocks_per_sm = 1;
  }
  const uint64_t warps_needed = (count + kChunk - 1) / kChunk;
  const uint64_t blocks_needed = (warps_needed + kThreads / 32 - 1) / (kThreads / 32);
  uint64_t grid = static_cast<uint64_t>(env.sms) * static_cast<uint64_t>(blocks_per_sm);
  if (blocks_needed < grid) grid = blocks_needed;
  if (grid == 0) return cudaSuccess;
  mandel_persistent<Real, R><<<static_cast<unsigned>(grid), kThreads, 0, env.stream>>>(
      make_viewport<Real>(p), first, count, static_cast<uint4*>(env.out[0]), env.ctrl);
  return cudaGetLastError();
}

}  // namespace

cudaError_t launch_mandelbrot(const KernelSpec& spec, const LaunchEnv& env, uint64_t first, uint64_t count) {
  if (count == 0) return cudaSuccess;
  if (spec.kind == KernelKind::MandelbrotF32) return launch_real<float, 16>(spec.mandel, env, first, count);
  return launch_real<double, 16>(spec.mandel, env, first, count);
}

}  // namespace ecl
