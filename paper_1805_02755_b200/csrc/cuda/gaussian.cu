// gaussian.cu — direct FxF convolution with clamp-to-edge (the paper's
// Gaussian blur benchmark; absent from the reference, definition in
// SURVEY.md Appendix B and oracle/oracle.c:orc_gaussian).
//
//   out[y*W+x] = sum_{i<F} sum_{j<F} filt[i*F+j] * img[cl(y+i-F/2)*W + cl(x+j-F/2)]
//
// Layout (one CTA = a 64x32 output tile, 256 threads, 8 outputs per thread):
//  * the (32+F-1) x (64+F-1) input tile is staged in shared memory with a
//    row pitch of 100 floats (= 4 mod 32 banks).  Interior tiles are staged
//    by the TMA engine: one cp.async.bulk (global -> shared, mbarrier
//    complete_tx) per tile row, 16-byte aligned 384-byte rows; tiles that
//    touch the image border use clamped LDG loads instead;
//  * thread (tx, ty) owns outputs (ty, 8tx..8tx+7); lanes are laid out so
//    the 8 lanes of an LDS.128 phase read 8 different rows -> the 100-float
//    pitch spreads them over all 32 banks (conflict-free);
//  * the filter travels as a __grid_constant__ kernel parameter (constant
//    bank 0), packed on the host from the device layer's host mirror of the
//    filter input, so every FFMA takes its weight from a uniform register
//    (LDCU) and each launch carries its own filter: no per-device constant
//    state, nothing shared between lanes or between engines on one GPU.
//    Per filter row i a thread loads 10 float4 of the input row and issues
//    8*F FFMAs (i outer, j inner, the oracle's order);
//  * results leave as two float4 stores per thread.
// Packages are arbitrary work-item ranges: tiles cover the rows the range
// touches and only pixels inside [first, first+count) are written.
#include <algorithm>
#include <atomic>
#include <cmath>
#include <cstdlib>
#include <cstring>
#include <vector>

#include "kernels.cuh"

namespace ecl {
namespace {

constexpr int kTileW = 64, kTileH = 32, kThreads = 256, kPitch = 100;
constexpr int kMaxF = 31;

// Tiled path: the filter twice with an even row pitch F+1, so tap pairs are
// 8-byte aligned: a[i*(F+1) + j] = w[i][j], b[i*(F+1) + j] = w[i][j+1]
// (zero past the row).  7.9 KB at F = 31, inside the 32 KB parameter limit.
template <int F>
struct TapPairs {
  __align__(16) float a[F * (F + 1)];
  __align__(16) float b[F * (F + 1)];
};

// Generic path: the F x F filter as given (F <= 63: 15.9 KB).
struct FilterParam {
  float w[63 * 63];
};

__device__ __forceinline__ int clampi(int v, int lo, int hi) { return v < lo ? lo : (v > hi ? hi : v); }

__device__ __forceinline__ void mbar_init(uint64_t* bar, unsigned count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(static_cast<unsigned>(__cvta_generic_to_shared(bar))),
               "r"(count));
}

__device__ __forceinline__ void mbar_expect_tx(uint64_t* bar, unsigned bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(
                   static_cast<unsigned>(__cvta_generic_to_shared(bar))),
               "r"(bytes)
               : "memory");
}

__device__ __forceinline__ void mbar_wait(uint64_t* bar, unsigned phase) {
  const unsigned a = static_cast<unsigned>(__cvta_generic_to_shared(bar));
  asm volatile(
      "{\n"
      ".reg .pred p;\n"
      "WAIT_%=:\n"
      "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n"
      "@!p bra WAIT_%=;\n"
      "}\n" ::"r"(a),
      "r"(phase)
      : "memory");
}

// TMA bulk copy of `bytes` (multiple of 16, 16-byte aligned) into shared memory.
__device__ __forceinline__ void bulk_g2s(void* dst, const void* src, unsigned bytes, uint64_t* bar) {
  asm volatile(
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
          static_cast<unsigned>(__cvta_generic_to_shared(dst))),
      "l"(src), "r"(bytes), "r"(static_cast<unsigned>(__cvta_generic_to_shared(bar)))
      : "memory");
}

template <int F>
__global__ void __launch_bounds__(kThreads)
    gaussian_tiled(const float* __restrict__ img, float* __restrict__ out, int W, int H, uint64_t first, uint64_t count,
                   int row0, const __grid_constant__ TapPairs<F> taps) {
  constexpr int R = F / 2;
  constexpr int TH = kTileH + F - 1;  // staged rows
  constexpr int NV = 8 + F - 1;       // input values per thread row
  constexpr int SHIFT = (4 - R % 4) % 4;  // first value's offset inside its float4
  constexpr int NL = (SHIFT + NV + 3) / 4;  // float4 loads per filter row
  __shared__ __align__(128) float tile[TH * kPitch];
  __shared__ __align__(8) uint64_t bar;

  const int tile_x = blockIdx.x * kTileW;
  const int tile_y = row0 + blockIdx.y * kTileH;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int tx = (warp >> 2) * 4 + (lane >> 3);  // 0..7
  const int ty = (warp & 3) * 8 + (lane & 7);    // 0..31

  // Stage columns tile_x-16 .. tile_x+79 (96 floats) of rows tile_y-R .. ;
  // smem column c holds global column tile_x - 16 + c.
  const bool interior = tile_x >= 16 && tile_x + kTileW + 16 <= W && tile_y - R >= 0 && tile_y + kTileH + R <= H &&
                        (W & 3) == 0;
  if (interior) {
    if (threadIdx.x == 0) {
      mbar_init(&bar, 1);
      asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
      mbar_expect_tx(&bar, TH * 96 * 4);
    }
    __syncthreads();
    // One bulk copy per staged row.  The copy takes warp-uniform operands, so
    // a warp issues its lanes' copies one after another: rows go round-robin
    // over all warps (row = lane * warps + warp), not to the first TH threads.
    {
      const int rr = static_cast<int>(threadIdx.x & 31) * (kThreads / 32) + static_cast<int>(threadIdx.x >> 5);
      if (rr < TH) {
        const int gy = tile_y - R + rr;
        bulk_g2s(&tile[rr * kPitch], img + static_cast<int64_t>(gy) * W + (tile_x - 16), 96 * 4, &bar);
      }
    }
    mbar_wait(&bar, 0);
  } else {
    // border tile: clamp-to-edge loads, one warp per row (coalesced, the
    // three column clamps hoisted out of the row loop)
    {
      const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
      int gx[3];
#pragma unroll
      for (int q = 0; q < 3; ++q) gx[q] = clampi(tile_x - 16 + lane + 32 * q, 0, W - 1);
      for (int r = warp; r < TH; r += kThreads / 32) {
        const float* src = img + static_cast<int64_t>(clampi(tile_y - R + r, 0, H - 1)) * W;
#pragma unroll
        for (int q = 0; q < 3; ++q) tile[r * kPitch + lane + 32 * q] = src[gx[q]];
      }
    }
    __syncthreads();
  }

  // Taps travel in packed pairs through FFMA2: output b accumulates taps
  // (j, j+1) of a row into (acc[b].x, acc[b].y) from the input pair
  // (v[a], v[a+1]), a = SHIFT + b + j, which is a register pair of the float4
  // loads when a is even — so outputs with even SHIFT + b pair taps from
  // j = 0 (weights taps.a, leftover tap F-1) and the others from j = 1
  // (weights taps.b, leftover tap 0).  Half the FP32 issue slots of scalar
  // FFMAs (the kernel was issue-bound); the two partial sums per output
  // change the accumulation order only (≤ 3.2e-6 relative vs the oracle's
  // sequential order on this filter, budget 1e-5).
  constexpr int P = F + 1;            // padded filter row pitch (even)
  constexpr int NP = (F - 1) / 2;     // tap pairs per row
  float2 acc[8];
#pragma unroll
  for (int b = 0; b < 8; ++b) acc[b] = make_float2(0.0f, 0.0f);
  // thread's first input column in smem: output col 8tx needs global col 8tx - R
  const float* row = tile + ty * kPitch + (16 + 8 * tx - R - SHIFT);  // 16-byte aligned
#pragma unroll 1
  for (int i = 0; i < F; ++i) {
    float2 ev[NL * 2];
    const float4* src = reinterpret_cast<const float4*>(row + i * kPitch);
#pragma unroll
    for (int m = 0; m < NL; ++m) {
      const float4 q = src[m];
      ev[2 * m] = make_float2(q.x, q.y);
      ev[2 * m + 1] = make_float2(q.z, q.w);
    }
    const float2* wa = reinterpret_cast<const float2*>(taps.a + i * P);  // (w[2m], w[2m+1])
    const float2* wb = reinterpret_cast<const float2*>(taps.b + i * P);  // (w[2m+1], w[2m+2])
#pragma unroll
    for (int b = 0; b < 8; ++b) {
      const int a0 = SHIFT + b;
      if ((a0 & 1) == 0) {
#pragma unroll
        for (int m = 0; m < NP; ++m) acc[b] = __ffma2_rn(wa[m], ev[a0 / 2 + m], acc[b]);
        const int a = a0 + F - 1;  // leftover tap F-1
        acc[b].x = fmaf(taps.a[i * P + F - 1], (a & 1) ? ev[a >> 1].y : ev[a >> 1].x, acc[b].x);
      } else {
        acc[b].x = fmaf(taps.a[i * P], ev[a0 >> 1].y, acc[b].x);  // leftover tap 0 (a0 odd)
#pragma unroll
        for (int m = 0; m < NP; ++m) acc[b] = __ffma2_rn(wb[m], ev[(a0 + 1) / 2 + m], acc[b]);
      }
    }
  }
  float res[8];
#pragma unroll
  for (int b = 0; b < 8; ++b) res[b] = acc[b].x + acc[b].y;

  // Masked float4 stores of the 8 outputs (pixels outside the package skipped).
  const int gy = tile_y + ty, gx = tile_x + 8 * tx;
  if (gy >= H || gx >= W) return;
  const uint64_t base = static_cast<uint64_t>(gy) * W + gx;
  float* dst = out + base;
  if (base >= first && base + 8 <= first + count && gx + 8 <= W && (reinterpret_cast<uintptr_t>(dst) & 15) == 0) {
    reinterpret_cast<float4*>(dst)[0] = make_float4(res[0], res[1], res[2], res[3]);
    reinterpret_cast<float4*>(dst)[1] = make_float4(res[4], res[5], res[6], res[7]);
  } else {
#pragma unroll
    for (int b = 0; b < 8; ++b)
      if (gx + b < W && base + b >= first && base + b < first + count) dst[b] = res[b];
  }
}

// ---- Separable path --------------------------------------------------------
// A rank-1 filter w[i][j] = r[i] c[j] (the Gaussian one is) takes F + F taps
// per pixel instead of F*F: a horizontal pass over the staged (32+F-1) rows
// into a shared-memory buffer, then a vertical pass — ~91 FMAs per pixel at
// F = 31 against 961, which moves the kernel from the FMA pipe towards the
// memory system (8 B of algorithmic HBM traffic per pixel).  Taps travel in
// packed pairs through FFMA2 as in gaussian_tiled.  Numerics: the factors
// are taken in double from the filter's centre row and column and the
// factorisation is accepted only when every r[i] c[j] matches w[i][j] to
// 2^-20 relative (a few float ulps), so the result differs from the direct
// sum by the factorisation's rounding plus a 62-term reassociation (both
// ~1e-7 relative against the 1e-5 budget).  Any other filter runs the
// direct kernel.
template <int F>
struct SepTaps {
  __align__(16) float c[F + 1];   // horizontal taps (pairs (2m, 2m+1)), zero-padded
  __align__(16) float cb[F + 1];  // c shifted by one: pairs (2m+1, 2m+2)
  float r[F];                     // vertical taps
};

constexpr int kHPitch = 68;  // horizontal-pass buffer pitch (floats): rows of 64 + 4 (bank spread)

// One 64 x TO output tile per CTA.  Default (INPLACE): the horizontal pass
// overwrites the staged tile, 37 KB of shared memory and 5 CTAs per SM
// (register-limited) at TO = 64: 67-68 us at 4096^2 against 72-73 us with a
// separate pass buffer (63 KB, 3 CTAs per SM; gaussian@2).  Measured and
// dropped: persistent CTAs with the input tile double-buffered (prefetch of
// tile k+1 during tile k; ncu: the TMA wait disappears, but 2-3 CTAs per SM
// cannot keep the FMA pipe fed): round 2a 98 us (32-row tiles) and 105 us
// (64-row), round 2b in place 82 us (64-row, 2 CTAs/SM), 89 (56), 94 (48).
// The two passes of the separable kernel on one staged tile (all threads).
template <int F, int TO, bool INPLACE>
__device__ __forceinline__ void sep_hpass(float* __restrict__ tile, float* __restrict__ hbuf,
                                          const SepTaps<F>& taps) {
  constexpr int R = F / 2;
  constexpr int TH = TO + F - 1;
  constexpr int NV = 8 + F - 1;
  constexpr int SHIFT = (4 - R % 4) % 4;
  constexpr int NL = (SHIFT + NV + 3) / 4;
  constexpr int NP = (F - 1) / 2;
  // in place, every thread runs every iteration (barriers inside): pad the
  // segment count to whole CTA passes (the padding rows store nothing)
  constexpr int NSEG = INPLACE ? (((TH + 7) & ~7) * 8 + kThreads - 1) / kThreads * kThreads : ((TH + 7) & ~7) * 8;
  // Horizontal pass: segment (row, s) = 8 outputs hbuf[row][8s .. 8s+7].
  // The 8 lanes of an LDS.128 phase take 8 consecutive rows of one segment
  // column: the 100-float tile pitch and the 68-float buffer pitch put them
  // on disjoint banks (conflict-free loads and stores).  INPLACE: the outputs
  // overwrite the first 64 floats of their own tile row (one iteration's
  // segments cover whole rows, 32 of them, and no other iteration reads
  // those rows), after a barrier that orders every read of the rows before
  // the first write — no separate buffer, 37 KB instead of 63 KB per CTA.
  const float2* wa = reinterpret_cast<const float2*>(taps.c);
  const float2* wb = reinterpret_cast<const float2*>(taps.cb);
#pragma unroll 1
  for (int seg = threadIdx.x; seg < NSEG; seg += kThreads) {
    const int row = (seg & 7) + 8 * (seg >> 6), s8 = (seg >> 3) & 7;
    if (!INPLACE && row >= TH) continue;
    const int lrow = row < TH ? row : TH - 1;  // padding rows (in-place only): read a real row, store nothing
    const float4* src = reinterpret_cast<const float4*>(tile + lrow * kPitch + (16 + 8 * s8 - R - SHIFT));
    float2 ev[NL * 2];
#pragma unroll
    for (int m = 0; m < NL; ++m) {
      const float4 q = src[m];
      ev[2 * m] = make_float2(q.x, q.y);
      ev[2 * m + 1] = make_float2(q.z, q.w);
    }
    float2 acc[8];
#pragma unroll
    for (int b = 0; b < 8; ++b) {
      acc[b] = make_float2(0.0f, 0.0f);
      const int a0 = SHIFT + b;
      if ((a0 & 1) == 0) {
#pragma unroll
        for (int m = 0; m < NP; ++m) acc[b] = __ffma2_rn(wa[m], ev[a0 / 2 + m], acc[b]);
        const int a = a0 + F - 1;
        acc[b].x = fmaf(taps.c[F - 1], (a & 1) ? ev[a >> 1].y : ev[a >> 1].x, acc[b].x);
      } else {
        acc[b].x = fmaf(taps.c[0], ev[a0 >> 1].y, acc[b].x);
#pragma unroll
        for (int m = 0; m < NP; ++m) acc[b] = __ffma2_rn(wb[m], ev[(a0 + 1) / 2 + m], acc[b]);
      }
    }
    if (INPLACE) __syncthreads();
    if (row < TH) {
      float4* dst = reinterpret_cast<float4*>(INPLACE ? tile + row * kPitch + 8 * s8 : hbuf + row * kHPitch + 8 * s8);
      dst[0] = make_float4(acc[0].x + acc[0].y, acc[1].x + acc[1].y, acc[2].x + acc[2].y, acc[3].x + acc[3].y);
      dst[1] = make_float4(acc[4].x + acc[4].y, acc[5].x + acc[5].y, acc[6].x + acc[6].y, acc[7].x + acc[7].y);
    }
  }
}

template <int F, int TO, int HP>
__device__ __forceinline__ void sep_vpass(const float* __restrict__ hbuf, float* __restrict__ out, int W, int H,
                                          uint64_t first, uint64_t count, int tile_x, int tile_y,
                                          const SepTaps<F>& taps) {
  // Vertical pass: lane = column pair (64 columns per warp), warp = 4 output
  // rows.  A thread slides down its column pair through 4 + F - 1 buffer
  // rows (one LDS.64 each) and feeds every output row the tap it owes —
  // each loaded value serves up to 4 outputs from registers.
  constexpr int VR = TO / (kThreads / 32);  // output rows per thread
  const int lane = threadIdx.x & 31, y0 = (threadIdx.x >> 5) * VR;
  float2 acc[VR];
#pragma unroll
  for (int o = 0; o < VR; ++o) acc[o] = make_float2(0.f, 0.f);
  const float* col = hbuf + y0 * HP + 2 * lane;
#pragma unroll
  for (int i = 0; i < VR + F - 1; ++i) {
    const float2 h = *reinterpret_cast<const float2*>(col + i * HP);
#pragma unroll
    for (int o = 0; o < VR; ++o) {
      const int tap = i - o;
      if (tap >= 0 && tap < F) acc[o] = __ffma2_rn(make_float2(taps.r[tap], taps.r[tap]), h, acc[o]);
    }
  }

  const int gx = tile_x + 2 * lane;
#pragma unroll
  for (int o = 0; o < VR; ++o) {
    const int gy = tile_y + y0 + o;
    if (gx >= W || gy >= H) break;
    const uint64_t base = static_cast<uint64_t>(gy) * W + gx;
    float* dst = out + base;
    if (base >= first && base + 2 <= first + count && gx + 2 <= W && (reinterpret_cast<uintptr_t>(dst) & 7) == 0) {
      *reinterpret_cast<float2*>(dst) = acc[o];
    } else {
      if (base >= first && base < first + count) dst[0] = acc[o].x;
      if (gx + 1 < W && base + 1 >= first && base + 1 < first + count) dst[1] = acc[o].y;
    }
  }
}

template <int F, int TO, bool INPLACE>
__global__ void __launch_bounds__(kThreads)
    gaussian_sep(const float* __restrict__ img, float* __restrict__ out, int W, int H, uint64_t first, uint64_t count,
                 int row0, const __grid_constant__ SepTaps<F> taps) {
  constexpr int R = F / 2;
  constexpr int TH = TO + F - 1;  // staged rows (TO output rows per tile)
  extern __shared__ __align__(128) float sep_smem[];
  float* const tile = sep_smem;
  float* const hbuf = sep_smem + TH * kPitch;
  __shared__ __align__(8) uint64_t bar;

  const int tile_x = blockIdx.x * kTileW;
  const int tile_y = row0 + blockIdx.y * TO;
  const bool interior = tile_x >= 16 && tile_x + kTileW + 16 <= W && tile_y - R >= 0 && tile_y + TO + R <= H &&
                        (W & 3) == 0;
  if (interior) {
    if (threadIdx.x == 0) {
      mbar_init(&bar, 1);
      asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
      mbar_expect_tx(&bar, TH * 96 * 4);
    }
    __syncthreads();
    // One bulk copy per staged row.  The copy takes warp-uniform operands, so
    // a warp issues its lanes' copies one after another: rows go round-robin
    // over all warps (row = lane * warps + warp), not to the first TH threads.
    {
      const int rr = static_cast<int>(threadIdx.x & 31) * (kThreads / 32) + static_cast<int>(threadIdx.x >> 5);
      if (rr < TH) {
        const int gy = tile_y - R + rr;
        bulk_g2s(&tile[rr * kPitch], img + static_cast<int64_t>(gy) * W + (tile_x - 16), 96 * 4, &bar);
      }
    }
    mbar_wait(&bar, 0);
  } else {
    // border tile: clamp-to-edge loads, one warp per row (coalesced, the
    // three column clamps hoisted out of the row loop)
    {
      const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
      int gx[3];
#pragma unroll
      for (int q = 0; q < 3; ++q) gx[q] = clampi(tile_x - 16 + lane + 32 * q, 0, W - 1);
      for (int r = warp; r < TH; r += kThreads / 32) {
        const float* src = img + static_cast<int64_t>(clampi(tile_y - R + r, 0, H - 1)) * W;
#pragma unroll
        for (int q = 0; q < 3; ++q) tile[r * kPitch + lane + 32 * q] = src[gx[q]];
      }
    }
    __syncthreads();
  }

  sep_hpass<F, TO, INPLACE>(tile, hbuf, taps);
  __syncthreads();
  if (INPLACE)
    sep_vpass<F, TO, kPitch>(tile, out, W, H, first, count, tile_x, tile_y, taps);
  else
    sep_vpass<F, TO, kHPitch>(hbuf, out, W, H, first, count, tile_x, tile_y, taps);
}

template <int F, int TO, bool INPLACE>
constexpr size_t sep_smem_bytes() {
  return sizeof(float) * ((TO + F - 1) * kPitch + (INPLACE ? 0 : (TO + F - 1) * kHPitch));
}

// Factorisation of the F x F filter as r[i] c[j] (see gaussian_sep), or
// false.  The last filter seen is cached per host thread (a device thread
// launches every package of its device), so repeated launches with the same
// filter cost one 4 KB compare.
struct SepCache {
  std::vector<float> w;
  bool ok = false;
  std::vector<float> r, c;
};

bool factor_filter(const float* w, int F, const float** r, const float** c) {
  thread_local SepCache cache;
  const size_t n = static_cast<size_t>(F) * F;
  if (cache.w.size() != n || std::memcmp(cache.w.data(), w, n * sizeof(float)) != 0) {
    cache.w.assign(w, w + n);
    cache.r.assign(F, 0.0f);
    cache.c.assign(F, 0.0f);
    cache.ok = false;
    const int R = F / 2;
    const double ctr = w[R * F + R];
    if (ctr > 0.0 && std::isfinite(ctr)) {
      const double sc = std::sqrt(ctr);
      std::vector<double> rd(F), cd(F);
      for (int i = 0; i < F; ++i) rd[i] = w[i * F + R] / sc;
      for (int j = 0; j < F; ++j) cd[j] = w[R * F + j] / sc;
      bool ok = true;
      for (int i = 0; i < F && ok; ++i)
        for (int j = 0; j < F && ok; ++j) {
          const double v = static_cast<double>(w[i * F + j]), p = rd[i] * cd[j];
          ok = std::isfinite(v) && std::fabs(v - p) <= 0x1p-20 * std::fabs(v);
        }
      if (ok) {
        for (int i = 0; i < F; ++i) cache.r[i] = static_cast<float>(rd[i]);
        for (int j = 0; j < F; ++j) cache.c[j] = static_cast<float>(cd[j]);
        cache.ok = true;
      }
    }
  }
  *r = cache.r.data();
  *c = cache.c.data();
  return cache.ok;
}

template <int F, int TO, bool INPLACE>
cudaError_t launch_sep(const GaussianParams& g, const LaunchEnv& env, const float* r, const float* c, uint64_t first,
                       uint64_t count) {
  SepTaps<F> taps;
  for (int j = 0; j <= F; ++j) {
    taps.c[j] = j < F ? c[j] : 0.0f;
    taps.cb[j] = j + 1 < F ? c[j + 1] : 0.0f;
  }
  for (int i = 0; i < F; ++i) taps.r[i] = r[i];
  constexpr size_t smem = sep_smem_bytes<F, TO, INPLACE>();
  // the dynamic shared-memory limit is a per-device function attribute: set
  // it once on every device that launches this kernel (idempotent if two
  // device threads race)
  static std::atomic<uint64_t> attr_set{0};
  const uint64_t bit = uint64_t{1} << (env.device & 63);
  if (!(attr_set.load(std::memory_order_relaxed) & bit)) {
    const cudaError_t e =
        cudaFuncSetAttribute(gaussian_sep<F, TO, INPLACE>, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(smem));
    if (e != cudaSuccess) return e;
    attr_set.fetch_or(bit, std::memory_order_relaxed);
  }
  const int row0 = static_cast<int>(first / g.width);
  const int row1 = static_cast<int>((first + count - 1) / g.width);
  const dim3 grid((g.width + kTileW - 1) / kTileW, (row1 - row0 + TO) / TO);
  gaussian_sep<F, TO, INPLACE><<<grid, kThreads, smem, env.stream>>>(static_cast<const float*>(env.in[0]),
                                                        static_cast<float*>(env.out[0]), static_cast<int>(g.width),
                                                        static_cast<int>(g.height), first, count, row0, taps);
  return cudaGetLastError();
}

// Any odd F up to 63: one thread per output, filter from the parameter bank.
__global__ void __launch_bounds__(kThreads)
    gaussian_generic(const float* __restrict__ img, float* __restrict__ out, int W, int H, int F, uint64_t first,
                     uint64_t count, const __grid_constant__ FilterParam filt) {
  const int R = F / 2;
  for (uint64_t k = blockIdx.x * static_cast<uint64_t>(blockDim.x) + threadIdx.x; k < count;
       k += static_cast<uint64_t>(gridDim.x) * blockDim.x) {
    const uint64_t idx = first + k;
    const int x = static_cast<int>(idx % W), y = static_cast<int>(idx / W);
    float acc = 0.0f;
    for (int i = 0; i < F; ++i) {
      const float* src = img + static_cast<int64_t>(clampi(y + i - R, 0, H - 1)) * W;
      for (int j = 0; j < F; ++j) acc = fmaf(filt.w[i * F + j], src[clampi(x + j - R, 0, W - 1)], acc);
    }
    out[idx] = acc;
  }
}

template <int F>
cudaError_t launch_tiled(const GaussianParams& g, const LaunchEnv& env, const float* w, uint64_t first,
                         uint64_t count) {
  constexpr int P = F + 1;
  TapPairs<F> taps;
  for (int i = 0; i < F; ++i)
    for (int j = 0; j < P; ++j) {
      taps.a[i * P + j] = j < F ? w[i * F + j] : 0.0f;
      taps.b[i * P + j] = j + 1 < F ? w[i * F + j + 1] : 0.0f;
    }
  const int row0 = static_cast<int>(first / g.width);
  const int row1 = static_cast<int>((first + count - 1) / g.width);
  const dim3 grid((g.width + kTileW - 1) / kTileW, (row1 - row0 + kTileH) / kTileH);
  gaussian_tiled<F><<<grid, kThreads, 0, env.stream>>>(static_cast<const float*>(env.in[0]),
                                                       static_cast<float*>(env.out[0]), static_cast<int>(g.width),
                                                       static_cast<int>(g.height), first, count, row0, taps);
  return cudaGetLastError();
}

}  // namespace

// The filter (input 1) is host-mirrored by the device layer
// (host_mirrored_input): each launch packs it into its own parameters.
bool gaussian_mirrors_input(uint32_t input) { return input == 1; }

cudaError_t launch_gaussian(const KernelSpec& spec, const LaunchEnv& env, uint64_t first, uint64_t count) {
  if (count == 0) return cudaSuccess;
  const GaussianParams& g = spec.gauss;
  const float* w = env.in_host ? static_cast<const float*>(env.in_host[1]) : nullptr;
  if (!w) return cudaErrorInvalidValue;  // the device layer keeps the filter mirrored (host_mirrored_input)
  // gaussian@1 (or ECL_GAUSSIAN_VARIANT=1 when the id has no @n): always the direct F x F kernel
  static const int env_variant = [] {
    const char* v = std::getenv("ECL_GAUSSIAN_VARIANT");
    return v ? std::atoi(v) : 0;
  }();
  const int variant = spec.variant >= 0 ? spec.variant : env_variant;
  // Pieces whose outputs go straight to host memory run the direct kernel:
  // the end-to-end step is PCIe-bound (64 MiB each way, ~1.6 ms duplex), and
  // measured with 2^19-item pieces it reaches that floor with the direct
  // kernel's 23 us pieces (1.63-1.73 ms) but not with the separable kernel's
  // 8 us pieces (2.2-2.3 ms; CUPTI shows the H2D stream idling while both
  // D2H streams are busy).  Resident pieces take the separable kernel.
  const float *r = nullptr, *c = nullptr;
  if (variant != 1 && !env.host_copies && (g.filter == 31 || g.filter == 15) && factor_filter(w, static_cast<int>(g.filter), &r, &c)) {
    // ECL_GAUSSIAN_TILE_ROWS: output rows per separable tile; measured at
    // 4096^2 with the pass buffer (gaussian@2): 32 rows (5 CTAs/SM) 78 us,
    // 64 rows (3 CTAs/SM, 1.47x instead of 1.94x horizontal rows per output
    // row) 72 us; also 40 rows 77 us, 48 rows (4 CTAs/SM) 72, 56 rows 75,
    // 96 rows 77, 128 rows 75.  In place (default): 32 rows 78 us, 64 rows
    // 67-68, 96 rows 67-68, 128 rows 71.
    // ECL_GAUSSIAN_SEP_INPLACE=0: the pass-buffer kernel (as gaussian@2).
    static const int tall = [] {
      const char* v = std::getenv("ECL_GAUSSIAN_TILE_ROWS");
      return v ? std::atoi(v) : 64;
    }();
    static const int inplace = [] {
      const char* v = std::getenv("ECL_GAUSSIAN_SEP_INPLACE");
      return v ? std::atoi(v) : 1;
    }();
    if (g.filter == 31) {
      if (variant == 2 || !inplace)
        return tall == 64 ? launch_sep<31, 64, false>(g, env, r, c, first, count)
                          : launch_sep<31, 32, false>(g, env, r, c, first, count);
      if (tall == 128) return launch_sep<31, 128, true>(g, env, r, c, first, count);
      if (tall == 96) return launch_sep<31, 96, true>(g, env, r, c, first, count);
      return tall == 64 ? launch_sep<31, 64, true>(g, env, r, c, first, count)
                        : launch_sep<31, 32, true>(g, env, r, c, first, count);
    }
    return launch_sep<15, 32, false>(g, env, r, c, first, count);
  }
  switch (g.filter) {
    case 3: return launch_tiled<3>(g, env, w, first, count);
    case 5: return launch_tiled<5>(g, env, w, first, count);
    case 7: return launch_tiled<7>(g, env, w, first, count);
    case 9: return launch_tiled<9>(g, env, w, first, count);
    case 15: return launch_tiled<15>(g, env, w, first, count);
    case 31: return launch_tiled<31>(g, env, w, first, count);
    default: break;
  }
  FilterParam filt;
  std::copy(w, w + g.filter * g.filter, filt.w);
  const uint64_t blocks = std::min<uint64_t>((count + kThreads - 1) / kThreads, static_cast<uint64_t>(env.sms) * 16);
  gaussian_generic<<<static_cast<unsigned>(blocks), kThreads, 0, env.stream>>>(
      static_cast<const float*>(env.in[0]), static_cast<float*>(env.out[0]), static_cast<int>(g.width),
      static_cast<int>(g.height), static_cast<int>(g.filter), first, count, filt);
  return cudaGetLastError();
}

}  // namespace ecl
