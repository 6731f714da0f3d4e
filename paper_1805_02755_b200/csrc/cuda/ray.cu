// ray.cu — Whitted ray tracer (the paper's Ray benchmark, Table 2
// PAPER.md:506-511; absent from the reference, definition frozen in
// oracle/oracle.c:orc_ray — SURVEY.md Appendix B).
//
// Parity: every float operation is an IEEE-rounded intrinsic (_rn) in the
// oracle's order and the specular power is x^16 by four squarings, so the
// device reproduces the oracle's pixels bit for bit (no FMA contraction,
// correctly rounded sqrt and division).
//
// Layout: the sphere and material arrays (2 x ns float4) are staged in
// shared memory once per CTA and read as warp-wide broadcasts.  Work is
// irregular (0..max_depth+1 bounces per pixel, shadow tests that stop at the
// first occluder), so warps are persistent and refill lanes per bounce:
// each warp claims 32-pixel chunks from a device counter and, after every
// bounce, lanes whose pixel finished store it and take the next pixel — a
// warp stays full until the package is exhausted instead of idling on its
// deepest reflection.
#include <cuda_runtime.h>

#include <atomic>
#include <cstdlib>

#include "kernels.cuh"

namespace ecl {
namespace {

constexpr unsigned kFull = 0xffffffffu;
constexpr int kThreads = 128;  // Table 2: lws 128
constexpr uint64_t kChunk = 32;
constexpr int kMaxSpheres = 256;

struct V3 {
  float x, y, z;
};

__device__ __forceinline__ float add(float a, float b) { return __fadd_rn(a, b); }
__device__ __forceinline__ float sub(float a, float b) { return __fsub_rn(a, b); }
__device__ __forceinline__ float mul(float a, float b) { return __fmul_rn(a, b); }
__device__ __forceinline__ float dvd(float a, float b) { return __fdiv_rn(a, b); }
__device__ __forceinline__ V3 vsub(V3 a, V3 b) { return {sub(a.x, b.x), sub(a.y, b.y), sub(a.z, b.z)}; }
__device__ __forceinline__ float vdot(V3 a, V3 b) { return add(add(mul(a.x, b.x), mul(a.y, b.y)), mul(a.z, b.z)); }
__device__ __forceinline__ V3 vnorm(V3 a) {
  const float len = __fsqrt_rn(vdot(a, a));
  return {dvd(a.x, len), dvd(a.y, len), dvd(a.z, len)};
}

// distance along (o, d) to sphere s; < 0 = miss (oracle: ray_sphere)
__device__ __forceinline__ float ray_sphere(V3 o, V3 d, float4 s) {
  const V3 oc = vsub(o, V3{s.x, s.y, s.z});
  const float b = vdot(oc, d);
  const float cc = sub(vdot(oc, oc), mul(s.w, s.w));
  const float disc = sub(mul(b, b), cc);
  if (disc < 0.0f) return -1.0f;
  const float sq = __fsqrt_rn(disc);
  float t = sub(-b, sq);
  if (t > 1e-3f) return t;
  t = add(-b, sq);
  return t > 1e-3f ? t : -1.0f;
}

// The same test for spheres s and s+1 at once: the arithmetic up to the
// discriminant runs on packed pairs (FADD2/FMUL2 round each component like
// the scalar _rn ops, in the same order), over structure-of-arrays sphere
// data (x, y, z, r*r) in shared memory.  The sqrt / root selection stays
// scalar per sphere.
__device__ __forceinline__ float2 neg2(float2 a) { return make_float2(-a.x, -a.y); }
// Packed product that ptxas cannot fuse into a following FADD2: it contracts
// mul.rn.f32x2 + add.rn.f32x2 into FFMA2 (even with -fmad=false), which would
// break parity.  x*y + (+0) rounds exactly like x*y except that a -0 product
// becomes +0; only b's sign of zero can change, and b enters the results only
// as b*b and as -b +/- sqrt(disc), where that sign is absorbed (see test).
__device__ __forceinline__ float2 pmul(float2 a, float2 b) { return __ffma2_rn(a, b, make_float2(0.0f, 0.0f)); }
__device__ __forceinline__ float root_of(float b, float disc) {
  if (disc < 0.0f) return -1.0f;
  const float sq = __fsqrt_rn(disc);
  float t = sub(-b, sq);
  if (t > 1e-3f) return t;
  t = add(-b, sq);
  return t > 1e-3f ? t : -1.0f;
}
// The packed part of the pair test: b and the discriminant of both spheres.
__device__ __forceinline__ void pair_disc(V3 o, V3 d, float4 r0, float4 r1, float2& b, float2& disc) {
  const float2 X = make_float2(r0.x, r0.y), Y = make_float2(r0.z, r0.w);
  const float2 Z = make_float2(r1.x, r1.y), RR = make_float2(r1.z, r1.w);
  const float2 ox = __fadd2_rn(make_float2(o.x, o.x), neg2(X));
  const float2 oy = __fadd2_rn(make_float2(o.y, o.y), neg2(Y));
  const float2 oz = __fadd2_rn(make_float2(o.z, o.z), neg2(Z));
  b = __fadd2_rn(__fadd2_rn(pmul(ox, make_float2(d.x, d.x)), pmul(oy, make_float2(d.y, d.y))),
                 pmul(oz, make_float2(d.z, d.z)));
  const float2 cc = __fadd2_rn(__fadd2_rn(__fadd2_rn(pmul(ox, ox), pmul(oy, oy)), pmul(oz, oz)), neg2(RR));
  disc = __fadd2_rn(pmul(b, b), neg2(cc));
}

// Candidate scan with a conservative FMA prefilter.  The exact test above
// costs 16 unfused lane-ops per sphere; the scan instead evaluates the same
// discriminant in a translation-free form with FMAs, per sphere pair
//   e    = o.d - s.d                      (o.d per ray, s.d: 3 FMA)
//   cc   = (|o|^2 + q) - 2 o.s            (q = |s|^2 - r^2 per sphere, o.s: 3 FMA)
//   disc'= e*e - cc
// (8 packed instructions per pair instead of 16, see scan_group) and rejects a sphere only
// when disc' < -M, M = 2^-17 ((|o|_1 + max|s|)^2 + max r^2).  Error bound
// (u = 2^-24, R >= |o| + |s|, |d| = 1): the IEEE-ordered exact path's disc
// is within 17.1 u R^2 + 3 u r^2 of the real-number discriminant, disc'
// within ~20 u (R^2 + r^2) — together < 40 u (R^2 + r^2) <= M / 3 — so
// disc' < -M implies the exact disc < 0: the exact test would miss too.
// Every sphere that survives goes through the exact test (pair_disc +
// root_of), so the image stays bit-identical; only provable misses are
// skipped.
struct RayPre {
  float2 ox, oy, oz, hx, hy, hz;  // (v, v) pairs: FFMA2 operands; h = d / 2
  float2 nod, moo;                // -(o.d) and M - |o|^2
  uint32_t all;                   // ~0u: M overflowed, every pair is a candidate
};
__device__ __forceinline__ RayPre ray_pre(V3 o, V3 d, float smax, float rmax2) {
  RayPre p;
  p.ox = make_float2(o.x, o.x);
  p.oy = make_float2(o.y, o.y);
  p.oz = make_float2(o.z, o.z);
  p.hx = make_float2(0.5f * d.x, 0.5f * d.x);  // exact: scaling by a power of two
  p.hy = make_float2(0.5f * d.y, 0.5f * d.y);
  p.hz = make_float2(0.5f * d.z, 0.5f * d.z);
  const float od = fmaf(o.z, d.z, fmaf(o.y, d.y, o.x * d.x));
  const float oo = fmaf(o.z, o.z, fmaf(o.y, o.y, o.x * o.x));
  const float R = fabsf(o.x) + fabsf(o.y) + fabsf(o.z) + smax;
  const float M = 0x1p-17f * fmaf(R, R, rmax2);
  p.nod = make_float2(-od, -od);
  p.moo = make_float2(M - oo, M - oo);
  // with M finite every magnitude below is finite (no NaN); otherwise skip nothing
  p.all = M < INFINITY ? 0u : ~0u;
  return p;
}
// pre[i] = (2x0, 2x1, 2y0, 2y1), (2z0, 2z1, q0, q1) for sphere pair i (the
// doubled centre 2s serves both products: (2s).(d/2) = s.d exactly, and
// (2s).o = 2 o.s).  Per pair, 8 packed FMA-pipe instructions:
//   e'  = (2s).(d/2) - o.d                      = -e   (3 FFMA2, from -o.d)
//   acc = (M - |o|^2 - q) + (2s).o                     (1 FADD2 + 3 FFMA2)
//   t   = e'^2 + acc = disc' + M                        (1 FFMA2)
// A sphere is rejected iff t < 0, a pair iff both are: the sign bits are
// collected with one AND of the two words and one funnel shift per pair,
// no compares.  Bit G-1-k of the collected word is pair k's "both rejected".
template <int G>
__device__ __forceinline__ uint32_t scan_group(const RayPre& p, const float4 (*pre)[2], uint32_t first) {
  static_assert(G >= 1 && G <= 32, "group of at most 32 pairs");
  uint32_t miss = 0;
#pragma unroll
  for (int k = 0; k < G; ++k) {
    const float4 r0 = pre[first + k][0], r1 = pre[first + k][1];
    const float2 X = make_float2(r0.x, r0.y), Y = make_float2(r0.z, r0.w);
    const float2 Z = make_float2(r1.x, r1.y), Q = make_float2(r1.z, r1.w);
    const float2 e = __ffma2_rn(Z, p.hz, __ffma2_rn(Y, p.hy, __ffma2_rn(X, p.hx, p.nod)));
    const float2 acc = __ffma2_rn(Z, p.oz, __ffma2_rn(Y, p.oy, __ffma2_rn(X, p.ox, __fadd2_rn(p.moo, neg2(Q)))));
    const float2 t = __ffma2_rn(e, e, acc);
    miss = __funnelshift_l(__float_as_uint(t.x) & __float_as_uint(t.y), miss, 1);
  }
  const uint32_t cand = (~miss | p.all) & (G == 32 ? ~0u : ((1u << G) - 1u));
  return __brev(cand) >> (32 - G);
}
// Candidate pairs among up to 32 from `first`, as a bit mask, branch-free.
// Groups of G pairs run unrolled; the loops over groups stay rolled (a
// 32-pair unroll of both scans overflowed the instruction cache: ncu "no
// instruction" was the top stall).  The rare candidates are then resolved
// exactly in increasing pair order, which keeps the oracle's
// first-lowest-index choice among equal distances.
__device__ __forceinline__ uint32_t scan_chunk(const RayPre& p, const float4 (*pre)[2], uint32_t first, uint32_t n) {
  constexpr int kGroup = 16;
  uint32_t mask = 0, q = 0;
#pragma unroll 1
  for (; q + kGroup <= n; q += kGroup) mask |= scan_group<kGroup>(p, pre, first + q) << q;
#pragma unroll 1
  for (; q < n; ++q) mask |= scan_group<1>(p, pre, first + q) << q;
  return mask;
}

struct Lane {
  V3 o, d;
  float r, g, b, weight;
  uint32_t depth, bounces;
};

// Shadow rays of one warp's bounce, compacted: lanes write the geometry of
// their up to 3 light rays (direction, distance) and their hit point; the
// (lane, light) pairs that need a shadow test are queued and the warp then
// tests them 32 at a time, so lanes whose pixel missed or faces away from a
// light do not idle through other lanes' shadow loops.  Only scheduling
// changes: every shadow test and shading term is the same arithmetic.
struct ShadowQueue {
  float4 ray[32][3];   // (ln.x, ln.y, ln.z, dist) per lane and light
  float4 point[32];    // hit point p per lane
  uint32_t entry[96];  // (lane << 2) | light
  uint8_t shadowed[32][4];
};

size_t ray_smem_bytes(uint32_t ns) {
  return sizeof(float4) * (2 * static_cast<size_t>(ns) + 4 * ((ns + 1) / 2)) +
         sizeof(ShadowQueue) * (kThreads / 32);
}

template <int MB>
__global__ void __launch_bounds__(kThreads, MB)
    ray_persistent(const float4* __restrict__ scene, uint32_t ns, uint32_t w, uint32_t h, uint32_t max_depth,
                   float4* __restrict__ out, uint64_t first, uint64_t count, unsigned* __restrict__ ctrl) {
  // Dynamic shared memory (ray_smem_bytes): spheres, materials, sphere-pair
  // records, then one ShadowQueue per warp.  Pair records are two 16-byte
  // records (x0, x1, y0, y1), (z0, z1, r0^2, r1^2), so a pair test reads two
  // LDS.128 off one pointer (packed operands aligned).
  extern __shared__ float4 smem[];
  __shared__ unsigned bound_bits[2];  // max |s| and max r^2 as float bits (>= 0: integer order = float order)
  float4* const sph = smem;
  float4* const mat = smem + ns;
  float4 (*const pair_rec)[2] = reinterpret_cast<float4 (*)[2]>(smem + 2 * ns);
  float4 (*const pre_rec)[2] = reinterpret_cast<float4 (*)[2]>(smem + 2 * ns + 2 * ((ns + 1) / 2));
  ShadowQueue* const sq = reinterpret_cast<ShadowQueue*>(smem + 2 * ns + 4 * ((ns + 1) / 2)) + (threadIdx.x >> 5);
  if (threadIdx.x < 2) bound_bits[threadIdx.x] = 0u;
  __syncthreads();
  for (uint32_t i = threadIdx.x; i < ns; i += kThreads) {
    const float4 c = scene[i];
    sph[i] = c;
    mat[i] = scene[ns + i];
    float* rec = reinterpret_cast<float*>(pair_rec[i / 2]);
    float* pre = reinterpret_cast<float*>(pre_rec[i / 2]);
    const uint32_t h = i & 1u;
    rec[0 + h] = c.x;
    rec[2 + h] = c.y;
    rec[4 + h] = c.z;
    pre[0 + h] = 2.0f * c.x;  // exact
    pre[2 + h] = 2.0f * c.y;
    pre[4 + h] = 2.0f * c.z;
    rec[6 + h] = mul(c.w, c.w);
    const double x = c.x, y = c.y, z = c.z, r = c.w;
    pre[6 + h] = static_cast<float>(x * x + y * y + z * z - r * r);  // q = |s|^2 - r^2
    // bounds rounded up (x 1.000001): M only has to dominate the error terms
    atomicMax(&bound_bits[0], __float_as_uint(static_cast<float>(sqrt(x * x + y * y + z * z) * 1.000001)));
    atomicMax(&bound_bits[1], __float_as_uint(static_cast<float>(r * r * 1.000001)));
  }
  // sphere pairs [0, pairs_end) go through pair_disc, an odd last one alone
  const uint32_t pairs_end = ns & ~1u, npairs = ns / 2;

  // camera, lights, floor material, shading constants and sky stay in shared
  // memory (broadcast reads where used): 28 registers the sphere scans need
  __shared__ float4 env[7];
  if (threadIdx.x < 7) env[threadIdx.x] = scene[2 * ns + threadIdx.x];
  const float4& cam = env[0];
  const float4* const lights = env + 1;
  const float4 &pmat = env[4], &shading = env[5], &sky = env[6];
  __syncthreads();
  const float smax = __uint_as_float(bound_bits[0]), rmax2 = __uint_as_float(bound_bits[1]);

  const unsigned lane_id = threadIdx.x & 31u;
  const unsigned below = (1u << lane_id) - 1u;
  const uint64_t nchunks = (count + kChunk - 1) / kChunk;
  uint64_t next = 0, end = 0;
  bool more = true;
  auto claim = [&]() {
    unsigned c = 0;
    if (lane_id == 0) c = atomicAdd(ctrl, 1u);
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

  const float aspect = dvd(static_cast<float>(w), static_cast<float>(h));
  bool valid = false;
  uint64_t idx = 0;
  Lane L{};
  for (;;) {
    unsigned need = __ballot_sync(kFull, !valid);
    while (need && more) {
      const unsigned rank = __popc(need & below);
      const uint64_t avail = end - next;
      if (!valid && rank < avail) {
        idx = first + next + rank;
        const uint32_t px = static_cast<uint32_t>(idx % w), py = static_cast<uint32_t>(idx / w);
        const float u = mul(mul(sub(dvd(mul(2.0f, add(static_cast<float>(px), 0.5f)), static_cast<float>(w)), 1.0f),
                                aspect),
                            cam.w);
        const float v =
            mul(sub(1.0f, dvd(mul(2.0f, add(static_cast<float>(py), 0.5f)), static_cast<float>(h))), cam.w);
        L.d = vnorm(V3{u, v, 1.0f});
        L.o = V3{cam.x, cam.y, cam.z};
        L.r = L.g = L.b = 0.0f;
        L.weight = 1.0f;
        L.depth = 0;
        L.bounces = 0;
        valid = true;
      }
      const uint64_t want = __popc(need);
      next += want < avail ? want : avail;
      if (next >= end) claim();
      need = __ballot_sync(kFull, !valid);
    }
    if (!__any_sync(kFull, valid)) break;

    bool finished = !valid;
    bool lit = false;  // hit a surface this bounce: shade it
    V3 p{0.0f, 0.0f, 0.0f}, n{0.0f, 0.0f, 0.0f};
    float cr = 0.0f, cg = 0.0f, cb = 0.0f, refl = 0.0f;
    float ndl[3] = {0.0f, 0.0f, 0.0f};
    if (valid) {
      // ---- one bounce (oracle: trace_pixel loop body) ----
      float tmin = 1e30f;
      int hit = -1;
      const RayPre rp = ray_pre(L.o, L.d, smax, rmax2);
      for (uint32_t c0 = 0; c0 < npairs; c0 += 32) {
        for (uint32_t m = scan_chunk(rp, pre_rec, c0, npairs - c0); m; m &= m - 1) {
          const uint32_t pq = c0 + static_cast<uint32_t>(__ffs(m)) - 1, s = 2 * pq;
          float2 b, disc;
          pair_disc(L.o, L.d, pair_rec[pq][0], pair_rec[pq][1], b, disc);
          const float2 t = make_float2(root_of(b.x, disc.x), root_of(b.y, disc.y));
          if (t.x > 0.0f && t.x < tmin) {
            tmin = t.x;
            hit = static_cast<int>(s);
          }
          if (t.y > 0.0f && t.y < tmin) {
            tmin = t.y;
            hit = static_cast<int>(s + 1);
          }
        }
      }
      if (pairs_end < ns) {
        const float t = ray_sphere(L.o, L.d, sph[pairs_end]);
        if (t > 0.0f && t < tmin) {
          tmin = t;
          hit = static_cast<int>(pairs_end);
        }
      }
      if (L.d.y < 0.0f) {
        const float tp = dvd(-L.o.y, L.d.y);
        if (tp > 1e-3f && tp < tmin) {
          tmin = tp;
          hit = static_cast<int>(ns);
        }
      }
      if (hit < 0) {
        L.r = add(L.r, mul(L.weight, sky.x));
        L.g = add(L.g, mul(L.weight, sky.y));
        L.b = add(L.b, mul(L.weight, sky.z));
        finished = true;
      } else {
        lit = true;
        p = V3{add(L.o.x, mul(tmin, L.d.x)), add(L.o.y, mul(tmin, L.d.y)), add(L.o.z, mul(tmin, L.d.z))};
        if (hit < static_cast<int>(ns)) {
          const float4 c = sph[hit], m = mat[hit];
          n = vnorm(vsub(p, V3{c.x, c.y, c.z}));
          cr = m.x;
          cg = m.y;
          cb = m.z;
          refl = m.w;
        } else {
          n = V3{0.0f, 1.0f, 0.0f};
          const int check = (static_cast<int>(floorf(p.x)) + static_cast<int>(floorf(p.z))) & 1;
          const float k = check ? 1.0f : 0.35f;
          cr = mul(pmat.x, k);
          cg = mul(pmat.y, k);
          cb = mul(pmat.z, k);
          refl = pmat.w;
        }
        sq->point[lane_id] = make_float4(p.x, p.y, p.z, 0.0f);
#pragma unroll
        for (int l = 0; l < 3; ++l) {
          const V3 Lv = vsub(V3{lights[l].x, lights[l].y, lights[l].z}, p);
          const float dist = __fsqrt_rn(vdot(Lv, Lv));
          const V3 ln{dvd(Lv.x, dist), dvd(Lv.y, dist), dvd(Lv.z, dist)};
          ndl[l] = vdot(n, ln);
          sq->ray[lane_id][l] = make_float4(ln.x, ln.y, ln.z, dist);
        }
      }
    }

    // ---- shadow rays of the whole warp, compacted (all lanes converged) ----
    __syncwarp();
    unsigned queued = 0;
#pragma unroll
    for (int l = 0; l < 3; ++l) {
      const bool need = lit && ndl[l] > 0.0f;
      const unsigned m = __ballot_sync(kFull, need);
      if (need) sq->entry[queued + __popc(m & below)] = (lane_id << 2) | static_cast<unsigned>(l);
      queued += __popc(m);
    }
    __syncwarp();
    for (unsigned base = 0; base < queued; base += 32) {
      const unsigned e = base + lane_id;
      if (e < queued) {
        const unsigned code = sq->entry[e], owner = code >> 2, l = code & 3u;
        const float4 g = sq->ray[owner][l], pp = sq->point[owner];
        const V3 po{pp.x, pp.y, pp.z}, ln{g.x, g.y, g.z};
        const float dist = g.w;
        bool shadow = false;
        const RayPre rp = ray_pre(po, ln, smax, rmax2);
        for (uint32_t c0 = 0; c0 < npairs && !shadow; c0 += 32) {
          for (uint32_t m = scan_chunk(rp, pre_rec, c0, npairs - c0); m && !shadow; m &= m - 1) {
            const uint32_t pq = c0 + static_cast<uint32_t>(__ffs(m)) - 1;
            float2 b, disc;
            pair_disc(po, ln, pair_rec[pq][0], pair_rec[pq][1], b, disc);
            const float2 t = make_float2(root_of(b.x, disc.x), root_of(b.y, disc.y));
            shadow = (t.x > 0.0f && t.x < dist) || (t.y > 0.0f && t.y < dist);
          }
        }
        if (!shadow && pairs_end < ns) {
          const float t = ray_sphere(po, ln, sph[pairs_end]);
          shadow = t > 0.0f && t < dist;
        }
        sq->shadowed[owner][l] = shadow ? 1 : 0;
      }
    }
    __syncwarp();

    if (lit) {
      float lr = mul(shading.x, cr), lg = mul(shading.x, cg), lb = mul(shading.x, cb);
#pragma unroll
      for (int l = 0; l < 3; ++l) {
        if (ndl[l] <= 0.0f) continue;
        if (sq->shadowed[lane_id][l]) continue;
        const float4 g = sq->ray[lane_id][l];
        const V3 ln{g.x, g.y, g.z};
        const float two_ndl = mul(2.0f, ndl[l]);
        const V3 rl{sub(mul(two_ndl, n.x), ln.x), sub(mul(two_ndl, n.y), ln.y), sub(mul(two_ndl, n.z), ln.z)};
        float sp = -add(add(mul(rl.x, L.d.x), mul(rl.y, L.d.y)), mul(rl.z, L.d.z));
        sp = sp > 0.0f ? sp : 0.0f;
        sp = mul(sp, sp);
        sp = mul(sp, sp);
        sp = mul(sp, sp);
        sp = mul(sp, sp);
        const float I = lights[l].w;
        lr = add(lr, mul(I, add(mul(cr, ndl[l]), mul(shading.y, sp))));
        lg = add(lg, mul(I, add(mul(cg, ndl[l]), mul(shading.y, sp))));
        lb = add(lb, mul(I, add(mul(cb, ndl[l]), mul(shading.y, sp))));
      }
      const float keep = mul(L.weight, sub(1.0f, refl));
      L.r = add(L.r, mul(keep, lr));
      L.g = add(L.g, mul(keep, lg));
      L.b = add(L.b, mul(keep, lb));
      L.bounces = L.depth + 1;
      L.weight = mul(L.weight, refl);
      if (!(refl > 0.0f) || L.weight < 1e-3f || L.depth + 1 > max_depth) {
        finished = true;
      } else {
        const float two_dn = mul(2.0f, vdot(L.d, n));
        L.d = V3{sub(L.d.x, mul(two_dn, n.x)), sub(L.d.y, mul(two_dn, n.y)), sub(L.d.z, mul(two_dn, n.z))};
        L.o = p;
        L.depth += 1;
      }
    }
    __syncwarp();  // the queue is rewritten next bounce
    if (valid && finished) {
      out[idx] = make_float4(L.r, L.g, L.b, static_cast<float>(L.bounces));
      valid = false;
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

template <int MB>
cudaError_t launch(const KernelSpec& spec, const LaunchEnv& env, uint64_t first, uint64_t count) {
  // Resident CTAs per SM depend on the scene's shared memory: cached as
  // (smem bytes << 8 | CTAs) for the last scene size seen (device threads
  // may race to fill it; every writer stores the same value for a size).
  static std::atomic<uint64_t> occ_cache{0};
  const size_t smem = ray_smem_bytes(spec.ray.spheres);
  if (smem > 48 * 1024) {
    const cudaError_t e = cudaFuncSetAttribute(ray_persistent<MB>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                               static_cast<int>(smem));
    if (e != cudaSuccess) return e;
  }
  uint64_t cached = occ_cache.load(std::memory_order_relaxed);
  int blocks_per_sm = static_cast<int>(cached & 0xffu);
  if ((cached >> 8) != smem || blocks_per_sm == 0) {
    const cudaError_t e =
        cudaOccupancyMaxActiveBlocksPerMultiprocessor(&blocks_per_sm, ray_persistent<MB>, kThreads, smem);
    if (e != cudaSuccess) return e;
    if (blocks_per_sm < 1) blocks_per_sm = 1;
    occ_cache.store((static_cast<uint64_t>(smem) << 8) | static_cast<uint64_t>(blocks_per_sm & 0xff),
                    std::memory_order_relaxed);
  }
  const uint64_t chunks = (count + kChunk - 1) / kChunk;
  const uint64_t blocks_needed = (chunks + kThreads / 32 - 1) / (kThreads / 32);
  uint64_t grid = static_cast<uint64_t>(env.sms) * static_cast<uint64_t>(blocks_per_sm);
  if (blocks_needed < grid) grid = blocks_needed;
  ray_persistent<MB><<<static_cast<unsigned>(grid), kThreads, smem, env.stream>>>(
      static_cast<const float4*>(env.in[0]), spec.ray.spheres, spec.ray.width, spec.ray.height, spec.ray.max_depth,
      static_cast<float4*>(env.out[0]), first, count, env.ctrl);
  return cudaGetLastError();
}

}  // namespace

cudaError_t launch_ray(const KernelSpec& spec, const LaunchEnv& env, uint64_t first, uint64_t count) {
  if (count == 0) return cudaSuccess;
  // ECL_RAY_MB: 128-thread CTAs per SM the registers are sized for.  Measured
  // (8192^2 native single launch, sign-bit prefiltered scans, scene constants
  // in shared memory): 6 -> 11.40 ms (80 registers, 8 B spilled),
  // 7 -> 11.15 (72, no spill), 8 -> 11.01 (64; 16 B of stack, 28 B of spill
  // loads, outside the sphere scans: the occupancy pays for them), 10 -> 11.87.
  // With the 8-instruction scan (bench step, two-lane pieces): 7 -> 9.38,
  // 8 -> 9.23, 10 -> 9.50.
  static const int env_mb = [] {
    const char* v = std::getenv("ECL_RAY_MB");
    return v ? std::atoi(v) : 0;
  }();
  // ray@1: 10 CTAs/SM (48 registers), ray@2: 6
  const int mb = spec.variant == 1 ? 10 : spec.variant == 2 ? 6 : spec.variant == 0 ? 8 : env_mb;
  switch (mb) {
    case 6: return launch<6>(spec, env, first, count);
    case 7: return launch<7>(spec, env, first, count);
    case 8: return launch<8>(spec, env, first, count);
    case 12: return launch<12>(spec, env, first, count);
    case 16: return launch<16>(spec, env, first, count);
    case 10: return launch<10>(spec, env, first, count);
    default: return launch<8>(spec, env, first, count);
  }
}

}  // namespace ecl
