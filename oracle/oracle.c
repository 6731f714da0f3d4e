/*
 * oracle.c — CPU restatement of the EngineCL/coexec hot-path arithmetic.
 *
 * TEST INFRASTRUCTURE ONLY.  This file is the checker the parity tests,
 * __graft_entry__.smoke() and bench.py's cpu_baseline leg compare the CUDA
 * path against.  Nothing in the product (libcoexec.so / libecl_cuda.so /
 * the paper_1805_02755_b200 package) links, loads or calls it.
 *
 * Build flags are pinned: -std=c11 -O2 -ffp-contract=off (no FMA contraction,
 * no -ffast-math) — SURVEY.md §8c "Required oracle build flags".
 *
 * Parity status per function:
 *   mandelbrot_f64, vecscale, synthetic, fill_f64: restate the reference
 *     (/root/reference/proj/include/coexec/workloads.hpp) and are PINNED by
 *     the reference's own known answers and by oracle/_ref (the reference
 *     headers compiled by oracle/Makefile) — see tests/test_oracle.py.
 *   mandelbrot_f32, gaussian, nbody, binomial, ray: the reference has NO
 *     implementation.  Their definitions are this repo's own
 *      — "parity unpinned" by the reference.
 */
#include <math.h>
#include <stdlib.h>
#include <stdint.h>
#include <string.h>

#ifdef _OPENMP
#include <omp.h>
#endif

/* ------------------------------------------------------------------------ */
/* splitmix64 input fill — workloads.hpp:261-283 (fill_default_inputs).      */
/* One generator state runs across all input buffers in order; doubles are  */
/* (z >> 11) * 2^-53.                                                        */

static uint64_t splitmix_next(uint64_t* state) {
  *state += 0x9e3779b97f4a7c15ull;
  uint64_t z = *state;
  z = (z ^ (z >> 30)) * 0xbf58476d1ce4e5b9ull;
  z = (z ^ (z >> 27)) * 0x94d049bb133111ebull;
  return z ^ (z >> 31);
}

/* Fills n doubles in [0,1); *state is advanced (workloads.hpp:272-274). */
void orc_fill_f64(uint64_t* state, uint64_t n, double* out) {
  for (uint64_t i = 0; i < n; ++i) out[i] = (double)(splitmix_next(state) >> 11) * 0x1.0p-53;
}

/* Non-double buffers get one byte per draw (workloads.hpp:276-277). */
void orc_fill_bytes(uint64_t* state, uint64_t n, uint8_t* out) {
  for (uint64_t i = 0; i < n; ++i) out[i] = (uint8_t)(splitmix_next(state) & 0xff);
}

/* FNV-1a 64 over raw bytes (SURVEY.md §8c checksum convention). */
uint64_t orc_fnv1a64(const void* data, uint64_t n, uint64_t h) {
  const uint8_t* p = (const uint8_t*)data;
  if (h == 0) h = 0xcbf29ce484222325ull;
  for (uint64_t i = 0; i < n; ++i) {
    h ^= p[i];
    h *= 0x100000001b3ull;
  }
  return h;
}

/* ------------------------------------------------------------------------ */
/* Mandelbrot, FP64 — workloads.hpp:78-100 (mandel_escape_count,            */
/* mandel_count_for_index).  Same operation order, no contraction.          */

static uint32_t escape_f64(double cx, double cy, uint32_t max_iter) {
  double zx = 0.0, zy = 0.0;
  uint32_t n = 0;
  while (n < max_iter) {
    const double xx = zx * zx;
    const double yy = zy * zy;
    if (xx + yy > 4.0) break;
    zy = 2.0 * zx * zy + cy; /* (2*zx)*zy + cy, left to right */
    zx = xx - yy + cx;       /* (xx - yy) + cx */
    ++n;
  }
  return n;
}

uint32_t orc_mandel_count_f64(uint64_t index, uint64_t w, uint64_t h, uint32_t max_iter, double x0,
                              double y0, double x1, double y1) {
  const uint64_t px = index % w, py = index / w;
  const double cx = x0 + (double)px * (x1 - x0) / (double)w;
  const double cy = y0 + (double)py * (y1 - y0) / (double)h;
  return escape_f64(cx, cy, max_iter);
}

/* counts[i - first] for i in [first, first+count): one count per pixel.
 * The reference kernel writes it 4 times (4:1 pattern, workloads.hpp:217-222);
 * tests expand when they compare against the device's 4:1 buffer. */
void orc_mandelbrot_f64(uint64_t w, uint64_t h, uint32_t max_iter, double x0, double y0, double x1,
                        double y1, uint64_t first, uint64_t count, uint32_t* counts) {
#pragma omp parallel for schedule(dynamic, 1024)
  for (int64_t k = 0; k < (int64_t)count; ++k)
    counts[k] = orc_mandel_count_f64(first + (uint64_t)k, w, h, max_iter, x0, y0, x1, y1);
}

/* ------------------------------------------------------------------------ */
/* Mandelbrot, FP32 variant (this repo's definition; parity unpinned by the  */
/* reference).  Viewport cast to float once; the map and the iteration keep */
/* the FP64 kernel's operation order in float.                              */

static uint32_t escape_f32(float cx, float cy, uint32_t max_iter) {
  float zx = 0.0f, zy = 0.0f;
  uint32_t n = 0;
  while (n < max_iter) {
    const float xx = zx * zx;
    const float yy = zy * zy;
    if (xx + yy > 4.0f) break;
    zy = 2.0f * zx * zy + cy;
    zx = xx - yy + cx;
    ++n;
  }
  return n;
}

uint32_t orc_mandel_count_f32(uint64_t index, uint64_t w, uint64_t h, uint32_t max_iter, double x0,
                              double y0, double x1, double y1) {
  const uint64_t px = index % w, py = index / w;
  const float fx0 = (float)x0, fy0 = (float)y0, fx1 = (float)x1, fy1 = (float)y1;
  const float cx = fx0 + (float)px * (fx1 - fx0) / (float)w;
  const float cy = fy0 + (float)py * (fy1 - fy0) / (float)h;
  return escape_f32(cx, cy, max_iter);
}

void orc_mandelbrot_f32(uint64_t w, uint64_t h, uint32_t max_iter, double x0, double y0, double x1,
                        double y1, uint64_t first, uint64_t count, uint32_t* counts) {
#pragma omp parallel for schedule(dynamic, 1024)
  for (int64_t k = 0; k < (int64_t)count; ++k)
    counts[k] = orc_mandel_count_f32(first + (uint64_t)k, w, h, max_iter, x0, y0, x1, y1);
}

/* Algorithmic FP64 flop count of a count array: 8 per iteration + 3 for the
 * failed escape test of every escaped pixel.  Also returns
 * the iteration sum and the number of pixels that reached max_iter. */
void orc_mandel_stats(const uint32_t* counts, uint64_t n, uint32_t max_iter, uint64_t* sum_count,
                      uint64_t* inside, double* flops) {
  uint64_t s = 0, in = 0;
  for (uint64_t i = 0; i < n; ++i) {
    s += counts[i];
    in += counts[i] >= max_iter;
  }
  *sum_count = s;
  *inside = in;
  *flops = 8.0 * (double)s + 3.0 * (double)(n - in);
}

/* ------------------------------------------------------------------------ */
/* vecscale — workloads.hpp:207-214: out[i] = a*in[i] + b (FP64, no FMA).   */

void orc_vecscale(double a, double b, const double* in, double* out, uint64_t first, uint64_t count) {
  for (uint64_t i = first; i < first + count; ++i) out[i] = a * in[i] + b;
}

/* synthetic cost profiles — workloads.hpp:136-149.  profile 0 constant (c),
 * 1 ramp (1 + i/gws), 2 step (1 below gws/2, `high` above). */
void orc_synthetic(int profile, double param, int has_param, uint64_t gws, double* out, uint64_t first,
                   uint64_t count) {
  for (uint64_t i = first; i < first + count; ++i) {
    double v = 1.0;
    if (profile == 0) v = has_param ? param : 1.0;
    else if (profile == 1) v = 1.0 + (double)i / (double)gws;
    else v = i < gws / 2 ? 1.0 : (has_param ? param : 10.0);
    out[i] = v;
  }
}

/* ------------------------------------------------------------------------ */
/* Gaussian blur (ABSENT in the reference).            */
/* out[y*W+x] = sum_{i<F} sum_{j<F} filt[i*F+j] * img[cl(y+i-F/2)*W + cl(x+j-F/2)] */
/* f32 accumulation, i outer, j inner, starting at 0.0f; clamp-to-edge.     */

void orc_gaussian_filter(uint32_t f, double sigma, float* filt) {
  const int r = (int)f / 2;
  double sum = 0.0;
  for (uint32_t i = 0; i < f; ++i)
    for (uint32_t j = 0; j < f; ++j) {
      const double di = (double)((int)i - r), dj = (double)((int)j - r);
      sum += exp(-(di * di + dj * dj) / (2.0 * sigma * sigma));
    }
  for (uint32_t i = 0; i < f; ++i)
    for (uint32_t j = 0; j < f; ++j) {
      const double di = (double)((int)i - r), dj = (double)((int)j - r);
      filt[i * f + j] = (float)(exp(-(di * di + dj * dj) / (2.0 * sigma * sigma)) / sum);
    }
}

static inline int64_t clampi(int64_t v, int64_t lo, int64_t hi) { return v < lo ? lo : (v > hi ? hi : v); }

void orc_gaussian(const float* img, const float* filt, float* out, uint32_t w, uint32_t h, uint32_t f,
                  uint64_t first, uint64_t count) {
  const int64_t r = (int64_t)f / 2;
#pragma omp parallel for schedule(static) if (count > 256)
  for (int64_t k = 0; k < (int64_t)count; ++k) {
    const uint64_t idx = first + (uint64_t)k;
    const int64_t x = (int64_t)(idx % w), y = (int64_t)(idx / w);
    float acc = 0.0f;
    for (int64_t i = 0; i < (int64_t)f; ++i) {
      const int64_t yy = clampi(y + i - r, 0, (int64_t)h - 1);
      for (int64_t j = 0; j < (int64_t)f; ++j) {
        const int64_t xx = clampi(x + j - r, 0, (int64_t)w - 1);
        acc += filt[i * f + j] * img[yy * (int64_t)w + xx];
      }
    }
    out[idx] = acc;
  }
}

/* ------------------------------------------------------------------------ */
/* NBody step (ABSENT in the reference; Listing 2 PAPER.md:403-440 and       */
/* SURVEY.md Appendix B).  pos = float4 (xyz, w = mass), vel = float4.      */
/* acc_i = sum_j m_j * r_ij / (|r_ij|^2 + eps2)^(3/2), r_ij = p_j - p_i.    */
/* The oracle accumulates in double (a more accurate reference than the    */
/* f32 device sum); tolerances are stated in tests/test_kernels_gpu.py.    */

void orc_nbody_step(const float* pos, const float* vel, uint64_t n, float dt, float eps2, float* npos,
                    float* nvel, uint64_t first, uint64_t count) {
#pragma omp parallel for schedule(dynamic, 16) if (count > 16)
  for (int64_t k = 0; k < (int64_t)count; ++k) {
    const uint64_t i = first + (uint64_t)k;
    const double px = pos[4 * i], py = pos[4 * i + 1], pz = pos[4 * i + 2];
    double ax = 0.0, ay = 0.0, az = 0.0;
    for (uint64_t j = 0; j < n; ++j) {
      const double rx = (double)pos[4 * j] - px, ry = (double)pos[4 * j + 1] - py,
                   rz = (double)pos[4 * j + 2] - pz;
      const double d2 = rx * rx + ry * ry + rz * rz + (double)eps2;
      const double inv = 1.0 / sqrt(d2);
      const double s = (double)pos[4 * j + 3] * inv * inv * inv;
      ax += s * rx;
      ay += s * ry;
      az += s * rz;
    }
    const double vx = vel[4 * i], vy = vel[4 * i + 1], vz = vel[4 * i + 2];
    const double hdt2 = 0.5 * (double)dt * (double)dt;
    npos[4 * i] = (float)(px + vx * dt + ax * hdt2);
    npos[4 * i + 1] = (float)(py + vy * dt + ay * hdt2);
    npos[4 * i + 2] = (float)(pz + vz * dt + az * hdt2);
    npos[4 * i + 3] = pos[4 * i + 3];
    nvel[4 * i] = (float)(vx + ax * dt);
    nvel[4 * i + 1] = (float)(vy + ay * dt);
    nvel[4 * i + 2] = (float)(vz + az * dt);
    nvel[4 * i + 3] = vel[4 * i + 3];
  }
}

/* NBody synthetic init: xyz U[3,50), w U[1,1000), vel 0;   */
/* one splitmix64 stream from `seed`, four draws per body in x,y,z,w order. */
void orc_nbody_init(uint64_t seed, uint64_t n, float* pos, float* vel) {
  uint64_t st = seed;
  for (uint64_t i = 0; i < n; ++i) {
    for (int c = 0; c < 3; ++c) {
      const double u = (double)(splitmix_next(&st) >> 11) * 0x1.0p-53;
      pos[4 * i + c] = (float)(3.0 + 47.0 * u);
    }
    const double u = (double)(splitmix_next(&st) >> 11) * 0x1.0p-53;
    pos[4 * i + 3] = (float)(1.0 + 999.0 * u);
    vel[4 * i] = vel[4 * i + 1] = vel[4 * i + 2] = vel[4 * i + 3] = 0.0f;
  }
}

/* ------------------------------------------------------------------------ */
/* Binomial options (ABSENT in the reference; Listing 1,   */
/* SURVEY.md Appendix B).  European call on a CRR lattice.  One float4 of   */
/* four options per work-group (out pattern 1:255 with lws = steps+1).      */
/* The oracle evaluates in double; the device in f32.                       */

void orc_binomial(const float* rand4, float* out4, uint32_t steps, uint64_t first_opt, uint64_t n_opt) {
  const double R = 0.02, V = 0.30;
#pragma omp parallel if (n_opt > 16)
  {
    double call[1024];
#pragma omp for schedule(static)
    for (int64_t k = 0; k < (int64_t)n_opt; ++k) {
      const uint64_t o = first_opt + (uint64_t)k;
      const double r = rand4[o];
      const double S = 5.0 * (1.0 - r) + 30.0 * r;
      const double K = 1.0 * (1.0 - r) + 100.0 * r;
      const double T = 0.25 * (1.0 - r) + 10.0 * r;
      const double dt = T / (double)steps;
      const double vsdt = V * sqrt(dt);
      const double a = exp(R * dt);
      const double u = exp(vsdt);
      const double d = 1.0 / u;
      const double pu = (a - d) / (u - d);
      const double pu_r = pu / a, pd_r = (1.0 - pu) / a;
      for (uint32_t t = 0; t <= steps; ++t) {
        const double st = S * exp(vsdt * (2.0 * (double)t - (double)steps)) - K;
        call[t] = st > 0.0 ? st : 0.0;
      }
      for (uint32_t j = steps; j > 0; --j)
        for (uint32_t t = 0; t < j; ++t) call[t] = pu_r * call[t + 1] + pd_r * call[t];
      out4[o] = (float)call[0];
    }
  }
}

/* Binomial synthetic input: r ~ U[0,1) per option from splitmix64(seed). */
void orc_binomial_init(uint64_t seed, uint64_t n_opt, float* rand4) {
  uint64_t st = seed;
  for (uint64_t i = 0; i < n_opt; ++i) rand4[i] = (float)((double)(splitmix_next(&st) >> 11) * 0x1.0p-53);
}

/* Ray synthetic scene (layout below): the same arithmetic as
 * paper_1805_02755_b200/workloads.py:ray_scene — doubles from splitmix64(seed),
 * eight draws per sphere, cast to float at the end — so bench.py's reference
 * arm builds the scene without the product package.  buf: (2*ns+8) float4. */
void orc_ray_scene(uint64_t seed, uint32_t ns, float* buf) {
  uint64_t st = seed;
  double* u = (double*)malloc(sizeof(double) * 8 * (size_t)ns);
  for (uint64_t i = 0; i < 8ull * ns; ++i) u[i] = (double)(splitmix_next(&st) >> 11) * 0x1.0p-53;
  for (uint64_t i = 0; i < 4ull * (2 * ns + 8); ++i) buf[i] = 0.0f;
  for (uint32_t k = 0; k < ns; ++k) {
    const double* v = u + 8 * (size_t)k;
    const double r = 0.3 + 1.2 * v[2];
    float* sp = buf + 4 * (size_t)k;
    float* mt = buf + 4 * ((size_t)ns + k);
    sp[0] = (float)(-8.0 + 16.0 * v[0]);
    sp[1] = (float)(r + 2.0 * v[3]);
    sp[2] = (float)(2.0 + 16.0 * v[1]);
    sp[3] = (float)r;
    for (int c = 0; c < 3; ++c) mt[c] = (float)(0.2 + 0.8 * v[4 + c]);
    mt[3] = (float)((k % 3) == 0 ? 0.6 + 0.3 * v[7] : 0.15 * v[7]);
  }
  free(u);
  static const float tail[7][4] = {{0.0f, 2.5f, -12.0f, 0.6f}, {-10.0f, 12.0f, -6.0f, 0.7f},
                                   {8.0f, 15.0f, 0.0f, 0.5f},   {0.0f, 20.0f, 10.0f, 0.4f},
                                   {0.9f, 0.9f, 0.9f, 0.3f},    {0.08f, 0.5f, 0.0f, 0.0f},
                                   {0.25f, 0.35f, 0.55f, 0.0f}};
  for (int t = 0; t < 7; ++t)
    for (int c = 0; c < 4; ++c) buf[4 * (2 * (size_t)ns + t) + c] = tail[t][c];
}

int orc_num_threads(void) {
#ifdef _OPENMP
  return omp_get_max_threads();
#else
  return 1;
#endif
}

/* ------------------------------------------------------------------------ */
/* Ray tracing (ABSENT in the reference; Table 2; this      */
/* repo's definition).  Whitted-style: nearest hit     */
/* over `ns` spheres and the ground plane y = 0, Phong shading with hard     */
/* shadows from 3 point lights, mirror reflection up to `max_depth` bounces. */
/* Every float operation is a single IEEE op in a fixed order (the oracle   */
/* is built with -ffp-contract=off and the device uses _rn intrinsics), the */
/* specular power is x^16 by four squarings, so the device can match the    */
/* oracle bit for bit.  Scene buffer (float4): spheres[ns] (cx,cy,cz,r),    */
/* materials[ns] (r,g,b,refl), then camera (ox,oy,oz,tan_half_fov),        */
/* lights[3] (x,y,z,intensity), plane material (r,g,b,refl), shading        */
/* (ambient, spec_k, 0, 0), sky (r,g,b,0).  Output float4 (r,g,b,bounces). */

typedef struct { float x, y, z; } v3;

static inline v3 v3sub(v3 a, v3 b) { v3 r = {a.x - b.x, a.y - b.y, a.z - b.z}; return r; }
static inline float v3dot(v3 a, v3 b) { return a.x * b.x + a.y * b.y + a.z * b.z; }
static inline v3 v3scale(v3 a, float s) { v3 r = {a.x * s, a.y * s, a.z * s}; return r; }
static inline v3 v3norm(v3 a) {
  const float len = sqrtf(v3dot(a, a));
  v3 r = {a.x / len, a.y / len, a.z / len};
  return r;
}

/* distance along (o,d) to sphere s (cx,cy,cz,r); < 0 = miss */
static inline float ray_sphere(v3 o, v3 d, const float* s) {
  const v3 c = {s[0], s[1], s[2]};
  const v3 oc = v3sub(o, c);
  const float b = v3dot(oc, d);
  const float cc = v3dot(oc, oc) - s[3] * s[3];
  const float disc = b * b - cc;
  if (disc < 0.0f) return -1.0f;
  const float sq = sqrtf(disc);
  float t = -b - sq;
  if (t > 1e-3f) return t;
  t = -b + sq;
  return t > 1e-3f ? t : -1.0f;
}

typedef struct { uint64_t sphere_tests, plane_tests, shades; } RayCounts;

static void trace_pixel(const float* scene, uint32_t ns, uint32_t w, uint32_t h, uint32_t max_depth, uint64_t idx,
                        float* out4, RayCounts* cnt) {
  const float* sph = scene;
  const float* mat = scene + 4 * ns;
  const float* cam = scene + 8 * ns;
  const float* lights = cam + 4;
  const float* pmat = cam + 16;
  const float* shading = cam + 20;
  const float* sky = cam + 24;
  const uint32_t px = (uint32_t)(idx % w), py = (uint32_t)(idx / w);
  const float tanf_ = cam[3];
  const float aspect = (float)w / (float)h;
  const float u = ((2.0f * ((float)px + 0.5f)) / (float)w - 1.0f) * aspect * tanf_;
  const float v = (1.0f - (2.0f * ((float)py + 0.5f)) / (float)h) * tanf_;
  v3 d0 = {u, v, 1.0f};
  v3 d = v3norm(d0);
  v3 o = {cam[0], cam[1], cam[2]};
  float r = 0.0f, g = 0.0f, b = 0.0f, weight = 1.0f;
  uint32_t bounces = 0;
  for (uint32_t depth = 0; depth <= max_depth; ++depth) {
    float tmin = 1e30f;
    int hit = -1;
    for (uint32_t s = 0; s < ns; ++s) {
      const float t = ray_sphere(o, d, sph + 4 * s);
      if (t > 0.0f && t < tmin) { tmin = t; hit = (int)s; }
    }
    cnt->sphere_tests += ns;
    cnt->plane_tests += 1;
    if (d.y < 0.0f) {
      const float tp = -o.y / d.y;
      if (tp > 1e-3f && tp < tmin) { tmin = tp; hit = (int)ns; }
    }
    if (hit < 0) {
      r += weight * sky[0];
      g += weight * sky[1];
      b += weight * sky[2];
      break;
    }
    const v3 p = {o.x + tmin * d.x, o.y + tmin * d.y, o.z + tmin * d.z};
    v3 n;
    float cr, cg, cb, refl;
    if (hit < (int)ns) {
      const v3 c = {sph[4 * hit], sph[4 * hit + 1], sph[4 * hit + 2]};
      n = v3norm(v3sub(p, c));
      cr = mat[4 * hit]; cg = mat[4 * hit + 1]; cb = mat[4 * hit + 2]; refl = mat[4 * hit + 3];
    } else {
      n.x = 0.0f; n.y = 1.0f; n.z = 0.0f;
      const int check = ((int)floorf(p.x) + (int)floorf(p.z)) & 1;
      const float k = check ? 1.0f : 0.35f;
      cr = pmat[0] * k; cg = pmat[1] * k; cb = pmat[2] * k; refl = pmat[3];
    }
    const float amb = shading[0], spec_k = shading[1];
    float lr = amb * cr, lg = amb * cg, lb = amb * cb;
    for (int l = 0; l < 3; ++l) {
      const v3 lp = {lights[4 * l], lights[4 * l + 1], lights[4 * l + 2]};
      const v3 L = v3sub(lp, p);
      const float dist = sqrtf(v3dot(L, L));
      const v3 ln = {L.x / dist, L.y / dist, L.z / dist};
      const float ndl = v3dot(n, ln);
      cnt->shades += 1;
      if (ndl <= 0.0f) continue;
      int shadow = 0;
      for (uint32_t s = 0; s < ns; ++s) {
        const float t = ray_sphere(p, ln, sph + 4 * s);
        if (t > 0.0f && t < dist) { shadow = 1; break; }
      }
      cnt->sphere_tests += ns; /* counted as a full pass (the device has no early exit per lane) */
      if (shadow) continue;
      /* specular: reflect -ln about n, dot with -d, ^16 */
      const float two_ndl = 2.0f * ndl;
      const v3 rl = {two_ndl * n.x - ln.x, two_ndl * n.y - ln.y, two_ndl * n.z - ln.z};
      float sp = -(rl.x * d.x + rl.y * d.y + rl.z * d.z);
      sp = sp > 0.0f ? sp : 0.0f;
      sp = sp * sp; sp = sp * sp; sp = sp * sp; sp = sp * sp;
      const float I = lights[4 * l + 3];
      lr += I * (cr * ndl + spec_k * sp);
      lg += I * (cg * ndl + spec_k * sp);
      lb += I * (cb * ndl + spec_k * sp);
    }
    const float keep = weight * (1.0f - refl);
    r += keep * lr;
    g += keep * lg;
    b += keep * lb;
    bounces = depth + 1;
    weight = weight * refl;
    if (!(refl > 0.0f) || weight < 1e-3f) break;
    const float two_dn = 2.0f * v3dot(d, n);
    const v3 nd = {d.x - two_dn * n.x, d.y - two_dn * n.y, d.z - two_dn * n.z};
    d = nd;
    o = p;
  }
  out4[0] = r; out4[1] = g; out4[2] = b; out4[3] = (float)bounces;
}

/* Renders pixels [first, first+count) into out4 (float4 per pixel, indexed
 * globally) and returns the instrumented operation counts. */
void orc_ray(const float* scene, uint32_t ns, uint32_t w, uint32_t h, uint32_t max_depth, float* out4,
             uint64_t first, uint64_t count, uint64_t* counts3) {
  uint64_t st = 0, pt = 0, sh = 0;
#pragma omp parallel for schedule(dynamic, 256) reduction(+ : st, pt, sh) if (count > 256)
  for (int64_t k = 0; k < (int64_t)count; ++k) {
    RayCounts c = {0, 0, 0};
    const uint64_t idx = first + (uint64_t)k;
    trace_pixel(scene, ns, w, h, max_depth, idx, out4 + 4 * idx, &c);
    st += c.sphere_tests;
    pt += c.plane_tests;
    sh += c.shades;
  }
  if (counts3) {
    counts3[0] = st;
    counts3[1] = pt;
    counts3[2] = sh;
  }
}
