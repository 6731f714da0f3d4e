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
#pragma omp parallel for schedule(static)
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
#pragma omp parallel for schedule(dynamic, 16)
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
#pragma omp parallel
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

int orc_num_threads(void) {
#ifdef _OPENMP
  return omp_get_max_threads();
#else
  return 1;
#endif
}
