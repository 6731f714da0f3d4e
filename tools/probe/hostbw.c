// Host memory bandwidth probe: expand u32[n] -> 4 x u32 per element (the
// Mandelbrot 4:1 layout) with T threads and non-temporal 128-bit stores.
#include <immintrin.h>
#include <pthread.h>
#include <stdint.h>
#include <stdio.h>
#include <stdlib.h>
#include <string.h>
#include <time.h>

typedef struct {
  const uint32_t* src;
  uint32_t* dst;
  size_t a, b;
} job;

static void* work(void* p) {
  job* j = (job*)p;
  for (size_t i = j->a; i < j->b; ++i) {
    __m128i v = _mm_set1_epi32((int)j->src[i]);
    _mm_stream_si128((__m128i*)(j->dst + 4 * i), v);
  }
  _mm_sfence();
  return 0;
}

static double now(void) {
  struct timespec t;
  clock_gettime(CLOCK_MONOTONIC, &t);
  return t.tv_sec + t.tv_nsec * 1e-9;
}

int main(void) {
  size_t n = (size_t)16384 * 16384;
  uint32_t* src = aligned_alloc(64, n * 4);
  uint32_t* dst = aligned_alloc(64, n * 16);
  memset(src, 1, n * 4);
  memset(dst, 0, n * 16);
  for (int T = 1; T <= 32; T *= 2) {
    pthread_t th[64];
    job jb[64];
    double best = 1e9;
    for (int rep = 0; rep < 3; ++rep) {
      double t0 = now();
      for (int t = 0; t < T; ++t) {
        jb[t] = (job){src, dst, n * t / T, n * (t + 1) / T};
        pthread_create(&th[t], 0, work, &jb[t]);
      }
      for (int t = 0; t < T; ++t) pthread_join(th[t], 0);
      double dt = now() - t0;
      if (dt < best) best = dt;
    }
    printf("threads %2d: %.1f ms  write %.1f GB/s\n", T, best * 1e3, n * 16 / best / 1e9);
  }
  return 0;
}
