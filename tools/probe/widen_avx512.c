// Host widening 1 -> 4 (Mandelbrot's replicated output): 16-byte SSE
// streaming stores (hostpool.cpp) vs 64-byte AVX-512 streaming stores (one
// full cache line per store).  T threads over a 4 GiB destination.
// Build: gcc -O2 -pthread widen_avx512.c -o widen_avx512
#include <immintrin.h>
#include <pthread.h>
#include <stdint.h>
#include <stdio.h>
#include <stdlib.h>
#include <string.h>
#include <sys/mman.h>
#include <time.h>

typedef struct { const uint32_t* src; uint32_t* dst; uint64_t n; int mode; } Job;

__attribute__((target("avx512f"))) static void widen512(const uint32_t* src, uint32_t* dst, uint64_t n) {
  const __m512i idx = _mm512_set_epi32(3, 3, 3, 3, 2, 2, 2, 2, 1, 1, 1, 1, 0, 0, 0, 0);
  uint64_t i = 0;
  for (; i + 4 <= n; i += 4) {
    const __m512i s = _mm512_castsi128_si512(_mm_loadu_si128((const __m128i*)(src + i)));
    _mm512_stream_si512((__m512i*)(dst + 4 * i), _mm512_permutexvar_epi32(idx, s));
  }
  for (; i < n; ++i) _mm_stream_si128((__m128i*)(dst + 4 * i), _mm_set1_epi32((int)src[i]));
  _mm_sfence();
}
static void widen128(const uint32_t* src, uint32_t* dst, uint64_t n) {
  for (uint64_t i = 0; i < n; ++i) _mm_stream_si128((__m128i*)(dst + 4 * i), _mm_set1_epi32((int)src[i]));
  _mm_sfence();
}
static void* run(void* p) {
  Job* j = (Job*)p;
  if (j->mode) widen512(j->src, j->dst, j->n); else widen128(j->src, j->dst, j->n);
  return NULL;
}
static double now(void) { struct timespec t; clock_gettime(CLOCK_MONOTONIC, &t); return t.tv_sec + 1e-9 * t.tv_nsec; }

int main(int argc, char** argv) {
  const uint64_t n = (argc > 1 ? strtoull(argv[1], NULL, 0) : 1ull << 27);  // items (default: 2 GiB destination)
  uint32_t* src = mmap(NULL, n * 4, PROT_READ | PROT_WRITE, MAP_PRIVATE | MAP_ANONYMOUS, -1, 0);
  uint32_t* dst = mmap(NULL, n * 16, PROT_READ | PROT_WRITE, MAP_PRIVATE | MAP_ANONYMOUS, -1, 0);
  if (src == MAP_FAILED || dst == MAP_FAILED) { perror("mmap"); return 1; }
  madvise(dst, n * 16, MADV_HUGEPAGE);
  madvise(src, n * 4, MADV_HUGEPAGE);
  for (uint64_t i = 0; i < n; ++i) src[i] = (uint32_t)i;
  memset(dst, 1, n * 16);
  const int avx = __builtin_cpu_supports("avx512f") ? 1 : 0;
  for (int mode = 0; mode <= avx; ++mode)
    for (int t = 8; t <= 16; t += 4) {
      double best = 1e9;
      for (int rep = 0; rep < 3; ++rep) {
        pthread_t th[64]; Job jb[64];
        const double t0 = now();
        for (int k = 0; k < t; ++k) {
          const uint64_t a = (n * k / t) & ~3ull, b = k + 1 == t ? n : (n * (k + 1) / t) & ~3ull;  // 64-B aligned chunks
          jb[k] = (Job){src + a, dst + 4 * a, b - a, mode};
          pthread_create(&th[k], NULL, run, &jb[k]);
        }
        for (int k = 0; k < t; ++k) pthread_join(th[k], NULL);
        const double dt = now() - t0;
        if (dt < best) best = dt;
      }
      for (uint64_t i = 0; i < n; i += 12345) if (dst[4 * i + 3] != (uint32_t)i) { printf("mismatch\n"); return 1; }
      printf("%s threads %2d: %.1f ms, write %.1f GB/s\n", mode ? "avx512 64B" : "sse 16B   ", t, best * 1e3,
             n * 16.0 / best / 1e9);
    }
  return 0;
}
