// Host widening bandwidth (u32 -> 4 x u32, NT stores, 16 threads) by the
// destination's page size: 4 KiB pages vs transparent huge pages.
#define _GNU_SOURCE
#include <immintrin.h>
#include <pthread.h>
#include <stdint.h>
#include <stdio.h>
#include <stdlib.h>
#include <string.h>
#include <sys/mman.h>
#include <time.h>

typedef struct {
  const uint32_t* src;
  uint32_t* dst;
  size_t a, b;
} job;

static void* work(void* p) {
  job* j = (job*)p;
  for (size_t i = j->a; i < j->b; ++i) _mm_stream_si128((__m128i*)(j->dst + 4 * i), _mm_set1_epi32((int)j->src[i]));
  _mm_sfence();
  return 0;
}

static double now(void) {
  struct timespec t;
  clock_gettime(CLOCK_MONOTONIC, &t);
  return t.tv_sec + t.tv_nsec * 1e-9;
}

static uint32_t* alloc(size_t bytes, int advice) {
  void* p = mmap(0, bytes, PROT_READ | PROT_WRITE, MAP_PRIVATE | MAP_ANONYMOUS, -1, 0);
  if (p == MAP_FAILED) return 0;
  if (advice) madvise(p, bytes, advice);
  memset(p, 0, bytes);
  return (uint32_t*)p;
}

static void run(const char* name, const uint32_t* src, uint32_t* dst, size_t n, int T) {
  pthread_t th[64];
  job jb[64];
  double best = 1e9;
  for (int rep = 0; rep < 4; ++rep) {
    double t0 = now();
    for (int t = 0; t < T; ++t) {
      jb[t] = (job){src, dst, n * t / T, n * (t + 1) / T};
      pthread_create(&th[t], 0, work, &jb[t]);
    }
    for (int t = 0; t < T; ++t) pthread_join(th[t], 0);
    double dt = now() - t0;
    if (rep && dt < best) best = dt;
  }
  printf("%-10s threads %2d: %.1f ms  write %.1f GB/s\n", name, T, best * 1e3, n * 16 / best / 1e9);
}

int main(void) {
  FILE* f = fopen("/sys/kernel/mm/transparent_hugepage/enabled", "r");
  char line[256] = "?";
  if (f) {
    if (!fgets(line, sizeof line, f)) line[0] = 0;
    fclose(f);
  }
  printf("THP: %s", line);
  size_t n = (size_t)16384 * 16384;
  uint32_t* src = alloc(n * 4, 0);
  memset(src, 1, n * 4);
  uint32_t* d4k = alloc(n * 16, MADV_NOHUGEPAGE);
  run("4k-pages", src, d4k, n, 14);
  munmap(d4k, n * 16);
  uint32_t* dhp = alloc(n * 16, MADV_HUGEPAGE);
  run("huge", src, dhp, n, 14);
  munmap(dhp, n * 16);
  return 0;
}
