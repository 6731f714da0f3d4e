// Host-side 4:1 widening of a 1 GiB compact D2H stream into a 4 GiB host
// buffer, two ways:
//   full  — the device layer's current scheme: the compact copy lands in a
//           1 GiB page-locked buffer, widen workers read it back from DRAM;
//   ring  — the copy lands in a small page-locked ring (R slots of S bytes)
//           that stays in the last-level cache (DMA writes allocate in LLC
//           when the platform does that), widen workers read it from cache
//           and free the slot for the next copy.
// Prints the wall time of each (data already on the device, no kernel).
// Build: nvcc -O3 -std=c++17 -gencode arch=compute_100a,code=sm_100a ring_widen.cu -o ring_widen -lpthread
#include <cuda_runtime.h>
#include <emmintrin.h>
#include <sys/mman.h>

#include <algorithm>
#include <atomic>
#include <chrono>
#include <cstdint>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <thread>
#include <vector>

#define CK(x)                                                              \
  do {                                                                     \
    cudaError_t e_ = (x);                                                  \
    if (e_ != cudaSuccess) {                                               \
      fprintf(stderr, "%s:%d %s\n", __FILE__, __LINE__, cudaGetErrorString(e_)); \
      exit(1);                                                             \
    }                                                                      \
  } while (0)

static void widen(const uint32_t* src, uint32_t* dst, uint64_t n) {
  auto* d = reinterpret_cast<__m128i*>(dst);
  for (uint64_t i = 0; i < n; ++i) _mm_stream_si128(d + i, _mm_set1_epi32(static_cast<int>(src[i])));
  _mm_sfence();
}

static double now_ms() {
  return std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now().time_since_epoch()).count();
}

static void* big_alloc(size_t bytes) {
  void* p = mmap(nullptr, bytes, PROT_READ | PROT_WRITE, MAP_PRIVATE | MAP_ANONYMOUS, -1, 0);
  madvise(p, bytes, MADV_HUGEPAGE);
  memset(p, 0, bytes);
  return p;
}

__global__ void fill(uint32_t* d, uint64_t n) {
  for (uint64_t i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x)
    d[i] = static_cast<uint32_t>(i * 2654435761u);
}

constexpr uint64_t kItems = 1ull << 28;  // 1 GiB of uint32

// Current scheme: chunked copies into a 1 GiB landing zone, T workers widen
// sub-chunks once their copy's event completed.
static double run_full(const uint32_t* dev, uint32_t* land, uint32_t* out, uint64_t chunk, int T) {
  const uint64_t nchunks = kItems / chunk;
  std::vector<cudaEvent_t> ev(nchunks);
  for (auto& e : ev) CK(cudaEventCreateWithFlags(&e, cudaEventDisableTiming));
  cudaStream_t s[2];
  for (auto& x : s) CK(cudaStreamCreateWithFlags(&x, cudaStreamNonBlocking));
  std::atomic<uint64_t> next{0};
  const uint64_t sub = 1 << 17;  // items per widen task (512 KiB compact)
  const uint64_t per = chunk / sub;
  const double t0 = now_ms();
  for (uint64_t c = 0; c < nchunks; ++c) {
    CK(cudaMemcpyAsync(land + c * chunk, dev + c * chunk, chunk * 4, cudaMemcpyDeviceToHost, s[c & 1]));
    CK(cudaEventRecord(ev[c], s[c & 1]));
  }
  std::vector<std::thread> th;
  for (int t = 0; t < T; ++t)
    th.emplace_back([&] {
      for (;;) {
        const uint64_t k = next.fetch_add(1);
        if (k >= nchunks * per) return;
        const uint64_t c = k / per;
        cudaEventSynchronize(ev[c]);
        const uint64_t o = k * sub;
        widen(land + o, out + 4 * o, sub);
      }
    });
  for (auto& x : th) x.join();
  const double t = now_ms() - t0;
  for (auto& e : ev) cudaEventDestroy(e);
  for (auto& x : s) cudaStreamDestroy(x);
  return t;
}

// Ring scheme: R slots of S items; a copy thread issues slot copies as slots
// free up, T workers widen landed slots and release them.
static double run_ring(const uint32_t* dev, uint32_t* ring, uint32_t* out, uint64_t S, int R, int T) {
  const uint64_t nchunks = kItems / S;
  std::vector<cudaEvent_t> ev(R);
  for (auto& e : ev) CK(cudaEventCreateWithFlags(&e, cudaEventDisableTiming | cudaEventBlockingSync));
  std::vector<std::atomic<int64_t>> slot_chunk(R);   // chunk landed/landing in slot, -1 = free
  std::vector<std::atomic<int64_t>> issued(R);       // chunk whose copy was issued into the slot
  for (int r = 0; r < R; ++r) {
    slot_chunk[r].store(-1);
    issued[r].store(-1);
  }
  cudaStream_t s[2];
  for (auto& x : s) CK(cudaStreamCreateWithFlags(&x, cudaStreamNonBlocking));
  std::atomic<uint64_t> next{0};
  const double t0 = now_ms();
  std::thread copier([&] {
    for (uint64_t c = 0; c < nchunks; ++c) {
      const int r = static_cast<int>(c % R);
      while (slot_chunk[r].load(std::memory_order_acquire) != -1) _mm_pause();  // slot still being widened
      slot_chunk[r].store(static_cast<int64_t>(c), std::memory_order_relaxed);
      CK(cudaMemcpyAsync(ring + r * S, dev + c * S, S * 4, cudaMemcpyDeviceToHost, s[c & 1]));
      CK(cudaEventRecord(ev[r], s[c & 1]));
      issued[r].store(static_cast<int64_t>(c), std::memory_order_release);
    }
  });
  std::vector<std::thread> th;
  for (int t = 0; t < T; ++t)
    th.emplace_back([&] {
      for (;;) {
        const uint64_t c = next.fetch_add(1);
        if (c >= nchunks) return;
        const int r = static_cast<int>(c % R);
        while (issued[r].load(std::memory_order_acquire) != static_cast<int64_t>(c)) _mm_pause();
        cudaEventSynchronize(ev[r]);
        widen(ring + r * S, out + 4 * c * S, S);
        slot_chunk[r].store(-1, std::memory_order_release);
      }
    });
  copier.join();
  for (auto& x : th) x.join();
  const double t = now_ms() - t0;
  for (auto& e : ev) cudaEventDestroy(e);
  for (auto& x : s) cudaStreamDestroy(x);
  return t;
}

static bool check(const uint32_t* out) {
  for (uint64_t i = 0; i < kItems; i += 4099) {
    const uint32_t v = static_cast<uint32_t>(i * 2654435761u);
    for (int r = 0; r < 4; ++r)
      if (out[4 * i + r] != v) return false;
  }
  return true;
}

int main(int argc, char** argv) {
  const int T = argc > 1 ? atoi(argv[1]) : 14;
  uint32_t* dev;
  CK(cudaMalloc(&dev, kItems * 4));
  fill<<<1184, 256>>>(dev, kItems);
  CK(cudaDeviceSynchronize());
  auto* out = static_cast<uint32_t*>(big_alloc(kItems * 16));
  auto* land = static_cast<uint32_t*>(big_alloc(kItems * 4));
  CK(cudaHostRegister(land, kItems * 4, cudaHostRegisterDefault));
  void* ringp;
  CK(cudaHostAlloc(&ringp, 64u << 20, cudaHostAllocDefault));
  auto* ring = static_cast<uint32_t*>(ringp);

  // pure D2H of 1 GiB
  {
    cudaEvent_t a, b;
    cudaEventCreate(&a);
    cudaEventCreate(&b);
    cudaEventRecord(a);
    CK(cudaMemcpyAsync(land, dev, kItems * 4, cudaMemcpyDeviceToHost));
    cudaEventRecord(b);
    cudaEventSynchronize(b);
    float ms;
    cudaEventElapsedTime(&ms, a, b);
    printf("d2h 1 GiB: %.2f ms (%.1f GB/s)\n", ms, kItems * 4 / ms / 1e6);
  }
  for (int rep = 0; rep < 2; ++rep) {
    for (uint64_t chunk : {1ull << 22}) {
      memset(out, 0, 64);
      const double t = run_full(dev, land, out, chunk, T);
      printf("full  chunk %5llu KiB T=%d: %.2f ms  ok=%d\n", (unsigned long long)(chunk * 4 >> 10), T, t, check(out));
    }
    for (auto [S, R] : std::vector<std::pair<uint64_t, int>>{{1 << 18, 32}, {1 << 18, 48}, {1 << 18, 64}, {1 << 19, 16}, {1 << 19, 24},
                                                             {1 << 19, 32}, {1 << 20, 8}, {1 << 20, 16}, {1 << 17, 96},
                                                             {1 << 17, 128}}) {
      memset(out, 0, 64);
      const double t = run_ring(dev, ring, out, S, R, T);
      printf("ring  slot %4llu KiB x %3d (%5.1f MiB) T=%d: %.2f ms  ok=%d\n", (unsigned long long)(S * 4 >> 10), R,
             S * 4.0 * R / (1 << 20), T, t, check(out));
    }
  }
  return 0;
}
