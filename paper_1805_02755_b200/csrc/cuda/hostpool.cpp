// hostpool.cpp — host-side widening of replicated outputs.
//
// The Mandelbrot kernel writes four identical uint32 counts per work-item
// (the reference's 4:1 out pattern, workloads.hpp:217-222).  Shipping all
// four over PCIe costs 16 B/pixel (4 GiB at the config, ~75 ms at 57 GB/s);
// the device layer instead copies the one count per pixel (2 B/pixel when
// max_iter < 65536, else 4) into
// page-locked staging slots (device.cu ring_setup) and this pool widens
// every piece into the caller's buffer as soon as its copy has landed, with
// non-temporal 128-bit stores on all host cores, overlapped with the
// remaining kernels and copies.  The caller's buffer ends up byte-identical to a full D2H.
#include <cuda_runtime.h>
#include <immintrin.h>

#include <sys/mman.h>

#include <algorithm>
#include <chrono>
#include <cstdlib>
#include <atomic>
#include <condition_variable>
#include <cstdint>
#include <deque>
#include <mutex>
#include <thread>
#include <vector>

#include "hostpool.h"

namespace ecl {
namespace {

struct Job {
  int device;
  cudaEvent_t ready;
  const void* src;
  uint32_t src_bytes;  // 4, or 2 (16-bit compact values)
  uint32_t* dst;
  uint64_t count;
  uint32_t rep;
  WidenTicket* ticket;
  uint32_t* release;
  uint32_t release_value;
};

// 1 -> 4 with one full cache line per streaming store (AVX-512): four
// source values permuted into 16 lanes.  Measured on the GPU box's 16-core
// host (tools/probe/widen_avx512.c, 4 GiB destination): 140.9 vs 129.1 GB/s
// for 16-byte SSE streaming stores at 12 threads, 128 vs 111 at 8.
__attribute__((target("avx512f"))) void widen4_avx512(const uint32_t* src, uint32_t* dst, uint64_t count) {
  uint64_t i = 0;
  // 16-byte stores until the destination is cache-line aligned
  for (; i < count && (reinterpret_cast<uintptr_t>(dst + 4 * i) & 63) != 0; ++i)
    _mm_stream_si128(reinterpret_cast<__m128i*>(dst + 4 * i), _mm_set1_epi32(static_cast<int>(src[i])));
  const __m512i idx = _mm512_set_epi32(3, 3, 3, 3, 2, 2, 2, 2, 1, 1, 1, 1, 0, 0, 0, 0);
  for (; i + 4 <= count; i += 4) {
    const __m512i s = _mm512_castsi128_si512(_mm_loadu_si128(reinterpret_cast<const __m128i*>(src + i)));
    _mm512_stream_si512(reinterpret_cast<__m512i*>(dst + 4 * i), _mm512_permutexvar_epi32(idx, s));
  }
  for (; i < count; ++i)
    _mm_stream_si128(reinterpret_cast<__m128i*>(dst + 4 * i), _mm_set1_epi32(static_cast<int>(src[i])));
  _mm_sfence();
}

// The same from 16-bit values: half the source bytes (the staging copies and
// their reads), the destination stores unchanged.
__attribute__((target("avx512f"))) void widen4_u16_avx512(const uint16_t* src, uint32_t* dst, uint64_t count) {
  uint64_t i = 0;
  for (; i < count && (reinterpret_cast<uintptr_t>(dst + 4 * i) & 63) != 0; ++i)
    _mm_stream_si128(reinterpret_cast<__m128i*>(dst + 4 * i), _mm_set1_epi32(static_cast<int>(src[i])));
  const __m512i idx = _mm512_set_epi32(3, 3, 3, 3, 2, 2, 2, 2, 1, 1, 1, 1, 0, 0, 0, 0);
  for (; i + 4 <= count; i += 4) {
    const __m128i w = _mm_cvtepu16_epi32(_mm_loadl_epi64(reinterpret_cast<const __m128i*>(src + i)));
    _mm512_stream_si512(reinterpret_cast<__m512i*>(dst + 4 * i), _mm512_permutexvar_epi32(idx, _mm512_castsi128_si512(w)));
  }
  for (; i < count; ++i)
    _mm_stream_si128(reinterpret_cast<__m128i*>(dst + 4 * i), _mm_set1_epi32(static_cast<int>(src[i])));
  _mm_sfence();
}

void widen16(const uint16_t* src, uint32_t* dst, uint64_t count, uint32_t rep) {
  if (rep == 4 && (reinterpret_cast<uintptr_t>(dst) & 15) == 0 && __builtin_cpu_supports("avx512f")) {
    widen4_u16_avx512(src, dst, count);
    return;
  }
  for (uint64_t i = 0; i < count; ++i)
    for (uint32_t r = 0; r < rep; ++r) dst[i * rep + r] = src[i];
}

void widen(const uint32_t* src, uint32_t* dst, uint64_t count, uint32_t rep) {
  static const bool avx512 = [] {  // ECL_WIDEN_SSE=1: 16-byte stores only (A/B)
    const char* v = std::getenv("ECL_WIDEN_SSE");
    return __builtin_cpu_supports("avx512f") != 0 && !(v && std::atoi(v) == 1);
  }();
  if (rep == 4 && (reinterpret_cast<uintptr_t>(dst) & 15) == 0) {
    if (avx512) {
      widen4_avx512(src, dst, count);
      return;
    }
    auto* d = reinterpret_cast<__m128i*>(dst);
    for (uint64_t i = 0; i < count; ++i) _mm_stream_si128(d + i, _mm_set1_epi32(static_cast<int>(src[i])));
    _mm_sfence();
    return;
  }
  for (uint64_t i = 0; i < count; ++i)
    for (uint32_t r = 0; r < rep; ++r) dst[i * rep + r] = src[i];
}

class Pool {
 public:
  Pool() {
    // Leave two cores for the engine's device threads and CUDA's own threads:
    // a descheduled widen worker stalls its piece for a whole time slice.
    // Under torchrun (one process per GPU, LOCAL_WORLD_SIZE processes on the
    // host) the cores are shared: each process takes its share after two
    // cores per process for device threads.
    const unsigned hw = std::max(1u, std::thread::hardware_concurrency());
    unsigned lw = 1;
    if (const char* v = std::getenv("LOCAL_WORLD_SIZE"); v && std::atoi(v) > 1) lw = static_cast<unsigned>(std::atoi(v));
    unsigned n = hw > 2 * lw + 2 ? (hw - 2 * lw) / lw : std::max(1u, hw / lw);
    if (const char* v = std::getenv("ECL_WIDEN_THREADS"); v && std::atoi(v) > 0) n = static_cast<unsigned>(std::atoi(v));
    for (unsigned i = 0; i < n; ++i) threads_.emplace_back([this] { loop(); });
  }
  ~Pool() {
    {
      std::lock_guard lock(m_);
      stop_ = true;
    }
    cv_.notify_all();
    for (auto& t : threads_) t.join();
  }
  unsigned size() const { return static_cast<unsigned>(threads_.size()); }

  void submit(const Job& j) {
    // split into ~2 MiB-of-output sub-jobs so every core takes part (ring
    // jobs stay whole: one release per staging slot)
    const uint64_t sub = j.release ? std::max<uint64_t>(1, j.count)
                                   : std::max<uint64_t>(1, (1u << 19) / std::max<uint32_t>(1, j.rep));
    std::vector<Job> parts;
    for (uint64_t o = 0; o < j.count; o += sub) {
      Job p = j;
      p.src = static_cast<const char*>(j.src) + o * j.src_bytes;
      p.dst = j.dst + o * j.rep;
      p.count = std::min(sub, j.count - o);
      parts.push_back(p);
    }
    j.ticket->pending.fetch_add(static_cast<int64_t>(parts.size()));
    {
      std::lock_guard lock(m_);
      for (auto& p : parts) q_.push_back(p);
    }
    cv_.notify_all();
  }

 private:
  void loop() {
    int current_device = -1;
    for (;;) {
      Job j;
      {
        std::unique_lock lock(m_);
        cv_.wait(lock, [&] { return stop_ || !q_.empty(); });
        if (stop_ && q_.empty()) return;
        // Prefer a piece whose copy already landed: pieces of the two compute
        // lanes complete out of submission order, FIFO would idle on the
        // older lane while the other lane's pieces wait.
        auto pick = q_.begin();
        const auto scan_end = q_.size() > 64 ? q_.begin() + 64 : q_.end();
        for (auto it = q_.begin(); it != scan_end; ++it) {
          if (cudaEventQuery(it->ready) == cudaSuccess) {
            pick = it;
            break;
          }
        }
        cudaGetLastError();
        j = *pick;
        q_.erase(pick);
      }
      if (j.device != current_device) {
        cudaSetDevice(j.device);
        current_device = j.device;
      }
      if (cudaEventSynchronize(j.ready) != cudaSuccess) {
        cudaGetLastError();
        j.ticket->failed.store(true);
      } else {
        if (j.src_bytes == 2)
          widen16(static_cast<const uint16_t*>(j.src), j.dst, j.count, j.rep);
        else
          widen(static_cast<const uint32_t*>(j.src), j.dst, j.count, j.rep);
      }
      if (j.release) __atomic_store_n(j.release, j.release_value, __ATOMIC_RELEASE);
      {
        // Decrement under the ticket's lock: widen_wait returns only after
        // taking the same lock, so the ticket (owned by a device slot that
        // ecl_gpu_close frees) outlives this worker's last touch of it.
        std::lock_guard lock(j.ticket->m);
        if (j.ticket->pending.fetch_sub(1) == 1) j.ticket->cv.notify_all();
      }
    }
  }

  std::vector<std::thread> threads_;
  std::mutex m_;
  std::condition_variable cv_;
  std::deque<Job> q_;
  bool stop_ = false;
};

Pool& pool() {
  static Pool p;
  return p;
}

}  // namespace

void widen_async(int device, cudaEvent_t ready, const void* src, uint32_t src_bytes, uint32_t* dst, uint64_t count,
                 uint32_t rep, WidenTicket* ticket, uint32_t* release, uint32_t release_value) {
  pool().submit(Job{device, ready, src, src_bytes == 2 ? 2u : 4u, dst, count, rep, ticket, release, release_value});
}

unsigned widen_workers() { return pool().size(); }

double widen_probe_ms(uint64_t items, uint32_t rep, uint32_t src_bytes) {
  // The pool's own arithmetic and thread count on fresh huge-page buffers,
  // without the CUDA event gating: what host DRAM sustains for widening.
  const unsigned n = std::max(1u, pool().size());
  std::vector<uint32_t> src(items);
  std::vector<uint16_t> src16(src_bytes == 2 ? items : 0);
  for (uint64_t i = 0; i < items; ++i) src[i] = static_cast<uint32_t>(i);
  for (uint64_t i = 0; i < src16.size(); ++i) src16[i] = static_cast<uint16_t>(i);
  // destination on transparent huge pages, like the page-locked output
  // buffers callers hand the engine (device.cu pinned_alloc)
  const size_t huge = size_t{2} << 20;
  const size_t len = (items * rep * sizeof(uint32_t) + huge - 1) / huge * huge;
  void* raw = mmap(nullptr, len, PROT_READ | PROT_WRITE, MAP_PRIVATE | MAP_ANONYMOUS, -1, 0);
  if (raw == MAP_FAILED) return -1.0;
  madvise(raw, len, MADV_HUGEPAGE);
  auto* dst = static_cast<uint32_t*>(raw);
  auto pass = [&] {
    std::vector<std::thread> ts;
    const uint64_t per = (items + n - 1) / n;
    for (unsigned t = 0; t < n; ++t) {
      const uint64_t a = std::min<uint64_t>(items, t * per), b = std::min<uint64_t>(items, a + per);
      ts.emplace_back([&, a, b] {
        if (src_bytes == 2)
          widen16(src16.data() + a, dst + a * rep, b - a, rep);
        else
          widen(src.data() + a, dst + a * rep, b - a, rep);
      });
    }
    for (auto& t : ts) t.join();
  };
  pass();  // first touch of the destination pages
  const auto t0 = std::chrono::steady_clock::now();
  pass();
  const double ms = std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now() - t0).count();
  munmap(raw, len);
  return ms;
}

bool widen_wait(WidenTicket* ticket) {
  std::unique_lock lock(ticket->m);  // always: see the worker's decrement
  ticket->cv.wait(lock, [&] { return ticket->pending.load() == 0; });
  return !ticket->failed.load();
}

}  // namespace ecl
