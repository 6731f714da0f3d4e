// hostpool.h — host thread pool that widens replicated outputs (see hostpool.cpp).
#pragma once

#include <cuda_runtime.h>

#include <atomic>
#include <condition_variable>
#include <cstdint>
#include <mutex>

namespace ecl {

// Outstanding widen jobs of one package.
struct WidenTicket {
  std::atomic<int64_t> pending{0};
  std::atomic<bool> failed{false};
  std::mutex m;
  std::condition_variable cv;
};

// After `ready` completes, writes `rep` copies of src[i] to dst[i*rep .. +rep)
// for i < count, on the pool's threads; src holds `src_bytes`-byte unsigned
// values (4, or 2 when every value fits 16 bits), zero-extended to uint32.  With `release`, the job runs as one
// piece and then stores `release_value` to *release (a page-locked word a
// copy stream waits on before it reuses src: the staging ring of
// device.cu) — also when the copy failed, so a waiting stream never hangs.
void widen_async(int device, cudaEvent_t ready, const void* src, uint32_t src_bytes, uint32_t* dst, uint64_t count,
                 uint32_t rep, WidenTicket* ticket, uint32_t* release = nullptr, uint32_t release_value = 0);

// Number of widen worker threads.
unsigned widen_workers();

// Milliseconds the pool's threads take to widen `items` values `rep`-fold
// between host buffers (second pass, pages already touched): the host-DRAM
// floor of an end-to-end run whose outputs are widened.
double widen_probe_ms(uint64_t items, uint32_t rep, uint32_t src_bytes = 4);

// Blocks until every job of the ticket finished; false if a copy failed.
bool widen_wait(WidenTicket* ticket);

}  // namespace ecl
