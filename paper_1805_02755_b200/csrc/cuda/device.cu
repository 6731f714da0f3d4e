// device.cu — the B200 device layer behind include/ecl_cuda.h.
//
// Replaces NativePool (engine.hpp:97-200): where the reference wakes W host
// threads, splits the package contiguously and waits on a condition variable
// (engine.hpp:120-136), a package here is one kernel launch bracketed by two
// timing events on one of the device's compute lanes (streams).
//
// Streams per device:
//   lane[0], lane[1]  compute.  Consecutive packages alternate lanes (queue
//                     depth >= 2), so package k+1's CTAs fill the SMs that
//                     package k's drain tail leaves idle; each lane has its
//                     own work-claim counters.  Depth 1 uses lane[0] only,
//                     the reference's strictly serial device.
//   copy[0], copy[1]  D2H of every package's out_range_for slice (one copy
//                     stream per lane, so one lane's copies never queue
//                     behind the other lane's kernels), waiting on the
//                     kernel (piece) events: copies overlap later kernels.
//                     Replicated outputs (Mandelbrot's 4 identical counts)
//                     copy one value per item and are widened by host
//                     threads (hostpool.cpp).
//   notify            completion callbacks, after the copies; kept off the
//                     copy stream so a host callback never stalls a DMA.
#include <cuda_runtime.h>

#include <sys/mman.h>

#include <algorithm>
#include <atomic>
#include <chrono>
#include <cstdlib>
#include <cstring>
#include <mutex>
#include <string>
#include <unordered_map>
#include <vector>

#include "ecl_cuda.h"
#include "hostpool.h"
#include "kernels.cuh"

struct ecl_kernel {
  ecl::KernelSpec spec;
};

namespace {

thread_local std::string t_error;

int fail(int code, const std::string& msg) {
  t_error = msg;
  return code;
}

int cuda_fail(cudaError_t e, const char* what) {
  t_error = std::string(what) + ": " + cudaGetErrorName(e) + " (" + cudaGetErrorString(e) + ")";
  return ECL_KERNEL_PANIC;
}

#define ECL_CK(call)                                    \
  do {                                                  \
    cudaError_t e_ = (call);                            \
    if (e_ != cudaSuccess) return cuda_fail(e_, #call); \
  } while (0)

constexpr uint32_t kSlots = 64;  // timing-event ring; >= 2 x max queue depth
constexpr int kLanes = 2;
constexpr size_t kCtrlWordsPerLane = 16;

struct Slot {
  cudaEvent_t start = nullptr;  // kernel start (first lane of the package)
  cudaEvent_t end = nullptr;    // kernel end (first lane)
  cudaEvent_t start2 = nullptr;  // pieces also ran on the other lane: its start / end
  cudaEvent_t end2 = nullptr;
  bool two_lanes = false;
  cudaEvent_t done = nullptr;   // copies + callback finished (notify stream)
  uint64_t seq = ~0ull;
  bool busy = false;
  bool timed = false;
  ecl_done_fn fn = nullptr;
  void* user = nullptr;
  ecl::WidenTicket widen;               // host widening of this package's copies
  std::vector<cudaEvent_t> piece_done;  // per-piece D2H completion (widen triggers)
};

void CUDART_CB on_package_done(void* arg) {
  Slot* s = static_cast<Slot*>(arg);
  if (s->fn) s->fn(s->user, s->seq, ECL_OK);
}

}  // namespace

struct ecl_gpu {
  int ordinal = 0;
  int sms = 0;
  uint32_t depth = 2;
  int lanes = 1;
  cudaStream_t lane[kLanes] = {nullptr, nullptr};
  cudaStream_t copy[kLanes] = {nullptr, nullptr};  // per lane: one lane's copies never queue behind the other's
  cudaStream_t notify = nullptr;
  cudaEvent_t epoch = nullptr;             // anchor event: device time <-> host steady clock
  cudaEvent_t ready = nullptr;             // last input/replication write on lane 0
  cudaEvent_t piece[kLanes] = {nullptr, nullptr};  // end of a sub-launch the copy stream drains
  cudaEvent_t copied[kLanes] = {nullptr, nullptr};  // copies of a lane's latest package
  double epoch_host_ms = -1.0;  // steady-clock ms of the anchor event; < 0 = not anchored
  Slot slots[kSlots];
  uint32_t next_slot = 0;  // per-device rotation: seqs are global across devices
  uint32_t next_lane = 0;
  const ecl::KernelSpec* spec = nullptr;
  std::vector<void*> in, out;
  std::vector<uint64_t> in_bytes, out_bytes;
  unsigned* ctrl = nullptr;  // kLanes x kCtrlWordsPerLane words
  void* scratch = nullptr;
  uint64_t scratch_cap = 0;
  uint32_t* tally = nullptr;
  uint64_t tally_items = 0;
  bool tally_on = false;
  double kernel_ms = 0.0;
  uint64_t launches = 0;
  std::vector<void*> peer_out;  // fused exchange: n_peers x outputs (ecl_gpu_set_peer_outputs)
  uint32_t n_peers = 0;
  uint64_t d2h_split_items = 1ull << 23;  // sub-launch size when copies are pipelined
  uint32_t* compact_dev = nullptr;        // replicate > 1: one value per work-item (device)
  uint32_t* compact_host = nullptr;       // page-locked landing zone of the compact copies
  uint64_t compact_items = 0;
  uint32_t widen_per_8 = 8;               // pieces (of 8) copied compact and widened on the host
  uint64_t widen_chunk_items = [] {       // compact D2H granularity (ECL_WIDEN_CHUNK, items)
    const char* v = std::getenv("ECL_WIDEN_CHUNK");
    const long long n = v ? std::atoll(v) : 0;
    return n > 0 ? static_cast<uint64_t>(n) : ~uint64_t{0};
  }();
  uint64_t piece_counter = 0;
  // Staging ring for the compact copies (ring_setup): instead of
  // a gws-sized landing zone, copies land in R page-locked slots of S items
  // that the widen workers release; a copy stream waits (cuStreamWaitValue32
  // on the slot's release counter) before it reuses a slot.
  uint32_t* ring = nullptr;           // R x S items, page-locked
  uint32_t* ring_released = nullptr;  // R counters, page-locked + mapped (widen workers bump them)
  void* ring_released_dev = nullptr;  // device address of ring_released
  std::vector<uint32_t> ring_uses;    // copies issued per slot
  uint32_t ring_slots = 0, ring_next = 0;
  bool ring_tried = false;
  uint64_t ring_items = 0;
  // Host mirrors of small inputs a launcher passes in its parameters
  // (ecl::host_mirrored_input: Gaussian's filter); empty for other inputs.
  std::vector<std::vector<char>> in_host;
  std::vector<const void*> in_host_ptr;  // LaunchEnv::in_host (nullptr: not mirrored)
  std::vector<bool> in_host_valid;       // false: the device copy changed on the device (swap_io)
  // Streamed inputs (ecl_gpu_set_streamed_inputs): uploads are enqueued on
  // `h2d` piece by piece, each piece's kernel waiting for the prefix it reads.
  bool streamed = false;
  cudaStream_t h2d = nullptr;
  cudaEvent_t up_ev = nullptr;         // after the latest streamed upload
  bool up_live = false;                // up_ev recorded in this run
  std::vector<const char*> pending_in;  // host source still streaming (nullptr: complete/resident)
  std::vector<uint64_t> up_bytes;       // bytes of each input already enqueued
};

namespace {

// Page-locked host memory on transparent huge pages: mmap + MADV_HUGEPAGE +
// cudaHostRegister.  The host widening streams 4 GiB per Mandelbrot step
// through such buffers; 2 MiB pages measured 126 vs 119 GB/s for 4 KiB
// pages (tools/probe/hostbw_thp.c).  Falls back to cudaHostAlloc.
std::mutex g_pinned_m;
std::unordered_map<void*, size_t> g_pinned;  // mmap'ed blocks -> bytes

cudaError_t pinned_alloc(void** ptr, size_t bytes) {
  *ptr = nullptr;
  const size_t huge = size_t{2} << 20;
  const size_t len = (bytes + huge - 1) / huge * huge;
  void* p = mmap(nullptr, len, PROT_READ | PROT_WRITE, MAP_PRIVATE | MAP_ANONYMOUS, -1, 0);
  if (p != MAP_FAILED) {
    madvise(p, len, MADV_HUGEPAGE);
    if (cudaHostRegister(p, len, cudaHostRegisterPortable) == cudaSuccess) {
      std::lock_guard lock(g_pinned_m);
      g_pinned[p] = len;
      *ptr = p;
      return cudaSuccess;
    }
    cudaGetLastError();
    munmap(p, len);
  }
  return cudaHostAlloc(ptr, bytes, cudaHostAllocPortable);
}

cudaError_t pinned_free(void* p) {
  if (!p) return cudaSuccess;
  size_t len = 0;
  {
    std::lock_guard lock(g_pinned_m);
    auto it = g_pinned.find(p);
    if (it != g_pinned.end()) {
      len = it->second;
      g_pinned.erase(it);
    }
  }
  if (!len) return cudaFreeHost(p);
  const cudaError_t e = cudaHostUnregister(p);
  munmap(p, len);
  return e;
}

// cuStreamWaitValue32 through the runtime's driver entry point (no libcuda
// link).  Returns nullptr when the driver does not offer it.
using WaitValueFn = int (*)(cudaStream_t, unsigned long long, uint32_t, unsigned);
WaitValueFn wait_value_fn() {
  static WaitValueFn fn = [] {
    void* p = nullptr;
    cudaDriverEntryPointQueryResult q{};
    if (cudaGetDriverEntryPoint("cuStreamWaitValue32", &p, cudaEnableDefault, &q) != cudaSuccess ||
        q != cudaDriverEntryPointSuccess) {
      cudaGetLastError();
      return static_cast<WaitValueFn>(nullptr);
    }
    return reinterpret_cast<WaitValueFn>(p);
  }();
  return fn;
}

// Sets up the staging ring once per device.  Slots of ECL_WIDEN_RING_SLOT_KB
// (2 MiB); ECL_WIDEN_RING_SLOTS sets their number, 0 turns the ring off
// (gws-sized landing zone), unset = two slots per widen worker plus four for
// copies in flight.  It pins 64 MiB instead of gws x 4 bytes (1 GiB at the
// Mandelbrot config, per device) and keeps the copies' landing data in the
// host's last-level cache.  Measured (1 B200, 16-core host, Mandelbrot
// 16384^2 e2e, three alternating runs): 32 slots 49.6-50.1 ms against
// 50.5-50.7 ms for the landing zone; one box gave 46.8 vs 49.3.  A ring with
// barely more slots than workers starves the copies (16 slots: 89 ms), hence
// the auto size.  The ring stays off when the driver lacks stream memory
// operations.
cudaError_t ring_setup(ecl_gpu* g) {
  static const long long ring_slots = [] {
    const char* v = std::getenv("ECL_WIDEN_RING_SLOTS");
    return v ? std::atoll(v) : -1ll;
  }();
  static const uint64_t slot_kb = [] {
    const char* v = std::getenv("ECL_WIDEN_RING_SLOT_KB");
    const long long n = v ? std::atoll(v) : 2048;
    return n > 0 ? static_cast<uint64_t>(n) : uint64_t{2048};
  }();
  if (g->ring || g->ring_tried || ring_slots == 0 || !wait_value_fn()) return cudaSuccess;
  g->ring_tried = true;  // one attempt per device: a refusal keeps the landing zone
  const uint64_t items = slot_kb * 1024 / 4;
  const uint64_t auto_slots = 2ull * ecl::widen_workers() + 4;
  const uint32_t slots =
      static_cast<uint32_t>(ring_slots < 0 ? auto_slots : std::max<long long>(1, ring_slots));
  void* p = nullptr;
  cudaError_t e = pinned_alloc(&p, slots * items * 4);
  if (e != cudaSuccess) return e;
  void* f = nullptr;
  e = cudaHostAlloc(&f, slots * sizeof(uint32_t), cudaHostAllocMapped | cudaHostAllocPortable);
  if (e != cudaSuccess) {
    pinned_free(p);
    return e;
  }
  std::memset(f, 0, slots * sizeof(uint32_t));
  void* fd = nullptr;
  e = cudaHostGetDevicePointer(&fd, f, 0);
  if (e != cudaSuccess) {
    pinned_free(p);
    cudaFreeHost(f);
    return e;
  }
  // Drivers can refuse stream memory operations (module option): probe with
  // a wait that is already satisfied and keep the landing zone if refused.
  if (wait_value_fn()(g->copy[0], reinterpret_cast<unsigned long long>(fd), 0, 0 /* GEQ */) != 0) {
    cudaGetLastError();
    pinned_free(p);
    cudaFreeHost(f);
    return cudaSuccess;
  }
  g->ring = static_cast<uint32_t*>(p);
  g->ring_released = static_cast<uint32_t*>(f);
  g->ring_released_dev = fd;
  g->ring_uses.assign(slots, 0);
  g->ring_slots = slots;
  g->ring_items = items;
  g->ring_next = 0;
  return cudaSuccess;
}

Slot* find_slot(ecl_gpu* g, uint64_t seq) {
  for (auto& s : g->slots)
    if (s.busy && s.seq == seq) return &s;
  return nullptr;
}

int set_device(const ecl_gpu* g) {
  ECL_CK(cudaSetDevice(g->ordinal));
  return ECL_OK;
}

ecl::LaunchEnv env_of(const ecl_gpu* g, int lane) {
  ecl::LaunchEnv env;
  env.stream = g->lane[lane];
  env.sms = g->sms;
  env.in = g->in.data();
  env.out = g->out.data();
  env.ctrl = g->ctrl + lane * kCtrlWordsPerLane;
  env.scratch = g->scratch;
  env.device = g->ordinal;
  env.in_host = g->in_host_ptr.data();
  env.extra_launches = const_cast<uint64_t*>(&g->launches);  // g itself is never a const object
  if (g->n_peers) {
    env.peer_out = g->peer_out.data();
    env.n_peers = g->n_peers;
  }
  return env;
}

// Makes every lane of g wait for the work queued so far on lane 0.
int fan_out_lane0(ecl_gpu* g) {
  ECL_CK(cudaEventRecord(g->ready, g->lane[0]));
  for (int l = 1; l < g->lanes; ++l) ECL_CK(cudaStreamWaitEvent(g->lane[l], g->ready, 0));
  return ECL_OK;
}

// Makes lane 0 wait for everything queued on the other lanes.
int join_lanes(ecl_gpu* g) {
  for (int l = 1; l < g->lanes; ++l) {
    ECL_CK(cudaEventRecord(g->piece[l], g->lane[l]));
    ECL_CK(cudaStreamWaitEvent(g->lane[0], g->piece[l], 0));
  }
  return ECL_OK;
}

// Host mirrors (in_host): refreshed from the caller's bytes on every upload
// path; a mirror whose device copy changed on the device (swap_io) is read
// back before the next launch.
void mirror_write(ecl_gpu* g, size_t i, uint64_t offset, const void* src, uint64_t bytes) {
  if (i >= g->in_host.size() || g->in_host[i].empty()) return;
  std::memcpy(g->in_host[i].data() + offset, src, bytes);
}

int sync_all(ecl_gpu* g);

int ensure_mirrors(ecl_gpu* g) {
  for (size_t i = 0; i < g->in_host.size(); ++i) {
    if (g->in_host[i].empty() || g->in_host_valid[i]) continue;
    if (int rc = sync_all(g)) return rc;
    ECL_CK(cudaMemcpy(g->in_host[i].data(), g->in[i], g->in_host[i].size(), cudaMemcpyDeviceToHost));
    g->in_host_valid[i] = true;
  }
  return ECL_OK;
}

// Enqueues the rest of every streamed input (nothing left pending).
int flush_streamed(ecl_gpu* g) {
  for (size_t i = 0; i < g->pending_in.size(); ++i) {
    if (!g->pending_in[i]) continue;
    const uint64_t up = g->up_bytes[i];
    if (g->in_bytes[i] > up)
      ECL_CK(cudaMemcpyAsync(static_cast<char*>(g->in[i]) + up, g->pending_in[i] + up, g->in_bytes[i] - up,
                             cudaMemcpyHostToDevice, g->h2d));
    g->up_bytes[i] = g->in_bytes[i];
    g->pending_in[i] = nullptr;
  }
  return ECL_OK;
}

int sync_all(ecl_gpu* g) {
  if (int rc = flush_streamed(g)) return rc;
  ECL_CK(cudaStreamSynchronize(g->h2d));
  g->up_live = false;
  for (int l = 0; l < g->lanes; ++l) {
    ECL_CK(cudaStreamSynchronize(g->lane[l]));
    ECL_CK(cudaStreamSynchronize(g->copy[l]));
  }
  ECL_CK(cudaStreamSynchronize(g->notify));
  bool ok = true;
  for (auto& s : g->slots) ok = ecl::widen_wait(&s.widen) && ok;  // host widening of the copies
  return ok ? ECL_OK : fail(ECL_KERNEL_PANIC, "host widening: a copy failed");
}

// out_range_for (core.hpp:172-185): the package's output-element range.
int out_range(const ecl::KernelSpec& s, uint64_t offset_wg, uint64_t size_wg, uint64_t* off, uint64_t* cnt) {
  const uint64_t items = size_wg * s.lws, first = offset_wg * s.lws;
  if ((items * s.out_indices) % s.out_work_items != 0 || (first * s.out_indices) % s.out_work_items != 0)
    return fail(ECL_INDIVISIBLE_PACKAGE, "package of " + std::to_string(items) + " work-items at offset " +
                                             std::to_string(first) + " is not divisible by out pattern " +
                                             std::to_string(s.out_indices) + ":" + std::to_string(s.out_work_items));
  *off = first * s.out_indices / s.out_work_items;
  *cnt = items * s.out_indices / s.out_work_items;
  return ECL_OK;
}

void free_buffers(ecl_gpu* g) {
  for (void* p : g->in) cudaFree(p);
  for (void* p : g->out) cudaFree(p);
  g->in.clear();
  g->out.clear();
  g->in_bytes.clear();
  g->out_bytes.clear();
}

// Peer access state per (dst, src) ordinal pair: 0 unknown, 1 enabled (dst
// reads/writes src's memory over NVLink), 2 not possible (copies then stage
// through the host).
std::mutex g_peer_m;
int g_peer[64][64] = {};

void enable_peer(int dst, int src) {
  if (dst == src) return;
  std::lock_guard lock(g_peer_m);
  if (g_peer[dst & 63][src & 63] != 0) return;
  cudaSetDevice(dst);
  int can = 0;
  cudaDeviceCanAccessPeer(&can, dst, src);
  cudaError_t e = cudaErrorPeerAccessUnsupported;
  if (can) e = cudaDeviceEnablePeerAccess(src, 0);
  g_peer[dst & 63][src & 63] = (e == cudaSuccess || e == cudaErrorPeerAccessAlreadyEnabled) ? 1 : 2;
  cudaGetLastError();
}

// ECL_FORCE_PEER_COPY=1: owner-slice copies between logical devices on ONE
// ordinal also go through cudaMemcpyPeerAsync (the multi-GPU call path),
// so a one-GPU box exercises it.
bool force_peer_copy() {
  static const bool on = [] {
    const char* v = std::getenv("ECL_FORCE_PEER_COPY");
    return v && std::string(v) == "1";
  }();
  return on;
}

}  // namespace

extern "C" {

const char* ecl_last_error(void) { return t_error.c_str(); }

int ecl_gpu_count(int* count) {
  *count = 0;
  cudaError_t e = cudaGetDeviceCount(count);
  if (e != cudaSuccess) {
    *count = 0;
    cudaGetLastError();
    return fail(ECL_CONFIG_ERROR, std::string("CUDA unavailable: ") + cudaGetErrorString(e));
  }
  return ECL_OK;
}

int ecl_gpu_open(int ordinal, uint32_t queue_depth, ecl_gpu** out) {
  *out = nullptr;
  int n = 0;
  if (ecl_gpu_count(&n) != ECL_OK) return ECL_CONFIG_ERROR;
  if (ordinal < 0 || ordinal >= n)
    return fail(ECL_CONFIG_ERROR, "CUDA device ordinal " + std::to_string(ordinal) + " out of range (" +
                                      std::to_string(n) + " visible)");
  if (queue_depth < 1 || queue_depth > kSlots / 2)
    return fail(ECL_CONFIG_ERROR, "queue_depth must lie in [1, " + std::to_string(kSlots / 2) + "]");
  auto* g = new ecl_gpu;
  g->ordinal = ordinal;
  g->depth = queue_depth;
  g->lanes = queue_depth >= 2 ? kLanes : 1;
  auto undo = [&](int rc) {
    ecl_gpu_close(g);
    return rc;
  };
  if (int rc = set_device(g)) return undo(rc);
  cudaError_t e = cudaDeviceGetAttribute(&g->sms, cudaDevAttrMultiProcessorCount, ordinal);
  if (e != cudaSuccess) return undo(cuda_fail(e, "cudaDeviceGetAttribute"));
  for (int l = 0; l < kLanes; ++l) {
    if ((e = cudaStreamCreateWithFlags(&g->lane[l], cudaStreamNonBlocking)) != cudaSuccess)
      return undo(cuda_fail(e, "cudaStreamCreate(lane)"));
    if ((e = cudaStreamCreateWithFlags(&g->copy[l], cudaStreamNonBlocking)) != cudaSuccess)
      return undo(cuda_fail(e, "cudaStreamCreate(copy)"));
  }
  if ((e = cudaStreamCreateWithFlags(&g->notify, cudaStreamNonBlocking)) != cudaSuccess)
    return undo(cuda_fail(e, "cudaStreamCreate(notify)"));
  if ((e = cudaStreamCreateWithFlags(&g->h2d, cudaStreamNonBlocking)) != cudaSuccess)
    return undo(cuda_fail(e, "cudaStreamCreate(h2d)"));
  if ((e = cudaEventCreate(&g->epoch)) != cudaSuccess) return undo(cuda_fail(e, "cudaEventCreate"));
  for (cudaEvent_t* ev : {&g->ready, &g->piece[0], &g->piece[1], &g->copied[0], &g->copied[1], &g->up_ev})
    if ((e = cudaEventCreateWithFlags(ev, cudaEventDisableTiming)) != cudaSuccess)
      return undo(cuda_fail(e, "cudaEventCreate"));
  for (auto& s : g->slots) {
    if ((e = cudaEventCreate(&s.start)) != cudaSuccess || (e = cudaEventCreate(&s.end)) != cudaSuccess ||
        (e = cudaEventCreate(&s.start2)) != cudaSuccess || (e = cudaEventCreate(&s.end2)) != cudaSuccess ||
        (e = cudaEventCreateWithFlags(&s.done, cudaEventDisableTiming)) != cudaSuccess)
      return undo(cuda_fail(e, "cudaEventCreate(slot)"));
  }
  const size_t ctrl_bytes = kLanes * kCtrlWordsPerLane * sizeof(unsigned);
  if ((e = cudaMalloc(&g->ctrl, ctrl_bytes)) != cudaSuccess) return undo(cuda_fail(e, "cudaMalloc(ctrl)"));
  if ((e = cudaMemset(g->ctrl, 0, ctrl_bytes)) != cudaSuccess) return undo(cuda_fail(e, "cudaMemset(ctrl)"));
  *out = g;
  return ECL_OK;
}

int ecl_gpu_close(ecl_gpu* g) {
  if (!g) return ECL_OK;
  cudaSetDevice(g->ordinal);
  for (int l = 0; l < kLanes; ++l) {
    if (g->lane[l]) cudaStreamSynchronize(g->lane[l]);
    if (g->copy[l]) cudaStreamSynchronize(g->copy[l]);
  }
  if (g->notify) cudaStreamSynchronize(g->notify);
  if (g->h2d) cudaStreamSynchronize(g->h2d);
  for (auto& s : g->slots) ecl::widen_wait(&s.widen);
  free_buffers(g);
  if (g->scratch) cudaFree(g->scratch);
  if (g->ctrl) cudaFree(g->ctrl);
  if (g->tally) cudaFree(g->tally);
  if (g->compact_dev) cudaFree(g->compact_dev);
  if (g->compact_host) pinned_free(g->compact_host);
  if (g->ring) pinned_free(g->ring);
  if (g->ring_released) cudaFreeHost(g->ring_released);
  for (auto& s : g->slots) {
    if (s.start) cudaEventDestroy(s.start);
    if (s.end) cudaEventDestroy(s.end);
    if (s.start2) cudaEventDestroy(s.start2);
    if (s.end2) cudaEventDestroy(s.end2);
    if (s.done) cudaEventDestroy(s.done);
    for (cudaEvent_t ev : s.piece_done) cudaEventDestroy(ev);
  }
  for (cudaEvent_t ev : {g->epoch, g->ready, g->piece[0], g->piece[1], g->copied[0], g->copied[1], g->up_ev})
    if (ev) cudaEventDestroy(ev);
  if (g->h2d) cudaStreamDestroy(g->h2d);
  for (int l = 0; l < kLanes; ++l) {
    if (g->lane[l]) cudaStreamDestroy(g->lane[l]);
    if (g->copy[l]) cudaStreamDestroy(g->copy[l]);
  }
  if (g->notify) cudaStreamDestroy(g->notify);
  delete g;
  cudaGetLastError();
  return ECL_OK;
}

int ecl_gpu_sm_count(const ecl_gpu* g, int* sms) {
  *sms = g->sms;
  return ECL_OK;
}

int ecl_gpu_ordinal(const ecl_gpu* g, int* ordinal) {
  *ordinal = g->ordinal;
  return ECL_OK;
}

int ecl_kernel_create(const char* kernel_id, uint64_t gws, uint64_t lws, const ecl_arg* args, uint32_t n_args,
                      const ecl_buffer_geom* inputs, uint32_t n_inputs, const ecl_buffer_geom* outputs,
                      uint32_t n_outputs, uint64_t out_indices, uint64_t out_work_items, ecl_kernel** out) {
  *out = nullptr;
  if (!kernel_id) return fail(ECL_UNKNOWN_KERNEL, "null kernel id");
  if (gws == 0 || lws == 0) return fail(ECL_CONFIG_ERROR, "global/local work size must be positive");
  if (gws % lws != 0) return fail(ECL_NON_DIVISIBLE_WORK_SIZE, "local_work_size does not divide global_work_size");
  if (out_indices == 0 || out_work_items == 0)
    return fail(ECL_BAD_OUT_PATTERN, "out_pattern components must be positive");
  auto* k = new ecl_kernel;
  ecl::KernelSpec& s = k->spec;
  s.id = kernel_id;
  s.gws = gws;
  s.lws = lws;
  s.out_indices = out_indices;
  s.out_work_items = out_work_items;
  s.args.assign(args, args + n_args);
  s.inputs.assign(inputs, inputs + n_inputs);
  s.outputs.assign(outputs, outputs + n_outputs);
  std::string err;
  const int rc = ecl::resolve_kernel(s, &err);
  if (rc != ECL_OK) {
    delete k;
    return fail(rc, err);
  }
  *out = k;
  return ECL_OK;
}

void ecl_kernel_destroy(ecl_kernel* k) { delete k; }

int ecl_kernel_register(const char* kernel_id, const void* image, size_t image_bytes, const char* entry) {
  (void)image_bytes;
  std::string err;
  const int rc = ecl::register_plugin(kernel_id ? kernel_id : "", image, entry ? entry : "", &err);
  return rc == ECL_OK ? rc : fail(rc, err);
}

int ecl_kernel_unregister(const char* kernel_id) {
  std::string err;
  const int rc = ecl::unregister_plugin(kernel_id ? kernel_id : "", &err);
  return rc == ECL_OK ? rc : fail(rc, err);
}

int ecl_kernel_is_plugin(const char* kernel_id) { return kernel_id && ecl::find_plugin(kernel_id) ? 1 : 0; }

int ecl_gpu_bind(ecl_gpu* g, const ecl_kernel* k) {
  if (int rc = set_device(g)) return rc;
  if (int rc = sync_all(g)) return rc;
  std::vector<uint64_t> want_in, want_out;
  for (const auto& b : k->spec.inputs) want_in.push_back(b.element_size_bytes * b.element_count);
  for (const auto& b : k->spec.outputs) want_out.push_back(b.element_size_bytes * b.element_count);
  if (want_in != g->in_bytes || want_out != g->out_bytes) {
    free_buffers(g);
    for (uint64_t bytes : want_in) {
      void* p = nullptr;
      ECL_CK(cudaMalloc(&p, std::max<uint64_t>(bytes, 16)));
      g->in.push_back(p);
    }
    for (uint64_t bytes : want_out) {
      void* p = nullptr;
      ECL_CK(cudaMalloc(&p, std::max<uint64_t>(bytes, 16)));
      g->out.push_back(p);
    }
    g->in_bytes = want_in;
    g->out_bytes = want_out;
  }
  g->spec = &k->spec;
  g->in_host.assign(g->in.size(), {});
  g->in_host_ptr.assign(g->in.size(), nullptr);
  g->in_host_valid.assign(g->in.size(), false);
  for (uint32_t i = 0; i < g->in.size(); ++i) {
    if (!ecl::host_mirrored_input(k->spec, i)) continue;
    g->in_host[i].assign(g->in_bytes[i], 0);
    g->in_host_ptr[i] = g->in_host[i].data();
  }
  const uint64_t scratch = ecl::scratch_bytes(k->spec);
  if (scratch > g->scratch_cap) {
    if (g->scratch) cudaFree(g->scratch);
    g->scratch = nullptr;
    g->scratch_cap = 0;
    ECL_CK(cudaMalloc(&g->scratch, scratch));
    g->scratch_cap = scratch;
  }
  if (k->spec.replicate > 1 && g->compact_items != k->spec.gws) {
    if (g->compact_dev) cudaFree(g->compact_dev);
    if (g->compact_host) pinned_free(g->compact_host);
    g->compact_dev = nullptr;
    g->compact_host = nullptr;  // the pinned landing zone is allocated on first host copy
    g->compact_items = 0;
    ECL_CK(cudaMalloc(&g->compact_dev, k->spec.gws * sizeof(uint32_t)));
    g->compact_items = k->spec.gws;
  }
  ECL_CK(cudaMemsetAsync(g->ctrl, 0, kLanes * kCtrlWordsPerLane * sizeof(unsigned), g->lane[0]));
  const cudaError_t e = ecl::prepare_kernel(k->spec, env_of(g, 0));
  if (e != cudaSuccess) return cuda_fail(e, "kernel prepare");
  ECL_CK(cudaStreamSynchronize(g->lane[0]));
  return ECL_OK;
}

int ecl_gpu_buffer(ecl_gpu* g, int is_output, uint32_t index, void** ptr) {
  const auto& v = is_output ? g->out : g->in;
  if (index >= v.size()) return fail(ECL_CONFIG_ERROR, "buffer index out of range");
  *ptr = v[index];
  return ECL_OK;
}

int ecl_gpu_swap_io(ecl_gpu* g, uint32_t i, uint32_t o) {
  if (i >= g->in.size() || o >= g->out.size()) return fail(ECL_CONFIG_ERROR, "buffer index out of range");
  if (g->in_bytes[i] != g->out_bytes[o]) return fail(ECL_CONFIG_ERROR, "swap_io needs equal buffer sizes");
  if (int rc = set_device(g)) return rc;
  if (int rc = sync_all(g)) return rc;
  std::swap(g->in[i], g->out[o]);
  if (i < g->in_host_valid.size()) g->in_host_valid[i] = false;  // produced on the device
  return ECL_OK;
}

int ecl_gpu_set_streamed_inputs(ecl_gpu* g, int enable) {
  g->streamed = enable != 0;
  return ECL_OK;
}

int ecl_gpu_upload_inputs(ecl_gpu* g, const void* const* host_inputs) {
  if (int rc = set_device(g)) return rc;
  if (int rc = join_lanes(g)) return rc;  // no kernel of an earlier run still reads the inputs
  if (g->streamed) {
    // Nothing moves yet: each piece enqueues (on h2d) the prefix it reads
    // and its kernel waits for it (ecl_gpu_submit); ecl_gpu_sync uploads
    // whatever no piece needed.
    if (int rc = flush_streamed(g)) return rc;  // a previous run's leftovers first
    ECL_CK(cudaEventRecord(g->ready, g->lane[0]));
    ECL_CK(cudaStreamWaitEvent(g->h2d, g->ready, 0));
    g->pending_in.assign(g->in.size(), nullptr);
    g->up_bytes.assign(g->in.size(), 0);
    for (size_t i = 0; i < g->in.size(); ++i) {
      if (!host_inputs || !host_inputs[i]) continue;
      g->pending_in[i] = static_cast<const char*>(host_inputs[i]);
      mirror_write(g, i, 0, host_inputs[i], g->in_bytes[i]);
      if (i < g->in_host_valid.size()) g->in_host_valid[i] = true;
    }
    return ECL_OK;
  }
  for (size_t i = 0; i < g->in.size(); ++i) {
    if (!host_inputs || !host_inputs[i]) continue;
    ECL_CK(cudaMemcpyAsync(g->in[i], host_inputs[i], g->in_bytes[i], cudaMemcpyHostToDevice, g->lane[0]));
    mirror_write(g, i, 0, host_inputs[i], g->in_bytes[i]);
    if (i < g->in_host_valid.size()) g->in_host_valid[i] = true;
  }
  return fan_out_lane0(g);
}

int ecl_replicate_inputs(ecl_gpu* const* gpus, uint32_t n, uint32_t root) {
  if (root >= n) return fail(ECL_CONFIG_ERROR, "replicate: root out of range");
  std::vector<ecl_gpu*> order;
  order.push_back(gpus[root]);
  for (uint32_t i = 0; i < n; ++i)
    if (i != root) order.push_back(gpus[i]);
  // Binary doubling over NVLink: in round r the first 2^r holders each feed one more.
  for (size_t have = 1; have < order.size(); have *= 2) {
    for (size_t i = 0; i < have && have + i < order.size(); ++i) {
      ecl_gpu* src = order[i];
      ecl_gpu* dst = order[have + i];
      if (src->in_bytes != dst->in_bytes) return fail(ECL_CONFIG_ERROR, "replicate: devices bound differently");
      enable_peer(dst->ordinal, src->ordinal);
      if (int rc = set_device(dst)) return rc;
      if (int rc = join_lanes(dst)) return rc;
      ECL_CK(cudaStreamWaitEvent(dst->lane[0], src->ready, 0));
      for (size_t b = 0; b < dst->in.size(); ++b)
        ECL_CK(cudaMemcpyPeerAsync(dst->in[b], dst->ordinal, src->in[b], src->ordinal, dst->in_bytes[b],
                                   dst->lane[0]));
      if (int rc = ensure_mirrors(src)) return rc;
      dst->in_host = src->in_host;
      dst->in_host_valid = src->in_host_valid;
      for (size_t b = 0; b < dst->in_host.size(); ++b)
        dst->in_host_ptr[b] = dst->in_host[b].empty() ? nullptr : dst->in_host[b].data();
      if (int rc = fan_out_lane0(dst)) return rc;
    }
  }
  return ECL_OK;
}

int ecl_broadcast_output_slice(ecl_gpu* const* gpus, uint32_t n, uint32_t src_i, uint32_t index,
                               uint64_t elem_offset, uint64_t elem_count) {
  if (src_i >= n) return fail(ECL_CONFIG_ERROR, "broadcast: source out of range");
  ecl_gpu* src = gpus[src_i];
  if (index >= src->out.size()) return fail(ECL_CONFIG_ERROR, "broadcast: output index out of range");
  const uint64_t esz = src->spec->outputs[index].element_size_bytes;
  if ((elem_offset + elem_count) * esz > src->out_bytes[index])
    return fail(ECL_CONFIG_ERROR, "broadcast: slice out of range");
  for (uint32_t d = 0; d < n; ++d) enable_peer(gpus[d]->ordinal, src->ordinal);
  if (int rc = set_device(src)) return rc;
  if (int rc = join_lanes(src)) return rc;
  for (uint32_t d = 0; d < n; ++d) {
    ecl_gpu* dst = gpus[d];
    if (d == src_i || dst->out.size() <= index) continue;
    char* to = static_cast<char*>(dst->out[index]) + elem_offset * esz;
    const char* from = static_cast<const char*>(src->out[index]) + elem_offset * esz;
    if (dst->ordinal == src->ordinal && !force_peer_copy())
      ECL_CK(cudaMemcpyAsync(to, from, elem_count * esz, cudaMemcpyDeviceToDevice, src->lane[0]));
    else
      ECL_CK(cudaMemcpyPeerAsync(to, dst->ordinal, from, src->ordinal, elem_count * esz, src->lane[0]));
  }
  if (int rc = fan_out_lane0(src)) return rc;
  for (uint32_t d = 0; d < n; ++d) {
    if (d == src_i) continue;
    if (int rc = set_device(gpus[d])) return rc;
    for (int l = 0; l < gpus[d]->lanes; ++l) ECL_CK(cudaStreamWaitEvent(gpus[d]->lane[l], src->ready, 0));
  }
  return ECL_OK;
}

int ecl_gpu_download_slice(ecl_gpu* g, uint32_t index, uint64_t elem_offset, uint64_t elem_count, void* host) {
  if (index >= g->out.size()) return fail(ECL_CONFIG_ERROR, "download: output index out of range");
  const uint64_t esz = g->spec->outputs[index].element_size_bytes;
  if ((elem_offset + elem_count) * esz > g->out_bytes[index])
    return fail(ECL_CONFIG_ERROR, "download: slice out of range");
  if (int rc = set_device(g)) return rc;
  if (int rc = sync_all(g)) return rc;
  ECL_CK(cudaMemcpyAsync(host, static_cast<const char*>(g->out[index]) + elem_offset * esz, elem_count * esz,
                         cudaMemcpyDeviceToHost, g->copy[0]));
  ECL_CK(cudaStreamSynchronize(g->copy[0]));
  return ECL_OK;
}

int ecl_peer_access(int dst, int src, int* can_access, int* enabled) {
  *can_access = 0;
  *enabled = 0;
  if (dst == src) {
    *can_access = *enabled = 1;
    return ECL_OK;
  }
  ECL_CK(cudaDeviceCanAccessPeer(can_access, dst, src));
  std::lock_guard lock(g_peer_m);
  *enabled = g_peer[dst & 63][src & 63] == 1;
  return ECL_OK;
}

int ecl_probe_host_widen(uint64_t items, uint32_t replicate, double* ms) {
  return ecl_probe_host_widen_width(items, replicate, 4, ms);
}

int ecl_probe_host_widen_width(uint64_t items, uint32_t replicate, uint32_t src_bytes, double* ms) {
  if (src_bytes != 2 && src_bytes != 4) return fail(ECL_CONFIG_ERROR, "widen probe: src_bytes must be 2 or 4");
  *ms = ecl::widen_probe_ms(items, replicate, src_bytes);
  return *ms >= 0.0 ? ECL_OK : fail(ECL_CONFIG_ERROR, "widen probe: allocation failed");
}

int ecl_host_register(void* ptr, size_t bytes) {
  cudaError_t e = cudaHostRegister(ptr, bytes, cudaHostRegisterPortable);
  if (e == cudaErrorHostMemoryAlreadyRegistered) {
    cudaGetLastError();
    return ECL_OK;
  }
  if (e != cudaSuccess) return cuda_fail(e, "cudaHostRegister");
  return ECL_OK;
}

int ecl_host_unregister(void* ptr) {
  cudaError_t e = cudaHostUnregister(ptr);
  if (e != cudaSuccess && e != cudaErrorHostMemoryNotRegistered) return cuda_fail(e, "cudaHostUnregister");
  cudaGetLastError();
  return ECL_OK;
}

int ecl_host_alloc(size_t bytes, void** ptr) {
  *ptr = nullptr;
  ECL_CK(pinned_alloc(ptr, bytes));
  return ECL_OK;
}

int ecl_host_free(void* ptr) {
  ECL_CK(pinned_free(ptr));
  return ECL_OK;
}

int ecl_gpu_alloc(ecl_gpu* g, size_t bytes, void** dptr) {
  *dptr = nullptr;
  if (int rc = set_device(g)) return rc;
  ECL_CK(cudaMalloc(dptr, std::max<size_t>(bytes, 16)));
  return ECL_OK;
}

int ecl_gpu_free(ecl_gpu* g, void* dptr) {
  if (int rc = set_device(g)) return rc;
  if (int rc = sync_all(g)) return rc;
  ECL_CK(cudaFree(dptr));
  return ECL_OK;
}

int ecl_gpu_upload(ecl_gpu* g, void* dst, const void* src, size_t bytes) {
  if (int rc = set_device(g)) return rc;
  if (int rc = join_lanes(g)) return rc;
  ECL_CK(cudaMemcpyAsync(dst, src, bytes, cudaMemcpyHostToDevice, g->lane[0]));
  // A raw upload into a mirrored input keeps the mirror in step.
  for (size_t i = 0; i < g->in_host.size(); ++i) {
    if (g->in_host[i].empty()) continue;
    const uintptr_t b0 = reinterpret_cast<uintptr_t>(g->in[i]), b1 = b0 + g->in_bytes[i];
    const uintptr_t d0 = reinterpret_cast<uintptr_t>(dst), d1 = d0 + bytes;
    const uintptr_t lo = std::max(b0, d0), hi = std::min(b1, d1);
    if (lo < hi) mirror_write(g, i, lo - b0, static_cast<const char*>(src) + (lo - d0), hi - lo);
  }
  return fan_out_lane0(g);
}

int ecl_gpu_download(ecl_gpu* g, void* dst, const void* src, size_t bytes) {
  if (int rc = set_device(g)) return rc;
  if (int rc = sync_all(g)) return rc;
  ECL_CK(cudaMemcpyAsync(dst, src, bytes, cudaMemcpyDeviceToHost, g->copy[0]));
  ECL_CK(cudaStreamSynchronize(g->copy[0]));
  return ECL_OK;
}

int ecl_gpu_launch(ecl_gpu* g, const ecl_kernel* k, uint64_t first_item, uint64_t item_count, uint64_t seq,
                   ecl_done_fn done, void* user) {
  if (!g->spec || &k->spec != g->spec) return fail(ECL_CONFIG_ERROR, "launch: kernel is not the one bound");
  const uint64_t lws = g->spec->lws;
  if (item_count == 0 || first_item % lws != 0 || item_count % lws != 0)
    return fail(ECL_INDIVISIBLE_PACKAGE, "launch: item range must be whole work-groups");
  return ecl_gpu_submit(g, seq, first_item / lws, item_count / lws, nullptr, done, user);
}

// Streamed inputs (ecl_gpu_set_streamed_inputs): enqueues on the H2D stream
// the prefix of every still-pending input that items [first, first+count)
// read, and makes `st` wait for the latest upload.
static int stream_inputs_for(ecl_gpu* g, const ecl::KernelSpec& s, uint64_t first, uint64_t count, cudaStream_t st) {
  bool moved = false;
  for (uint32_t i = 0; i < g->pending_in.size(); ++i) {
    if (!g->pending_in[i]) continue;
    const uint64_t need = ecl::input_bytes_needed(s, i, first, count), up = g->up_bytes[i];
    if (need > up) {
      ECL_CK(cudaMemcpyAsync(static_cast<char*>(g->in[i]) + up, g->pending_in[i] + up, need - up,
                             cudaMemcpyHostToDevice, g->h2d));
      g->up_bytes[i] = need;
      moved = true;
    }
    if (g->up_bytes[i] >= g->in_bytes[i]) g->pending_in[i] = nullptr;
  }
  if (moved) {
    ECL_CK(cudaEventRecord(g->up_ev, g->h2d));
    g->up_live = true;
  }
  if (g->up_live) ECL_CK(cudaStreamWaitEvent(st, g->up_ev, 0));
  return ECL_OK;
}

// The compact copies of one piece (items [first, first+count), one value of
// s.compact_bytes each) on copy stream `cp`, and the host widening of each into `dst` (the
// piece's slice of the caller's output, `replicate` values per item).  The
// copy may go in chunks (ECL_WIDEN_CHUNK), each widened as soon as it lands;
// measured on the 16-core Xeon host: 2^20-item chunks = whole pieces (54.5
// vs 54.9 ms), smaller chunks slower (API cost), so without the staging ring
// the default is one copy per piece.  With the ring, every chunk is one slot.
static int enqueue_compact_copies(ecl_gpu* g, Slot& slot, const ecl::KernelSpec& s, uint64_t first, uint64_t count,
                                  uint32_t* dst, cudaStream_t cp, size_t* piece_no) {
  const uint64_t chunk = g->ring ? g->ring_items : g->widen_chunk_items;
  const uint32_t cb = s.compact_bytes;  // 2: 16-bit counts
  for (uint64_t c0 = 0; c0 < count; c0 += chunk) {
    const uint64_t cn = std::min(chunk, count - c0);
    char* land = g->compact_host ? reinterpret_cast<char*>(g->compact_host) + (first + c0) * cb : nullptr;
    uint32_t* release = nullptr;
    uint32_t release_value = 0;
    if (g->ring) {  // next staging slot, once its previous contents are widened
      const uint32_t r = g->ring_next;
      g->ring_next = (r + 1) % g->ring_slots;
      const uint32_t uses = g->ring_uses[r]++;
      const unsigned long long flag = reinterpret_cast<unsigned long long>(g->ring_released_dev) + 4ull * r;
      if (wait_value_fn()(cp, flag, uses, 0 /* CU_STREAM_WAIT_VALUE_GEQ */) != 0)
        return fail(ECL_KERNEL_PANIC, "staging ring: stream wait failed");
      land = reinterpret_cast<char*>(g->ring + static_cast<uint64_t>(r) * g->ring_items);
      release = g->ring_released + r;
      release_value = uses + 1;
    }
    ECL_CK(cudaMemcpyAsync(land, reinterpret_cast<const char*>(g->compact_dev) + (first + c0) * cb, cn * cb,
                           cudaMemcpyDeviceToHost, cp));
    if (slot.piece_done.size() <= *piece_no) {
      cudaEvent_t ev;
      // blocking-sync: widen workers sleep on it instead of spinning a core
      ECL_CK(cudaEventCreateWithFlags(&ev, cudaEventDisableTiming | cudaEventBlockingSync));
      slot.piece_done.push_back(ev);
    }
    cudaEvent_t ev = slot.piece_done[(*piece_no)++];
    ECL_CK(cudaEventRecord(ev, cp));
    ecl::widen_async(g->ordinal, ev, land, cb, dst + c0 * s.replicate, cn, s.replicate, &slot.widen, release,
                     release_value);
  }
  return ECL_OK;
}

int ecl_gpu_submit(ecl_gpu* g, uint64_t seq, uint64_t offset_wg, uint64_t size_wg, void* const* host_outputs,
                   ecl_done_fn done, void* user) {
  if (!g->spec) return fail(ECL_CONFIG_ERROR, "submit before bind");
  const ecl::KernelSpec& s = *g->spec;
  if (size_wg == 0 || (offset_wg + size_wg) * s.lws > s.gws)
    return fail(ECL_SCHEDULER_ERROR, "package outside the work-group range");
  uint64_t o_off = 0, o_cnt = 0;
  if (int rc = out_range(s, offset_wg, size_wg, &o_off, &o_cnt)) return rc;
  if (int rc = set_device(g)) return rc;
  if (int rc = ensure_mirrors(g)) return rc;
  if (find_slot(g, seq)) return fail(ECL_SCHEDULER_ERROR, "package seq submitted twice");
  Slot& slot = g->slots[g->next_slot];
  g->next_slot = (g->next_slot + 1) % (kSlots - 1);  // the last slot is reserved for native_run
  // Ring wrapped: the slot's previous package must be retired, copies and
  // widening included (a package timed by package_times may still be copying).
  ECL_CK(cudaEventSynchronize(slot.done));
  if (!ecl::widen_wait(&slot.widen)) return fail(ECL_KERNEL_PANIC, "host widening: a copy failed");
  slot.widen.failed.store(false);
  slot.seq = seq;
  slot.busy = true;
  slot.timed = false;
  slot.fn = done;
  slot.user = user;
  const int lane = static_cast<int>(g->next_lane);
  g->next_lane = (g->next_lane + 1) % static_cast<uint32_t>(g->lanes);

  bool copies = false;
  for (size_t b = 0; host_outputs && b < g->out.size(); ++b) copies = copies || host_outputs[b] != nullptr;

  // With host outputs the package runs as sub-launches of ~d2h_split_items
  // work-items, each followed on its lane's copy stream by the D2H of its own
  // slice, so the PCIe copy of piece i overlaps the kernels of later pieces.
  // Pieces alternate between the two compute lanes so one piece's drain tail
  // overlaps the next piece's ramp (the timing events bracket the package
  // across both lanes).
  uint64_t piece_wg = size_wg;
  bool streaming = false;
  for (const char* p : g->pending_in) streaming = streaming || p != nullptr;
  const uint64_t compute_split = g->lanes > 1 ? s.compute_split_items : 0;
  const uint64_t split_items = copies ? g->d2h_split_items
                                      : (compute_split ? compute_split : (streaming ? g->d2h_split_items : 0));
  if (split_items > 0) {
    piece_wg = std::max<uint64_t>(1, split_items / s.lws);
    uint64_t po = 0, pc = 0;
    if (out_range(s, offset_wg, std::min(piece_wg, size_wg), &po, &pc) != ECL_OK) piece_wg = size_wg;
  }
  // Replicated outputs (4 identical uint32 per item): copy one value per item
  // and widen on the host (hostpool.cpp) — a quarter of the PCIe bytes.
  const bool widen = copies && s.replicate > 1 && g->compact_dev && s.outputs.size() == 1 &&
                     s.outputs[0].element_size_bytes == 4 && s.out_indices == s.replicate &&
                     s.out_work_items == 1 && g->widen_per_8 > 0;
  if (widen) ECL_CK(ring_setup(g));
  if (widen && !g->ring && !g->compact_host) {
    void* p = nullptr;
    ECL_CK(pinned_alloc(&p, g->compact_items * 4));
    g->compact_host = static_cast<uint32_t*>(p);
  }
  const int other = (lane + 1) % g->lanes;
  slot.two_lanes = g->lanes > 1 && piece_wg < size_wg;
  ECL_CK(cudaEventRecord(slot.start, g->lane[lane]));
  if (slot.two_lanes) ECL_CK(cudaEventRecord(slot.start2, g->lane[other]));
  size_t piece_no = 0, piece_idx = 0;
  for (uint64_t wg = offset_wg; wg < offset_wg + size_wg; wg += piece_wg, ++piece_idx) {
    const int pl = slot.two_lanes && (piece_idx & 1) ? other : lane;
    cudaStream_t st = g->lane[pl];
    cudaStream_t cp = g->copy[pl];
    ecl::LaunchEnv env = env_of(g, pl);
    if (widen) {
      env.compact = g->compact_dev;
      env.compact_bytes = s.compact_bytes;
    }
    env.host_copies = copies;
    const uint64_t n_wg = std::min(piece_wg, offset_wg + size_wg - wg);
    const uint64_t first = wg * s.lws, count = n_wg * s.lws;
    if (streaming || g->up_live) {
      if (int rc = stream_inputs_for(g, s, first, count, st)) return rc;
    }
    cudaError_t e = ecl::launch_kernel(s, env, first, count);
    if (e != cudaSuccess) return cuda_fail(e, "kernel launch");
    g->launches += 1;  // every kernel launch (a package may run as several pieces)
    if (g->tally_on) {
      e = ecl::launch_tally(g->tally, first, count, st);
      if (e != cudaSuccess) return cuda_fail(e, "tally launch");
    }
    if (!copies) continue;
    uint64_t p_off = o_off, p_cnt = o_cnt;
    if (piece_wg != size_wg && out_range(s, wg, n_wg, &p_off, &p_cnt) != ECL_OK) return ECL_INDIVISIBLE_PACKAGE;
    ECL_CK(cudaEventRecord(g->piece[pl], st));
    ECL_CK(cudaStreamWaitEvent(cp, g->piece[pl], 0));  // captures this recording
    // widen_per_8 of every 8 pieces go compact + host widening, the rest are
    // copied whole: balances PCIe bytes against host-DRAM traffic.
    if (widen && (g->piece_counter++ % 8) < g->widen_per_8) {
      if (int rc = enqueue_compact_copies(g, slot, s, first, count, static_cast<uint32_t*>(host_outputs[0]) + p_off,
                                          cp, &piece_no))
        return rc;
      continue;
    }
    for (size_t b = 0; b < g->out.size(); ++b) {
      if (!host_outputs[b]) continue;
      const uint64_t esz = s.outputs[b].element_size_bytes;
      ECL_CK(cudaMemcpyAsync(static_cast<char*>(host_outputs[b]) + p_off * esz,
                             static_cast<const char*>(g->out[b]) + p_off * esz, p_cnt * esz,
                             cudaMemcpyDeviceToHost, cp));
    }
  }
  ECL_CK(cudaEventRecord(slot.end, g->lane[lane]));
  ECL_CK(cudaStreamWaitEvent(g->notify, slot.end, 0));
  if (slot.two_lanes) {
    ECL_CK(cudaEventRecord(slot.end2, g->lane[other]));
    ECL_CK(cudaStreamWaitEvent(g->notify, slot.end2, 0));
  }
  if (copies) {
    for (int l : {lane, other}) {
      if (l == other && !slot.two_lanes) continue;
      ECL_CK(cudaEventRecord(g->copied[l], g->copy[l]));
      ECL_CK(cudaStreamWaitEvent(g->notify, g->copied[l], 0));
    }
  }
  if (done) ECL_CK(cudaLaunchHostFunc(g->notify, on_package_done, &slot));
  ECL_CK(cudaEventRecord(slot.done, g->notify));
  return ECL_OK;
}

int ecl_gpu_poll(ecl_gpu* g, uint64_t seq) {
  Slot* sp = find_slot(g, seq);
  if (!sp) return fail(ECL_CONFIG_ERROR, "poll: unknown package");
  cudaSetDevice(g->ordinal);
  cudaError_t e = cudaEventQuery(sp->done);
  if (e == cudaSuccess) {
    if (sp->widen.pending.load() != 0) return ECL_PENDING;
    return sp->widen.failed.load() ? fail(ECL_KERNEL_PANIC, "host widening: a copy failed") : ECL_OK;
  }
  if (e == cudaErrorNotReady) {
    cudaGetLastError();
    return ECL_PENDING;
  }
  return cuda_fail(e, "package completion");
}

int ecl_gpu_package_times(ecl_gpu* g, uint64_t seq, double* t_start, double* t_end) {
  Slot* sp = find_slot(g, seq);
  if (!sp) return fail(ECL_CONFIG_ERROR, "package_times: unknown package");
  Slot& slot = *sp;
  if (int rc = set_device(g)) return rc;
  ECL_CK(cudaEventSynchronize(slot.end));  // kernel times only: copies may still be in flight
  if (slot.two_lanes) ECL_CK(cudaEventSynchronize(slot.end2));
  float a = 0.f, b = 0.f, k = 0.f;
  ECL_CK(cudaEventElapsedTime(&a, g->epoch, slot.start));
  ECL_CK(cudaEventElapsedTime(&b, g->epoch, slot.end));
  if (slot.two_lanes) {  // the package spans both lanes: earliest start, latest end
    float a2 = 0.f, b2 = 0.f;
    ECL_CK(cudaEventElapsedTime(&a2, g->epoch, slot.start2));
    ECL_CK(cudaEventElapsedTime(&b2, g->epoch, slot.end2));
    a = std::min(a, a2);
    b = std::max(b, b2);
  }
  k = b - a;
  *t_start = g->epoch_host_ms + a;
  *t_end = g->epoch_host_ms + b;
  if (!slot.timed) {
    g->kernel_ms += k;
    slot.timed = true;
  }
  slot.busy = false;
  return ECL_OK;
}

int ecl_gpu_set_epoch(ecl_gpu* g, double (*host_now_ms)(void*), void* clock_user) {
  (void)host_now_ms;
  (void)clock_user;
  // Anchor device event time to the host steady clock.  Cheap when fresh:
  // re-anchoring (an event record + synchronize on an idle lane) happens only
  // every 2 s so cudaEventElapsedTime's float stays sub-microsecond.
  const double now = std::chrono::duration<double, std::milli>(
                         std::chrono::steady_clock::now().time_since_epoch()).count();
  if (g->epoch_host_ms >= 0.0 && now - g->epoch_host_ms < 2000.0) return ECL_OK;
  if (int rc = set_device(g)) return rc;
  if (int rc = sync_all(g)) return rc;
  ECL_CK(cudaEventRecord(g->epoch, g->lane[0]));
  ECL_CK(cudaEventSynchronize(g->epoch));
  g->epoch_host_ms = std::chrono::duration<double, std::milli>(
                         std::chrono::steady_clock::now().time_since_epoch()).count();
  return ECL_OK;
}

int ecl_gpu_wait(ecl_gpu* g, uint64_t seq) {
  Slot* sp = find_slot(g, seq);
  if (!sp) return fail(ECL_CONFIG_ERROR, "wait: unknown package");
  if (int rc = set_device(g)) return rc;
  ECL_CK(cudaEventSynchronize(sp->done));
  if (!ecl::widen_wait(&sp->widen)) return fail(ECL_KERNEL_PANIC, "host widening: a copy failed");
  return ECL_OK;
}

// Completion wait of a package's kernels: poll the event for a short while
// before blocking.  A blocking wait wakes the device thread ~5 us after the
// kernel ends (measured with CUPTI on a 72 us Gaussian step); polling costs
// one host core for at most ~0.5 ms per package, then falls back.
static cudaError_t await_event(cudaEvent_t ev) {
  for (int i = 0; i < 1500; ++i) {
    const cudaError_t q = cudaEventQuery(ev);
    if (q != cudaErrorNotReady) return q;
  }
  return cudaEventSynchronize(ev);
}

int ecl_gpu_wait_compute(ecl_gpu* g, uint64_t seq) {
  Slot* sp = find_slot(g, seq);
  if (!sp) return fail(ECL_CONFIG_ERROR, "wait_compute: unknown package");
  if (int rc = set_device(g)) return rc;
  ECL_CK(await_event(sp->end));
  if (sp->two_lanes) ECL_CK(await_event(sp->end2));
  return ECL_OK;
}

int ecl_gpu_sync(ecl_gpu* g) {
  if (int rc = set_device(g)) return rc;
  return sync_all(g);
}

int ecl_gpu_enable_tally(ecl_gpu* g, int enable) {
  if (int rc = set_device(g)) return rc;
  g->tally_on = enable != 0;
  if (!g->tally_on) return ECL_OK;
  if (!g->spec) return fail(ECL_CONFIG_ERROR, "tally before bind");
  if (int rc = join_lanes(g)) return rc;
  if (g->tally_items != g->spec->gws) {
    if (g->tally) cudaFree(g->tally);
    g->tally = nullptr;
    ECL_CK(cudaMalloc(&g->tally, g->spec->gws * sizeof(uint32_t)));
    g->tally_items = g->spec->gws;
  }
  ECL_CK(cudaMemsetAsync(g->tally, 0, g->tally_items * sizeof(uint32_t), g->lane[0]));
  return fan_out_lane0(g);
}

int ecl_gpu_download_tally(ecl_gpu* g, uint32_t* host) {
  if (!g->tally) return fail(ECL_CONFIG_ERROR, "tally not enabled");
  if (int rc = set_device(g)) return rc;
  if (int rc = sync_all(g)) return rc;
  ECL_CK(cudaMemcpy(host, g->tally, g->tally_items * sizeof(uint32_t), cudaMemcpyDeviceToHost));
  return ECL_OK;
}

int ecl_gpu_set_peer_outputs(ecl_gpu* g, void* const* ptrs, uint32_t n_peers) {
  if (!g->spec) return fail(ECL_CONFIG_ERROR, "peer outputs before bind");
  if (n_peers == 0) {
    g->peer_out.clear();
    g->n_peers = 0;
    return ECL_OK;
  }
  if (!g->spec->peer_writes) return fail(ECL_CONFIG_ERROR, "the bound kernel does not write to peer buffers");
  if (n_peers > ecl::kMaxPeerWrites) return fail(ECL_CONFIG_ERROR, "too many peers for a fused exchange");
  const size_t n = static_cast<size_t>(n_peers) * g->out.size();
  for (size_t k = 0; k < n; ++k) {
    if (!ptrs[k]) continue;
    cudaPointerAttributes a{};
    if (cudaPointerGetAttributes(&a, ptrs[k]) != cudaSuccess || a.type != cudaMemoryTypeDevice) {
      cudaGetLastError();
      return fail(ECL_CONFIG_ERROR, "peer output is not device memory");
    }
    if (a.device != g->ordinal) {
      enable_peer(g->ordinal, a.device);
      std::lock_guard lock(g_peer_m);
      if (g_peer[g->ordinal & 63][a.device & 63] != 1)
        return fail(ECL_CONFIG_ERROR, "no peer access to the device of a peer output");
    }
  }
  if (int rc = set_device(g)) return rc;
  if (int rc = join_lanes(g)) return rc;  // launches already queued keep the previous targets
  g->peer_out.assign(ptrs, ptrs + n);
  g->n_peers = n_peers;
  return fan_out_lane0(g);
}

int ecl_gpu_peer_writes(const ecl_gpu* g, int* supported) {
  if (!g->spec) return fail(ECL_CONFIG_ERROR, "peer_writes before bind");
  *supported = g->spec->peer_writes ? 1 : 0;
  return ECL_OK;
}

int ecl_gpu_export_buffer(ecl_gpu* g, int is_output, uint32_t index, void* handle) {
  if (!g->spec) return fail(ECL_CONFIG_ERROR, "export before bind");
  const auto& bufs = is_output ? g->out : g->in;
  if (index >= bufs.size()) return fail(ECL_CONFIG_ERROR, "export: buffer index out of range");
  if (int rc = set_device(g)) return rc;
  static_assert(sizeof(cudaIpcMemHandle_t) == ECL_IPC_HANDLE_BYTES, "IPC handle size");
  cudaIpcMemHandle_t h;
  ECL_CK(cudaIpcGetMemHandle(&h, bufs[index]));
  std::memcpy(handle, &h, sizeof(h));
  return ECL_OK;
}

int ecl_gpu_import_buffer(ecl_gpu* g, const void* handle, void** dptr) {
  if (int rc = set_device(g)) return rc;
  cudaIpcMemHandle_t h;
  std::memcpy(&h, handle, sizeof(h));
  ECL_CK(cudaIpcOpenMemHandle(dptr, h, cudaIpcMemLazyEnablePeerAccess));
  return ECL_OK;
}

int ecl_gpu_release_import(ecl_gpu* g, void* dptr) {
  if (int rc = set_device(g)) return rc;
  ECL_CK(cudaIpcCloseMemHandle(dptr));
  return ECL_OK;
}

int ecl_gpu_pull_output_slice(ecl_gpu* g, uint32_t index, const void* src_base, uint64_t elem_offset,
                              uint64_t elem_count) {
  if (!g->spec || index >= g->out.size()) return fail(ECL_CONFIG_ERROR, "pull: output index out of range");
  const uint64_t esz = g->spec->outputs[index].element_size_bytes;
  if ((elem_offset + elem_count) * esz > g->out_bytes[index]) return fail(ECL_CONFIG_ERROR, "pull: slice out of range");
  if (int rc = set_device(g)) return rc;
  if (int rc = join_lanes(g)) return rc;
  ECL_CK(cudaMemcpyAsync(static_cast<char*>(g->out[index]) + elem_offset * esz,
                         static_cast<const char*>(src_base) + elem_offset * esz, elem_count * esz, cudaMemcpyDefault,
                         g->lane[0]));
  return fan_out_lane0(g);
}

int ecl_gpu_native_run(ecl_gpu* g, float* kernel_ms) {
  if (!g->spec) return fail(ECL_CONFIG_ERROR, "native run before bind");
  if (int rc = set_device(g)) return rc;
  if (int rc = ensure_mirrors(g)) return rc;
  if (int rc = join_lanes(g)) return rc;
  // Inputs whole before the one launch (streamed uploads finish first; the
  // kernel timing below starts after them).
  if (int rc = flush_streamed(g)) return rc;
  ECL_CK(cudaEventRecord(g->up_ev, g->h2d));
  ECL_CK(cudaStreamWaitEvent(g->lane[0], g->up_ev, 0));
  Slot& slot = g->slots[kSlots - 1];
  ECL_CK(cudaEventRecord(slot.start, g->lane[0]));
  cudaError_t e = ecl::launch_kernel(*g->spec, env_of(g, 0), 0, g->spec->gws);
  if (e != cudaSuccess) return cuda_fail(e, "kernel launch");
  ECL_CK(cudaEventRecord(slot.end, g->lane[0]));
  ECL_CK(cudaEventSynchronize(slot.end));
  float ms = 0.f;
  ECL_CK(cudaEventElapsedTime(&ms, slot.start, slot.end));
  *kernel_ms = ms;
  g->kernel_ms += ms;
  g->launches += 1;
  return fan_out_lane0(g);
}

int ecl_gpu_native_run_split(ecl_gpu* g, uint64_t items_per_launch, float* kernel_ms) {
  if (!g->spec) return fail(ECL_CONFIG_ERROR, "native run before bind");
  const uint64_t lws = g->spec->lws, gws = g->spec->gws;
  uint64_t piece = items_per_launch / lws * lws;
  if (piece == 0) piece = lws;
  if (int rc = set_device(g)) return rc;
  if (int rc = ensure_mirrors(g)) return rc;
  if (int rc = join_lanes(g)) return rc;
  if (int rc = flush_streamed(g)) return rc;
  ECL_CK(cudaEventRecord(g->up_ev, g->h2d));
  ECL_CK(cudaStreamWaitEvent(g->lane[0], g->up_ev, 0));
  Slot& slot = g->slots[kSlots - 1];
  ECL_CK(cudaEventRecord(slot.start, g->lane[0]));
  if (int rc = fan_out_lane0(g)) return rc;  // every lane starts after the start event
  uint64_t launches = 0;
  for (uint64_t first = 0; first < gws; first += piece, ++launches) {
    const uint64_t count = first + piece < gws ? piece : gws - first;
    cudaError_t e = ecl::launch_kernel(*g->spec, env_of(g, static_cast<int>(launches % g->lanes)), first, count);
    if (e != cudaSuccess) return cuda_fail(e, "kernel launch");
  }
  if (int rc = join_lanes(g)) return rc;
  ECL_CK(cudaEventRecord(slot.end, g->lane[0]));
  ECL_CK(cudaEventSynchronize(slot.end));
  float ms = 0.f;
  ECL_CK(cudaEventElapsedTime(&ms, slot.start, slot.end));
  *kernel_ms = ms;
  g->kernel_ms += ms;
  g->launches += launches;
  return fan_out_lane0(g);
}

int ecl_gpu_kernel_time(ecl_gpu* g, double* total_ms, uint64_t* launches, int reset) {
  *total_ms = g->kernel_ms;
  *launches = g->launches;
  if (reset) {
    g->kernel_ms = 0.0;
    g->launches = 0;
  }
  return ECL_OK;
}

int ecl_gpu_set_copy_split(ecl_gpu* g, uint64_t items) {
  g->d2h_split_items = items;
  return ECL_OK;
}

int ecl_gpu_set_widen_fraction(ecl_gpu* g, uint32_t per_8) {
  if (per_8 > 8) return fail(ECL_CONFIG_ERROR, "widen fraction is per 8 pieces (0..8)");
  g->widen_per_8 = per_8;
  return ECL_OK;
}

}  // extern "C"
