// shared.cpp — SharedCoordinator: the decision log in POSIX shared memory.
#include "coexec/shared.hpp"

#include <fcntl.h>
#include <pthread.h>
#include <sys/mman.h>
#include <sys/stat.h>
#include <unistd.h>

#include <algorithm>
#include <atomic>
#include <cerrno>
#include <chrono>
#include <cstring>
#include <thread>

namespace coexec {

namespace {

constexpr std::uint64_t kMagic = 0x45434c5348524431ull;  // "ECLSHRD1"
constexpr std::uint64_t kMaxLog = 1u << 16;

struct LogEntry {
  std::uint32_t kind;  // 0 = grant to `device`, 1 = observation
  std::uint32_t device;
  std::uint64_t items;
  double ms;
};

struct DoneRec {
  std::uint64_t seq;
  std::uint32_t device;
  std::uint32_t pad;
  std::uint64_t offset_wg, size_wg;
  double t_enqueue, t_start, t_end;
};

double steady_now_ms() {
  return std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now().time_since_epoch()).count();
}

[[noreturn]] void sys_fail(const std::string& what) {
  throw Error(ErrorCode::ConfigError, what + ": " + std::strerror(errno));
}

class Lock {
 public:
  explicit Lock(pthread_mutex_t* m) : m_(m) { pthread_mutex_lock(m_); }
  ~Lock() { pthread_mutex_unlock(m_); }

 private:
  pthread_mutex_t* m_;
};

}  // namespace

struct SharedCoordinator::Region {
  std::atomic<std::uint64_t> magic;
  std::uint32_t world;
  std::uint32_t failed;
  pthread_mutex_t mu;
  pthread_cond_t cv;
  std::uint64_t barrier_gen;
  std::uint32_t barrier_count;
  std::uint32_t pad;
  double epoch_ms;
  std::uint64_t log_len;
  std::uint64_t grants;
  std::uint64_t n_done;
  LogEntry log[kMaxLog];
  DoneRec done[kMaxLog];
  unsigned char blobs[SharedCoordinator::kMaxRanks][SharedCoordinator::kBlobSlots][SharedCoordinator::kBlobBytes];
};

SharedCoordinator::SharedCoordinator(SharedConfig cfg) : cfg_(std::move(cfg)) {
  if (cfg_.world < 1 || cfg_.rank >= cfg_.world || cfg_.world > kMaxRanks)
    throw Error(ErrorCode::ConfigError, "shared: bad rank/world");
  if (cfg_.name.empty() || cfg_.name[0] != '/') throw Error(ErrorCode::ConfigError, "shared: name must start with '/'");
  bytes_ = sizeof(Region);
  int fd = -1;
  if (cfg_.rank == 0) {
    fd = shm_open(cfg_.name.c_str(), O_CREAT | O_RDWR | O_TRUNC, 0600);
    if (fd < 0) sys_fail("shm_open(" + cfg_.name + ")");
    if (ftruncate(fd, static_cast<off_t>(bytes_)) != 0) sys_fail("ftruncate");
  } else {
    const auto deadline = std::chrono::steady_clock::now() + std::chrono::duration<double>(cfg_.barrier_timeout_s);
    while ((fd = shm_open(cfg_.name.c_str(), O_RDWR, 0600)) < 0) {
      if (std::chrono::steady_clock::now() > deadline) sys_fail("shm_open(" + cfg_.name + ") waiting for rank 0");
      std::this_thread::sleep_for(std::chrono::milliseconds(2));
    }
    struct stat st{};
    while (fstat(fd, &st) == 0 && static_cast<std::size_t>(st.st_size) < bytes_) {
      if (std::chrono::steady_clock::now() > deadline) sys_fail("shared segment never sized");
      std::this_thread::sleep_for(std::chrono::milliseconds(2));
    }
  }
  void* p = mmap(nullptr, bytes_, PROT_READ | PROT_WRITE, MAP_SHARED, fd, 0);
  close(fd);
  if (p == MAP_FAILED) sys_fail("mmap");
  region_ = static_cast<Region*>(p);
  if (cfg_.rank == 0) {
    pthread_mutexattr_t ma;
    pthread_mutexattr_init(&ma);
    pthread_mutexattr_setpshared(&ma, PTHREAD_PROCESS_SHARED);
    pthread_mutex_init(&region_->mu, &ma);
    pthread_mutexattr_destroy(&ma);
    pthread_condattr_t ca;
    pthread_condattr_init(&ca);
    pthread_condattr_setpshared(&ca, PTHREAD_PROCESS_SHARED);
    pthread_condattr_setclock(&ca, CLOCK_MONOTONIC);
    pthread_cond_init(&region_->cv, &ca);
    pthread_condattr_destroy(&ca);
    region_->world = cfg_.world;
    region_->barrier_gen = 0;
    region_->barrier_count = 0;
    region_->failed = 0;
    region_->log_len = region_->grants = region_->n_done = 0;
    region_->magic.store(kMagic, std::memory_order_release);
  } else {
    const auto deadline = std::chrono::steady_clock::now() + std::chrono::duration<double>(cfg_.barrier_timeout_s);
    while (region_->magic.load(std::memory_order_acquire) != kMagic) {
      if (std::chrono::steady_clock::now() > deadline) throw Error(ErrorCode::ConfigError, "shared: rank 0 never initialized");
      std::this_thread::sleep_for(std::chrono::milliseconds(1));
    }
    if (region_->world != cfg_.world) throw Error(ErrorCode::ConfigError, "shared: world size mismatch");
  }
}

SharedCoordinator::~SharedCoordinator() {
  if (region_) munmap(region_, bytes_);
  if (cfg_.rank == 0) shm_unlink(cfg_.name.c_str());
}

void SharedCoordinator::barrier() {
  Lock lock(&region_->mu);
  const std::uint64_t gen = region_->barrier_gen;
  if (++region_->barrier_count == region_->world) {
    region_->barrier_count = 0;
    ++region_->barrier_gen;
    pthread_cond_broadcast(&region_->cv);
    return;
  }
  timespec ts{};
  clock_gettime(CLOCK_MONOTONIC, &ts);
  ts.tv_sec += static_cast<time_t>(cfg_.barrier_timeout_s);
  while (gen == region_->barrier_gen) {
    if (pthread_cond_timedwait(&region_->cv, &region_->mu, &ts) == ETIMEDOUT && gen == region_->barrier_gen) {
      region_->failed = 1;
      throw Error(ErrorCode::KernelPanic, "shared: barrier timed out (a peer rank died or stalled)");
    }
  }
}

double SharedCoordinator::begin_run(const SchedulerConfig& sched, std::uint64_t total_wg,
                                    const std::vector<DeviceProfile>& devices) {
  barrier();  // every rank has finished reading the previous run
  if (cfg_.rank == 0) {
    Lock lock(&region_->mu);
    region_->log_len = region_->grants = region_->n_done = 0;
    region_->failed = 0;
    region_->epoch_ms = steady_now_ms();
  }
  barrier();
  sched_ = make_scheduler(sched, total_wg, devices);
  replayed_ = 0;
  device_ids_.clear();
  for (const DeviceProfile& d : devices) device_ids_.push_back(d.id);
  Lock lock(&region_->mu);
  return region_->epoch_ms;
}

void SharedCoordinator::replay() {
  for (; replayed_ < region_->log_len; ++replayed_) {
    const LogEntry& e = region_->log[replayed_];
    if (e.kind == 0) sched_->next(e.device);
    else sched_->observe(e.device, e.items, e.ms);
  }
}

bool SharedCoordinator::next(std::uint32_t device, PackageRange* range, std::uint64_t* seq) {
  Lock lock(&region_->mu);
  if (region_->failed) return false;
  replay();
  const auto r = sched_->next(device);
  if (!r) return false;
  if (region_->log_len >= kMaxLog) throw Error(ErrorCode::SchedulerError, "shared: decision log full");
  region_->log[region_->log_len++] = LogEntry{0, device, 0, 0.0};
  ++replayed_;
  *range = *r;
  *seq = region_->grants++;
  return true;
}

void SharedCoordinator::observe(std::uint32_t device, std::uint64_t items, double busy_ms) {
  Lock lock(&region_->mu);
  replay();
  if (region_->log_len >= kMaxLog) return;
  sched_->observe(device, items, busy_ms);
  region_->log[region_->log_len++] = LogEntry{1, device, items, busy_ms};
  ++replayed_;
}

void SharedCoordinator::complete(const Package& p) {
  Lock lock(&region_->mu);
  if (region_->n_done >= kMaxLog) return;
  region_->done[region_->n_done++] =
      DoneRec{p.seq, p.device_index, 0, p.offset_wg, p.size_wg, p.t_enqueue_ms, p.t_start_ms, p.t_end_ms};
}

void SharedCoordinator::fail() {
  Lock lock(&region_->mu);
  region_->failed = 1;
}

std::vector<Package> SharedCoordinator::end_run(bool* peer_failed) {
  barrier();  // every rank has completed its packages
  std::vector<Package> out;
  Lock lock(&region_->mu);
  replay();  // every rank's scheduler ends in the same state (learned powers)
  *peer_failed = region_->failed != 0;
  for (std::uint64_t i = 0; i < region_->n_done; ++i) {
    const DoneRec& r = region_->done[i];
    Package p;
    p.seq = r.seq;
    p.device_index = r.device;
    p.device_id = r.device < device_ids_.size() ? device_ids_[r.device] : std::to_string(r.device);
    p.offset_wg = r.offset_wg;
    p.size_wg = r.size_wg;
    p.t_enqueue_ms = r.t_enqueue;
    p.t_start_ms = r.t_start;
    p.t_end_ms = r.t_end;
    out.push_back(std::move(p));
  }
  std::sort(out.begin(), out.end(), [](const Package& a, const Package& b) { return a.seq < b.seq; });
  return out;
}

void SharedCoordinator::publish(std::uint32_t slot, const void* data, std::size_t n) {
  if (slot >= kBlobSlots || n > kBlobBytes) throw Error(ErrorCode::ConfigError, "shared: blob slot/size out of range");
  Lock lock(&region_->mu);
  std::memcpy(region_->blobs[cfg_.rank][slot], data, n);
}

void SharedCoordinator::fetch(std::uint32_t rank, std::uint32_t slot, void* data, std::size_t n) const {
  if (rank >= cfg_.world || slot >= kBlobSlots || n > kBlobBytes)
    throw Error(ErrorCode::ConfigError, "shared: blob rank/slot/size out of range");
  Lock lock(&region_->mu);
  std::memcpy(data, region_->blobs[rank][slot], n);
}

std::uint64_t SharedCoordinator::remaining() const {
  Lock lock(&region_->mu);
  const_cast<SharedCoordinator*>(this)->replay();
  return sched_ ? sched_->remaining_work_groups() : 0;
}

}  // namespace coexec
