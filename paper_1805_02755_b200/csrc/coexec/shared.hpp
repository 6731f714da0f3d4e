// shared.hpp — cross-process coordinator for one-process-per-GPU co-execution.
//
// The reference serializes scheduler access between its per-device threads
// with one mutex (engine.hpp:357,370).  When every B200 is driven by its own
// process (torchrun: one rank per GPU), the equivalent is a POSIX
// shared-memory segment holding a process-shared mutex and the run's
// *decision log*: every grant ("device d asked, got the next package") and
// every throughput observation, in order.  Each process keeps its own
// scheduler instance and replays the log entries it has not seen before
// deciding, so all ranks drive the very same Static/Dynamic/HGuided code
// (schedulers.hpp) and agree on every package without serializing scheduler
// state.  Completed packages are appended to the segment so every rank can
// assemble the whole run's trace.  No data-path collective: outputs land in
// disjoint slices on each rank's GPU.
#pragma once

#include <cstdint>
#include <memory>
#include <optional>
#include <string>
#include <vector>

#include "coexec/core.hpp"
#include "coexec/schedulers.hpp"

namespace coexec {

struct SharedConfig {
  std::string name;                     // shm object name, e.g. "/ecl_run_1234"
  std::uint32_t rank = 0;               // this process
  std::uint32_t world = 1;              // processes sharing the run
  std::vector<std::uint32_t> local;     // device indices (into the device list) this process drives
  double barrier_timeout_s = 120.0;
};

class SharedCoordinator {
 public:
  explicit SharedCoordinator(SharedConfig cfg);  // rank 0 creates the segment, others attach
  ~SharedCoordinator();
  SharedCoordinator(const SharedCoordinator&) = delete;
  SharedCoordinator& operator=(const SharedCoordinator&) = delete;

  /// Collective: starts a run; returns the shared run epoch (steady-clock ms).
  double begin_run(const SchedulerConfig& sched, std::uint64_t total_wg, const std::vector<DeviceProfile>& devices);
  /// Next package for `device` (replays peers' decisions first); false when drained or aborted.
  bool next(std::uint32_t device, PackageRange* range, std::uint64_t* seq);
  void observe(std::uint32_t device, std::uint64_t items, double busy_ms);
  void complete(const Package& pkg);
  void fail();
  /// Collective: ends the run; returns every rank's packages (seq order) and
  /// whether any rank failed.
  std::vector<Package> end_run(bool* peer_failed);
  void barrier();
  /// Small per-rank blobs (CUDA IPC handles, device lists) exchanged through
  /// the segment: publish writes this rank's slot; after a barrier() every
  /// rank can fetch any rank's slot.  n <= kBlobBytes, slot < kBlobSlots.
  static constexpr std::size_t kBlobBytes = 64, kBlobSlots = 16, kMaxRanks = 64;
  void publish(std::uint32_t slot, const void* data, std::size_t n);
  void fetch(std::uint32_t rank, std::uint32_t slot, void* data, std::size_t n) const;

  /// The run's adaptive-HGuided powers (identical on every rank: end_run
  /// replays the whole decision log first); empty if not learned.
  std::vector<double> learned_powers() const { return sched_ ? sched_->learned_powers() : std::vector<double>{}; }
  const SharedConfig& config() const { return cfg_; }
  std::uint64_t remaining() const;

 private:
  struct Region;
  void replay();  // caller holds the lock
  SharedConfig cfg_;
  Region* region_ = nullptr;
  std::size_t bytes_ = 0;
  std::unique_ptr<Scheduler> sched_;
  std::uint64_t replayed_ = 0;
  std::vector<std::string> device_ids_;
};

}  // namespace coexec
