// engine.hpp — the co-execution engine (reference: engine.hpp:21-446).
//
// Same surface — Engine(EngineConfig, ValidatedProgram).run(inputs) ->
// RunResult{outputs, trace} — with the device executor replaced: each Cuda
// device is one B200 behind include/ecl_cuda.h, driven by one persistent
// host thread that pulls packages from the mutex-serialized scheduler with
// up to Backend::queue_depth packages in flight, so the next package is
// already queued on the GPU when the current one ends.
//
// Additions for the B200 build:
//   run_into()     caller-owned host outputs (the paper's program.out(v),
//                  PAPER.md:366) — pinned buffers get async D2H per package
//                  overlapped with the next package's kernel; nullptr
//                  outputs keep results device-resident (gather() later).
//   run_virtual()  the virtual-clock replay (engine.hpp:306-338) with
//                  caller-supplied per-item costs; trace only.
//   native_run()   one launch over the whole grid: the overhead denominator;
//   native_run_split()  the same grid as plain sub-launches on two streams.
#pragma once

#include <cstddef>
#include <cstdint>
#include <functional>
#include <memory>
#include <string>
#include <span>
#include <utility>
#include <vector>

#include <optional>

#include "coexec/core.hpp"
#include "coexec/schedulers.hpp"
#include "coexec/shared.hpp"

namespace coexec {

struct EngineConfig {
  std::vector<DeviceProfile> devices;
  SchedulerConfig scheduler;
  ClockMode clock_mode = ClockMode::Wall;
  std::uint64_t seed = 0;
  bool exclude_init_from_total = false;
  bool tally = false;  // exactly-once check (also enabled by COEXEC_TALLY=1)
  // One process per GPU: this process drives shared->local of `devices` and
  // co-schedules with its peers through the shared-memory decision log
  // (coexec/shared.hpp).  Unset = one process drives every device.
  std::optional<SharedConfig> shared;
};

struct RunResult {
  std::vector<std::vector<std::byte>> outputs;
  ExecutionTrace trace;
};

struct NativeResult {
  double kernel_ms = 0.0;  // CUDA-event time of the single launch
  double total_ms = 0.0;   // host wall time: first H2D -> last D2H
};

/// A device kernel by id — the B200 form of the reference's KernelFn
/// (workloads.hpp:44): a built-in ("vecscale", "mandelbrot@3", ...) or a
/// kernel registered with register_device_kernel (include/ecl_plugin.h ABI).
struct DeviceKernel {
  std::string id;
};

/// Per-work-item cost for the virtual clock (reference CostFn, workloads.hpp:47).
using CostFn = std::function<double(std::uint64_t index)>;

/// Registers a device kernel image (cubin / fatbin / NUL-terminated PTX for
/// sm_100a) whose `entry` follows include/ecl_plugin.h; throws Error.
DeviceKernel register_device_kernel(const std::string& id, std::span<const std::byte> image, const std::string& entry);
/// The same from a file (a .cubin / .fatbin / .ptx written by nvcc).
DeviceKernel register_device_kernel_file(const std::string& id, const std::string& path, const std::string& entry);

struct KernelTiming {
  double kernel_ms = 0.0;  // summed CUDA-event time of every package launch
  std::uint64_t launches = 0;
};

class Engine {
 public:
  Engine(EngineConfig cfg, ValidatedProgram prog);
  ~Engine();
  Engine(const Engine&) = delete;
  Engine& operator=(const Engine&) = delete;

  /// Reference semantics (engine.hpp:219-256): engine-allocated outputs.
  RunResult run(std::span<const std::vector<std::byte>> inputs);

  /// The reference's run(inputs, kernel, cost) (engine.hpp:223): this run
  /// executes `kernel` (same program geometry) on every device instead of the
  /// program's kernel; `cost` is the virtual clock's model, which a wall run
  /// does not use (as in drive_wall).  Virtual engines throw ConfigError
  /// (trace only: run_virtual(cost)).
  RunResult run(std::span<const std::vector<std::byte>> inputs, const DeviceKernel& kernel, const CostFn& cost);
  /// run_into with a kernel override (caller-owned buffers).
  ExecutionTrace run_into(std::span<const void* const> inputs, std::span<void* const> outputs,
                          const DeviceKernel& kernel);

  /// Caller-owned buffers; inputs[i] must hold in_buffers[i].size_bytes()
  /// bytes.  outputs empty (or all null) = device-resident run.
  ExecutionTrace run_into(std::span<const void* const> inputs, std::span<void* const> outputs);

  /// Iterative program: `steps` passes; between passes every (input i,
  /// output o) pair in `swaps` is exchanged across devices (owner slices over
  /// NVLink) and swapped in place.  Outputs gathered after the last pass.
  ExecutionTrace run_steps(std::span<const void* const> inputs, std::span<void* const> outputs, std::uint32_t steps,
                           std::span<const std::pair<std::uint32_t, std::uint32_t>> swaps);

  /// Virtual clock (simulated devices): per-item costs, one per work-item;
  /// empty = the analytic cost of vecscale/synthetic kernels.
  ExecutionTrace run_virtual(std::span<const double> item_costs);
  /// The same with a cost function evaluated per work-item.
  ExecutionTrace run_virtual(const CostFn& cost);

  /// Copies the last device-resident run's slices to host buffers.
  void gather(std::span<void* const> outputs);

  /// One kernel launch over the whole grid on the first device, same
  /// uploads/downloads as run_into (outputs may be empty).
  NativeResult native_run(std::span<const void* const> inputs, std::span<void* const> outputs);
  // The same kernel as launches of items_per_launch work-items alternating
  // over the first device's compute lanes (resident outputs, no scheduler):
  // returns the kernel span in ms.
  double native_run_split(std::uint64_t items_per_launch);

  KernelTiming kernel_timing(bool reset);
  /// Adaptive HGuided: the per-device work-items/ms the last run measured,
  /// which seed the next run (empty before a run measured every device).
  std::vector<double> learned_powers() const;
  const ExecutionTrace& last_trace() const;
  double init_ms() const;
  const ValidatedProgram& program() const;
  const EngineConfig& config() const;

 private:
  struct Impl;
  std::unique_ptr<Impl> impl_;
};

/// Reference free function (engine.hpp:440-444).
inline RunResult run(const EngineConfig& cfg, const ValidatedProgram& prog,
                     std::span<const std::vector<std::byte>> inputs) {
  Engine engine(cfg, prog);
  return engine.run(inputs);
}

}  // namespace coexec
