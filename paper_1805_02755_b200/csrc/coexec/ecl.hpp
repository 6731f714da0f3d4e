// ecl.hpp — the EngineCL programming interface over the
// B200 co-execution engine.
//
//   ecl::EngineCL engine;
//   engine.use(ecl::Device(0), ecl::Device(1));          // B200 ordinals
//   engine.work_items(gws, lws);                          // or global_/local_work_items
//   engine.scheduler(ecl::Scheduler::HGuided(2.0));       // Static(props) / Dynamic(n)
//   ecl::Program program;
//   program.in(in_vec);  program.out(out_vec);            // caller-owned containers
//   program.out_pattern(1, lws);
//   program.kernel("binomial");                           // registered sm_100a kernel id
//   program.args(steps);                                  // scalar args (positional: arg(i, v))
//   engine.program(std::move(program));
//   engine.run();
//   if (engine.has_errors()) for (auto& e : engine.get_errors()) ...
//
// Listing 1/2 differences: kernels are ids of the compiled sm_100a registry
// (no OpenCL source strings); buffers passed to args() are ignored (they are
// bound by in()/out() order, as in Table 2); LocalAlloc arguments are
// accepted and ignored (the kernels size their shared memory themselves).
// Types map onto coexec: Program -> ProgramSpec, Device -> DeviceProfile
// (BackendKind::Cuda), errors -> EngineFailure.
#pragma once

#include <cstdint>
#include <cstring>
#include <memory>
#include <string>
#include <type_traits>
#include <utility>
#include <variant>
#include <vector>

#include "coexec/engine.hpp"

namespace ecl {

/// One B200 (paper: Device(platform, device[, kernel])).  `power` seeds
/// HGuided (work-items/ms); queue_depth 1 restores one package in flight.
struct Device {
  explicit Device(int ordinal = 0, double power = 1.0, std::uint32_t queue_depth = 2,
                  std::uint64_t min_package_work_groups = 0)
      : ordinal(ordinal), power(power), queue_depth(queue_depth), min_package_work_groups(min_package_work_groups) {}
  /// Paper: Device(platform, device, kernel) — this device runs its own
  /// specialization of the program's kernel ("<kernel>@<variant>").
  Device(int ordinal, std::string kernel) : Device(ordinal) { this->kernel = std::move(kernel); }
  int ordinal;
  double power;
  std::uint32_t queue_depth;
  std::uint64_t min_package_work_groups;  // 0 = coexec's power-ratio heuristic
  std::string kernel;                     // "" = the program's kernel
};

/// Scheduler selection.
struct Scheduler {
  static coexec::SchedulerConfig Static(std::vector<double> props = {}) {
    return coexec::StaticConfig{std::move(props), {}};
  }
  static coexec::SchedulerConfig Dynamic(std::uint64_t packages) { return coexec::DynamicConfig{packages}; }
  static coexec::SchedulerConfig HGuided(double k = 2.0, bool measured_powers = false) {
    coexec::HGuidedConfig c;
    c.k = k;
    c.adaptive = measured_powers;
    return c;
  }
};

enum class Arg { LocalAlloc };

class Program {
 public:
  template <typename T>
  Program& in(std::vector<T>& v) {
    ins_.push_back(Buf{v.data(), sizeof(T), v.size()});
    return *this;
  }
  template <typename T>
  Program& out(std::vector<T>& v) {
    outs_.push_back(Buf{v.data(), sizeof(T), v.size()});
    return *this;
  }
  Program& out_pattern(std::uint64_t out_indices, std::uint64_t work_items) {
    pattern_ = {out_indices, work_items};
    return *this;
  }
  Program& kernel(std::string id) {
    kernel_ = std::move(id);
    return *this;
  }
  /// Aggregate argument: scalars append a kernel argument; containers are
  /// the in()/out() buffers and are skipped (Listing 1).
  template <typename T>
  Program& arg(const T& v) {
    push(v);
    return *this;
  }
  /// Positional argument: index i of the scalar argument list.
  template <typename T>
  Program& arg(std::size_t i, const T& v) {
    if constexpr (std::is_arithmetic_v<T>) {
      if (args_.size() <= i) args_.resize(i + 1, std::int64_t{0});
      args_[i] = to_arg(v);
    }
    return *this;
  }
  Program& arg(std::size_t /*bytes*/, Arg) { return *this; }  // LocalAlloc: sized by the kernel
  Program& arg(std::size_t /*index*/, std::size_t /*bytes*/, Arg) { return *this; }
  template <typename... Ts>
  Program& args(const Ts&... vs) {
    (push(vs), ...);
    return *this;
  }

 private:
  friend class EngineCL;
  struct Buf {
    void* data;
    std::uint64_t elem;
    std::uint64_t count;
  };
  template <typename T>
  static coexec::ArgValue to_arg(const T& v) {
    if constexpr (std::is_integral_v<T>) return static_cast<std::int64_t>(v);
    else return static_cast<double>(v);
  }
  template <typename T>
  void push(const T& v) {
    if constexpr (std::is_arithmetic_v<T>) args_.push_back(to_arg(v));
  }
  std::vector<Buf> ins_, outs_;
  coexec::OutPattern pattern_{1, 1};
  std::string kernel_;
  std::vector<coexec::ArgValue> args_;
};

class EngineCL {
 public:
  template <typename... Ds>
  void use(Ds&&... ds) {
    (devices_.push_back(std::forward<Ds>(ds)), ...);
  }
  void work_items(std::uint64_t gws, std::uint64_t lws) {
    gws_ = gws;
    lws_ = lws;
  }
  void global_work_items(std::uint64_t gws) { gws_ = gws; }
  void local_work_items(std::uint64_t lws) { lws_ = lws; }
  void scheduler(coexec::SchedulerConfig s) { sched_ = std::move(s); }
  void program(Program p) { prog_ = std::move(p); }
  void use(Program p) { prog_ = std::move(p); }  // Listing 1 spells it engine.use(std::move(program))

  /// Runs the program; errors are collected, not thrown (has_errors()).
  void run() {
    errors_.clear();
    try {
      if (!engine_) build();
      std::vector<const void*> in;
      for (const auto& b : prog_.ins_) in.push_back(b.data);
      std::vector<void*> out;
      for (const auto& b : prog_.outs_) out.push_back(b.data);
      trace_ = engine_->run_into(in, out);
    } catch (const coexec::EngineFailure& f) {
      errors_ = f.errors();
    } catch (const coexec::Error& e) {
      errors_.push_back(e);
    }
  }

  bool has_errors() const { return !errors_.empty(); }
  const std::vector<coexec::Error>& get_errors() const { return errors_; }
  /// The run's introspection data: packages, timestamps, times.
  const coexec::ExecutionTrace& trace() const { return trace_; }

 private:
  void build() {
    coexec::ProgramSpec spec;
    spec.global_work_size = gws_;
    spec.local_work_size = lws_;
    for (const auto& b : prog_.ins_) spec.in_buffers.push_back({"in", b.elem, b.count, coexec::BufferRole::Input});
    for (const auto& b : prog_.outs_)
      spec.out_buffers.push_back({"out", b.elem, b.count, coexec::BufferRole::Output});
    spec.out_pattern = prog_.pattern_;
    spec.kernel = prog_.kernel_;
    spec.args = prog_.args_;
    coexec::EngineConfig cfg;
    for (std::size_t i = 0; i < devices_.size(); ++i) {
      coexec::DeviceProfile d;
      d.id = "gpu" + std::to_string(i);
      d.name = d.id;
      d.computing_power = devices_[i].power;
      d.backend.kind = coexec::BackendKind::Cuda;
      d.backend.ordinal = devices_[i].ordinal;
      d.backend.queue_depth = devices_[i].queue_depth;
      d.min_package_work_groups = devices_[i].min_package_work_groups;
      d.kernel = devices_[i].kernel;
      cfg.devices.push_back(d);
    }
    if (cfg.devices.empty()) {
      coexec::DeviceProfile d;
      d.id = "gpu0";
      d.name = d.id;
      d.backend.kind = coexec::BackendKind::Cuda;
      cfg.devices.push_back(d);
    }
    coexec::apply_default_min_package(cfg.devices);
    cfg.scheduler = sched_;
    cfg.clock_mode = coexec::ClockMode::Wall;
    engine_ = std::make_unique<coexec::Engine>(std::move(cfg), coexec::validate_program(std::move(spec)));
  }

  std::vector<Device> devices_;
  std::uint64_t gws_ = 0, lws_ = 1;
  coexec::SchedulerConfig sched_ = coexec::StaticConfig{};
  Program prog_;
  std::unique_ptr<coexec::Engine> engine_;
  std::vector<coexec::Error> errors_;
  coexec::ExecutionTrace trace_;
};

}  // namespace ecl
