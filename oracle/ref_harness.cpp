// ref_harness.cpp — C entry points over the UNMODIFIED reference headers.
//
// TEST INFRASTRUCTURE ONLY.  oracle/Makefile compiles this file against
// /root/reference/proj/include (read in place, never copied) into
// oracle/_ref/libcoexec_ref.so.  It lets the tests and bench.py's reference
// arm call the reference's own code paths:
//   * kernel arithmetic   — mandel_count_for_index      workloads.hpp:94-100
//   * schedulers          — make_scheduler + the drain emulator of
//                           test_schedulers.cpp:27-49
//   * engine (virtual)    — Engine::run / drive_virtual  engine.hpp:219-338
//   * engine (wall)       — Engine::run / drive_wall     engine.hpp:354-405
//   * metrics             — make_report                  metrics.hpp:104-117
// Nothing in the product loads this library.

#include <chrono>
#include <cmath>
#include <cstring>
#include <string>

#include "coexec/config.hpp"
#include "coexec/engine.hpp"
#include "coexec/experiment.hpp"
#include "coexec/metrics.hpp"
#include "coexec/trace_io.hpp"
#include "coexec/workloads.hpp"

using namespace coexec;

// This repo's C restatements (oracle/oracle.c), linked into the same library.
extern "C" {
void orc_gaussian(const float* img, const float* filt, float* out, uint32_t w, uint32_t h, uint32_t f, uint64_t first,
                  uint64_t count);
void orc_nbody_step(const float* pos, const float* vel, uint64_t n, float dt, float eps2, float* npos, float* nvel,
                    uint64_t first, uint64_t count);
void orc_binomial(const float* rand4, float* out4, uint32_t steps, uint64_t first_opt, uint64_t n_opt);
void orc_ray(const float* scene, uint32_t ns, uint32_t w, uint32_t h, uint32_t max_depth, float* out4, uint64_t first,
             uint64_t count, uint64_t* counts3);
}

namespace {

thread_local std::string g_error;

int64_t copy_out(const std::string& s, char* out, uint64_t cap) {
  if (out && cap > s.size()) std::memcpy(out, s.c_str(), s.size() + 1);
  return static_cast<int64_t>(s.size());
}

std::vector<DeviceProfile> devices_from(const json& arr) {
  std::vector<DeviceProfile> devices;
  for (const auto& d : arr) devices.push_back(device_from_json(d));
  apply_default_min_package(devices);
  return devices;
}

uint64_t fnv1a(const std::vector<std::vector<std::byte>>& bufs) {
  uint64_t h = 0xcbf29ce484222325ull;
  for (const auto& b : bufs)
    for (std::byte c : b) {
      h ^= static_cast<uint8_t>(c);
      h *= 0x100000001b3ull;
    }
  return h;
}

}  // namespace

extern "C" {

const char* ref_last_error() { return g_error.c_str(); }

void ref_mandelbrot_counts(uint64_t w, uint64_t h, uint32_t iters, double x0, double y0, double x1,
                           double y1, uint64_t first, uint64_t count, uint32_t* out) {
  const MandelParams p{w, h, iters, x0, y0, x1, y1};
  for (uint64_t k = 0; k < count; ++k) out[k] = mandel_count_for_index(first + k, p);
}

// Drains a scheduler the way test_schedulers.cpp:27-49 does (every idle device
// asks in index order).  out receives (device, offset, size) triples.
int64_t ref_drain(const char* sched_json, const char* devices_json, uint64_t total_wg, uint64_t* out,
                  uint64_t cap) {
  try {
    auto devices = devices_from(json::parse(devices_json));
    auto sched = make_scheduler(scheduler_from_json(json::parse(sched_json)), total_wg, devices);
    uint64_t n = 0;
    bool granted = true;
    while (granted) {
      granted = false;
      for (uint32_t d = 0; d < devices.size(); ++d) {
        if (auto r = sched->next(d)) {
          if (3 * n + 2 < cap) {
            out[3 * n] = d;
            out[3 * n + 1] = r->offset_wg;
            out[3 * n + 2] = r->size_wg;
          }
          ++n;
          granted = true;
        }
      }
    }
    return static_cast<int64_t>(n);
  } catch (const std::exception& e) {
    g_error = e.what();
    return -1;
  }
}

// Runs the reference Engine on {"program", "devices", "scheduler",
// "clock_mode", "seed", "exclude_init"} with fill_default_inputs(seed) and
// returns the trace JSON (schema 1); *fnv gets FNV-1a-64 over the outputs.
int64_t ref_run_json(const char* config_json, char* out, uint64_t cap, uint64_t* fnv) {
  try {
    const json j = json::parse(config_json);
    EngineConfig cfg;
    cfg.devices = devices_from(j.at("devices"));
    cfg.scheduler = scheduler_from_json(j.at("scheduler"));
    cfg.clock_mode = j.value("clock_mode", std::string("virtual")) == "wall" ? ClockMode::Wall
                                                                             : ClockMode::Virtual;
    cfg.seed = j.value("seed", uint64_t{0});
    cfg.exclude_init_from_total = j.value("exclude_init", false);
    const auto prog = validate_program(program_from_json(j.at("program")));
    const auto inputs = fill_default_inputs(prog, cfg.seed);
    const auto result = run(cfg, prog, inputs);
    if (fnv) *fnv = fnv1a(result.outputs);
    return copy_out(trace_to_json_string(result.trace), out, cap);
  } catch (const std::exception& e) {
    g_error = e.what();
    return -1;
  }
}

// CPU baseline: the reference engine in Wall mode with `devices` NativePool
// devices of `workers` threads each and Dynamic{num_packages}.  Returns the
// wall seconds of Engine::run (construction excluded), -1 on error.
double ref_wall_run(const char* program_json, uint32_t devices, uint32_t workers, uint64_t num_packages,
                    uint64_t seed, uint64_t* fnv) {
  try {
    const auto prog = validate_program(program_from_json(json::parse(program_json)));
    EngineConfig cfg;
    for (uint32_t d = 0; d < devices; ++d) {
      DeviceProfile dev;
      dev.id = "cpu" + std::to_string(d);
      dev.name = dev.id;
      dev.backend = {BackendKind::NativePool, workers};
      cfg.devices.push_back(dev);
    }
    cfg.scheduler = DynamicConfig{num_packages};
    cfg.clock_mode = ClockMode::Wall;
    cfg.seed = seed;
    const auto inputs = fill_default_inputs(prog, seed);
    Engine engine(cfg, prog);
    const auto t0 = std::chrono::steady_clock::now();
    const auto result = engine.run(inputs);
    const double s = std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
    if (fnv) *fnv = fnv1a(result.outputs);
    return s;
  } catch (const std::exception& e) {
    g_error = e.what();
    return -1.0;
  }
}

// The same with any scheduler (config.hpp:41 scheduler_from_json), so the
// reference arm runs the very configuration the B200 arm runs (HGuided k=2
// for Mandelbrot).  `devices` NativePool devices x `workers` threads each.
double ref_wall_run_sched(const char* program_json, const char* scheduler_json, uint32_t devices, uint32_t workers,
                          uint64_t seed, uint64_t* fnv) {
  try {
    const auto prog = validate_program(program_from_json(json::parse(program_json)));
    EngineConfig cfg;
    for (uint32_t d = 0; d < devices; ++d) {
      DeviceProfile dev;
      dev.id = "cpu" + std::to_string(d);
      dev.name = dev.id;
      dev.backend = {BackendKind::NativePool, workers};
      cfg.devices.push_back(dev);
    }
    apply_default_min_package(cfg.devices);
    cfg.scheduler = scheduler_from_json(json::parse(scheduler_json));
    cfg.clock_mode = ClockMode::Wall;
    cfg.seed = seed;
    const auto inputs = fill_default_inputs(prog, seed);
    Engine engine(cfg, prog);
    const auto t0 = std::chrono::steady_clock::now();
    const auto result = engine.run(inputs);
    const double s = std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
    if (fnv) *fnv = fnv1a(result.outputs);
    return s;
  } catch (const std::exception& e) {
    g_error = e.what();
    return -1.0;
  }
}

// make_report over a trace JSON; reference_ms < 0 means "no overhead".
int64_t ref_report_json(const char* trace_json, const double* solo, uint32_t nsolo, double reference_ms,
                        char* out, uint64_t cap) {
  try {
    const auto trace = trace_from_json(json::parse(trace_json));
    std::optional<double> ref;
    if (reference_ms >= 0.0) ref = reference_ms;
    const auto report = make_report(trace, std::span<const double>(solo, nsolo), ref);
    return copy_out(to_json(report).dump(), out, cap);
  } catch (const std::exception& e) {
    g_error = e.what();
    return -1;
  }
}

// CPU baseline for the kernels the reference does not have (SURVEY §8d,
// BASELINE.md §3): the reference engine itself in wall mode (devices x 1
// worker, the given scheduler; NULL = Dynamic{max(64,16*devices)}) drives
// this repo's C restatement, injected as a KernelFn through
// Engine::run(inputs, kernel, cost) (engine.hpp:223).  Work-item i of the
// program is item i*stride of the real workload (stride 1 = the whole
// workload).  Returns wall seconds of Engine::run, -1 on error.
double ref_wall_run_restated(const char* kind, const void* in0, const void* in1, void* out, uint64_t sample,
                             uint64_t stride, const double* p, uint32_t devices, const char* scheduler_json) {
  try {
    const std::string k = kind;
    KernelFn fn;
    std::vector<float> scratch;
    if (k == "gaussian") {
      fn = [=](std::uint64_t i, std::span<const ArgValue>, const KernelBuffers&) {
        orc_gaussian(static_cast<const float*>(in0), static_cast<const float*>(in1), static_cast<float*>(out),
                     static_cast<uint32_t>(p[0]), static_cast<uint32_t>(p[1]), static_cast<uint32_t>(p[2]), i * stride, 1);
      };
    } else if (k == "nbody") {
      scratch.resize(4 * static_cast<size_t>(p[0]));
      float* nvel = scratch.data();
      fn = [=](std::uint64_t i, std::span<const ArgValue>, const KernelBuffers&) {
        orc_nbody_step(static_cast<const float*>(in0), static_cast<const float*>(in1), static_cast<uint64_t>(p[0]),
                       static_cast<float>(p[1]), static_cast<float>(p[2]), static_cast<float*>(out), nvel, i * stride, 1);
      };
    } else if (k == "binomial") {
      fn = [=](std::uint64_t i, std::span<const ArgValue>, const KernelBuffers&) {
        orc_binomial(static_cast<const float*>(in0), static_cast<float*>(out), static_cast<uint32_t>(p[0]), i * stride, 1);
      };
    } else if (k == "ray") {
      fn = [=](std::uint64_t i, std::span<const ArgValue>, const KernelBuffers&) {
        orc_ray(static_cast<const float*>(in0), static_cast<uint32_t>(p[2]), static_cast<uint32_t>(p[0]),
                static_cast<uint32_t>(p[1]), static_cast<uint32_t>(p[3]), static_cast<float*>(out), i * stride, 1,
                nullptr);
      };
    } else {
      throw Error(ErrorCode::UnknownKernel, "restated kernel '" + k + "'");
    }
    ProgramSpec spec;
    spec.kernel = "synthetic:constant";
    spec.global_work_size = sample;
    spec.local_work_size = 1;
    spec.out_buffers.push_back({"unused", 8, sample, BufferRole::Output});
    const auto prog = validate_program(spec);
    EngineConfig cfg;
    for (uint32_t d = 0; d < devices; ++d) {
      DeviceProfile dev;
      dev.id = "cpu" + std::to_string(d);
      dev.name = dev.id;
      dev.backend = {BackendKind::NativePool, 1};
      cfg.devices.push_back(dev);
    }
    if (scheduler_json)
      cfg.scheduler = scheduler_from_json(json::parse(scheduler_json));
    else
      cfg.scheduler = DynamicConfig{std::max<uint64_t>(64, 16ull * devices)};
    cfg.clock_mode = ClockMode::Wall;
    Engine engine(cfg, prog);
    const CostFn cost = [](std::uint64_t) { return 1.0; };
    const auto t0 = std::chrono::steady_clock::now();
    engine.run({}, fn, cost);
    return std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
  } catch (const std::exception& e) {
    g_error = e.what();
    return -1.0;
  }
}

// out_range_for / validate_program probes for the boundary tests.
int ref_out_range(const char* program_json, uint64_t offset_wg, uint64_t size_wg, uint64_t* off,
                  uint64_t* count) {
  try {
    const auto prog = validate_program(program_from_json(json::parse(program_json)));
    Package pkg;
    pkg.offset_wg = offset_wg;
    pkg.size_wg = size_wg;
    const auto r = out_range_for(pkg, prog);
    *off = r.offset;
    *count = r.count;
    return 0;
  } catch (const Error& e) {
    g_error = e.what();
    return 1 + static_cast<int>(e.code());
  } catch (const std::exception& e) {
    g_error = e.what();
    return -1;
  }
}

// The reference's experiment harness (experiment.hpp:67-181) on one
// experiment file, output_dir overridden; returns 0 or -1 (message in out).
int ref_run_experiment(const char* config_path, const char* out_dir, char* out, uint64_t cap) {
  try {
    coexec::ExperimentConfig cfg = coexec::load_experiment(config_path);
    cfg.output_dir = out_dir;
    coexec::RunOptions opts;
    coexec::run_experiment(cfg, opts);
    return 0;
  } catch (const std::exception& e) {
    copy_out(e.what(), out, cap);
    return -1;
  }
}

}  // extern "C"
