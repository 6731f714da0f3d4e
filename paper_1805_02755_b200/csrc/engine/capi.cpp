// capi.cpp — include/ecl_engine.h over the C++ engine.  Exceptions stop here:
// coexec::Error becomes its negative status, EngineFailure keeps its error
// list on the engine handle (ecl_engine_error*), anything else is a
// KernelPanic.
#include <cstring>
#include <memory>
#include <string>
#include <vector>

#include "coexec/chart.hpp"
#include "coexec/engine.hpp"
#include "coexec/experiment.hpp"
#include "coexec/json_io.hpp"
#include "ecl_engine.h"

using namespace coexec;

struct ecl_engine {
  std::unique_ptr<Engine> engine;
  std::vector<Error> errors;
};

struct ecl_scheduler {
  std::unique_ptr<Scheduler> impl;
};

namespace {

thread_local std::string t_error;

int64_t emit(const std::string& s, char* buf, uint64_t cap) {
  if (buf && cap > s.size()) std::memcpy(buf, s.c_str(), s.size() + 1);
  return static_cast<int64_t>(s.size());
}

template <typename F>
int guarded(ecl_engine* e, F&& body) {
  try {
    if (e) e->errors.clear();
    body();
    return ECL_OK;
  } catch (const EngineFailure& f) {
    t_error = f.what();
    if (e) e->errors = f.errors();
    return f.errors().empty() ? ECL_KERNEL_PANIC : status_of(f.errors().front().code());
  } catch (const Error& err) {
    t_error = err.what();  // a single Error, not an EngineFailure aggregate
    return status_of(err.code());
  } catch (const json::exception& je) {
    t_error = std::string("ConfigError: ") + je.what();
    return status_of(ErrorCode::ConfigError);
  } catch (const std::exception& ex) {
    t_error = std::string("KernelPanic: ") + ex.what();
    return status_of(ErrorCode::KernelPanic);
  }
}

template <typename F>
int64_t guarded_string(F&& body, char* buf, uint64_t cap) {
  std::string out;
  const int rc = guarded(nullptr, [&] { out = body(); });
  return rc == ECL_OK ? emit(out, buf, cap) : rc;
}

std::vector<DeviceProfile> devices_from(const json& arr) {
  std::vector<DeviceProfile> d;
  for (const json& x : arr) d.push_back(device_from_json(x));
  apply_default_min_package(d);
  return d;
}

}  // namespace

extern "C" {

const char* ecl_engine_last_error(void) { return t_error.c_str(); }

int ecl_engine_create(const char* config_json, ecl_engine** out) {
  *out = nullptr;
  auto handle = std::make_unique<ecl_engine>();
  const int rc = guarded(handle.get(), [&] {
    const json j = json::parse(config_json);
    if (j.value("schema", 1) != 1) throw Error(ErrorCode::ConfigError, "unsupported config schema version");
    EngineConfig cfg;
    cfg.devices = devices_from(j.at("devices"));
    cfg.scheduler = scheduler_from_json(j.at("scheduler"));
    cfg.clock_mode = j.value("clock_mode", std::string("wall")) == "virtual" ? ClockMode::Virtual : ClockMode::Wall;
    cfg.seed = j.value("seed", std::uint64_t{0});
    cfg.exclude_init_from_total = j.value("exclude_init", false);
    cfg.tally = j.value("tally", false);
    if (j.contains("shared")) {
      const json& s = j.at("shared");
      SharedConfig sc;
      sc.name = s.at("name").get<std::string>();
      sc.rank = s.at("rank").get<std::uint32_t>();
      sc.world = s.at("world").get<std::uint32_t>();
      sc.local = s.at("local_devices").get<std::vector<std::uint32_t>>();
      sc.barrier_timeout_s = s.value("barrier_timeout_s", 120.0);
      cfg.shared = sc;
    }
    handle->engine = std::make_unique<Engine>(std::move(cfg), validate_program(program_from_json(j.at("program"))));
  });
  if (rc == ECL_OK) *out = handle.release();
  return rc;
}

void ecl_engine_destroy(ecl_engine* e) { delete e; }

int ecl_engine_run(ecl_engine* e, const void* const* inputs, uint32_t n_in, void* const* outputs, uint32_t n_out) {
  return guarded(e, [&] {
    std::span<const void* const> in(inputs, inputs ? n_in : 0);
    std::span<void* const> out(outputs, outputs ? n_out : 0);
    e->engine->run_into(in, out);
  });
}

int ecl_engine_run_kernel(ecl_engine* e, const char* kernel_id, const void* const* inputs, uint32_t n_in,
                          void* const* outputs, uint32_t n_out) {
  return guarded(e, [&] {
    if (!kernel_id) throw coexec::Error(coexec::ErrorCode::UnknownKernel, "null kernel id");
    std::span<const void* const> in(inputs, inputs ? n_in : 0);
    std::span<void* const> out(outputs, outputs ? n_out : 0);
    e->engine->run_into(in, out, coexec::DeviceKernel{kernel_id});
  });
}

int ecl_engine_learned_powers(const ecl_engine* e, double* powers, uint32_t cap, uint32_t* n) {
  const std::vector<double> p = e->engine->learned_powers();
  *n = static_cast<uint32_t>(p.size());
  for (uint32_t i = 0; i < p.size() && i < cap; ++i) powers[i] = p[i];
  return ECL_OK;
}

int ecl_engine_run_steps(ecl_engine* e, const void* const* inputs, uint32_t n_in, void* const* outputs,
                         uint32_t n_out, uint32_t steps, const uint32_t* swap_in, const uint32_t* swap_out,
                         uint32_t n_swaps) {
  return guarded(e, [&] {
    std::vector<std::pair<std::uint32_t, std::uint32_t>> swaps;
    for (uint32_t k = 0; k < n_swaps; ++k) swaps.emplace_back(swap_in[k], swap_out[k]);
    e->engine->run_steps(std::span<const void* const>(inputs, inputs ? n_in : 0),
                         std::span<void* const>(outputs, outputs ? n_out : 0), steps, swaps);
  });
}

int ecl_engine_run_virtual(ecl_engine* e, const double* costs, uint64_t n) {
  return guarded(e, [&] { e->engine->run_virtual(std::span<const double>(costs, costs ? n : 0)); });
}

int ecl_engine_gather(ecl_engine* e, void* const* outputs, uint32_t n_out) {
  return guarded(e, [&] { e->engine->gather(std::span<void* const>(outputs, n_out)); });
}

int64_t ecl_engine_trace_json(ecl_engine* e, char* buf, uint64_t cap) {
  return guarded_string([&] { return trace_to_json_string(e->engine->last_trace()); }, buf, cap);
}

int ecl_engine_native_run(ecl_engine* e, const void* const* inputs, uint32_t n_in, void* const* outputs,
                          uint32_t n_out, double* kernel_ms, double* total_ms) {
  return guarded(e, [&] {
    const NativeResult r = e->engine->native_run(std::span<const void* const>(inputs, inputs ? n_in : 0),
                                                 std::span<void* const>(outputs, outputs ? n_out : 0));
    *kernel_ms = r.kernel_ms;
    *total_ms = r.total_ms;
  });
}

int ecl_engine_native_run_split(ecl_engine* e, uint64_t items_per_launch, double* kernel_ms) {
  return guarded(e, [&] { *kernel_ms = e->engine->native_run_split(items_per_launch); });
}

int ecl_engine_kernel_time(ecl_engine* e, double* kernel_ms, uint64_t* launches, int reset) {
  return guarded(e, [&] {
    const KernelTiming t = e->engine->kernel_timing(reset != 0);
    *kernel_ms = t.kernel_ms;
    *launches = t.launches;
  });
}

double ecl_engine_init_ms(const ecl_engine* e) { return e->engine->init_ms(); }

uint32_t ecl_engine_error_count(const ecl_engine* e) { return static_cast<uint32_t>(e->errors.size()); }

int64_t ecl_engine_error(const ecl_engine* e, uint32_t i, int* status, char* buf, uint64_t cap) {
  if (i >= e->errors.size()) return status_of(ErrorCode::ConfigError);
  *status = status_of(e->errors[i].code());
  return emit(e->errors[i].what(), buf, cap);
}

struct ecl_shared {
  std::unique_ptr<SharedCoordinator> coord;
  SchedulerConfig sched;
  std::uint64_t total_wg = 0;
  std::vector<DeviceProfile> devices;
};

int ecl_shared_open(const char* text, ecl_shared** out) {
  *out = nullptr;
  auto h = std::make_unique<ecl_shared>();
  const int rc = guarded(nullptr, [&] {
    const json j = json::parse(text);
    SharedConfig sc;
    sc.name = j.at("name").get<std::string>();
    sc.rank = j.at("rank").get<std::uint32_t>();
    sc.world = j.at("world").get<std::uint32_t>();
    sc.local = j.value("local_devices", std::vector<std::uint32_t>{});
    sc.barrier_timeout_s = j.value("barrier_timeout_s", 60.0);
    h->sched = scheduler_from_json(j.at("scheduler"));
    h->total_wg = j.at("total_work_groups").get<std::uint64_t>();
    h->devices = devices_from(j.at("devices"));
    h->coord = std::make_unique<SharedCoordinator>(sc);
  });
  if (rc == ECL_OK) *out = h.release();
  return rc;
}

void ecl_shared_close(ecl_shared* h) { delete h; }

int ecl_shared_begin(ecl_shared* h, double* epoch_ms) {
  return guarded(nullptr, [&] { *epoch_ms = h->coord->begin_run(h->sched, h->total_wg, h->devices); });
}

int ecl_shared_next(ecl_shared* h, uint32_t device, uint64_t* offset_wg, uint64_t* size_wg, uint64_t* seq) {
  int granted = 0;
  const int rc = guarded(nullptr, [&] {
    PackageRange r;
    if (h->coord->next(device, &r, seq)) {
      *offset_wg = r.offset_wg;
      *size_wg = r.size_wg;
      granted = 1;
    }
  });
  return rc == ECL_OK ? granted : rc;
}

int ecl_shared_observe(ecl_shared* h, uint32_t device, uint64_t items, double ms) {
  return guarded(nullptr, [&] { h->coord->observe(device, items, ms); });
}

int ecl_shared_complete(ecl_shared* h, uint64_t seq, uint32_t device, uint64_t offset_wg, uint64_t size_wg,
                        double t_start_ms, double t_end_ms) {
  return guarded(nullptr, [&] {
    Package p;
    p.seq = seq;
    p.device_index = device;
    p.offset_wg = offset_wg;
    p.size_wg = size_wg;
    p.t_start_ms = p.t_enqueue_ms = t_start_ms;
    p.t_end_ms = t_end_ms;
    h->coord->complete(p);
  });
}

int ecl_shared_fail(ecl_shared* h) {
  return guarded(nullptr, [&] { h->coord->fail(); });
}

int64_t ecl_shared_end(ecl_shared* h, uint64_t* quads, uint64_t cap, int* peer_failed) {
  int64_t n = 0;
  const int rc = guarded(nullptr, [&] {
    bool failed = false;
    const auto all = h->coord->end_run(&failed);
    *peer_failed = failed ? 1 : 0;
    for (const Package& p : all) {
      if (4 * static_cast<uint64_t>(n) + 3 < cap) {
        quads[4 * n] = p.seq;
        quads[4 * n + 1] = p.device_index;
        quads[4 * n + 2] = p.offset_wg;
        quads[4 * n + 3] = p.size_wg;
      }
      ++n;
    }
  });
  return rc == ECL_OK ? n : rc;
}

int ecl_scheduler_create(const char* text, ecl_scheduler** out) {
  *out = nullptr;
  auto s = std::make_unique<ecl_scheduler>();
  const int rc = guarded(nullptr, [&] {
    const json j = json::parse(text);
    s->impl = make_scheduler(scheduler_from_json(j.at("scheduler")), j.at("total_work_groups").get<std::uint64_t>(),
                             devices_from(j.at("devices")));
  });
  if (rc == ECL_OK) *out = s.release();
  return rc;
}

void ecl_scheduler_destroy(ecl_scheduler* s) { delete s; }

int ecl_scheduler_next(ecl_scheduler* s, uint32_t device, uint64_t* offset_wg, uint64_t* size_wg) {
  int granted = 0;
  const int rc = guarded(nullptr, [&] {
    if (auto r = s->impl->next(device)) {
      *offset_wg = r->offset_wg;
      *size_wg = r->size_wg;
      granted = 1;
    }
  });
  return rc == ECL_OK ? granted : rc;
}

uint64_t ecl_scheduler_remaining(const ecl_scheduler* s) { return s->impl->remaining_work_groups(); }

int ecl_scheduler_observe(ecl_scheduler* s, uint32_t device, uint64_t items, double ms) {
  return guarded(nullptr, [&] { s->impl->observe(device, items, ms); });
}

int64_t ecl_scheduler_unclamped(const ecl_scheduler* s, uint64_t pending, uint32_t device) {
  const auto* h = dynamic_cast<const HGuidedScheduler*>(s->impl.get());
  if (!h) return -1;
  int64_t v = -1;
  guarded(nullptr, [&] { v = static_cast<int64_t>(h->unclamped_size(pending, device)); });
  return v;
}

int64_t ecl_describe_scheduler(const char* text, char* buf, uint64_t cap) {
  return guarded_string([&] { return describe(scheduler_from_json(json::parse(text))); }, buf, cap);
}

int64_t ecl_resolve_static(const char* sched, const char* devs, char* buf, uint64_t cap) {
  return guarded_string(
      [&] {
        const SchedulerConfig c = scheduler_from_json(json::parse(sched));
        if (!std::holds_alternative<StaticConfig>(c)) throw Error(ErrorCode::BadSchedulerConfig, "not a static config");
        const StaticConfig r = resolve_static(std::get<StaticConfig>(c), devices_from(json::parse(devs)));
        return json{{"proportions", r.proportions}, {"device_order", r.device_order}}.dump();
      },
      buf, cap);
}

int64_t ecl_apply_default_min_package(const char* devs, char* buf, uint64_t cap) {
  return guarded_string(
      [&] {
        json arr = json::array();
        for (const DeviceProfile& d : devices_from(json::parse(devs))) arr.push_back(to_json(d));
        return arr.dump();
      },
      buf, cap);
}

int ecl_validate_program(const char* text, uint64_t* total_wg) {
  return guarded(nullptr, [&] { *total_wg = validate_program(program_from_json(json::parse(text))).total_work_groups(); });
}

int ecl_out_range_for(const char* text, uint64_t offset_wg, uint64_t size_wg, uint64_t* offset, uint64_t* count) {
  return guarded(nullptr, [&] {
    const ValidatedProgram p = validate_program(program_from_json(json::parse(text)));
    Package pkg;
    pkg.offset_wg = offset_wg;
    pkg.size_wg = size_wg;
    const OutRange r = out_range_for(pkg, p);
    *offset = r.offset;
    *count = r.count;
  });
}

int ecl_tiles_exactly(const uint64_t* offsets, const uint64_t* sizes, uint64_t n, uint64_t total_wg) {
  std::vector<Package> pk(n);
  for (uint64_t i = 0; i < n; ++i) {
    pk[i].offset_wg = offsets[i];
    pk[i].size_wg = sizes[i];
  }
  return tiles_exactly(std::move(pk), total_wg) ? 1 : 0;
}

int64_t ecl_metrics_report(const char* trace_json, const double* solo, uint32_t n_solo, double reference_ms,
                           char* buf, uint64_t cap) {
  return guarded_string(
      [&] {
        const ExecutionTrace t = trace_from_json(json::parse(trace_json));
        std::optional<double> ref;
        if (reference_ms >= 0.0) ref = reference_ms;
        return to_json(make_report(t, std::span<const double>(solo, n_solo), ref)).dump();
      },
      buf, cap);
}

int64_t ecl_trace_csv(const char* trace_json, char* buf, uint64_t cap) {
  return guarded_string([&] { return trace_to_csv(trace_from_json(json::parse(trace_json))); }, buf, cap);
}

int64_t ecl_chart_svg(const char* trace_json, char* buf, uint64_t cap) {
  return guarded_string([&] { return render_svg(trace_from_json(json::parse(trace_json))); }, buf, cap);
}

int ecl_experiment_run(const char* config_path, const char* overrides_json, char* path_buf, uint64_t cap) {
  return guarded(nullptr, [&] {
    ExperimentConfig cfg = load_experiment(config_path);
    RunOptions opts;
    if (overrides_json && *overrides_json) {
      const json o = json::parse(overrides_json);
      if (o.contains("scheduler")) {
        SchedulerConfig s = scheduler_from_json(o.at("scheduler"));
        if (auto* st = std::get_if<StaticConfig>(&s)) *st = resolve_static(*st, cfg.devices);
        cfg.schedulers = {s};
      }
      if (o.contains("out_dir")) cfg.output_dir = o.at("out_dir").get<std::string>();
      cfg.exclude_init = o.value("exclude_init", cfg.exclude_init);
      opts.write_traces = o.value("write_traces", opts.write_traces);
      opts.write_csv = o.value("write_csv", opts.write_csv);
      opts.write_charts = o.value("write_charts", opts.write_charts);
      opts.dump_pgm = o.value("dump_pgm", opts.dump_pgm);
    }
    const ExperimentResult r = run_experiment(cfg, opts);
    const std::string path = r.summary_file.string();
    if (!path_buf || cap <= path.size()) throw Error(ErrorCode::ConfigError, "summary path buffer too small");
    std::memcpy(path_buf, path.c_str(), path.size() + 1);
  });
}

int64_t ecl_experiment_validate(const char* config_path, char* buf, uint64_t cap) {
  return guarded_string([&] { return describe_experiment(load_experiment(config_path)); }, buf, cap);
}

}  // extern "C"
