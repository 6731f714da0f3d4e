// experiment.cpp — coexec/experiment.hpp: the repetition protocol, solo
// baselines, medians, traces / charts / summary.json (reference
// experiment.hpp:67-181, config.hpp:159-195).
#include "coexec/experiment.hpp"

#include <algorithm>
#include <cmath>
#include <cstdio>
#include <cstring>
#include <fstream>
#include <numeric>
#include <sstream>

#include "coexec/chart.hpp"
#include "coexec/engine.hpp"

namespace coexec {

namespace {

json read_json(const std::filesystem::path& path) {
  std::ifstream in(path);
  if (!in) throw Error(ErrorCode::ConfigError, "cannot open '" + path.string() + "'");
  try {
    return json::parse(in);
  } catch (const json::exception& e) {
    throw Error(ErrorCode::ConfigError, std::string(e.what()) + " in '" + path.string() + "'");
  }
}

void write_file(const std::filesystem::path& path, const std::string& text) {
  std::ofstream out(path, std::ios::binary);
  if (!out) throw Error(ErrorCode::IoError, "cannot open '" + path.string() + "' for writing");
  out << text;
  if (!out) throw Error(ErrorCode::IoError, "failed writing '" + path.string() + "'");
}

// Lower median by (value, run order).
std::size_t median_of(const std::vector<double>& v) {
  std::vector<std::size_t> idx(v.size());
  std::iota(idx.begin(), idx.end(), std::size_t{0});
  std::stable_sort(idx.begin(), idx.end(), [&](std::size_t a, std::size_t b) { return v[a] < v[b]; });
  return idx[(idx.size() - 1) / 2];
}

std::uint64_t splitmix(std::uint64_t& state) {
  state += 0x9e3779b97f4a7c15ull;
  std::uint64_t z = state;
  z = (z ^ (z >> 30)) * 0xbf58476d1ce4e5b9ull;
  z = (z ^ (z >> 27)) * 0x94d049bb133111ebull;
  return z ^ (z >> 31);
}

std::uint64_t arg_u64(const ProgramSpec& s, std::size_t i) {
  if (i >= s.args.size()) throw Error(ErrorCode::BadKernelArgs, "missing kernel argument " + std::to_string(i));
  return std::visit([](auto v) { return static_cast<std::uint64_t>(v); }, s.args[i]);
}

// One repetition: a fresh engine (construction is part of the protocol,
// reference experiment.hpp:73), then one run.
struct Rep {
  ExecutionTrace trace;
  std::vector<std::vector<std::byte>> outputs;
};

Rep run_once(const EngineConfig& ecfg, const ValidatedProgram& prog, const std::vector<std::vector<std::byte>>& inputs,
             const std::vector<double>& costs, bool resident) {
  Engine engine(ecfg, prog);
  Rep r;
  if (ecfg.clock_mode == ClockMode::Virtual) {
    r.trace = engine.run_virtual(costs);
  } else if (resident) {
    std::vector<const void*> in;
    for (const auto& v : inputs) in.push_back(v.data());
    r.trace = engine.run_into(in, {});
  } else {
    RunResult res = engine.run(inputs);
    r.trace = std::move(res.trace);
    r.outputs = std::move(res.outputs);
  }
  return r;
}

std::vector<Rep> repetitions(const EngineConfig& ecfg, const ValidatedProgram& prog,
                             const std::vector<std::vector<std::byte>>& inputs, const std::vector<double>& costs,
                             const ExperimentConfig& cfg) {
  std::vector<Rep> kept;
  for (std::uint32_t rep = 0; rep < cfg.repetitions; ++rep) {
    Rep r = run_once(ecfg, prog, inputs, costs, cfg.resident_outputs);
    if (rep >= cfg.warmup_discard) kept.push_back(std::move(r));
  }
  return kept;
}

EngineConfig engine_config(const ExperimentConfig& cfg, std::vector<DeviceProfile> devices, SchedulerConfig sched) {
  EngineConfig e;
  e.devices = std::move(devices);
  e.scheduler = std::move(sched);
  e.clock_mode = cfg.clock_mode;
  e.seed = cfg.seed;
  e.exclude_init_from_total = cfg.exclude_init;
  return e;
}

}  // namespace

std::vector<DeviceProfile> load_device_profiles(const std::filesystem::path& path) {
  const json j = read_json(path);
  std::vector<DeviceProfile> devices;
  try {
    for (const json& d : j.at("devices")) devices.push_back(device_from_json(d));
  } catch (const json::exception& e) {
    throw Error(ErrorCode::ConfigError, std::string(e.what()) + " in '" + path.string() + "'");
  }
  if (devices.empty()) throw Error(ErrorCode::ConfigError, "profile '" + path.string() + "' lists no devices");
  apply_default_min_package(devices);
  for (const DeviceProfile& d : devices) validate_device(d);
  return devices;
}

ExperimentConfig experiment_from_json(const json& j, const std::filesystem::path& base_dir) {
  ExperimentConfig cfg;
  try {
    if (j.value("schema", 1) != 1) throw Error(ErrorCode::ConfigError, "unsupported config schema version");
    cfg.program = program_from_json(j.at("program"));
    if (j.contains("devices_file")) {
      const std::filesystem::path f = j.at("devices_file").get<std::string>();
      cfg.devices = load_device_profiles(f.is_relative() ? base_dir / f : f);
    } else {
      for (const json& d : j.at("devices")) cfg.devices.push_back(device_from_json(d));
      apply_default_min_package(cfg.devices);
    }
    for (const json& s : j.at("schedulers")) cfg.schedulers.push_back(scheduler_from_json(s));
    cfg.repetitions = j.value("repetitions", 1u);
    cfg.warmup_discard = j.value("warmup_discard", 0u);
    cfg.clock_mode = j.value("clock_mode", std::string("virtual")) == "wall" ? ClockMode::Wall : ClockMode::Virtual;
    cfg.seed = j.value("seed", std::uint64_t{0});
    cfg.exclude_init = j.value("exclude_init", false);
    const std::string outputs = j.value("outputs", std::string("host"));
    if (outputs != "host" && outputs != "resident")
      throw Error(ErrorCode::ConfigError, "outputs must be 'host' or 'resident'");
    cfg.resident_outputs = outputs == "resident";
    cfg.output_dir = j.value("output_dir", std::string("out"));
  } catch (const json::exception& e) {
    throw Error(ErrorCode::ConfigError, e.what());
  }
  if (cfg.devices.empty()) throw Error(ErrorCode::ConfigError, "no devices configured");
  for (const DeviceProfile& d : cfg.devices) validate_device(d);
  if (cfg.schedulers.empty()) throw Error(ErrorCode::ConfigError, "no schedulers configured");
  if (cfg.repetitions < 1) throw Error(ErrorCode::ConfigError, "repetitions must be >= 1");
  if (cfg.warmup_discard >= cfg.repetitions)
    throw Error(ErrorCode::ConfigError, "warmup_discard must be smaller than repetitions");
  (void)validate_program(cfg.program);  // work-size errors surface at load
  for (SchedulerConfig& s : cfg.schedulers)
    if (auto* st = std::get_if<StaticConfig>(&s)) *st = resolve_static(*st, cfg.devices);
  return cfg;
}

ExperimentConfig load_experiment(const std::filesystem::path& path) {
  const json j = read_json(path);
  try {
    return experiment_from_json(j, path.parent_path());
  } catch (const Error& e) {
    if (e.code() == ErrorCode::ConfigError) throw Error(ErrorCode::ConfigError, std::string(e.what()) + " in '" + path.string() + "'");
    throw;
  }
}

std::vector<std::vector<std::byte>> fill_default_inputs(const ValidatedProgram& prog, std::uint64_t seed) {
  std::vector<std::vector<std::byte>> inputs;
  std::uint64_t state = seed;  // one stream across buffers, in buffer order
  const ProgramSpec& spec = prog.spec();
  for (std::size_t bi = 0; bi < spec.in_buffers.size(); ++bi) {
    const BufferDesc& b = spec.in_buffers[bi];
    if (spec.kernel == "gaussian" && bi == 1 && b.element_size_bytes == 4) {
      // the filter: a normalized Gaussian, sigma = F/6 (F = 31 -> 5, the paper's config)
      const std::uint64_t f = static_cast<std::uint64_t>(std::llround(std::sqrt(double(b.element_count))));
      std::vector<std::byte> bytes(b.size_bytes());
      std::vector<double> w(b.element_count);
      const double sigma = double(f) / 6.0, r = double(f / 2);
      double sum = 0;
      for (std::uint64_t i = 0; i < b.element_count; ++i) {
        const double y = double(i / f) - r, x = double(i % f) - r;
        w[i] = std::exp(-(x * x + y * y) / (2 * sigma * sigma));
        sum += w[i];
      }
      for (std::uint64_t i = 0; i < b.element_count; ++i) {
        const float v = static_cast<float>(w[i] / sum);
        std::memcpy(bytes.data() + 4 * i, &v, 4);
      }
      inputs.push_back(std::move(bytes));
      continue;
    }
    std::vector<std::byte> bytes(b.size_bytes());
    if (b.element_size_bytes == 8) {
      for (std::uint64_t i = 0; i < b.element_count; ++i) {
        const double v = static_cast<double>(splitmix(state) >> 11) * 0x1.0p-53;
        std::memcpy(bytes.data() + 8 * i, &v, 8);
      }
    } else if (b.element_size_bytes == 4 || b.element_size_bytes == 16) {
      for (std::uint64_t i = 0; i < b.size_bytes() / 4; ++i) {
        const float v = static_cast<float>(splitmix(state) >> 40) * 0x1.0p-24f;
        std::memcpy(bytes.data() + 4 * i, &v, 4);
      }
    } else {
      for (std::byte& x : bytes) x = static_cast<std::byte>(splitmix(state) & 0xff);
    }
    inputs.push_back(std::move(bytes));
  }
  return inputs;
}

std::vector<double> virtual_item_costs(const ValidatedProgram& prog) {
  const ProgramSpec& s = prog.spec();
  if (s.kernel == "vecscale" || s.kernel.rfind("synthetic", 0) == 0) return {};
  const std::uint64_t gws = prog.global_work_size();
  if (s.kernel != "mandelbrot") return std::vector<double>(gws, 1.0);
  // Mandelbrot's cost is its escape count: evaluate the kernel once on the
  // first B200 (a one-device static run) and read the 4:1 counts back.
  DeviceProfile gpu;
  gpu.id = "cost-eval";
  gpu.name = "cost table (CUDA device 0)";
  gpu.backend.kind = BackendKind::Cuda;
  gpu.backend.ordinal = 0;
  gpu.min_package_work_groups = 1;
  EngineConfig ecfg;
  ecfg.devices = {gpu};
  ecfg.scheduler = StaticConfig{{1.0}, {gpu.id}};
  ecfg.clock_mode = ClockMode::Wall;
  Engine engine(ecfg, prog);
  std::vector<std::uint32_t> counts(s.out_buffers.at(0).element_count);
  void* out[] = {counts.data()};
  engine.run_into({}, out);
  const std::uint64_t per = s.out_pattern.out_indices / s.out_pattern.work_items;
  std::vector<double> costs(gws);
  for (std::uint64_t i = 0; i < gws; ++i) costs[i] = static_cast<double>(counts[i * per]);
  return costs;
}

std::string render_table(const MetricsReport& r) {
  std::string out;
  char line[160];
  auto row = [&](const char* name, double v) {
    std::snprintf(line, sizeof line, "%-12s %10.4f\n", name, v);
    out += line;
  };
  row("balance", r.balance);
  row("speedup", r.speedup);
  row("s_max", r.s_max);
  row("efficiency", r.efficiency);
  if (r.overhead_pct) row("overhead_pct", *r.overhead_pct);
  for (const auto& [id, share] : r.work_share) {
    const int pad = id.size() <= 10 ? static_cast<int>(10 - id.size()) : 0;
    std::snprintf(line, sizeof line, "share[%s]%*s %7.2f%%\n", id.c_str(), pad, "", share * 100.0);
    out += line;
  }
  for (const std::string& n : r.notes) out += "note: " + n + "\n";
  return out;
}

std::string describe_experiment(const ExperimentConfig& cfg) {
  const ValidatedProgram prog = validate_program(cfg.program);
  std::ostringstream o;
  o << "ok: " << cfg.program.kernel << ", gws " << prog.global_work_size() << ", lws " << prog.local_work_size()
    << ", " << prog.total_work_groups() << " work-groups, " << cfg.devices.size() << " devices, "
    << cfg.schedulers.size() << " schedulers, " << cfg.repetitions << " repetitions (" << cfg.warmup_discard
    << " warm-up)\n";
  for (const SchedulerConfig& s : cfg.schedulers) o << "  " << describe(s) << "\n";
  return o.str();
}

void write_pgm(const std::filesystem::path& path, const std::uint32_t* counts, std::uint64_t width,
               std::uint64_t height, std::uint32_t max_iterations) {
  std::string img = "P5\n" + std::to_string(width) + " " + std::to_string(height) + "\n255\n";
  const std::size_t header = img.size();
  img.resize(header + width * height);
  for (std::uint64_t i = 0; i < width * height; ++i) {
    const std::uint32_t c = counts[4 * i];
    img[header + i] = static_cast<char>(c >= max_iterations ? 0 : 255 - (c * 255) / max_iterations);
  }
  write_file(path, img);
}

ExperimentResult run_experiment(const ExperimentConfig& cfg, const RunOptions& opts) {
  const ValidatedProgram prog = validate_program(cfg.program);
  const auto inputs = fill_default_inputs(prog, cfg.seed);
  const std::vector<double> costs =
      cfg.clock_mode == ClockMode::Virtual ? virtual_item_costs(prog) : std::vector<double>{};
  std::filesystem::create_directories(cfg.output_dir);
  ExperimentResult result;

  // Solo baselines: each device alone, everything in one static package.
  for (const DeviceProfile& d : cfg.devices) {
    const auto runs = repetitions(engine_config(cfg, {d}, StaticConfig{{1.0}, {d.id}}), prog, inputs, costs, cfg);
    std::vector<double> totals;
    for (const Rep& r : runs) totals.push_back(r.trace.t_total_ms);
    result.solo_ms[d.id] = totals[median_of(totals)];
  }
  std::vector<double> solo;
  for (const auto& [id, t] : result.solo_ms) solo.push_back(t);

  for (std::size_t i = 0; i < cfg.schedulers.size(); ++i) {
    SchedulerOutcome oc;
    oc.config = cfg.schedulers[i];
    oc.name = "s" + std::to_string(i) + "-" + scheduler_kind(oc.config);
    auto runs = repetitions(engine_config(cfg, cfg.devices, oc.config), prog, inputs, costs, cfg);
    for (std::size_t r = 0; r < runs.size(); ++r) {
      oc.t_totals_ms.push_back(runs[r].trace.t_total_ms);
      if (!opts.write_traces) continue;
      const std::string stem = (cfg.output_dir / (oc.name + "-rep" + std::to_string(r))).string();
      write_file(stem + ".trace.json", trace_to_json_string(runs[r].trace));
      oc.trace_files.emplace_back(stem + ".trace.json");
      if (opts.write_csv) write_file(stem + ".trace.csv", trace_to_csv(runs[r].trace));
    }
    oc.median_index = median_of(oc.t_totals_ms);
    oc.median_trace = runs[oc.median_index].trace;
    oc.report = make_report(oc.median_trace, solo);
    if (opts.write_charts) write_file(cfg.output_dir / (oc.name + "-median.svg"), render_svg(oc.median_trace));
    if (opts.dump_pgm && cfg.program.kernel == "mandelbrot" && !runs[oc.median_index].outputs.empty()) {
      const auto& bytes = runs[oc.median_index].outputs.at(0);
      write_pgm(cfg.output_dir / (oc.name + ".pgm"), reinterpret_cast<const std::uint32_t*>(bytes.data()),
                arg_u64(cfg.program, 0), arg_u64(cfg.program, 1), static_cast<std::uint32_t>(arg_u64(cfg.program, 2)));
    }
    if (!opts.quiet) {
      std::printf("%s  %s\n  t_total (median): %s ms over %zu retained runs\n%s", oc.name.c_str(),
                  describe(oc.config).c_str(), format_double(oc.t_totals_ms[oc.median_index]).c_str(),
                  oc.t_totals_ms.size(), render_table(oc.report).c_str());
    }
    result.outcomes.push_back(std::move(oc));
  }

  json summary{{"schema", 1},
               {"clock_mode", std::string(clock_mode_name(cfg.clock_mode))},
               {"seed", cfg.seed},
               {"repetitions", cfg.repetitions},
               {"warmup_discard", cfg.warmup_discard},
               {"program", to_json(cfg.program)},
               {"solo_ms", result.solo_ms}};
  json outcomes = json::array();
  for (const SchedulerOutcome& oc : result.outcomes) {
    json files = json::array();
    for (const auto& f : oc.trace_files) files.push_back(f.filename().string());
    outcomes.push_back({{"name", oc.name},
                        {"scheduler", to_json(oc.config)},
                        {"description", describe(oc.config)},
                        {"t_totals_ms", oc.t_totals_ms},
                        {"median_t_total_ms", oc.t_totals_ms[oc.median_index]},
                        {"median_trace", oc.trace_files.empty()
                                             ? json(nullptr)
                                             : json(oc.trace_files[oc.median_index].filename().string())},
                        {"metrics", to_json(oc.report)},
                        {"trace_files", std::move(files)}});
  }
  summary["outcomes"] = std::move(outcomes);
  result.summary_json = summary.dump(2) + "\n";
  result.summary_file = cfg.output_dir / "summary.json";
  write_file(result.summary_file, result.summary_json);
  return result;
}

}  // namespace coexec
