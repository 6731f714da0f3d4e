// experiment.hpp — the paper's measurement protocol as a harness (reference:
// config.hpp:15-195, experiment.hpp:20-181, coexec_main.cpp:40-108):
// an experiment file names one program, a device list (inline or a profile
// file), a scheduler matrix and the repetition protocol; run_experiment runs
// one solo baseline per device plus every scheduler, discards the warm-up
// repetitions, keeps the median run's trace, writes traces / charts and a
// summary.json with the co-execution metrics.
//
// Same file formats as the reference, so its experiment files run here and
// its virtual-clock outputs are reproduced exactly.  B200 specifics:
//   * devices with backend "cuda" run on B200s (wall clock);
//   * virtual-clock Mandelbrot needs its per-pixel cost table (the
//     iteration counts, workloads.hpp:243-246): it is computed once per
//     experiment by the B200 kernel on CUDA device 0 — no CPU fallback;
//   * "outputs": "resident" (wall clock) keeps results in HBM instead of
//     copying them to engine-allocated host buffers each repetition.
#pragma once

#include <cstdint>
#include <filesystem>
#include <map>
#include <optional>
#include <string>
#include <vector>

#include "coexec/core.hpp"
#include "coexec/json_io.hpp"
#include "coexec/metrics.hpp"
#include "coexec/schedulers.hpp"

namespace coexec {

struct ExperimentConfig {
  ProgramSpec program;
  std::vector<DeviceProfile> devices;
  std::vector<SchedulerConfig> schedulers;
  std::uint32_t repetitions = 1;
  std::uint32_t warmup_discard = 0;
  ClockMode clock_mode = ClockMode::Virtual;
  std::uint64_t seed = 0;
  bool exclude_init = false;
  bool resident_outputs = false;  // "outputs": "resident" (B200 addition)
  std::filesystem::path output_dir = "out";
};

struct RunOptions {
  bool write_traces = true;
  bool write_csv = false;
  bool write_charts = true;
  bool dump_pgm = false;
  bool quiet = true;
};

struct SchedulerOutcome {
  std::string name;  // "s<i>-<kind>"
  SchedulerConfig config;
  std::vector<double> t_totals_ms;  // retained repetitions in run order
  std::size_t median_index = 0;
  ExecutionTrace median_trace;
  MetricsReport report;
  std::vector<std::filesystem::path> trace_files;
};

struct ExperimentResult {
  std::map<std::string, double> solo_ms;  // device id -> median solo t_total
  std::vector<SchedulerOutcome> outcomes;
  std::filesystem::path summary_file;
  std::string summary_json;
};

/// Parses an experiment file (schema 1); relative "devices_file" paths are
/// resolved against the file's directory.  Static proportions are resolved
/// (normalized, n-1 rule, device order) as the reference does at load.
ExperimentConfig load_experiment(const std::filesystem::path& path);
ExperimentConfig experiment_from_json(const json& j, const std::filesystem::path& base_dir);
std::vector<DeviceProfile> load_device_profiles(const std::filesystem::path& path);

/// Reference input recipe (workloads.hpp:261-283): splitmix64(seed) doubles
/// in [0,1) for 8-byte elements, random bytes otherwise.  B200 additions:
/// 4- and 16-byte elements (f32 / float4 kernels) get floats in [0,1), and
/// Gaussian's filter is a normalized Gaussian with sigma = F/6.
std::vector<std::vector<std::byte>> fill_default_inputs(const ValidatedProgram& prog, std::uint64_t seed);

/// Per-work-item virtual-clock costs (reference cost model,
/// workloads.hpp:238-257): empty for vecscale / synthetic (the engine's
/// analytic model), Mandelbrot's iteration counts computed on CUDA device 0,
/// 1.0 per item for the regular kernels added here.
std::vector<double> virtual_item_costs(const ValidatedProgram& prog);

ExperimentResult run_experiment(const ExperimentConfig& cfg, const RunOptions& opts = {});

/// Text report of one outcome's metrics (reference metrics.hpp:142-161 layout).
std::string render_table(const MetricsReport& r);

/// One line per scheduler; what `coexec validate` prints.
std::string describe_experiment(const ExperimentConfig& cfg);

/// Binary PGM of Mandelbrot counts (4:1 layout), gray = 255 - 255·count/max.
void write_pgm(const std::filesystem::path& path, const std::uint32_t* counts_4to1, std::uint64_t width,
               std::uint64_t height, std::uint32_t max_iterations);

}  // namespace coexec
