// coexec — command-line front end of the experiment harness (reference
// tools/coexec_main.cpp:40-175): `run`, `validate` and `chart`, the same
// flags and exit codes (1 = configuration error, 2 = runtime error).
//
//   coexec run experiments/b200-mandelbrot.json [--scheduler hguided --k 2]
//   coexec validate experiments/b200-mandelbrot.json
//   coexec chart out/b200-mandelbrot/s0-static-rep0.trace.json -o chart.svg
#include <cstdio>
#include <cstring>
#include <fstream>
#include <iostream>
#include <sstream>
#include <string>
#include <vector>

#include "coexec/chart.hpp"
#include "coexec/engine.hpp"
#include "coexec/experiment.hpp"

using namespace coexec;

namespace {

const char* kUsage =
    "co-execution runtime on B200s: partition one data-parallel kernel across devices\n"
    "usage:\n"
    "  coexec run CONFIG [--scheduler static|dynamic|hguided] [--props a,b,...]\n"
    "                    [--num-packages N] [--k K] [--exclude-init] [--out-dir DIR]\n"
    "                    [--format table|json|csv] [--dump-pgm]\n"
    "  coexec validate CONFIG\n"
    "  coexec chart TRACE [-o|--output SVG]\n";

struct Args {
  std::vector<std::string> positional;
  std::vector<std::pair<std::string, std::string>> options;  // (flag, value or "")
  bool has(const std::string& f) const {
    for (const auto& [k, v] : options)
      if (k == f) return true;
    return false;
  }
  std::string get(const std::string& f, const std::string& dflt = "") const {
    for (const auto& [k, v] : options)
      if (k == f) return v;
    return dflt;
  }
};

Args parse(int argc, char** argv, const std::vector<std::string>& valued, const std::vector<std::string>& flags) {
  Args a;
  for (int i = 2; i < argc; ++i) {
    const std::string s = argv[i];
    auto in = [&](const std::vector<std::string>& v) {
      for (const auto& x : v)
        if (x == s) return true;
      return false;
    };
    if (in(valued)) {
      if (i + 1 >= argc) throw Error(ErrorCode::ConfigError, s + " needs a value");
      a.options.emplace_back(s, argv[++i]);
    } else if (in(flags)) {
      a.options.emplace_back(s, "");
    } else if (!s.empty() && s[0] == '-') {
      throw Error(ErrorCode::ConfigError, "unknown option '" + s + "'");
    } else {
      a.positional.push_back(s);
    }
  }
  return a;
}

std::vector<double> parse_props(const std::string& csv) {
  std::vector<double> v;
  std::stringstream in(csv);
  std::string item;
  while (std::getline(in, item, ',')) {
    try {
      std::size_t used = 0;
      v.push_back(std::stod(item, &used));
      if (used != item.size()) throw std::invalid_argument(item);
    } catch (const std::exception&) {
      throw Error(ErrorCode::ConfigError, "--props expects comma-separated reals");
    }
  }
  return v;
}

std::uint64_t parse_u64(const std::string& s, const char* what) {
  try {
    std::size_t used = 0;
    const unsigned long long v = std::stoull(s, &used);
    if (used == s.size()) return v;
  } catch (const std::exception&) {
  }
  throw Error(ErrorCode::ConfigError, std::string(what) + " expects an unsigned integer");
}

double parse_real(const std::string& s, const char* what) {
  try {
    std::size_t used = 0;
    const double v = std::stod(s, &used);
    if (used == s.size()) return v;
  } catch (const std::exception&) {
  }
  throw Error(ErrorCode::ConfigError, std::string(what) + " expects a real number");
}

int cmd_run(const Args& a) {
  if (a.positional.size() != 1) throw Error(ErrorCode::ConfigError, "run: exactly one experiment file expected");
  ExperimentConfig cfg = load_experiment(a.positional[0]);
  if (a.has("--scheduler")) {
    const std::string kind = a.get("--scheduler");
    if (kind == "static") {
      StaticConfig s;
      if (a.has("--props")) s.proportions = parse_props(a.get("--props"));
      cfg.schedulers = {resolve_static(s, cfg.devices)};
    } else if (kind == "dynamic") {
      cfg.schedulers = {DynamicConfig{parse_u64(a.get("--num-packages", "50"), "--num-packages")}};
    } else if (kind == "hguided") {
      HGuidedConfig h;
      h.k = parse_real(a.get("--k", "2"), "--k");
      cfg.schedulers = {h};
    } else {
      throw Error(ErrorCode::ConfigError, "--scheduler must be static, dynamic or hguided");
    }
  }
  if (a.has("--exclude-init")) cfg.exclude_init = true;
  if (a.has("--out-dir")) cfg.output_dir = a.get("--out-dir");
  const std::string format = a.get("--format", "table");
  if (format != "table" && format != "json" && format != "csv")
    throw Error(ErrorCode::ConfigError, "--format must be table, json or csv");
  RunOptions opts;
  opts.write_csv = format == "csv";
  opts.dump_pgm = a.has("--dump-pgm");
  opts.quiet = format == "json";
  std::fflush(stdout);
  const ExperimentResult r = run_experiment(cfg, opts);
  if (format == "json") {
    std::cout << r.summary_json;
  } else {
    std::cout << "solo baselines (median t_total):\n";
    for (const auto& [id, ms] : r.solo_ms) std::cout << "  " << id << ": " << format_double(ms) << " ms\n";
    std::cout << "summary: " << r.summary_file.string() << "\n";
  }
  return 0;
}

int cmd_validate(const Args& a) {
  if (a.positional.size() != 1) throw Error(ErrorCode::ConfigError, "validate: exactly one experiment file expected");
  std::cout << describe_experiment(load_experiment(a.positional[0]));
  return 0;
}

int cmd_chart(const Args& a) {
  if (a.positional.size() != 1) throw Error(ErrorCode::ConfigError, "chart: exactly one trace file expected");
  const std::filesystem::path in = a.positional[0];
  std::ifstream f(in);
  if (!f) throw Error(ErrorCode::IoError, "cannot open '" + in.string() + "'");
  json j;
  try {
    j = json::parse(f);
  } catch (const json::exception& e) {
    throw Error(ErrorCode::MalformedTrace, std::string(e.what()) + " in '" + in.string() + "'");
  }
  std::string out = a.get("-o", a.get("--output"));
  if (out.empty()) out = std::filesystem::path(in).replace_extension(".svg").string();
  std::ofstream o(out, std::ios::binary);
  if (!o) throw Error(ErrorCode::IoError, "cannot open '" + out + "' for writing");
  o << render_svg(trace_from_json(j));
  if (!o) throw Error(ErrorCode::IoError, "failed writing '" + out + "'");
  std::cout << out << "\n";
  return 0;
}

bool is_config_error(ErrorCode c) {
  switch (c) {
    case ErrorCode::ConfigError:
    case ErrorCode::NonDivisibleWorkSize:
    case ErrorCode::BadOutPattern:
    case ErrorCode::EmptyProgram:
    case ErrorCode::BadSchedulerConfig:
    case ErrorCode::UnknownKernel:
    case ErrorCode::UnknownProfile:
    case ErrorCode::BadKernelArgs:
    case ErrorCode::MalformedTrace:
      return true;
    default:
      return false;
  }
}

}  // namespace

int main(int argc, char** argv) {
  if (argc < 2 || !std::strcmp(argv[1], "-h") || !std::strcmp(argv[1], "--help")) {
    std::cout << kUsage;
    return argc < 2 ? 1 : 0;
  }
  const std::string cmd = argv[1];
  try {
    if (cmd == "run")
      return cmd_run(parse(argc, argv, {"--scheduler", "--props", "--num-packages", "--k", "--out-dir", "--format"},
                           {"--exclude-init", "--dump-pgm"}));
    if (cmd == "validate") return cmd_validate(parse(argc, argv, {}, {}));
    if (cmd == "chart") return cmd_chart(parse(argc, argv, {"-o", "--output"}, {}));
    std::cerr << "error: unknown subcommand '" << cmd << "'\n" << kUsage;
    return 1;
  } catch (const EngineFailure& f) {
    std::cerr << "error: engine failed with " << f.errors().size() << " error(s):\n";
    for (const Error& e : f.errors()) std::cerr << "  " << e.what() << "\n";
    return 2;
  } catch (const Error& e) {
    std::cerr << "error: " << e.what() << "\n";
    return is_config_error(e.code()) ? 1 : 2;
  } catch (const std::exception& e) {
    std::cerr << "error: " << e.what() << "\n";
    return 2;
  }
}
