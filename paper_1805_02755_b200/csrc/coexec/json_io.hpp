// json_io.hpp — the reference's JSON schema 1 for programs, device profiles,
// scheduler configs and traces (reference: config.hpp:41-153,
// trace_io.hpp:26-175), so experiment files and traces are interchangeable
// with the reference's.  Backend kind "cuda" is the B200 addition.
#pragma once

#include <charconv>
#include <string>
#include <vector>

#include "coexec/core.hpp"
#include "coexec/metrics.hpp"
#include "coexec/schedulers.hpp"
#include "json.hpp"

namespace coexec {

using json = nlohmann::json;

inline std::string format_double(double v) {
  char buf[32];
  auto [end, ec] = std::to_chars(buf, buf + sizeof buf, v);
  return std::string(buf, end);
}

inline json to_json(const Backend& b) {
  if (b.kind == BackendKind::Simulated) return json{{"kind", "simulated"}};
  return json{{"kind", "cuda"},
              {"ordinal", b.ordinal},
              {"queue_depth", b.queue_depth},
              {"copy_split_items", b.copy_split_items},
              {"widen_per_8", b.widen_per_8}};
}

inline Backend backend_from_json(const json& j) {
  Backend b;
  const std::string kind = j.at("kind").get<std::string>();
  if (kind == "simulated") {
    b.kind = BackendKind::Simulated;
  } else if (kind == "cuda") {
    b.kind = BackendKind::Cuda;
    b.ordinal = j.value("ordinal", 0);
    b.queue_depth = j.value("queue_depth", 2u);
    b.copy_split_items = j.value("copy_split_items", std::uint64_t{1} << 23);
    b.widen_per_8 = j.value("widen_per_8", 8u);
  } else if (kind == "native_pool") {
    throw Error(ErrorCode::ConfigError,
                "backend 'native_pool' (host thread pools) is replaced by 'cuda' in the B200 build");
  } else {
    throw Error(ErrorCode::ConfigError, "unknown backend kind '" + kind + "'");
  }
  return b;
}

inline json to_json(const DeviceProfile& d) {
  json j{{"id", d.id},
         {"name", d.name},
         {"computing_power", d.computing_power},
         {"launch_overhead_ms", d.launch_overhead_ms},
         {"bandwidth_bytes_per_ms", d.bandwidth_bytes_per_ms},
         {"backend", to_json(d.backend)},
         {"min_package_work_groups", d.min_package_work_groups}};
  if (!d.kernel.empty()) j["kernel"] = d.kernel;  // absent for reference-shaped profiles
  return j;
}

inline DeviceProfile device_from_json(const json& j) {
  DeviceProfile d;
  d.id = j.at("id").get<std::string>();
  d.name = j.value("name", d.id);
  d.computing_power = j.value("computing_power", 1.0);
  d.launch_overhead_ms = j.value("launch_overhead_ms", 0.0);
  d.bandwidth_bytes_per_ms = j.value("bandwidth_bytes_per_ms", 1.0);
  if (j.contains("backend")) d.backend = backend_from_json(j.at("backend"));
  d.min_package_work_groups = j.value("min_package_work_groups", std::uint64_t{0});  // 0 = heuristic
  d.kernel = j.value("kernel", std::string());
  return d;
}

inline SchedulerConfig scheduler_from_json(const json& j) {
  const std::string type = j.at("type").get<std::string>();
  if (type == "static") {
    StaticConfig c;
    if (j.contains("proportions")) c.proportions = j.at("proportions").get<std::vector<double>>();
    if (j.contains("device_order")) c.device_order = j.at("device_order").get<std::vector<std::string>>();
    return c;
  }
  if (type == "dynamic") return DynamicConfig{j.at("num_packages").get<std::uint64_t>()};
  if (type == "hguided") {
    HGuidedConfig c;
    c.k = j.value("k", 2.0);
    if (j.contains("powers")) c.powers = j.at("powers").get<std::vector<double>>();
    c.include_device_count = j.value("include_device_count", true);
    c.adaptive = j.value("adaptive", false);
    c.ema_alpha = j.value("ema_alpha", 0.5);
    return c;
  }
  throw Error(ErrorCode::ConfigError, "unknown scheduler type '" + type + "'");
}

inline json to_json(const SchedulerConfig& cfg) {
  if (const auto* s = std::get_if<StaticConfig>(&cfg)) {
    json j{{"type", "static"}};
    if (!s->proportions.empty()) j["proportions"] = s->proportions;
    if (!s->device_order.empty()) j["device_order"] = s->device_order;
    return j;
  }
  if (const auto* d = std::get_if<DynamicConfig>(&cfg)) return json{{"type", "dynamic"}, {"num_packages", d->num_packages}};
  const auto& h = std::get<HGuidedConfig>(cfg);
  json j{{"type", "hguided"}, {"k", h.k}, {"include_device_count", h.include_device_count}};
  if (!h.powers.empty()) j["powers"] = h.powers;
  if (h.adaptive) {
    j["adaptive"] = true;
    j["ema_alpha"] = h.ema_alpha;
  }
  return j;
}

inline ProgramSpec program_from_json(const json& j) {
  ProgramSpec s;
  s.kernel = j.at("kernel").get<std::string>();
  s.global_work_size = j.at("global_work_size").get<std::uint64_t>();
  s.local_work_size = j.at("local_work_size").get<std::uint64_t>();
  if (j.contains("out_pattern")) {
    s.out_pattern.out_indices = j.at("out_pattern").at("out_indices").get<std::uint64_t>();
    s.out_pattern.work_items = j.at("out_pattern").at("work_items").get<std::uint64_t>();
  }
  auto read_buffers = [&](const char* key, BufferRole role, std::vector<BufferDesc>& into) {
    if (!j.contains(key)) return;
    for (const json& b : j.at(key))
      into.push_back(BufferDesc{b.at("name").get<std::string>(), b.at("element_size_bytes").get<std::uint64_t>(),
                                b.at("element_count").get<std::uint64_t>(), role});
  };
  read_buffers("in_buffers", BufferRole::Input, s.in_buffers);
  read_buffers("out_buffers", BufferRole::Output, s.out_buffers);
  if (j.contains("args"))
    for (const json& a : j.at("args")) {
      if (a.is_number_integer()) s.args.emplace_back(a.get<std::int64_t>());
      else if (a.is_number()) s.args.emplace_back(a.get<double>());
      else throw Error(ErrorCode::ConfigError, "kernel args must be scalars");
    }
  return s;
}

inline json to_json(const ProgramSpec& s) {
  json args = json::array();
  for (const ArgValue& a : s.args) std::visit([&](auto v) { args.push_back(v); }, a);
  auto buffers = [](const std::vector<BufferDesc>& v) {
    json arr = json::array();
    for (const BufferDesc& b : v)
      arr.push_back({{"name", b.name}, {"element_size_bytes", b.element_size_bytes}, {"element_count", b.element_count}});
    return arr;
  };
  return json{{"kernel", s.kernel},
              {"global_work_size", s.global_work_size},
              {"local_work_size", s.local_work_size},
              {"out_pattern", {{"out_indices", s.out_pattern.out_indices}, {"work_items", s.out_pattern.work_items}}},
              {"in_buffers", buffers(s.in_buffers)},
              {"out_buffers", buffers(s.out_buffers)},
              {"args", std::move(args)}};
}

inline json to_json(const Package& p) {
  return json{{"seq", p.seq},
              {"device_index", p.device_index},
              {"device_id", p.device_id},
              {"offset_wg", p.offset_wg},
              {"size_wg", p.size_wg},
              {"t_enqueue_ms", p.t_enqueue_ms},
              {"t_start_ms", p.t_start_ms},
              {"t_end_ms", p.t_end_ms}};
}

inline json to_json(const ExecutionTrace& t) {
  json devices = json::array(), packages = json::array();
  for (const DeviceProfile& d : t.devices) devices.push_back(to_json(d));
  for (const Package& p : t.packages) packages.push_back(to_json(p));
  return json{{"schema", t.schema},
              {"program",
               {{"kernel", t.program.kernel},
                {"global_work_size", t.program.global_work_size},
                {"local_work_size", t.program.local_work_size},
                {"total_work_groups", t.program.total_work_groups},
                {"out_pattern",
                 {{"out_indices", t.program.out_pattern.out_indices}, {"work_items", t.program.out_pattern.work_items}}}}},
              {"devices", std::move(devices)},
              {"scheduler", t.scheduler},
              {"clock_mode", std::string(clock_mode_name(t.clock_mode))},
              {"seed", t.seed},
              {"init_ms", t.init_ms},
              {"init_in_total", t.init_in_total},
              {"packages", std::move(packages)},
              {"t_total_ms", t.t_total_ms},
              {"per_device_time_ms", t.per_device_time_ms}};
}

inline ExecutionTrace trace_from_json(const json& j) {
  try {
    ExecutionTrace t;
    t.schema = j.at("schema").get<std::uint32_t>();
    const json& p = j.at("program");
    t.program = ProgramSummary{p.at("kernel").get<std::string>(), p.at("global_work_size").get<std::uint64_t>(),
                               p.at("local_work_size").get<std::uint64_t>(), p.at("total_work_groups").get<std::uint64_t>(),
                               OutPattern{p.at("out_pattern").at("out_indices").get<std::uint64_t>(),
                                          p.at("out_pattern").at("work_items").get<std::uint64_t>()}};
    for (const json& d : j.at("devices")) t.devices.push_back(device_from_json(d));
    t.scheduler = j.at("scheduler").get<std::string>();
    t.clock_mode = j.at("clock_mode").get<std::string>() == "wall" ? ClockMode::Wall : ClockMode::Virtual;
    t.seed = j.at("seed").get<std::uint64_t>();
    t.init_ms = j.at("init_ms").get<double>();
    t.init_in_total = j.at("init_in_total").get<bool>();
    for (const json& q : j.at("packages")) {
      Package k;
      k.seq = q.at("seq").get<std::uint64_t>();
      k.device_index = q.at("device_index").get<std::uint32_t>();
      k.device_id = q.at("device_id").get<std::string>();
      k.offset_wg = q.at("offset_wg").get<std::uint64_t>();
      k.size_wg = q.at("size_wg").get<std::uint64_t>();
      k.t_enqueue_ms = q.at("t_enqueue_ms").get<double>();
      k.t_start_ms = q.at("t_start_ms").get<double>();
      k.t_end_ms = q.at("t_end_ms").get<double>();
      t.packages.push_back(std::move(k));
    }
    t.t_total_ms = j.at("t_total_ms").get<double>();
    t.per_device_time_ms = j.at("per_device_time_ms").get<std::map<std::string, double>>();
    return t;
  } catch (const json::exception& e) {
    throw Error(ErrorCode::MalformedTrace, e.what());
  } catch (const Error& e) {
    throw Error(ErrorCode::MalformedTrace, e.what());
  }
}

inline std::string trace_to_json_string(const ExecutionTrace& t) { return to_json(t).dump(2) + "\n"; }

inline std::string trace_to_csv(const ExecutionTrace& t) {
  std::string out = "seq,device_id,offset_wg,size_wg,t_enqueue_ms,t_start_ms,t_end_ms\n";
  for (const Package& p : t.packages)
    out += std::to_string(p.seq) + ',' + p.device_id + ',' + std::to_string(p.offset_wg) + ',' +
           std::to_string(p.size_wg) + ',' + format_double(p.t_enqueue_ms) + ',' + format_double(p.t_start_ms) + ',' +
           format_double(p.t_end_ms) + '\n';
  return out;
}

inline json to_json(const MetricsReport& r) {
  json j{{"balance", r.balance},       {"speedup", r.speedup},       {"s_max", r.s_max},
         {"efficiency", r.efficiency}, {"work_share", r.work_share}, {"notes", r.notes}};
  if (r.overhead_pct) j["overhead_pct"] = *r.overhead_pct;
  return j;
}

}  // namespace coexec
