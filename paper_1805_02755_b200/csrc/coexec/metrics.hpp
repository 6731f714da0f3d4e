// metrics.hpp — co-execution metrics (reference: metrics.hpp:19-164;
// paper definitions PAPER.md:522 overhead, :683 balance, :725 efficiency).
#pragma once

#include <algorithm>
#include <cstdint>
#include <map>
#include <optional>
#include <span>
#include <string>
#include <utility>
#include <vector>

#include "coexec/core.hpp"
#include "coexec/error.hpp"

namespace coexec {

/// Per-device busy span: first enqueue -> last end (engine.hpp:418-427).
inline std::map<std::string, std::pair<double, double>> device_spans(const ExecutionTrace& trace) {
  std::map<std::string, std::pair<double, double>> spans;
  for (const Package& p : trace.packages) {
    auto [it, fresh] = spans.try_emplace(p.device_id, p.t_enqueue_ms, p.t_end_ms);
    if (!fresh) {
      it->second.first = std::min(it->second.first, p.t_enqueue_ms);
      it->second.second = std::max(it->second.second, p.t_end_ms);
    }
  }
  return spans;
}

/// Busy span of the first device to finish over that of the last one.
inline double balance(const ExecutionTrace& trace) {
  if (trace.packages.empty()) throw Error(ErrorCode::EmptyTrace, "trace has no packages");
  const auto spans = device_spans(trace);
  // Ties keep the first device in id order, like the reference's strict
  // comparisons (metrics.hpp:35-45).
  const std::pair<double, double>* first = nullptr;
  const std::pair<double, double>* last = nullptr;
  for (const auto& [id, s] : spans) {
    if (!first || s.second < first->second) first = &s;
    if (!last || s.second > last->second) last = &s;
  }
  return (first->second - first->first) / (last->second - last->first);
}

/// sum T_i / max T_i over the devices' solo times.
inline double s_max(std::span<const double> solo_ms) {
  if (solo_ms.empty()) throw Error(ErrorCode::NonPositiveTime, "no solo times");
  double sum = 0.0, hi = 0.0;
  for (double t : solo_ms) {
    if (!(t > 0.0)) throw Error(ErrorCode::NonPositiveTime, "solo times must be > 0");
    sum += t;
    hi = std::max(hi, t);
  }
  return sum / hi;
}

/// Speedup over the fastest solo device and its share of s_max.
inline std::pair<double, double> speedup_and_efficiency(const ExecutionTrace& trace, std::span<const double> solo_ms) {
  if (trace.packages.empty()) throw Error(ErrorCode::EmptyTrace, "trace has no packages");
  if (solo_ms.empty()) throw Error(ErrorCode::MissingBaseline, "no solo baseline times");
  const double base = *std::min_element(solo_ms.begin(), solo_ms.end());
  if (!(base > 0.0)) throw Error(ErrorCode::NonPositiveTime, "baseline must be > 0");
  const double speedup = base / trace.t_total_ms;
  return {speedup, speedup / s_max(solo_ms)};
}

/// (T - T_ref) / T_ref * 100.
inline double overhead_pct(double t_ms, double t_reference_ms) {
  if (!(t_reference_ms > 0.0)) throw Error(ErrorCode::NonPositiveReference, "reference time must be > 0");
  return (t_ms - t_reference_ms) / t_reference_ms * 100.0;
}

inline std::map<std::string, double> work_share_of(const ExecutionTrace& trace) {
  std::map<std::string, double> share;
  std::uint64_t total = 0;
  for (const Package& p : trace.packages) {
    share[p.device_id] += static_cast<double>(p.size_wg);
    total += p.size_wg;
  }
  for (auto& [id, v] : share) v /= static_cast<double>(total);
  return share;
}

struct MetricsReport {
  double balance = 1.0;
  double speedup = 1.0;
  double s_max = 1.0;
  double efficiency = 1.0;
  std::optional<double> overhead_pct;
  std::map<std::string, double> work_share;
  std::vector<std::string> notes;
  bool operator==(const MetricsReport&) const = default;
};

inline MetricsReport make_report(const ExecutionTrace& trace, std::span<const double> solo_ms,
                                 std::optional<double> reference_ms = std::nullopt) {
  MetricsReport r;
  r.balance = balance(trace);
  std::tie(r.speedup, r.efficiency) = speedup_and_efficiency(trace, solo_ms);
  r.s_max = s_max(solo_ms);
  if (reference_ms) r.overhead_pct = overhead_pct(trace.t_total_ms, *reference_ms);
  r.work_share = work_share_of(trace);
  if (r.efficiency > 1.001) r.notes.push_back("efficiency above s_max by more than 0.1%; trace anomaly");
  return r;
}

}  // namespace coexec
