// chart.hpp — the Introspector's package chart as SVG (reference:
// chart.hpp:52-154): one lane per device, one mark per
// package (x = its [t_start, t_end) interval, height ∝ size_wg), a 0..t_max
// time axis with 11 ticks and the per-device work-share bar underneath.
//
// The output is byte-identical to the reference's for the same trace
// (tests/test_experiment.py), so B200 charts diff against reference charts.
#pragma once

#include <algorithm>
#include <cstdio>
#include <map>
#include <sstream>
#include <string>
#include <string_view>
#include <utility>
#include <vector>

#include "coexec/core.hpp"
#include "coexec/error.hpp"
#include "coexec/metrics.hpp"

namespace coexec {

namespace svg {

// Two-decimal coordinate (the chart's fixed precision).
inline std::string num(double v) {
  char b[40];
  std::snprintf(b, sizeof b, "%.2f", v);
  return b;
}

// Layout constants printed with the stream's default formatting ("960").
inline std::string raw(double v) {
  std::ostringstream o;
  o << v;
  return o.str();
}

inline std::string escaped(std::string_view s) {
  std::string r;
  r.reserve(s.size());
  for (char c : s) {
    if (c == '&') r += "&amp;";
    else if (c == '<') r += "&lt;";
    else if (c == '>') r += "&gt;";
    else if (c == '"') r += "&quot;";
    else r += c;
  }
  return r;
}

// Lane colours (seaborn "muted"), cycling after eight devices.
inline const char* lane_colour(std::size_t lane) {
  static constexpr const char* kColours[8] = {"#4878cf", "#ee854a", "#6acc65", "#d65f5f",
                                              "#956cb4", "#8c613c", "#dc7ec0", "#797979"};
  return kColours[lane % 8];
}

using Attrs = std::vector<std::pair<const char*, std::string>>;

// One element per line: <name a="v" ...>body</name> or <name .../>.
class Doc {
 public:
  void element(const char* name, const Attrs& attrs, const std::string* body = nullptr) {
    out_ << '<' << name;
    for (const auto& [k, v] : attrs) out_ << ' ' << k << "=\"" << v << '"';
    if (body) out_ << '>' << *body << "</" << name << ">\n";
    else out_ << "/>\n";
  }
  void text(const Attrs& attrs, const std::string& body) { element("text", attrs, &body); }
  void open(const Attrs& attrs) {
    out_ << "<svg";
    for (const auto& [k, v] : attrs) out_ << ' ' << k << "=\"" << v << '"';
    out_ << ">\n";
  }
  std::string close() {
    out_ << "</svg>\n";
    return out_.str();
  }

 private:
  std::ostringstream out_;
};

}  // namespace svg

inline std::string render_svg(const ExecutionTrace& trace) {
  if (trace.packages.empty()) throw Error(ErrorCode::MalformedTrace, "trace has no packages");
  // Geometry (px).
  const double W = 960.0, left = 110.0, right = 20.0, lane_h = 46.0, gap = 8.0, top = 54.0;
  const double plot_w = W - left - right;
  const std::size_t n_lanes = trace.devices.size();
  const double bar_y = top + static_cast<double>(n_lanes) * (lane_h + gap) + 36.0;
  const double H = bar_y + 66.0;

  double t_max = trace.t_total_ms;
  std::uint64_t biggest = 1;
  for (const Package& p : trace.packages) {
    t_max = std::max(t_max, p.t_end_ms);
    biggest = std::max(biggest, p.size_wg);
  }
  if (!(t_max > 0.0)) t_max = 1.0;
  auto x_at = [&](double t) { return left + t / t_max * plot_w; };
  auto lane_y = [&](std::size_t lane) { return top + static_cast<double>(lane) * (lane_h + gap); };
  std::map<std::string, std::size_t> lane_index;
  for (std::size_t i = 0; i < n_lanes; ++i) lane_index.emplace(trace.devices[i].id, i);

  const std::string sans = "sans-serif";
  svg::Doc doc;
  doc.open({{"xmlns", "http://www.w3.org/2000/svg"},
            {"width", svg::raw(W)},
            {"height", svg::raw(H)},
            {"viewBox", "0 0 " + svg::raw(W) + " " + svg::raw(H)}});
  doc.element("rect", {{"width", svg::raw(W)}, {"height", svg::raw(H)}, {"fill", "#ffffff"}});
  doc.text({{"x", svg::raw(left)}, {"y", "22"}, {"font-family", sans}, {"font-size", "15"}},
           svg::escaped(trace.program.kernel) + " — " + svg::escaped(trace.scheduler) + " (" +
               std::string(clock_mode_name(trace.clock_mode)) + " clock, t_total " + svg::num(trace.t_total_ms) +
               " ms)");

  for (int k = 0; k <= 10; ++k) {  // time axis: grid line + label per tenth
    const double t = t_max * k / 10.0;
    const std::string x = svg::num(x_at(t));
    doc.element("line", {{"x1", x}, {"y1", svg::raw(top - 8)}, {"x2", x}, {"y2", svg::raw(bar_y - 24)},
                         {"stroke", "#dddddd"}, {"stroke-width", "1"}});
    doc.text({{"x", x}, {"y", svg::raw(top - 12)}, {"font-family", sans}, {"font-size", "10"},
              {"text-anchor", "middle"}, {"fill", "#555555"}},
             svg::num(t));
  }

  for (std::size_t i = 0; i < n_lanes; ++i) {  // lane labels and baselines
    const double y0 = lane_y(i);
    doc.text({{"x", "8"}, {"y", svg::num(y0 + lane_h / 2 + 4)}, {"font-family", sans}, {"font-size", "12"}},
             svg::escaped(trace.devices[i].id));
    doc.element("line", {{"x1", svg::raw(left)}, {"y1", svg::num(y0 + lane_h)}, {"x2", svg::raw(W - right)},
                         {"y2", svg::num(y0 + lane_h)}, {"stroke", "#bbbbbb"}, {"stroke-width", "1"}});
  }

  for (const Package& p : trace.packages) {  // one mark per package, hover title
    const auto it = lane_index.find(p.device_id);
    if (it == lane_index.end())
      throw Error(ErrorCode::MalformedTrace, "package on unknown device '" + p.device_id + "'");
    const std::size_t lane = it->second;
    const double h = std::max(2.0, lane_h * static_cast<double>(p.size_wg) / static_cast<double>(biggest));
    const double x = x_at(p.t_start_ms);
    const double w = std::max(0.75, x_at(p.t_end_ms) - x);
    const std::string title = "<title>seq " + std::to_string(p.seq) + ": wg [" + std::to_string(p.offset_wg) + ", " +
                              std::to_string(p.end_wg()) + ") on " + svg::escaped(p.device_id) + ", " +
                              svg::num(p.t_start_ms) + "-" + svg::num(p.t_end_ms) + " ms</title>";
    doc.element("rect",
                {{"class", "pkg"}, {"x", svg::num(x)}, {"y", svg::num(lane_y(lane) + lane_h - h)},
                 {"width", svg::num(w)}, {"height", svg::num(h)}, {"fill", svg::lane_colour(lane)},
                 {"fill-opacity", "0.85"}},
                &title);
  }

  const auto share = work_share_of(trace);  // stacked work-share bar
  doc.text({{"x", "8"}, {"y", svg::num(bar_y - 6)}, {"font-family", sans}, {"font-size", "12"}}, "work share");
  double x = left;
  for (std::size_t i = 0; i < n_lanes; ++i) {
    const auto s = share.find(trace.devices[i].id);
    if (s == share.end()) continue;
    const double w = s->second * plot_w;
    doc.element("rect", {{"class", "share"}, {"x", svg::num(x)}, {"y", svg::num(bar_y)}, {"width", svg::num(w)},
                         {"height", "22"}, {"fill", svg::lane_colour(i)}});
    if (w > 36.0) {
      char label[96];
      std::snprintf(label, sizeof label, "%s %.1f%%", trace.devices[i].id.c_str(), s->second * 100.0);
      doc.text({{"x", svg::num(x + w / 2)}, {"y", svg::num(bar_y + 15)}, {"font-family", sans},
                {"font-size", "11"}, {"text-anchor", "middle"}, {"fill", "#ffffff"}},
               svg::escaped(label));
    }
    x += w;
  }
  return doc.close();
}

}  // namespace coexec
