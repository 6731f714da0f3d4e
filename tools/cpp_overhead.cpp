// Per-run host overhead of the C++ engine without Python: device-resident
// Gaussian 4096^2 runs, wall time per run vs the package's kernel interval.
#include <chrono>
#include <cstdio>
#include <vector>

#include "coexec/engine.hpp"

int main() {
  using namespace coexec;
  const uint64_t W = 4096, H = 4096, F = 31;
  ProgramSpec s;
  s.kernel = "gaussian";
  s.global_work_size = W * H;
  s.local_work_size = 128;
  s.in_buffers = {{"image", 4, W * H, BufferRole::Input}, {"filter", 4, F * F, BufferRole::Input}};
  s.out_buffers = {{"out", 4, W * H, BufferRole::Output}};
  s.args = {int64_t(W), int64_t(H), int64_t(F)};
  EngineConfig cfg;
  DeviceProfile d;
  d.id = "gpu0";
  d.backend.kind = BackendKind::Cuda;
  d.min_package_work_groups = 1;
  cfg.devices = {d};
  cfg.scheduler = StaticConfig{};
  Engine e(cfg, validate_program(s));
  std::vector<float> img(W * H, 0.5f), filt(F * F, 1.0f / (F * F));
  const void* in[] = {img.data(), filt.data()};
  e.run_into(in, {});
  double wall = 0, kern = 0, tot = 0, pre = 0, post = 0;
  const int n = 200;
  for (int i = 0; i < n; ++i) {
    const auto t0 = std::chrono::steady_clock::now();
    const ExecutionTrace t = e.run_into({}, {});
    const double w = std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now() - t0).count();
    wall += w;
    kern += t.packages[0].t_end_ms - t.packages[0].t_start_ms;
    tot += t.t_total_ms;
    pre += t.packages[0].t_start_ms;          // run entry -> kernel start (run epoch = entry)
    post += w - t.packages[0].t_end_ms;       // kernel end -> run return
  }
  std::printf("C++ run_into: wall %.4f ms  t_total %.4f ms  kernel %.4f ms  -> host overhead %.1f us/run "
              "(entry->kernel start %.1f us, kernel end->return %.1f us)\n",
              wall / n, tot / n, kern / n, (wall - kern) / n * 1e3, pre / n * 1e3, post / n * 1e3);
  return 0;
}
