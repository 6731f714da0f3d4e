// test_facade.cpp — the paper's listings written against ecl.hpp (the
// EngineCL drop-in surface) and checked against the CPU oracle.
//
//   Listing 1: Binomial on one device.
//   Listing 2: NBody on three devices, Static({0.08, 0.3}).
//   Mandelbrot co-executed with HGuided, bit-exact with the reference kernel.
//
// Usage: test_facade [--no-gpu | --plugin <plugins.cubin>]   (exit 0 = all checks passed)
#include <cmath>
#include <cstdint>
#include <cstdio>
#include <cstring>
#include <vector>

#include "coexec/ecl.hpp"
#include "ecl_cuda.h"

extern "C" {  // tests only: the CPU oracle (oracle/oracle.c)
void orc_binomial(const float* rand4, float* out4, uint32_t steps, uint64_t first_opt, uint64_t n_opt);
void orc_binomial_init(uint64_t seed, uint64_t n_opt, float* rand4);
void orc_nbody_init(uint64_t seed, uint64_t n, float* pos, float* vel);
void orc_nbody_step(const float* pos, const float* vel, uint64_t n, float dt, float eps2, float* npos, float* nvel,
                    uint64_t first, uint64_t count);
void orc_mandelbrot_f64(uint64_t w, uint64_t h, uint32_t max_iter, double x0, double y0, double x1, double y1,
                        uint64_t first, uint64_t count, uint32_t* counts);
}

struct float4_ {
  float x, y, z, w;
};

static int failures = 0;
#define CHECK(cond, ...)                          \
  do {                                            \
    if (!(cond)) {                                \
      std::printf("FAIL %s:%d: ", __FILE__, __LINE__); \
      std::printf(__VA_ARGS__);                   \
      std::printf("\n");                          \
      ++failures;                                 \
    }                                             \
  } while (0)

static int gpus() {
  int n = 0;
  return ecl_gpu_count(&n) == 0 ? n : 0;
}

static void listing1_binomial(int ng) {
  const int samples = 4 * 2048, steps = 254, steps1 = steps + 1, lws = steps1;
  const int samples_by4 = samples / 4;
  const uint64_t gws = static_cast<uint64_t>(lws) * samples_by4;
  std::vector<float4_> in(samples_by4), out(samples_by4);
  orc_binomial_init(42, samples, reinterpret_cast<float*>(in.data()));

  ecl::EngineCL engine;
  engine.use(ecl::Device(0));
  engine.global_work_items(gws);
  engine.local_work_items(lws);
  ecl::Program program;
  program.in(in);
  program.out(out);
  program.out_pattern(1, lws);
  program.kernel("binomial");
  program.arg(0, steps);  // positional
  program.arg(in);        // aggregate (buffers are bound by in()/out())
  program.arg(out);
  program.arg(steps1 * sizeof(float4_), ecl::Arg::LocalAlloc);
  program.arg(4, steps * sizeof(float4_), ecl::Arg::LocalAlloc);
  engine.use(std::move(program));
  engine.run();
  CHECK(!engine.has_errors(), "binomial: %s", engine.has_errors() ? engine.get_errors()[0].what() : "");
  std::vector<float> exp(samples);
  orc_binomial(reinterpret_cast<const float*>(in.data()), exp.data(), steps, 0, samples);
  const float* got = reinterpret_cast<const float*>(out.data());
  double worst = 0;
  for (int i = 0; i < samples; ++i) {
    const double err = std::fabs(got[i] - exp[i]) - 1e-6;
    worst = std::max(worst, err / std::max(1e-30, std::fabs(double(exp[i]))));
  }
  CHECK(worst <= 1e-5, "binomial: max rel err %g", worst);
  (void)ng;
}

static void listing2_nbody(int ng) {
  const int bodies = 8192;
  const float del_t = 0.005f, esp_sqr = 500.0f;
  const int lws = 64, gws = bodies;
  std::vector<float4_> in_pos(bodies), in_vel(bodies), out_pos(bodies), out_vel(bodies);
  orc_nbody_init(42, bodies, reinterpret_cast<float*>(in_pos.data()), reinterpret_cast<float*>(in_vel.data()));

  ecl::EngineCL engine;
  engine.use(ecl::Device(0 % ng), ecl::Device(1 % ng), ecl::Device(2 % ng));
  engine.work_items(gws, lws);
  auto props = {0.08, 0.3};
  engine.scheduler(ecl::Scheduler::Static(props));
  ecl::Program program;
  program.in(in_pos);
  program.in(in_vel);
  program.out(out_pos);
  program.out(out_vel);
  program.kernel("nbody");
  program.args(in_pos, in_vel, bodies, del_t, esp_sqr, out_pos, out_vel);
  engine.program(std::move(program));
  engine.run();
  CHECK(!engine.has_errors(), "nbody: %s", engine.has_errors() ? engine.get_errors()[0].what() : "");
  CHECK(engine.trace().packages.size() == 3, "nbody: static gives one package per device");
  std::vector<float4_> ep(bodies), ev(bodies);
  orc_nbody_step(reinterpret_cast<const float*>(in_pos.data()), reinterpret_cast<const float*>(in_vel.data()),
                 bodies, del_t, esp_sqr, reinterpret_cast<float*>(ep.data()), reinterpret_cast<float*>(ev.data()), 0,
                 bodies);
  double worst = 0;
  for (int i = 0; i < bodies; ++i)
    worst = std::max(worst, std::fabs(double(out_pos[i].x) - ep[i].x) / std::fabs(double(ep[i].x)));
  CHECK(worst <= 1e-4, "nbody: position rel err %g", worst);
}

static void mandelbrot_hguided(int ng) {
  const uint64_t w = 512, h = 384;
  std::vector<uint32_t> counts(w * h * 4);
  ecl::EngineCL engine;
  // the second device runs a specialization of the kernel (two pixels per
  // lane), the paper's Device(platform, device, kernel)
  engine.use(ecl::Device(0 % ng), ecl::Device(1 % ng, "mandelbrot@5"));
  engine.work_items(w * h, 256);
  engine.scheduler(ecl::Scheduler::HGuided(2.0));
  ecl::Program program;
  program.out(counts);
  program.out_pattern(4, 1);
  program.kernel("mandelbrot");
  program.args(static_cast<int64_t>(w), static_cast<int64_t>(h), int64_t{512}, -2.5, -1.25, 1.0, 1.25);
  engine.program(std::move(program));
  engine.run();
  CHECK(!engine.has_errors(), "mandelbrot: %s", engine.has_errors() ? engine.get_errors()[0].what() : "");
  std::vector<uint32_t> exp(w * h);
  orc_mandelbrot_f64(w, h, 512, -2.5, -1.25, 1.0, 1.25, 0, w * h, exp.data());
  uint64_t bad = 0;
  for (uint64_t i = 0; i < w * h; ++i)
    for (int c = 0; c < 4; ++c) bad += counts[4 * i + c] != exp[i];
  CHECK(bad == 0, "mandelbrot: %llu mismatching counts", static_cast<unsigned long long>(bad));
  CHECK(coexec::tiles_exactly(engine.trace().packages, w * h / 256), "mandelbrot: tiling");
}

// The reference's plugin overload Engine::run(inputs, kernel, cost)
// (engine.hpp:223) with a user kernel compiled out of tree
// (tests/plugins/plugins.cu -> _build/plugins.cubin, include/ecl_plugin.h).
static void plugin_kernel_run(int ng, const char* cubin) {
  const std::uint64_t n = 1 << 16;
  coexec::ProgramSpec spec;
  spec.global_work_size = n;
  spec.local_work_size = 128;
  spec.in_buffers.push_back({"x", 8, n, coexec::BufferRole::Input});
  spec.out_buffers.push_back({"y", 8, n, coexec::BufferRole::Output});
  spec.kernel = "vecscale";
  spec.args = {2.5, -1.0};
  coexec::EngineConfig cfg;
  for (int i = 0; i < 2; ++i) {
    coexec::DeviceProfile d;
    d.id = "gpu" + std::to_string(i);
    d.name = d.id;
    d.backend.kind = coexec::BackendKind::Cuda;
    d.backend.ordinal = i % ng;
    cfg.devices.push_back(d);
  }
  cfg.scheduler = coexec::DynamicConfig{8};
  std::vector<std::vector<std::byte>> inputs(1, std::vector<std::byte>(n * 8));
  auto* x = reinterpret_cast<double*>(inputs[0].data());
  for (std::uint64_t i = 0; i < n; ++i) x[i] = static_cast<double>(i) * 0.25 - 100.0;
  try {
    const coexec::DeviceKernel k = coexec::register_device_kernel_file("cpp_vecscale", cubin, "vecscale_plugin");
    coexec::Engine engine(cfg, coexec::validate_program(spec));
    const coexec::CostFn cost = [](std::uint64_t) { return 1.0; };
    const coexec::RunResult r = engine.run(inputs, k, cost);
    const auto* y = reinterpret_cast<const double*>(r.outputs[0].data());
    std::uint64_t bad = 0;
    for (std::uint64_t i = 0; i < n; ++i) bad += y[i] != 2.5 * x[i] + -1.0;
    CHECK(bad == 0, "plugin vecscale: %llu wrong items", static_cast<unsigned long long>(bad));
    CHECK(coexec::tiles_exactly(r.trace.packages, n / 128), "plugin vecscale: tiling");
    ecl_kernel_unregister("cpp_vecscale");
  } catch (const std::exception& e) {
    CHECK(false, "plugin run threw: %s", e.what());
  }
}

static void errors_are_collected() {
  std::vector<double> out(1024);
  ecl::EngineCL engine;
  engine.use(ecl::Device(0));
  engine.work_items(1024, 64);
  ecl::Program program;
  program.out(out);
  program.kernel("warp-drive");
  engine.program(std::move(program));
  engine.run();
  CHECK(engine.has_errors(), "unknown kernel must be reported");
  if (engine.has_errors()) {
    const auto code = engine.get_errors()[0].code();
    CHECK(code == coexec::ErrorCode::UnknownKernel || code == coexec::ErrorCode::ConfigError,
          "unexpected error %s", engine.get_errors()[0].what());
  }
}

int main(int argc, char** argv) {
  const bool no_gpu = argc > 1 && std::strcmp(argv[1], "--no-gpu") == 0;
  const int ng = gpus();
  errors_are_collected();
  if (!no_gpu) {
    if (ng < 1) {
      std::printf("FAIL: no CUDA device\n");
      return 1;
    }
    listing1_binomial(ng);
    listing2_nbody(ng);
    mandelbrot_hguided(ng);
    if (argc > 2 && std::strcmp(argv[1], "--plugin") == 0) plugin_kernel_run(ng, argv[2]);
  }
  std::printf("%s (%d failures)\n", failures ? "FAILED" : "OK", failures);
  return failures ? 1 : 0;
}
