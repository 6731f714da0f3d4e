// kernels.cuh — the sm_100a kernel registry shared by the device layer.
//
// Every kernel is a pure function of (global work-item index, args, read-only
// inputs) that writes only the out_range_for slice of the items it is given —
// the contract of the reference's KernelFn (workloads.hpp:42-44) — launched
// over one package [first_item, first_item + item_count).
#pragma once

#include <cuda_runtime.h>
#include <stdint.h>

#include <memory>
#include <string>
#include <vector>

#include "ecl_cuda.h"

namespace ecl {

enum class KernelKind { VecScale, Mandelbrot, MandelbrotF32, Synthetic, Gaussian, NBody, Binomial, Ray, Fault, Plugin };

// A user kernel registered with ecl_kernel_register (plugin.cu).
struct PluginKernel;

enum class SyntheticProfile { Constant = 0, Ramp = 1, Step = 2 };

// Mandelbrot args [W, H, max_iter, x0, y0, x1, y1] (workloads.hpp:102-120).
struct MandelParams {
  uint64_t width = 0, height = 0;
  uint32_t max_iterations = 1;
  double x0 = -2.5, y0 = -1.25, x1 = 1.0, y1 = 1.25;
};

struct GaussianParams {
  uint32_t width = 0, height = 0, filter = 0;
};

struct NBodyParams {
  uint64_t bodies = 0;
  float dt = 0.005f, eps2 = 500.0f;
};

struct BinomialParams {
  uint32_t steps = 254;
  uint64_t options = 0;  // scalar options (4 per work-group)
};

struct RayParams {
  uint32_t width = 0, height = 0, spheres = 0, max_depth = 0;
};

// Resolved kernel: the device-independent half of ecl_kernel.
struct KernelSpec {
  KernelKind kind = KernelKind::VecScale;
  SyntheticProfile profile = SyntheticProfile::Constant;
  std::string id;
  int variant = -1;  // "<kernel>@<n>" tuning variant; -1 = default (or the ECL_* env hook)
  uint64_t gws = 0, lws = 1, out_indices = 1, out_work_items = 1;
  // > 1: each work-item's out_indices uint32 outputs are identical copies
  // (Mandelbrot's 4:1 pattern); the kernel also writes one compact value per
  // item (LaunchEnv::compact) so host copies move 1/replicate of the bytes.
  uint32_t replicate = 1;
  // Bytes per compact value: 2 when every value fits 16 bits (Mandelbrot
  // counts with max_iterations < 65536), halving the compact D2H copies and
  // the host's reads of them; 4 otherwise.
  uint32_t compact_bytes = 4;
  // > 0: even with resident outputs a package runs as sub-launches of about
  // this many work-items alternating over the device's two compute lanes.
  // Set for kernels whose single long launch is measurably slower than the
  // same work as two-stream pieces (Ray: 11.0 ms vs 9.9 ms at 8192^2).
  uint64_t compute_split_items = 0;
  // The kernel can store its outputs into peer devices' buffers as it
  // computes them (LaunchEnv::peer_out): an iterative run then needs no
  // separate per-step exchange of those outputs.
  bool peer_writes = false;
  std::vector<ecl_arg> args;
  std::vector<ecl_buffer_geom> inputs, outputs;
  // parsed arguments
  MandelParams mandel;
  double a = 0.0, b = 0.0;  // vecscale
  double synth_param = 1.0;
  bool synth_has_param = false;
  uint64_t fault_item = 0;  // "fault" test kernel: the work-item that traps
  GaussianParams gauss;
  NBodyParams nbody;
  BinomialParams binom;
  RayParams ray;
  std::shared_ptr<const PluginKernel> plugin;  // KernelKind::Plugin: keeps the loaded image alive
};

// Everything a launcher needs from the device context.
struct LaunchEnv {
  cudaStream_t stream = nullptr;
  int sms = 148;
  void* const* in = nullptr;   // device pointers of the bound inputs
  void* const* out = nullptr;  // device pointers of the bound outputs
  unsigned* ctrl = nullptr;    // zeroed per-device control words (work counters)
  void* scratch = nullptr;     // per-device, per-binding kernel scratch (scratch_bytes())
  uint32_t* compact = nullptr;  // replicate > 1 and host copies pending: one value per item
  uint32_t compact_bytes = 4;   // KernelSpec::compact_bytes: 2 = the values are stored as uint16
  int device = 0;               // CUDA ordinal
  // Host mirrors of the inputs host_mirrored_input() names (nullptr for the
  // others): small inputs a launcher passes by value in its parameters.
  const void* const* in_host = nullptr;
  // The piece's outputs are copied to host memory right after it (e2e runs).
  bool host_copies = false;
  // Fused exchange (kernels with KernelSpec::peer_writes): the current output
  // buffers of the other devices of an iterative run, n_peers x outputs
  // pointers (peer-major; nullptr = none); the kernel stores its results
  // there too, over NVLink, as it computes them.
  void* const* peer_out = nullptr;
  uint32_t n_peers = 0;
  // The device's kernel-launch counter: the caller counts one launch per
  // launch_kernel call, a launcher that issues more kernels adds the rest.
  uint64_t* extra_launches = nullptr;
};

constexpr uint32_t kMaxPeerWrites = 8;  // peers a fused-exchange kernel writes to

// The compact output a replicating kernel writes (LaunchEnv::compact,
// compact_bytes): one value per item, 16- or 32-bit.
struct CompactOut {
  void* p = nullptr;
  uint32_t bytes = 4;
  __host__ __device__ explicit operator bool() const { return p != nullptr; }
  __device__ __forceinline__ void put(uint64_t i, uint32_t v) const {
    if (bytes == 2)
      static_cast<uint16_t*>(p)[i] = static_cast<uint16_t>(v);
    else
      static_cast<uint32_t*>(p)[i] = v;
  }
};
inline CompactOut compact_of(const LaunchEnv& env) { return CompactOut{env.compact, env.compact_bytes}; }

// Device scratch a kernel needs per binding (e.g. Mandelbrot coordinate tables),
// filled once by prepare_kernel when the program is bound to a device.
uint64_t scratch_bytes(const KernelSpec& spec);
cudaError_t prepare_kernel(const KernelSpec& spec, const LaunchEnv& env);
uint64_t mandelbrot_scratch_bytes(const KernelSpec& spec);
uint64_t binomial_scratch_bytes(const KernelSpec& spec);
cudaError_t prepare_mandelbrot(const KernelSpec& spec, const LaunchEnv& env);

// Prefix of input `input` (bytes) the work-items [first, first+count) read:
// lets the device layer stream an input up ahead of the pieces that need it
// (Gaussian rows + halo, Binomial options, vecscale elements); other
// kernels read whole buffers.
uint64_t input_bytes_needed(const KernelSpec& spec, uint32_t input, uint64_t first, uint64_t count);

// Inputs the device layer keeps a host copy of (LaunchEnv::in_host), kept in
// step with every way the device copy changes (upload, replication, raw
// upload, swap): Gaussian's filter, which each launch carries in its
// parameters instead of a per-device constant bank.
bool host_mirrored_input(const KernelSpec& spec, uint32_t input);
bool gaussian_mirrors_input(uint32_t input);

// Parses and validates (kernel_for + check_buffer_shapes semantics).
// Returns ECL_OK or a negative status with *err filled.
int resolve_kernel(KernelSpec& spec, std::string* err);

// Launches the kernel over work-items [first, first + count) on env.stream.
cudaError_t launch_kernel(const KernelSpec& spec, const LaunchEnv& env, uint64_t first, uint64_t count);

// Per-kind launchers (one translation unit each).
cudaError_t launch_mandelbrot(const KernelSpec& spec, const LaunchEnv& env, uint64_t first, uint64_t count);
cudaError_t launch_vecscale(const KernelSpec& spec, const LaunchEnv& env, uint64_t first, uint64_t count);
cudaError_t launch_synthetic(const KernelSpec& spec, const LaunchEnv& env, uint64_t first, uint64_t count);
cudaError_t launch_gaussian(const KernelSpec& spec, const LaunchEnv& env, uint64_t first, uint64_t count);
cudaError_t launch_nbody(const KernelSpec& spec, const LaunchEnv& env, uint64_t first, uint64_t count);
cudaError_t launch_binomial(const KernelSpec& spec, const LaunchEnv& env, uint64_t first, uint64_t count);
cudaError_t launch_ray(const KernelSpec& spec, const LaunchEnv& env, uint64_t first, uint64_t count);

// Plugins (plugin.cu): the registered kernel named `id` (null if none), the
// launch-shape checks, and the launcher (include/ecl_plugin.h ABI).
std::shared_ptr<const PluginKernel> find_plugin(const std::string& id);
int register_plugin(const std::string& id, const void* image, const std::string& entry, std::string* err);
int unregister_plugin(const std::string& id, std::string* err);
int check_plugin_spec(const KernelSpec& spec, std::string* err);
cudaError_t launch_plugin(const KernelSpec& spec, const LaunchEnv& env, uint64_t first, uint64_t count);
bool is_builtin_kernel_id(const std::string& id);

// Test hook (ECL_FAULT_INJECTION=1 only): the work-item `fault_item` executes
// a trap, so the device faults mid-run (reference test_engine.cpp:236-254).
cudaError_t launch_fault(const KernelSpec& spec, const LaunchEnv& env, uint64_t first, uint64_t count);
// Exactly-once tally: tally[i] += 1 for i in [first, first + count).
cudaError_t launch_tally(uint32_t* tally, uint64_t first, uint64_t count, cudaStream_t stream);

}  // namespace ecl
