// plugin.cu — user device kernels co-executed like the built-in ones.
//
// The reference's plugin seam is a per-work-item host function:
// Engine::run(inputs, KernelFn, CostFn) (engine.hpp:223; KernelFn/CostFn at
// workloads.hpp:44,47) and kernel_for(prog) (workloads.hpp:203) resolving an
// id.  Here the per-item function is a CUDA kernel compiled out of tree for
// sm_100a (cubin / fatbin / PTX) with the launch ABI of include/ecl_plugin.h.
// ecl_kernel_register loads the image once as a context-independent CUDA
// library (cudaLibraryLoadData): it is loaded into each device's context on
// first launch there, so one registration serves every B200.  The registry
// holds shared references, so a kernel created from an id keeps its image
// loaded even after the id is unregistered.
#include <cuda_runtime.h>

#include <algorithm>
#include <map>
#include <mutex>

#include "ecl_plugin.h"
#include "kernels.cuh"

namespace ecl {

struct PluginKernel {
  std::string id, entry;
  cudaLibrary_t lib = nullptr;
  cudaKernel_t fn = nullptr;
  ~PluginKernel() {
    if (lib) cudaLibraryUnload(lib);
    cudaGetLastError();
  }
};

namespace {

std::mutex g_m;
// Never destroyed: libraries must not be unloaded during CUDA's own teardown.
auto* g_plugins = new std::map<std::string, std::shared_ptr<const PluginKernel>>();

}  // namespace

std::shared_ptr<const PluginKernel> find_plugin(const std::string& id) {
  std::lock_guard lock(g_m);
  auto it = g_plugins->find(id);
  return it == g_plugins->end() ? nullptr : it->second;
}

int register_plugin(const std::string& id, const void* image, const std::string& entry, std::string* err) {
  if (id.empty() || !image || entry.empty()) {
    *err = "kernel_register: id, image and entry are required";
    return ECL_CONFIG_ERROR;
  }
  if (is_builtin_kernel_id(id)) {
    *err = "kernel_register: '" + id + "' is a built-in kernel id";
    return ECL_CONFIG_ERROR;
  }
  {
    std::lock_guard lock(g_m);
    if (g_plugins->count(id)) {
      *err = "kernel_register: '" + id + "' is already registered";
      return ECL_CONFIG_ERROR;
    }
  }
  int n = 0;
  if (cudaGetDeviceCount(&n) != cudaSuccess || n < 1) {
    cudaGetLastError();
    *err = "kernel_register: CUDA unavailable";
    return ECL_CONFIG_ERROR;
  }
  auto pk = std::make_shared<PluginKernel>();
  pk->id = id;
  pk->entry = entry;
  cudaError_t e = cudaLibraryLoadData(&pk->lib, image, nullptr, nullptr, 0, nullptr, nullptr, 0);
  if (e != cudaSuccess) {
    pk->lib = nullptr;
    cudaGetLastError();
    *err = "kernel_register: image does not load (" + std::string(cudaGetErrorName(e)) + ")";
    return ECL_UNKNOWN_KERNEL;
  }
  e = cudaLibraryGetKernel(&pk->fn, pk->lib, entry.c_str());
  if (e != cudaSuccess) {
    cudaGetLastError();
    *err = "kernel_register: no entry '" + entry + "' in the image (" + std::string(cudaGetErrorName(e)) + ")";
    return ECL_UNKNOWN_KERNEL;
  }
  std::lock_guard lock(g_m);
  if (!g_plugins->emplace(id, std::move(pk)).second) {
    *err = "kernel_register: '" + id + "' is already registered";
    return ECL_CONFIG_ERROR;
  }
  return ECL_OK;
}

int unregister_plugin(const std::string& id, std::string* err) {
  std::lock_guard lock(g_m);
  if (!g_plugins->erase(id)) {
    *err = "kernel_unregister: no plugin '" + id + "'";
    return ECL_UNKNOWN_KERNEL;
  }
  return ECL_OK;
}

int check_plugin_spec(const KernelSpec& s, std::string* err) {
  auto bad = [&](const std::string& m) {
    *err = s.id + ": " + m;
    return ECL_BAD_KERNEL_ARGS;
  };
  if (s.lws == 0 || s.lws > 1024) return bad("plugin kernels run one CTA per work-group: local_work_size <= 1024");
  if (s.inputs.size() > ECL_PLUGIN_MAX_BUFFERS || s.outputs.size() > ECL_PLUGIN_MAX_BUFFERS)
    return bad("at most " + std::to_string(ECL_PLUGIN_MAX_BUFFERS) + " input and output buffers");
  if (s.args.size() > ECL_PLUGIN_MAX_ARGS) return bad("at most " + std::to_string(ECL_PLUGIN_MAX_ARGS) + " args");
  return ECL_OK;
}

cudaError_t launch_plugin(const KernelSpec& s, const LaunchEnv& env, uint64_t first, uint64_t count) {
  if (count == 0) return cudaSuccess;
  ecl_plugin_launch p{};
  p.global_work_size = s.gws;
  p.local_work_size = s.lws;
  p.out_indices = s.out_indices;
  p.out_work_items = s.out_work_items;
  p.n_args = static_cast<uint32_t>(s.args.size());
  p.n_inputs = static_cast<uint32_t>(s.inputs.size());
  p.n_outputs = static_cast<uint32_t>(s.outputs.size());
  p.device = env.device;
  for (uint32_t i = 0; i < p.n_inputs; ++i) p.inputs[i] = env.in[i];
  for (uint32_t i = 0; i < p.n_outputs; ++i) p.outputs[i] = env.out[i];
  std::copy(s.args.begin(), s.args.end(), p.args);
  // Packages and pieces are whole work-groups; grids beyond 2^31-1 CTAs go
  // as several launches.
  const uint64_t groups = (count + s.lws - 1) / s.lws, max_grid = 0x7fffffffull;
  for (uint64_t g0 = 0; g0 < groups; g0 += max_grid) {
    const uint64_t g = std::min(max_grid, groups - g0);
    p.first_item = first + g0 * s.lws;
    p.item_count = std::min(g * s.lws, count - g0 * s.lws);
    void* args[] = {&p};
    const cudaError_t e = cudaLaunchKernel(reinterpret_cast<const void*>(s.plugin->fn), dim3(static_cast<unsigned>(g)),
                                           dim3(static_cast<unsigned>(s.lws)), args, 0, env.stream);
    if (e != cudaSuccess) return e;
  }
  return cudaSuccess;
}

}  // namespace ecl
