/*
 * ecl_plugin.h — launch ABI of user device kernels ("binary kernels").
 *
 * The reference lets a caller co-execute ANY per-work-item function:
 *   Engine::run(inputs, const KernelFn& kernel, const CostFn& cost)
 *   — /root/reference/proj/include/coexec/engine.hpp:223, with
 *   KernelFn = void(uint64_t index, span<const ArgValue> args, const KernelBuffers&)
 *   and CostFn = double(uint64_t index) (workloads.hpp:44,47) —
 * and the paper's Device(platform, device, kernel) runs a per-device binary
 * kernel.  On B200 the per-item function is a CUDA kernel
 * compiled out of tree for sm_100a (cubin, fatbin or PTX) and registered by
 * id with ecl_kernel_register (include/ecl_cuda.h); a program whose kernel id
 * names it is co-executed like the built-in kernels.
 *
 * The entry must be
 *     extern "C" __global__ void entry(const __grid_constant__ ecl_plugin_launch p)
 * (the parameter stays in the constant parameter bank) and is launched once
 * per package piece with blockDim.x = local_work_size (<= 1024) and one CTA
 * per work-group of the piece, so work-item
 *     index = p.first_item + blockIdx.x * blockDim.x + threadIdx.x
 * (ecl_plugin_item() below) — the OpenCL-style global id the reference's
 * KernelFn receives.  Each work-item writes only its out_range_for slice
 * (core.hpp:172-185) of the full-extent outputs, at global offsets.
 * Plain C, usable from host code and from nvcc device code.
 */
#ifndef ECL_PLUGIN_H
#define ECL_PLUGIN_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

/* A kernel argument: coexec::ArgValue = variant<int64_t, double> (core.hpp:75). */
typedef struct {
  int32_t is_double;
  int32_t reserved;
  int64_t i;
  double d;
} ecl_arg;

#define ECL_PLUGIN_MAX_BUFFERS 8
#define ECL_PLUGIN_MAX_ARGS 16

/* The single by-value parameter of a plugin entry (kernel parameter space). */
typedef struct {
  uint64_t first_item;        /* first work-item of this launch (work-group aligned) */
  uint64_t item_count;        /* work-items of this launch */
  uint64_t global_work_size;  /* the program's index space */
  uint64_t local_work_size;
  uint64_t out_indices;       /* out pattern out_indices : work_items */
  uint64_t out_work_items;
  uint32_t n_args, n_inputs, n_outputs;
  int32_t device;             /* CUDA ordinal */
  const void* inputs[ECL_PLUGIN_MAX_BUFFERS]; /* this device's replica of every input */
  void* outputs[ECL_PLUGIN_MAX_BUFFERS];      /* this device's output partition (full extent) */
  ecl_arg args[ECL_PLUGIN_MAX_ARGS];
} ecl_plugin_launch;

#if defined(__CUDACC__)
/* Global work-item index of the calling thread. */
static __device__ __forceinline__ uint64_t ecl_plugin_item(const ecl_plugin_launch* p) {
  return p->first_item + (uint64_t)blockIdx.x * blockDim.x + threadIdx.x;
}
/* Argument i as a double (integers converted), arg_as_double (workloads.hpp:49). */
static __device__ __forceinline__ double ecl_plugin_arg_f64(const ecl_plugin_launch* p, uint32_t i) {
  return p->args[i].is_double ? p->args[i].d : (double)p->args[i].i;
}
#endif

#ifdef __cplusplus
}
#endif

#endif /* ECL_PLUGIN_H */
