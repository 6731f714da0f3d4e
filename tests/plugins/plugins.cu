// Out-of-tree device kernels for the plugin-seam tests (include/ecl_plugin.h
// ABI), compiled by tests/plugins/Makefile into a cubin, a fatbin and PTX
// that the tests register at run time with ecl_kernel_register — the B200
// form of handing the reference's Engine::run(inputs, kernel, cost)
// (engine.hpp:223) a user KernelFn.
#include <cstdint>

#include "ecl_plugin.h"

// vecscale (workloads.hpp:207-214): out[i] = a*in[i] + b on doubles, without
// FMA contraction, like the oracle (oracle.c:orc_vecscale, -ffp-contract=off).
extern "C" __global__ void vecscale_plugin(const __grid_constant__ ecl_plugin_launch p) {
  const uint64_t i = ecl_plugin_item(&p);
  if (i >= p.first_item + p.item_count) return;
  const double a = ecl_plugin_arg_f64(&p, 0), b = ecl_plugin_arg_f64(&p, 1);
  const double* in = static_cast<const double*>(p.inputs[0]);
  double* out = static_cast<double*>(p.outputs[0]);
  out[i] = __dadd_rn(__dmul_rn(a, in[i]), b);
}

// One output per `out_work_items` items (an out pattern 1:G): item i adds
// (double)i into out[i / G].  Used with G > local_work_size to reproduce the
// reference's runtime IndivisiblePackage failure (test_engine.cpp:256-278).
extern "C" __global__ void group_sum_plugin(const __grid_constant__ ecl_plugin_launch p) {
  const uint64_t i = ecl_plugin_item(&p);
  if (i >= p.first_item + p.item_count) return;
  atomicAdd(static_cast<double*>(p.outputs[0]) + i / p.out_work_items, static_cast<double>(i));
}

// Writes the work-item index and the launch's device ordinal: lets a test see
// which device ran which package and that every item ran exactly once.
extern "C" __global__ void whoami_plugin(const __grid_constant__ ecl_plugin_launch p) {
  const uint64_t i = ecl_plugin_item(&p);
  if (i >= p.first_item + p.item_count) return;
  static_cast<uint64_t*>(p.outputs[0])[i] = (i << 8) | static_cast<uint64_t>(p.device & 0xff);
}
