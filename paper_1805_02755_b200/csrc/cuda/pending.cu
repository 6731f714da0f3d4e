// pending.cu — launchers of the paper benchmarks not yet on the device.
// Each returns cudaErrorNotSupported, which the device layer reports as
// ECL_KERNEL_PANIC: there is no CPU fallback.
#include "kernels.cuh"

namespace ecl {

cudaError_t launch_ray(const KernelSpec&, const LaunchEnv&, uint64_t, uint64_t) { return cudaErrorNotSupported; }

}  // namespace ecl
