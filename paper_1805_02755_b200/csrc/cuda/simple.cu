// simple.cu — the reference's regular kernels on sm_100a.
//
//   vecscale   out[i] = a*in[i] + b                workloads.hpp:207-214
//   synthetic  out[i] = cost(i)                    workloads.hpp:136-149,224-230
//   tally      exactly-once counter per work-item  engine.hpp:165-167,228-252
//
// All three are HBM-bound streams: 16 B/item (vecscale), 8 B/item
// (synthetic).  Each thread handles two consecutive items so the 8-byte
// elements move as 16-byte vectors; the grid is sized to a whole number of
// waves (SMs x resident blocks) and strides over the package.
#include <algorithm>

#include "kernels.cuh"

namespace ecl {
namespace {

constexpr int kThreads = 256;

unsigned stride_grid(const LaunchEnv& env, uint64_t pairs) {
  const uint64_t cap = static_cast<uint64_t>(env.sms) * 8;  // 8 x 256 threads resident per SM
  const uint64_t need = (pairs + kThreads - 1) / kThreads;
  return static_cast<unsigned>(need < cap ? (need ? need : 1) : cap);
}

// out[i] = a*in[i] + b with a separate multiply and add (no contraction:
// the reference is built with -ffp-contract=off semantics on x86-64).
__global__ void __launch_bounds__(kThreads)
    vecscale_kernel(const double* __restrict__ in, double* __restrict__ out, double a, double b, uint64_t first,
                    uint64_t count) {
  const uint64_t stride = static_cast<uint64_t>(gridDim.x) * blockDim.x;
  const uint64_t end = first + count;
  // Peel so the vector loop starts on a 16-byte boundary.
  uint64_t head = first;
  if (head & 1) {
    if (blockIdx.x == 0 && threadIdx.x == 0) out[head] = __dadd_rn(__dmul_rn(a, in[head]), b);
    ++head;
  }
  const uint64_t pairs = (end - head) / 2;
  const double2* in2 = reinterpret_cast<const double2*>(in + head);
  double2* out2 = reinterpret_cast<double2*>(out + head);
  for (uint64_t p = static_cast<uint64_t>(blockIdx.x) * blockDim.x + threadIdx.x; p < pairs; p += stride) {
    const double2 v = __ldcs(in2 + p);
    double2 r;
    r.x = __dadd_rn(__dmul_rn(a, v.x), b);
    r.y = __dadd_rn(__dmul_rn(a, v.y), b);
    __stcs(out2 + p, r);
  }
  const uint64_t tail = head + 2 * pairs;
  if (tail < end && blockIdx.x == 0 && threadIdx.x == 0) out[tail] = __dadd_rn(__dmul_rn(a, in[tail]), b);
}

__device__ __forceinline__ double synthetic_cost(int profile, uint64_t i, uint64_t gws, double param,
                                                 bool has_param) {
  switch (profile) {
    case 0:
      return has_param ? param : 1.0;
    case 1:
      return __dadd_rn(1.0, __ddiv_rn(__ull2double_rn(i), __ull2double_rn(gws)));
    default:
      return i < gws / 2 ? 1.0 : (has_param ? param : 10.0);
  }
}

__global__ void __launch_bounds__(kThreads)
    synthetic_kernel(double* __restrict__ out, int profile, uint64_t gws, double param, bool has_param,
                     uint64_t first, uint64_t count) {
  const uint64_t stride = static_cast<uint64_t>(gridDim.x) * blockDim.x;
  for (uint64_t k = static_cast<uint64_t>(blockIdx.x) * blockDim.x + threadIdx.x; k < count; k += stride) {
    const uint64_t i = first + k;
    out[i] = synthetic_cost(profile, i, gws, param, has_param);
  }
}

__global__ void __launch_bounds__(kThreads) tally_kernel(uint32_t* __restrict__ tally, uint64_t first, uint64_t count) {
  const uint64_t stride = static_cast<uint64_t>(gridDim.x) * blockDim.x;
  for (uint64_t k = static_cast<uint64_t>(blockIdx.x) * blockDim.x + threadIdx.x; k < count; k += stride)
    tally[first + k] += 1u;  // packages on one device are stream-ordered
}

}  // namespace

cudaError_t launch_vecscale(const KernelSpec& spec, const LaunchEnv& env, uint64_t first, uint64_t count) {
  if (count == 0) return cudaSuccess;
  vecscale_kernel<<<stride_grid(env, count / 2 + 1), kThreads, 0, env.stream>>>(
      static_cast<const double*>(env.in[0]), static_cast<double*>(env.out[0]), spec.a, spec.b, first, count);
  return cudaGetLastError();
}

cudaError_t launch_synthetic(const KernelSpec& spec, const LaunchEnv& env, uint64_t first, uint64_t count) {
  if (count == 0) return cudaSuccess;
  synthetic_kernel<<<stride_grid(env, count), kThreads, 0, env.stream>>>(
      static_cast<double*>(env.out[0]), static_cast<int>(spec.profile), spec.gws, spec.synth_param,
      spec.synth_has_param, first, count);
  return cudaGetLastError();
}

namespace {
__global__ void fault_kernel(double* __restrict__ out, uint64_t first, uint64_t count, uint64_t trap_item) {
  for (uint64_t k = blockIdx.x * static_cast<uint64_t>(blockDim.x) + threadIdx.x; k < count;
       k += static_cast<uint64_t>(gridDim.x) * blockDim.x) {
    if (first + k == trap_item) __trap();
    out[first + k] = 0.0;
  }
}
}  // namespace

cudaError_t launch_fault(const KernelSpec& spec, const LaunchEnv& env, uint64_t first, uint64_t count) {
  if (count == 0) return cudaSuccess;
  const uint64_t blocks = std::min<uint64_t>((count + 255) / 256, static_cast<uint64_t>(env.sms) * 8);
  fault_kernel<<<static_cast<unsigned>(blocks), 256, 0, env.stream>>>(static_cast<double*>(env.out[0]), first, count,
                                                                     spec.fault_item);
  return cudaGetLastError();
}

cudaError_t launch_tally(uint32_t* tally, uint64_t first, uint64_t count, cudaStream_t stream) {
  if (count == 0) return cudaSuccess;
  LaunchEnv env;
  env.sms = 148;
  tally_kernel<<<stride_grid(env, count), kThreads, 0, stream>>>(tally, first, count);
  return cudaGetLastError();
}

}  // namespace ecl
