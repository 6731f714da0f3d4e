// registry.cu — kernel-id resolution and argument/buffer-shape validation.
//
// Mirrors parse_kernel_id / check_buffer_shapes / kernel_for
// (workloads.hpp:154-233) for the reference's kernels and fixes the shapes of
// the paper's other benchmarks (Table 2).
#include <algorithm>
#include <cstring>

#include <cstdlib>

#include "kernels.cuh"

namespace ecl {
namespace {

bool arg_double(const KernelSpec& s, size_t i, double* v, std::string* err) {
  if (i >= s.args.size()) {
    *err = s.id + ": missing argument " + std::to_string(i);
    return false;
  }
  const ecl_arg& a = s.args[i];
  *v = a.is_double ? a.d : static_cast<double>(a.i);
  return true;
}

bool arg_u64(const KernelSpec& s, size_t i, uint64_t* v, std::string* err) {
  if (i >= s.args.size()) {
    *err = s.id + ": missing argument " + std::to_string(i);
    return false;
  }
  const ecl_arg& a = s.args[i];
  if (a.is_double || a.i < 0) {
    *err = s.id + ": argument " + std::to_string(i) + " must be a non-negative integer";
    return false;
  }
  *v = static_cast<uint64_t>(a.i);
  return true;
}

bool one_to_one(const KernelSpec& s) { return s.out_indices == 1 && s.out_work_items == 1; }

int bad(std::string* err, const std::string& msg) {
  *err = msg;
  return ECL_BAD_KERNEL_ARGS;
}

}  // namespace

bool is_builtin_kernel_id(const std::string& full) {
  const std::string id = full.substr(0, full.find('@'));
  return id == "vecscale" || id == "mandelbrot" || id == "mandelbrot_f32" || id == "synthetic" ||
         id.rfind("synthetic:", 0) == 0 || id == "gaussian" || id == "nbody" || id == "binomial" || id == "ray" ||
         id == "fault";
}

int resolve_kernel(KernelSpec& s, std::string* err) {
  // A registered device kernel (ecl_kernel_register): the program's own
  // kernel, or a per-device binary kernel.
  if (auto pk = find_plugin(s.id)) {
    s.kind = KernelKind::Plugin;
    s.plugin = std::move(pk);
    s.variant = -1;
    return check_plugin_spec(s, err);
  }
  // "<kernel>@<n>": the same kernel's tuning variant n (per-device kernel
  // specialization) — identical results, different code.
  std::string id = s.id;
  s.variant = -1;
  if (const auto at = id.find('@'); at != std::string::npos) {
    const std::string v = id.substr(at + 1);
    char* end = nullptr;
    const long n = v.empty() ? -1 : std::strtol(v.c_str(), &end, 10);
    if (v.empty() || *end != '\0' || n < 0 || n > 15) {
      *err = "kernel variant must be '<kernel>@<0..15>', got '" + s.id + "'";
      return ECL_UNKNOWN_KERNEL;
    }
    s.variant = static_cast<int>(n);
    id = id.substr(0, at);
  }
  if (id == "vecscale") {
    s.kind = KernelKind::VecScale;
  } else if (id == "mandelbrot") {
    s.kind = KernelKind::Mandelbrot;
  } else if (id == "mandelbrot_f32") {
    s.kind = KernelKind::MandelbrotF32;
  } else if (id == "synthetic" || id.rfind("synthetic:", 0) == 0) {
    s.kind = KernelKind::Synthetic;
    const std::string prof = id == "synthetic" ? "constant" : id.substr(10);
    if (prof == "constant") s.profile = SyntheticProfile::Constant;
    else if (prof == "ramp") s.profile = SyntheticProfile::Ramp;
    else if (prof == "step") s.profile = SyntheticProfile::Step;
    else {
      *err = "no synthetic cost profile named '" + prof + "'";
      return ECL_UNKNOWN_PROFILE;
    }
  } else if (id == "gaussian") {
    s.kind = KernelKind::Gaussian;
  } else if (id == "nbody") {
    s.kind = KernelKind::NBody;
  } else if (id == "binomial") {
    s.kind = KernelKind::Binomial;
  } else if (id == "ray") {
    s.kind = KernelKind::Ray;
  } else if (id == "fault" && std::getenv("ECL_FAULT_INJECTION") && std::string(std::getenv("ECL_FAULT_INJECTION")) == "1") {
    s.kind = KernelKind::Fault;  // test hook only, see kernels.cuh
  } else {
    *err = "no kernel registered as '" + id + "'";
    return ECL_UNKNOWN_KERNEL;
  }

  {
    int max_variant = 0;  // per kind: the variants its launcher implements
    switch (s.kind) {
      case KernelKind::Mandelbrot: max_variant = 15; break;
      case KernelKind::MandelbrotF32: max_variant = 2; break;
      case KernelKind::Binomial: max_variant = 5; break;
      case KernelKind::NBody: max_variant = 1; break;
      case KernelKind::Ray: max_variant = 2; break;
      case KernelKind::Gaussian: max_variant = 2; break;
      default: break;
    }
    if (s.variant > max_variant) {
      *err = "kernel '" + id + "' has variants 0.." + std::to_string(max_variant);
      return ECL_UNKNOWN_KERNEL;
    }
  }

  switch (s.kind) {
    case KernelKind::VecScale:
      if (s.inputs.size() != 1 || s.inputs[0].element_size_bytes != 8 || s.inputs[0].element_count != s.gws)
        return bad(err, "vecscale expects one double input buffer of global_work_size elements");
      if (s.outputs.size() != 1 || s.outputs[0].element_size_bytes != 8)
        return bad(err, "vecscale expects one double output buffer");
      if (!one_to_one(s)) return bad(err, "vecscale writes with a 1:1 out pattern");
      if (!arg_double(s, 0, &s.a, err) || !arg_double(s, 1, &s.b, err)) return ECL_BAD_KERNEL_ARGS;
      return ECL_OK;
    case KernelKind::Mandelbrot:
    case KernelKind::MandelbrotF32: {
      if (!s.inputs.empty()) return bad(err, "mandelbrot reads no input buffers");
      if (s.outputs.size() != 1 || s.outputs[0].element_size_bytes != 4)
        return bad(err, "mandelbrot expects one uint32 output buffer");
      if (s.out_indices != 4 || s.out_work_items != 1) return bad(err, "mandelbrot writes with a 4:1 out pattern");
      uint64_t w, h, it;
      if (!arg_u64(s, 0, &w, err) || !arg_u64(s, 1, &h, err) || !arg_u64(s, 2, &it, err)) return ECL_BAD_KERNEL_ARGS;
      s.mandel.width = w;
      s.mandel.height = h;
      s.mandel.max_iterations = static_cast<uint32_t>(it);
      if (s.args.size() >= 7) {
        if (!arg_double(s, 3, &s.mandel.x0, err) || !arg_double(s, 4, &s.mandel.y0, err) ||
            !arg_double(s, 5, &s.mandel.x1, err) || !arg_double(s, 6, &s.mandel.y1, err))
          return ECL_BAD_KERNEL_ARGS;
      }
      if (w == 0 || h == 0 || s.mandel.max_iterations == 0)
        return bad(err, "mandelbrot: width, height and max_iterations must be positive");
      if (w * h != s.gws) return bad(err, "mandelbrot: width*height must equal global_work_size");
      s.replicate = 4;  // four identical counts per pixel (workloads.hpp:217-222)
      s.compact_bytes = s.mandel.max_iterations < 65536u ? 2 : 4;  // a count is <= max_iterations
      return ECL_OK;
    }
    case KernelKind::Synthetic:
      if (!s.inputs.empty()) return bad(err, "synthetic kernels read no input buffers");
      if (s.outputs.size() != 1 || s.outputs[0].element_size_bytes != 8)
        return bad(err, "synthetic kernels expect one double output buffer");
      if (!one_to_one(s)) return bad(err, "synthetic kernels write with a 1:1 out pattern");
      if (!s.args.empty()) {
        s.synth_has_param = true;
        if (!arg_double(s, 0, &s.synth_param, err)) return ECL_BAD_KERNEL_ARGS;
      }
      return ECL_OK;
    case KernelKind::Gaussian: {
      // args [W, H, F]; in: image f32 W*H, filter f32 F*F; out f32 W*H, 1:1.
      uint64_t w, h, f;
      if (!arg_u64(s, 0, &w, err) || !arg_u64(s, 1, &h, err) || !arg_u64(s, 2, &f, err)) return ECL_BAD_KERNEL_ARGS;
      if (w == 0 || h == 0 || f == 0 || (f % 2) == 0 || f > 63)
        return bad(err, "gaussian: W, H positive and F odd in [1, 63]");
      if (w * h != s.gws) return bad(err, "gaussian: W*H must equal global_work_size");
      if (s.inputs.size() != 2 || s.inputs[0].element_size_bytes != 4 || s.inputs[0].element_count != w * h ||
          s.inputs[1].element_size_bytes != 4 || s.inputs[1].element_count != f * f)
        return bad(err, "gaussian expects inputs (float image[W*H], float filter[F*F])");
      if (s.outputs.size() != 1 || s.outputs[0].element_size_bytes != 4)
        return bad(err, "gaussian expects one float output buffer");
      if (!one_to_one(s)) return bad(err, "gaussian writes with a 1:1 out pattern");
      s.gauss = GaussianParams{static_cast<uint32_t>(w), static_cast<uint32_t>(h), static_cast<uint32_t>(f)};
      return ECL_OK;
    }
    case KernelKind::NBody: {
      // args [N, dt, eps2]; in: pos float4[N], vel float4[N]; out: newPos, newVel.
      uint64_t n;
      double dt, eps2;
      if (!arg_u64(s, 0, &n, err) || !arg_double(s, 1, &dt, err) || !arg_double(s, 2, &eps2, err))
        return ECL_BAD_KERNEL_ARGS;
      if (n != s.gws) return bad(err, "nbody: bodies must equal global_work_size");
      if (s.inputs.size() != 2 || s.outputs.size() != 2) return bad(err, "nbody expects 2 inputs and 2 outputs");
      for (const auto* v : {&s.inputs, &s.outputs})
        for (const auto& g : *v)
          if (g.element_size_bytes != 16 || g.element_count != n)
            return bad(err, "nbody buffers are float4[bodies]");
      if (!one_to_one(s)) return bad(err, "nbody writes with a 1:1 out pattern");
      s.nbody = NBodyParams{n, static_cast<float>(dt), static_cast<float>(eps2)};
      s.peer_writes = true;  // fused per-step exchange (nbody.cu)
      return ECL_OK;
    }
    case KernelKind::Binomial: {
      // args [steps]; lws = steps + 1; one float4 of options per work-group.
      uint64_t steps;
      if (!arg_u64(s, 0, &steps, err)) return ECL_BAD_KERNEL_ARGS;
      if (steps < 1 || steps > 255) return bad(err, "binomial: steps must lie in [1, 255]");
      if (s.lws != steps + 1) return bad(err, "binomial: local_work_size must be steps + 1");
      if (s.out_indices != 1 || s.out_work_items != s.lws) return bad(err, "binomial writes with a 1:lws out pattern");
      const uint64_t groups = s.gws / s.lws;
      if (s.inputs.size() != 1 || s.inputs[0].element_size_bytes != 16 || s.inputs[0].element_count != groups)
        return bad(err, "binomial expects one float4 input per work-group");
      if (s.outputs.size() != 1 || s.outputs[0].element_size_bytes != 16)
        return bad(err, "binomial expects one float4 output buffer");
      s.binom = BinomialParams{static_cast<uint32_t>(steps), groups * 4};
      return ECL_OK;
    }
    case KernelKind::Fault:
      // args [item]; one double output, 1:1 (the synthetic kernels' shape).
      if (!s.inputs.empty() || s.outputs.size() != 1 || s.outputs[0].element_size_bytes != 8 || !one_to_one(s))
        return bad(err, "fault expects no inputs and one double output, 1:1");
      if (!arg_u64(s, 0, &s.fault_item, err)) return ECL_BAD_KERNEL_ARGS;
      return ECL_OK;
    case KernelKind::Plugin:
      return check_plugin_spec(s, err);
    case KernelKind::Ray: {
      // args [W, H, spheres, max_depth]; in: scene float4 buffer; out: float4 RGBA per pixel.
      uint64_t w, h, ns, depth;
      if (!arg_u64(s, 0, &w, err) || !arg_u64(s, 1, &h, err) || !arg_u64(s, 2, &ns, err) ||
          !arg_u64(s, 3, &depth, err))
        return ECL_BAD_KERNEL_ARGS;
      if (w * h != s.gws) return bad(err, "ray: W*H must equal global_work_size");
      if (ns == 0 || ns > 256 || depth > 8) return bad(err, "ray: spheres in [1,256], depth <= 8");
      if (s.inputs.size() != 1 || s.inputs[0].element_size_bytes != 16 || s.inputs[0].element_count < 2 * ns + 8)
        return bad(err, "ray expects one float4 scene buffer of >= 2*spheres+8 elements");
      if (s.outputs.size() != 1 || s.outputs[0].element_size_bytes != 16)
        return bad(err, "ray expects one float4 output buffer");
      if (!one_to_one(s)) return bad(err, "ray writes with a 1:1 out pattern");
      s.ray = RayParams{static_cast<uint32_t>(w), static_cast<uint32_t>(h), static_cast<uint32_t>(ns),
                        static_cast<uint32_t>(depth)};
      // resident packages as 2^20-item two-lane pieces (see compute_split_items)
      s.compute_split_items = 1u << 20;
      return ECL_OK;
    }
  }
  return ECL_UNKNOWN_KERNEL;
}

uint64_t scratch_bytes(const KernelSpec& spec) {
  switch (spec.kind) {
    case KernelKind::Mandelbrot:
    case KernelKind::MandelbrotF32: return mandelbrot_scratch_bytes(spec);
    case KernelKind::Binomial: return binomial_scratch_bytes(spec);  // option records (binomial@5)
    default: return 0;
  }
}

cudaError_t prepare_kernel(const KernelSpec& spec, const LaunchEnv& env) {
  switch (spec.kind) {
    case KernelKind::Mandelbrot:
    case KernelKind::MandelbrotF32: return prepare_mandelbrot(spec, env);
    default: return cudaSuccess;
  }
}

uint64_t input_bytes_needed(const KernelSpec& spec, uint32_t input, uint64_t first, uint64_t count) {
  const ecl_buffer_geom& g = spec.inputs[input];
  const uint64_t whole = g.element_size_bytes * g.element_count;
  const uint64_t end = first + count;  // work-items [first, end)
  switch (spec.kind) {
    case KernelKind::VecScale:  // in[i] for item i
      return std::min(whole, end * g.element_size_bytes);
    case KernelKind::Gaussian: {
      if (input != 0) return whole;  // the filter
      const uint64_t w = spec.gauss.width, r = spec.gauss.filter / 2;
      const uint64_t last_row = (end - 1) / w;  // clamp-to-edge reads rows up to last_row + R
      return std::min(whole, (last_row + r + 1) * w * g.element_size_bytes);
    }
    case KernelKind::Binomial:  // one float4 of options per work-group
      return std::min(whole, ((end + spec.lws - 1) / spec.lws) * g.element_size_bytes);
    default:
      return whole;
  }
}

bool host_mirrored_input(const KernelSpec& spec, uint32_t input) {
  return spec.kind == KernelKind::Gaussian && gaussian_mirrors_input(input);
}

cudaError_t launch_kernel(const KernelSpec& spec, const LaunchEnv& env, uint64_t first, uint64_t count) {
  switch (spec.kind) {
    case KernelKind::VecScale: return launch_vecscale(spec, env, first, count);
    case KernelKind::Mandelbrot:
    case KernelKind::MandelbrotF32: return launch_mandelbrot(spec, env, first, count);
    case KernelKind::Synthetic: return launch_synthetic(spec, env, first, count);
    case KernelKind::Gaussian: return launch_gaussian(spec, env, first, count);
    case KernelKind::NBody: return launch_nbody(spec, env, first, count);
    case KernelKind::Binomial: return launch_binomial(spec, env, first, count);
    case KernelKind::Ray: return launch_ray(spec, env, first, count);
    case KernelKind::Fault: return launch_fault(spec, env, first, count);
    case KernelKind::Plugin: return launch_plugin(spec, env, first, count);
  }
  return cudaErrorInvalidValue;
}

}  // namespace ecl
