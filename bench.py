#!/usr/bin/env python3
"""bench.py — BASELINE.json's benchmarks on B200 through the co-execution engine.

Default (the driver's line): Mandelbrot 16384^2 x 2048 (FP64, the reference
kernel workloads.hpp:78-100) co-executed with HGuided over N B200s.
`--workload` selects the other BASELINE configs (gaussian, nbody, binomial,
ray, mandelbrot_f32); same JSON contract.

One step = one Engine run over the whole index space (NBody: 10 timesteps).
  value   inputs already resident in HBM, outputs left in each GPU's
          partition; CUDA events on the bench stream around K steps.
  e2e     the same run through the C-ABI with HOST buffers: page-locked
          inputs are uploaded (H2D + NVLink replication) and every package's
          out_range_for slice is copied D2H inside the timed region.
  roofline   algorithmic flops per step / step time, against
          the vector peak measured on this device (ecl_probe_vector_peaks;
          MEASURED_PEAKS.json has HBM and bf16 only).
  cpu_baseline   the reference engine itself (oracle/_ref: wall mode, H
          NativePool devices x 1 worker, the same scheduler) on the full
          config (NBody: a bounded sample); for the kernels the reference
          lacks it drives this repo's C restatement as an injected KernelFn.
--impl reference times that CPU reference as the reference arm, on the same
config; it loads only oracle/_ref (inputs from oracle/oracle.c, the same
bytes as workloads.py's generators), never the product package.
"""
from __future__ import annotations

import argparse
import ctypes
import json
import os
import subprocess
import sys
import threading

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "work-items/s at 1/2/4/8 B200 + HGuided co-exec efficiency & overhead vs native"


def env_int(name, default):
    try:
        return int(os.environ.get(name, default))
    except ValueError:
        return default


def cpu_threads():
    try:
        return len(os.sched_getaffinity(0))
    except AttributeError:
        return os.cpu_count() or 1


def load_json(rel):
    with open(os.path.join(ROOT, rel)) as f:
        return json.load(f)


# ---------------------------------------------------------------------------
# workloads (BASELINE.json configs)

def describe_doc(doc):
    """Scheduler description (the engine's describe(), schedulers.hpp:18-30) of
    a schema-1 scheduler dict, without loading the product library."""
    t = doc["type"]
    if t == "static":
        return "static(props=power)"
    if t == "dynamic":
        return f"dynamic(packages={doc['num_packages']})"
    s = f"hguided(k={doc.get('k', 2.0):g}"
    if doc.get("adaptive"):
        s += f";adaptive={doc.get('ema_alpha', 0.5):g}"
    return s + ")"


class OracleInputs:
    """The synthetic inputs of workloads.py (gaussian_inputs, nbody_inputs,
    binomial_inputs, ray_scene) made by oracle/oracle.c instead — the same
    bytes (tests/test_bench_cpu.py checks) — so the reference arm builds its
    inputs without loading the product package."""

    def __init__(self, orc, np):
        self.o, self.np = orc, np

    def gaussian_inputs(self, w, h, f=31, seed=42):
        return [self.o.fill_f64(seed, w * h).astype(self.np.float32), self.o.gaussian_filter(f, 5.0)]

    def nbody_inputs(self, n, seed=42):
        return list(self.o.nbody_init(seed, n))

    def binomial_inputs(self, n, seed=42):
        return [self.o.binomial_init(seed, n)]

    def ray_scene(self, spheres=64, seed=42):
        return self.o.ray_scene(seed, spheres)


class Workload:
    name = ""
    LWS_CFG = 1
    workload = ""
    dtype = "f32"
    bound = "fp32"
    steps_per_run = 1
    swaps = ()
    copy_split = 1 << 23  # work-items per sub-launch when copies / streamed inputs pipeline

    def __init__(self, P, W, np):
        self.P, self.W, self.np = P, W, np

    def scheduler(self, n):
        return self.P.HGuidedConfig()

    def sched_doc(self, n):
        """The scheduler as a schema-1 dict (both arms; config.hpp:41-62)."""
        return {"type": "hguided", "k": 2.0}

    def min_package(self, n):
        return 1

    def host_inputs(self):
        return []

    def cpu_run(self, ref, inputs, threads, full=True):
        """Reference engine on this workload: (seconds, work-items, what ran)."""
        raise NotImplementedError

    def check(self, outputs):
        return True

    def config(self, n, sched_doc=None):
        """The `config` object both arms print (identical for the same N)."""
        return {"workload": self.workload, "scheduler": describe_doc(sched_doc or self.sched_doc(n)),
                "lws": self.LWS_CFG, "work_items_per_step": self.units(),
                "l2": "GPU arm: L2 flushed before every timed step on every GPU (512 MiB write each, outside "
                      "the step's CUDA events)"}


class Mandelbrot(Workload):
    # attainable fraction of the FP64 DFMA peak and why (bench line roofline.ceiling_*)
    ceiling = (8.0 / 12.0, "8 counted flops in 6 unfused FP64 instructions per iteration (bit-exact: no contraction)")
    name = "mandelbrot"
    W_PX, ITERS, LWS = 16384, 2048, 256
    LWS_CFG = LWS
    VIEWPORT = (-2.5, -1.25, 1.0, 1.25)
    SUM_COUNT, INSIDE = 96_141_151_663, 46_275_993  # SURVEY §8c golden facts
    dtype = "f64"
    bound = "fp64"
    kernel = "mandelbrot"
    workload = "mandelbrot 16384x16384 max_iter 2048 viewport (-2.5,-1.25)-(1,1.25), 4:1 uint32 out"

    def spec(self):
        return self.W.mandelbrot_spec(self.W_PX, self.W_PX, self.ITERS, lws=self.LWS, kernel=self.kernel)

    def units(self):
        return self.W_PX * self.W_PX

    def flops(self):
        return 8.0 * self.SUM_COUNT + 3.0 * (self.units() - self.INSIDE)

    def min_package(self, n):
        return 148 * 8

    def scheduler(self, n):
        return self.P.HGuidedConfig(k=2.0)

    def check(self, outputs):
        counts = outputs[0].view(self.np.uint32).reshape(-1, 4)[:, 0]
        return (int(counts.sum(dtype=self.np.uint64)) == self.SUM_COUNT and
                int((counts >= self.ITERS).sum()) == self.INSIDE)

    def cpu_run(self, ref, inputs, threads, full=True):
        # the reference's own Mandelbrot kernel (workloads.hpp:78-100) in its
        # own engine, same program and scheduler as the B200 arm; warm-up
        # passes take a 4096^2 sub-grid of the same viewport
        sw = self.W_PX if full else 4096
        prog = {"kernel": "mandelbrot", "global_work_size": sw * sw, "local_work_size": self.LWS,
                "out_pattern": {"out_indices": 4, "work_items": 1},
                "out_buffers": [{"name": "counts", "element_size_bytes": 4, "element_count": sw * sw * 4}],
                "args": [sw, sw, self.ITERS] + list(self.VIEWPORT)}
        s, _ = ref.wall_run_sched(prog, self.sched_doc(1), threads, 1)
        what = (f"full {sw}x{sw} x {self.ITERS} config" if full else
                f"{sw}x{sw} sub-grid of the same viewport (warm-up)")
        return s, sw * sw, f"{what}; reference kernel workloads.hpp:78-100 in the reference Engine::run"


class MandelbrotPeriodic(Mandelbrot):
    # mandelbrot@14: the same counts (checked below), with the exact early exit
    # for orbits that became periodic in FP64 (mandelbrot.cu mandel_persistent)
    name = "mandelbrot_periodic"
    kernel = "mandelbrot@14"
    workload = ("mandelbrot 16384x16384 max_iter 2048, kernel mandelbrot@14: exact early exit for FP64-periodic "
                "orbits (identical counts; not every reference iteration is executed)")
    roofline_note = ("effective rate: algorithmic flops of the reference's full iteration count over the step time; "
                     "this variant skips provably redundant iterations, so frac is not a pipe utilisation")


class MandelbrotF32(Mandelbrot):
    name = "mandelbrot_f32"
    kernel = "mandelbrot_f32"
    dtype = "f32"
    bound = "fp32"
    SUM_COUNT = 96_141_248_575  # FP32 restatement
    ceiling = (8.0 / 12.0, "8 counted flops in 6 unfused FP32 lane-ops per iteration (packed pairs)")
    workload = "mandelbrot_f32 16384x16384 max_iter 2048 (FP32 restatement, parity unpinned)"

    def flops(self):
        return 8.0 * self.SUM_COUNT + 3.0 * (self.units() - self.INSIDE)

    def check(self, outputs):
        counts = outputs[0].view(self.np.uint32).reshape(-1, 4)[:, 0]
        return int(counts.sum(dtype=self.np.uint64)) == self.SUM_COUNT


class Gaussian(Workload):
    # separable path (the filter is rank 1): 8 B of image + output per pixel
    # against ~38 FFMA2 executed per pixel (2F taps per pass, 1.47x rows of
    # horizontal pass per output row with 64-row tiles) — at the FFMA2 peak
    # that is 35.9 us per 4096^2 step against 20.5 us of HBM traffic, so the
    # kernel can reach at most 0.57 of HBM bandwidth
    ceiling = (20.5 / 35.9, "8 B/px of HBM (20.5 us at 6546 GB/s) vs 38.3 executed FFMA2/px (35.9 us at the "
                            "FFMA peak): the separable kernel's attainable fraction of HBM bandwidth")
    bound = "hbm"
    name = "gaussian"
    WIDTH = HEIGHT = 4096
    F = 31
    LWS_CFG = 128
    workload = "gaussian 4096x4096 float image, 31x31 filter (sigma 5), clamp-to-edge, static, single device"
    # 32 row bands: H2D of band k+1 and D2H of band k-1 overlap band k (e2e measured:
    # 2^19 items 1.66-1.74 ms, 2^20 1.81-1.89, 2^21 1.96, 2^18 1.93, 2^17 2.30)
    copy_split = 1 << 19

    def spec(self):
        return self.W.gaussian_spec(self.WIDTH, self.HEIGHT, self.F)

    def scheduler(self, n):
        return self.P.StaticConfig()

    def sched_doc(self, n):
        return {"type": "static"}

    def units(self):
        return self.WIDTH * self.HEIGHT

    def flops(self):
        return self.W.gaussian_flops(self.WIDTH, self.HEIGHT, self.F)

    def host_inputs(self):
        return self.W.gaussian_inputs(self.WIDTH, self.HEIGHT, self.F, seed=42)

    def roofline_override(self, ms_dev, n, f32_peak_per_gpu):
        """HBM roofline of the separable kernel, with the executed-algorithm
        FP32 rate and the direct-form effective rate beside it (SURVEY §8d:
        a separable variant reports against the direct-form flop count)."""
        px = float(self.units())
        nbytes = 8.0 * px  # image read once + output written once
        gbs = nbytes / (ms_dev * 1e-3) / 1e9
        try:
            peak = float(load_json("MEASURED_PEAKS.json").get("hbm_gbs", 0.0) or 0.0) * n
            src = "MEASURED_PEAKS.json hbm_gbs (driver-measured copy bandwidth)"
        except (OSError, ValueError):
            peak, src = 6549.8 * n, "SURVEY §8d measured copy bandwidth (MEASURED_PEAKS.json absent)"
        sep = 4.0 * self.F * px  # 2 flops x (F + F) taps
        direct = self.flops()
        tf = lambda f: f / (ms_dev * 1e-3) / 1e12  # noqa: E731
        return {"bound": "hbm", "achieved": gbs, "peak": peak or None, "unit": "GB/s",
                "frac": gbs / peak if peak else None,
                "peak_source": src, "peak_per_gpu": peak / n,
                "algorithmic_bytes_per_step": nbytes,
                "separable_fp32": {"flops_per_step": sep, "achieved_tflops": tf(sep),
                                   "frac_of_ffma_peak": tf(sep) / (f32_peak_per_gpu * n)},
                "direct_form": {"flops_per_step": direct, "effective_tflops": tf(direct),
                                "effective_frac_of_ffma_peak": tf(direct) / (f32_peak_per_gpu * n),
                                "note": "the 31x31 direct count (1922 flop/px); the kernel runs the separable form"}}

    def check(self, outputs):
        out = outputs[0].view(self.np.float32)
        # a normalized positive filter over U[0,1) keeps pixels in [0,1) with mean ~0.5
        return bool(self.np.isfinite(out).all() and out.min() >= 0 and out.max() < 1 and abs(out.mean() - 0.5) < 0.01)

    def cpu_run(self, ref, inputs, threads, full=True):
        n = self.units()
        out = self.np.zeros(n, self.np.float32)
        s = ref.wall_run_restated("gaussian", inputs, out, n, 1, [self.WIDTH, self.HEIGHT, self.F], threads,
                                  self.sched_doc(1))
        return s, n, "full 4096x4096 image; restated kernel oracle.c:orc_gaussian injected as KernelFn"


class NBody(Workload):
    ceiling = (20.0 / 24.0, "20 counted flops per interaction in 12 FP32 lane-ops (+1 MUFU)")
    name = "nbody"
    N = 1 << 20
    LWS_CFG = 64
    steps_per_run = 10
    swaps = ((0, 0), (1, 1))
    workload = "nbody 1048576 bodies x 10 timesteps, dt 0.005, eps2 500, dynamic, NVLink owner-slice exchange"

    def spec(self):
        return self.W.nbody_spec(self.N)

    def scheduler(self, n):
        return self.P.DynamicConfig(max(8, 4 * n))

    def sched_doc(self, n):
        return {"type": "dynamic", "num_packages": max(8, 4 * n)}

    def units(self):
        return self.N * self.steps_per_run

    def flops(self):
        return self.W.nbody_flops(self.N, self.steps_per_run)

    def host_inputs(self):
        return self.W.nbody_inputs(self.N, seed=42)

    def check(self, outputs):
        pos = outputs[0].view(self.np.float32).reshape(-1, 4)
        return bool(self.np.isfinite(pos).all() and (pos[:, 3] >= 1).all())

    def cpu_run(self, ref, inputs, threads, full=True):
        # the full config is 1.1e13 interactions (~40 min on 16 cores): always a sample
        targets = 8192 if full else 1024
        out = self.np.zeros((self.N, 4), self.np.float32)
        s = ref.wall_run_restated("nbody", inputs, out, targets, self.N // targets, [self.N, 0.005, 500.0], threads)
        return s, targets, (f"{targets} target bodies (stride {self.N // targets}) x all {self.N} sources x 1 step "
                            "(sampled: the full 10-step config takes ~40 min on the host); "
                            "restated kernel oracle.c:orc_nbody_step")


class Binomial(Workload):
    ceiling = (1.5 * 64770.0 / 73152.0,
               "full lattice: 3 counted flops per node in one FMA lane-op (scaled lattice); 64770 live of 73152 "
               "slots per pair of round 1's 32-lane phases")
    name = "binomial"
    OPTIONS = 8 * 1024 * 1024
    STEPS = 254
    LWS_CFG = STEPS + 1
    workload = "binomial 8388608 options x 254 steps (2097152 float4 work-groups of 255), hguided"

    def spec(self):
        return self.W.binomial_spec(self.OPTIONS, self.STEPS)

    def units(self):
        return self.OPTIONS

    def flops(self):
        return self.W.binomial_flops(self.OPTIONS, self.STEPS)

    def min_package(self, n):
        return 148 * 8

    def host_inputs(self):
        return self.W.binomial_inputs(self.OPTIONS, seed=42)

    def skip_ceiling(self):
        """The same bound for a lattice that skips the exact zeros below the
        strike (the default kernel's window): at level j only nodes
        t >= t0 - (steps - j) can be nonzero (t0 = first positive leaf), so an
        option needs steps(steps+1)/2 - t0(t0-1)/2 node updates (one FMA
        lane-op each) for its 3 steps(steps+1)/2 counted flops."""
        np, n = self.np, self.STEPS
        rv = self.host_inputs()[0].astype(np.float64)
        S, K, T = 5 * (1 - rv) + 30 * rv, 1 * (1 - rv) + 100 * rv, 0.25 * (1 - rv) + 10 * rv
        vsdt = 0.30 * np.sqrt(T / n)
        # first t with S u^(2t - n) > K
        t0 = np.clip(np.floor(0.5 * (n + np.log(K / S) / vsdt)) + 1, 0, n + 1)
        live = n * (n + 1) / 2 - t0 * (t0 - 1) / 2
        counted = 3.0 * n * (n + 1) / 2 * rv.size
        c = counted / (2.0 * live.sum())
        return c, (f"3 counted flops per node, one FMA lane-op per NONZERO node update: {live.mean():.0f} "
                   f"of {n * (n + 1) // 2} node updates per option are nonzero at this input")

    def check(self, outputs):
        call = outputs[0].view(self.np.float32)
        return bool(self.np.isfinite(call).all() and (call >= 0).all() and (call <= 30.0001).all())

    def cpu_run(self, ref, inputs, threads, full=True):
        stride = 1 if full else 64
        n = self.OPTIONS // stride
        out = self.np.zeros(self.OPTIONS, self.np.float32)
        s = ref.wall_run_restated("binomial", inputs, out, n, stride, [self.STEPS], threads, self.sched_doc(1))
        what = "all 8388608 options" if full else f"{n} options (every {stride}th, warm-up)"
        return s, n, f"{what} x {self.STEPS} steps; restated kernel oracle.c:orc_binomial"


class Ray(Workload):
    ceiling = (17.0 / 16.0, "17 counted flops per sphere test in the 8 FMA-pipe lane-ops of the conservative "
                            "fused scan (candidates then run the exact 16-op IEEE test; shading not counted here)")
    name = "ray"
    WIDTH = HEIGHT = 8192
    SPHERES, DEPTH = 64, 4
    LWS_CFG = 128
    workload = "ray 8192x8192, 64 spheres + plane, 3 lights, shadows, reflections depth 4, hguided"
    # smaller sub-launches shorten the last copy's tail (e2e measured: 2^20 items
    # 19.7-19.8 ms, 2^21 19.9-20.2, 2^22 19.9-20.0, 2^23 20.3-20.4)
    copy_split = 1 << 20

    def spec(self):
        return self.W.ray_spec(self.WIDTH, self.HEIGHT, self.SPHERES, self.DEPTH)

    def units(self):
        return self.WIDTH * self.HEIGHT

    def flops(self):
        return load_json("tests/golden/ray_counts.json")["8192x8192"]["flops"]

    def min_package(self, n):
        # 4 work-groups per SM per GPU in the job: the same package count per
        # device at every N (virtual model, tools/virtual_scaling_ray.py:
        # HGuided 0.957 at 8 GPUs with 4736 vs 0.919 with 592)
        return 148 * 4 * max(1, n)

    def host_inputs(self):
        return [self.W.ray_scene(self.SPHERES, seed=42)]

    def check(self, outputs):
        g = load_json("tests/golden/ray_counts.json")["8192x8192"]
        img = outputs[0].view(self.np.float32).reshape(-1, 4)
        hist = self.np.bincount(img[:, 3].astype(int), minlength=len(g["bounce_histogram"]))
        return [int(x) for x in hist] == g["bounce_histogram"]

    def cpu_run(self, ref, inputs, threads, full=True):
        stride = 1 if full else 16
        n = self.units() // stride
        out = self.np.zeros((self.units(), 4), self.np.float32)
        s = ref.wall_run_restated("ray", inputs, out, n, stride,
                                  [self.WIDTH, self.HEIGHT, self.SPHERES, self.DEPTH], threads, self.sched_doc(1))
        what = "all 8192^2 pixels" if full else f"{n} pixels (every {stride}th, warm-up)"
        return s, n, f"{what}; restated kernel oracle.c:orc_ray"


WORKLOADS = {c.name: c for c in (Mandelbrot, MandelbrotPeriodic, MandelbrotF32, Gaussian, NBody, Binomial, Ray)}


# ---------------------------------------------------------------------------
# clocks

class ClockSampler:
    """SM clocks and clock-event (throttle) reasons sampled in-process through
    NVML every ~2 ms during the timed region, so even a few-millisecond region
    gets samples (nvidia-smi's process start alone takes longer)."""

    PERIOD_S = 0.002

    def __init__(self, gpu_index: int):
        self.gpu = gpu_index
        self.samples = []  # (sm_mhz, max_mhz, power_w, reasons bitmask)
        self._stop = threading.Event()
        self._thread = None
        self._nvml = None
        self._handle = None
        self._error = None

    def _open(self):
        import pynvml
        pynvml.nvmlInit()
        self._nvml = pynvml
        try:  # NVML enumerates physical GPUs: map through the PCI bus id
            import torch
            props = torch.cuda.get_device_properties(self.gpu)
            bus = f"{props.pci_domain_id:08x}:{props.pci_bus_id:02x}:{props.pci_device_id:02x}.0"
            self._handle = pynvml.nvmlDeviceGetHandleByPciBusId(bus.encode())
        except Exception:
            self._handle = pynvml.nvmlDeviceGetHandleByIndex(self.gpu)

    def start(self):
        try:
            self._open()
        except Exception as e:  # no NVML: reported, not silently ignored
            self._error = f"nvml unavailable: {e}"
            return self
        self._sample()  # one sample at the start of the region
        self._thread = threading.Thread(target=self._loop, daemon=True)
        self._thread.start()
        return self

    def _sample(self):
        n, h = self._nvml, self._handle
        try:
            sm = n.nvmlDeviceGetClockInfo(h, n.NVML_CLOCK_SM)
            mx = n.nvmlDeviceGetMaxClockInfo(h, n.NVML_CLOCK_SM)
            try:
                pw = n.nvmlDeviceGetPowerUsage(h) / 1000.0
            except Exception:
                pw = None
            try:
                rs = n.nvmlDeviceGetCurrentClocksEventReasons(h)
            except Exception:
                rs = n.nvmlDeviceGetCurrentClocksThrottleReasons(h)
            self.samples.append((sm, mx, pw, rs))
        except Exception as e:
            self._error = f"nvml sample failed: {e}"

    def _loop(self):
        while not self._stop.wait(self.PERIOD_S):
            self._sample()

    def stop(self):
        if self._thread:
            self._stop.set()
            self._thread.join(timeout=5)
            self._sample()  # and one at the end
        return self.summary()

    def summary(self):
        if not self.samples:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": [self._error or "no samples"], "samples": 0}
        n = self._nvml
        bits = {"hw_slowdown": getattr(n, "nvmlClocksEventReasonHwSlowdown", 0x8),
                "hw_thermal_slowdown": getattr(n, "nvmlClocksEventReasonHwThermalSlowdown", 0x40),
                "hw_power_brake_slowdown": getattr(n, "nvmlClocksEventReasonHwPowerBrakeSlowdown", 0x80),
                "sw_thermal_slowdown": getattr(n, "nvmlClocksEventReasonSwThermalSlowdown", 0x20),
                "sw_power_cap": getattr(n, "nvmlClocksEventReasonSwPowerCap", 0x4)}
        sm = sorted(s[0] for s in self.samples)
        reasons = sorted({name for s in self.samples for name, b in bits.items() if s[3] & b})
        power = [s[2] for s in self.samples if s[2] is not None]
        return {"sm_mhz": sm[len(sm) // 2], "sm_max_mhz": max(s[1] for s in self.samples), "reasons": reasons,
                "samples": len(self.samples), "source": "nvml", "power_w_max": max(power) if power else None}


def merge_clocks(*cs, per_gpu=None):
    """One clocks object over several samplers (several GPUs and/or timed
    regions): the lowest median SM clock, every reason seen; with per_gpu
    (the ordinals of cs, in order) also each GPU's own summary."""
    cs = [c for c in cs if c]
    sm = [c["sm_mhz"] for c in cs if c.get("sm_mhz")]
    out = {"sm_mhz": min(sm) if sm else None, "sm_max_mhz": max((c["sm_max_mhz"] or 0) for c in cs) or None,
           "reasons": sorted(set().union(*[set(c["reasons"]) for c in cs])),
           "samples": sum(c["samples"] for c in cs),
           "power_w_max": max((c.get("power_w_max") or 0) for c in cs) or None}
    if per_gpu is not None:
        out["per_gpu"] = {str(d): {k: c.get(k) for k in ("sm_mhz", "sm_max_mhz", "reasons", "samples")}
                          for d, c in zip(per_gpu, cs)}
    else:
        merged = {}
        for c in cs:
            merged.update(c.get("per_gpu", {}))
        if merged:
            out["per_gpu"] = merged
    return out


def busy_per_device(trace):
    """Device busy time of one run: the union of its packages' kernel
    intervals per device (packages overlap on the two lanes, so a plain sum
    double-counts)."""
    iv = {}
    for p in trace.packages:
        iv.setdefault(p.device_id, []).append((p.t_start_ms, p.t_end_ms))
    out = {}
    for dev, xs in iv.items():
        xs.sort()
        total, cur0, cur1 = 0.0, None, None
        for a, b in xs:
            if cur1 is None or a > cur1:
                if cur1 is not None:
                    total += cur1 - cur0
                cur0, cur1 = a, b
            else:
                cur1 = max(cur1, b)
        if cur1 is not None:
            total += cur1 - cur0
        out[dev] = total
    return out


def pcie_d2h_gbps(torch, ordinal, nbytes=256 << 20):
    """Device-to-pinned-host copy rate of one GPU (CUDA events)."""
    src = torch.empty(nbytes, dtype=torch.uint8, device=torch.device("cuda", ordinal))
    dst = torch.empty(nbytes, dtype=torch.uint8, pin_memory=True)
    with torch.cuda.device(ordinal):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        dst.copy_(src, non_blocking=True)
        torch.cuda.synchronize()
        e0.record()
        for _ in range(3):
            dst.copy_(src, non_blocking=True)
        e1.record()
        e1.synchronize()
        return 3 * nbytes / (e0.elapsed_time(e1) * 1e-3) / 1e9


# ---------------------------------------------------------------------------
# arms

L2_FLUSH_BYTES = 512 << 20

NCU_KERNEL = {"mandelbrot": "mandel_persistent<double", "mandelbrot_f32": "mandel_x2<float",
              "gaussian": "gaussian_sep", "binomial": "binomial_hw", "nbody": "nbody_step",
              "ray": "ray_persistent"}


def ncu_traffic(workload):
    """DRAM bytes (read + write) of the workload's kernel from the committed
    ncu --set full capture of one launch (profiles/r2/ncu_summary.json)."""
    path = os.path.join(os.path.dirname(os.path.abspath(__file__)), "profiles", "r2", "ncu_summary.json")
    scale = {"byte": 1.0, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}
    try:
        rows = json.load(open(path))
    except (OSError, ValueError):
        return None, "no ncu capture committed"
    for r in rows:
        if NCU_KERNEL.get(workload, "?") in r.get("kernel", ""):
            def val(k):
                v, u = r[k].split()
                return float(v) * scale[u]
            t = val("dram__bytes_read.sum") + val("dram__bytes_write.sum")
            return t, (f"dram__bytes_read.sum + dram__bytes_write.sum of one captured launch "
                       f"({r['gpu__time_duration.sum']}) of {NCU_KERNEL[workload]}, bytes per launch "
                       f"(profiles/r2/ncu_summary.json)")
    return None, "kernel not in the committed ncu capture"


def init_dist():
    return env_int("WORLD_SIZE", 1), env_int("RANK", 0), env_int("LOCAL_RANK", 0)


def reference_runner(np):
    """(reference library, synthetic-input maker): oracle/_ref and oracle.c only."""
    from tests import _oracle
    ref = _oracle.Reference.load()
    if ref is None:
        raise RuntimeError("oracle/_ref is not built (make -C oracle where /root/reference exists)")
    return ref, OracleInputs(_oracle.Oracle(), np)


def run_reference(args, world, rank):
    """The reference arm: the reference's own engine (oracle/_ref, wall mode,
    H NativePool devices x 1 worker) on the same workload, program and
    scheduler as the B200 arm, on this box's host cores.  Warm-up passes run
    a smaller sample; every timed pass runs the full config (NBody: a
    bounded sample, the full config is ~40 min).  Loads no product code."""
    if rank != 0:
        return 0
    import numpy as np
    ref, synth = reference_runner(np)
    wl = WORKLOADS[args.workload](None, synth, np)
    h = cpu_threads()
    inputs = wl.host_inputs()
    for _ in range(args.warmup):
        wl.cpu_run(ref, inputs, h, full=False)
    secs, units, sample = [], 0, ""
    for _ in range(args.steps):
        s, units, sample = wl.cpu_run(ref, inputs, h, full=True)
        secs.append(s)
    sec = sum(secs) / len(secs)
    value = units / sec
    line = {"impl": "reference", "metric": METRIC, "value": value, "unit": "work-items/s", "n_gpus": args.gpus,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": 1e3 * sec, "higher_is_better": True,
            "scaling": "strong", "vs_baseline": None, "dtype": wl.dtype, "data": "synthetic",
            "config": wl.config(args.gpus),
            "reference": {"engine": f"reference coexec::Engine (oracle/_ref), wall mode, {h} NativePool devices "
                                    "x 1 worker", "sample": sample,
                          "warmup": "warm-up passes on a smaller sample of the same workload"},
            "cpu_baseline": {"value": value, "unit": "work-items/s", "cores": h, "kind": "reference",
                             "sample": sample},
            "e2e": {"value": value, "unit": "work-items/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(line), flush=True)
    return 0


def shared_out_dir(args):
    """Directory for the ranks' shared output file: /dev/shm when it has room
    for the workload's outputs (plus 10 %), else the first of $TMPDIR, /tmp
    that has."""
    import numpy as np
    import paper_1805_02755_b200 as P
    from paper_1805_02755_b200 import workloads as W
    need = 1.1 * sum(b.size_bytes() for b in WORKLOADS[args.workload](P, W, np).spec().out_buffers)
    for d in ("/dev/shm", os.environ.get("TMPDIR", ""), "/tmp"):
        if d and os.path.isdir(d):
            st = os.statvfs(d)
            if st.f_bavail * st.f_frsize >= need:
                return d
    return "/dev/shm"


class SharedHostBuffer:
    """A /dev/shm-backed host buffer every rank maps and page-locks: each
    process D2H-copies its own packages' slices into the one result."""

    def __init__(self, path, nbytes, create, P, np):
        import mmap
        self.path, self.P = path, P
        fd = os.open(path, os.O_RDWR | (os.O_CREAT if create else 0), 0o600)
        if create:
            os.ftruncate(fd, nbytes)
        self.mm = mmap.mmap(fd, nbytes, mmap.MAP_SHARED, mmap.PROT_READ | mmap.PROT_WRITE)
        os.close(fd)
        self.array = np.frombuffer(self.mm, dtype=np.uint8)
        P.host_register(self.array)
        self.create = create

    def free(self):
        self.P.host_unregister(self.array)
        self.array = None
        try:
            self.mm.close()
        except BufferError:  # numpy views still alive; the mapping goes with them
            pass
        if self.create and os.path.exists(self.path):
            os.unlink(self.path)


def run_ours(args, world, rank, local):
    import numpy as np
    import torch

    import paper_1805_02755_b200 as P
    from paper_1805_02755_b200 import _native as N
    from paper_1805_02755_b200 import workloads as W

    if P.gpu_count() < 1:
        print(json.dumps({"error": "no CUDA device visible"}))
        return 1
    dist = world > 1
    shared = None
    if dist:
        # One process per GPU (torchrun): every rank drives its own B200 and
        # the ranks co-schedule one index space through the shared-memory
        # decision log (coexec/shared.hpp) — no data-path collective.
        import torch.distributed as td
        ndev = torch.cuda.device_count()
        torch.cuda.set_device(local % ndev)
        if world <= ndev:
            td.init_process_group("nccl", device_id=torch.device("cuda", local))
        else:  # more ranks than GPUs (a one-GPU test box): NCCL refuses shared devices
            td.init_process_group("gloo")
        # rank 0 names the run and picks where the shared output lives: /dev/shm
        # unless that tmpfs is too small for the outputs (a container default
        # of 64 MB would SIGBUS when the buffer is page-locked), then /tmp
        tag = [f"{os.getpid():x}{int.from_bytes(os.urandom(4), 'little'):x}", shared_out_dir(args)] \
            if rank == 0 else [None, None]
        td.broadcast_object_list(tag, src=0)
        shared = {"name": f"/ecl_bench_{tag[0]}", "rank": rank, "world": world, "local_devices": [rank],
                  "host_buffer": os.path.join(tag[1], f"ecl_bench_out_{tag[0]}")}
    n = world if dist else args.gpus
    torch.cuda.set_device((local % torch.cuda.device_count()) if dist else 0)

    def barrier():
        torch.cuda.synchronize()
        if dist:
            torch.distributed.barrier()

    def max_over_ranks(x):
        if not dist:
            return x
        dev = "cuda" if torch.distributed.get_backend() == "nccl" else "cpu"
        t = torch.tensor([x], dtype=torch.float64, device=dev)
        torch.distributed.all_reduce(t, op=torch.distributed.ReduceOp.MAX)
        return float(t.item())

    wl = WORKLOADS[args.workload](P, W, np)
    line = bench_engine(args, n, wl, P, N, np, torch, barrier, max_over_ranks, shared, rank)
    if not dist and n == 1 and args.workload == "mandelbrot" and not args.no_other_workloads:
        # the other BASELINE configs, measured in the same run so the driver's
        # own bench record carries them (compact: no CPU baseline, NBody with
        # two timed 10-step runs)
        line["other_workloads"] = {}
        for name in ("ray", "binomial", "gaussian", "nbody"):
            sub = argparse.Namespace(**vars(args))
            sub.workload, sub.no_cpu_baseline, sub.copy_split, sub.min_package = name, True, 0, 0
            if name == "nbody":  # 4.3 s per run: two timed runs, the contract's minimum of 3 warm-ups
                sub.steps = min(sub.steps, 2)
                sub.warmup = min(sub.warmup, 3)
            w2 = WORKLOADS[name](P, W, np)
            full = bench_engine(sub, n, w2, P, N, np, torch, barrier, max_over_ranks, shared, rank)
            line["other_workloads"][name] = compact_line(full)
    if dist:
        torch.distributed.destroy_process_group()
    if rank == 0:
        print(json.dumps(line), flush=True)
    return 0


def compact_line(full):
    """The fields of a workload's bench line that summarise it inside another
    line (other_workloads)."""
    r, c = full["roofline"], full["coexec"]
    keep_r = ("bound", "achieved", "peak", "unit", "frac", "ceiling_frac", "frac_of_ceiling", "skip_ceiling_frac",
              "frac_of_skip_ceiling")
    return {"workload": full["config"]["workload"], "value": full["value"], "unit": full["unit"],
            "ms_per_step": full["ms_per_step"], "steps": full["steps"], "warmup": full["warmup"],
            "dtype": full["dtype"], "e2e": {k: full["e2e"][k] for k in ("value", "ms_per_step")},
            "step_ms": full.get("step_ms"), "roofline": {k: r[k] for k in keep_r if k in r},
            "coexec": {k: c.get(k) for k in ("native_kernel_ms", "overhead_pct_device", "packages_per_step",
                                             "outputs_sane")},
            "gpu_launches": full["gpu_launches"],
            "clocks": {k: full["clocks"].get(k) for k in ("sm_mhz", "sm_max_mhz", "reasons")}}


def bench_engine(args, n, wl, P, N, np, torch, barrier, max_over_ranks, shared, rank):
    min_wg = args.min_package if args.min_package else wl.min_package(n)
    copy_split = args.copy_split if args.copy_split else wl.copy_split
    ngpu = P.gpu_count()
    devs = [P.cuda_device(f"gpu{i}", ordinal=i % ngpu, power=1.0, queue_depth=args.queue_depth,
                          min_package_work_groups=min_wg, widen_per_8=args.widen,
                          copy_split_items=copy_split) for i in range(n)]
    sched = wl.scheduler(n)
    if isinstance(sched, P.HGuidedConfig):
        sched.k = args.k
        sched.adaptive = args.adaptive
    prog = P.validate_program(wl.spec())
    eng_shared = {k: v for k, v in shared.items() if k != "host_buffer"} if shared else None
    eng = P.Engine(P.EngineConfig(devs, sched, shared=eng_shared), prog)
    stream = torch.cuda.current_stream()

    # page-locked host buffers (inputs for the e2e H2D, outputs for the D2H)
    host_in = wl.host_inputs()
    pinned_in = []
    for a in host_in:
        pb = P.PinnedBuffer(a.nbytes, np.uint8)
        pb.array[:] = np.ascontiguousarray(a).reshape(-1).view(np.uint8)
        pinned_in.append(pb)
    in_arrays = [pb.array for pb in pinned_in]
    if shared:
        if rank == 0:
            pinned_out = [SharedHostBuffer(shared["host_buffer"] + f"_{i}", b.size_bytes(), True, P, np)
                          for i, b in enumerate(prog.spec().out_buffers)]
            barrier()
        else:
            barrier()
            pinned_out = [SharedHostBuffer(shared["host_buffer"] + f"_{i}", b.size_bytes(), False, P, np)
                          for i, b in enumerate(prog.spec().out_buffers)]
    else:
        pinned_out = [P.PinnedBuffer(b.size_bytes(), np.uint8) for b in prog.spec().out_buffers]
    out_arrays = [pb.array for pb in pinned_out]

    def run(inputs, outputs):
        if wl.steps_per_run > 1:
            eng.run_steps(inputs, outputs, wl.steps_per_run, wl.swaps, want_trace=False)
        else:
            eng.run_into(inputs, outputs, want_trace=False)

    # L2 flush between timed steps: a 512 MiB write (4x the 126 MB L2) on
    # every GPU this process drives, before every step, outside the step's events.
    my_gpus = [rank % ngpu] if shared else sorted({i % ngpu for i in range(n)})
    flush_bufs = [torch.empty(L2_FLUSH_BYTES, dtype=torch.uint8, device=torch.device("cuda", d)) for d in my_gpus]

    def flush_l2():
        for b in flush_bufs:
            b.zero_()
        for d in my_gpus:
            torch.cuda.synchronize(d)

    step_log = {}

    def timed(fn, steps, tag, after=None):
        e0 = torch.cuda.Event(enable_timing=True)
        e1 = torch.cuda.Event(enable_timing=True)
        per = []
        for _ in range(steps):
            flush_l2()
            barrier()
            e0.record(stream)
            fn()
            e1.record(stream)
            e1.synchronize()
            per.append(e0.elapsed_time(e1))
            if after is not None:
                after()  # outside the step's events
        torch.cuda.synchronize()
        barrier()
        step_log[tag] = per
        return sum(per) / steps

    # --- device-resident (value): inputs uploaded once before timing ---
    run(in_arrays, None)
    for _ in range(max(0, args.warmup - 1)):
        run(None, None)
    my_gpu = my_gpus[0]
    samplers = [ClockSampler(d).start() for d in my_gpus]
    # one more untimed step once the samplers run: the sampler threads'
    # start-up otherwise lands in the first timed step (measured +30-130 us)
    flush_l2()
    run(None, None)
    barrier()
    eng.kernel_timing(reset=True)
    # kernel time per step: the union of the step's kernel intervals on each
    # device (CUDA events recorded on the launching lane streams around every
    # package), max over devices — what the roofline's `achieved` divides by
    busy_steps = []
    ms_dev = max_over_ranks(timed(lambda: run(None, None), args.steps, "resident",
                                  after=lambda: busy_steps.append(max(busy_per_device(eng.last_trace()).values(),
                                                                      default=0.0))))
    step_log["resident_kernel_busy"] = busy_steps
    ms_kernel = sum(busy_steps) / len(busy_steps) if busy_steps and min(busy_steps) > 0 else 0.0
    ms_kernel = max_over_ranks(ms_kernel) or ms_dev
    clocks = merge_clocks(*[c.stop() for c in samplers], per_gpu=my_gpus)
    clocks["region"] = "device-resident"
    kernel_ms, launches = eng.kernel_timing(reset=True)
    last = eng.last_trace()
    bal = P.balance(last) if n > 1 else 1.0
    busy = busy_per_device(last)

    # --- end to end through the C-ABI with page-locked host buffers ---
    for _ in range(args.warmup):
        run(in_arrays, out_arrays)
    samplers2 = [ClockSampler(d).start() for d in my_gpus]
    run(in_arrays, out_arrays)  # untimed, as above
    barrier()
    if rank == 0:  # the timed runs must write every output themselves
        for a in out_arrays:
            a[:] = 0
    ms_e2e = max_over_ranks(timed(lambda: run(in_arrays, out_arrays), args.steps, "e2e"))
    clocks2 = merge_clocks(*[c.stop() for c in samplers2], per_gpu=my_gpus)
    eng.kernel_timing(reset=True)
    sane = wl.check(out_arrays) if rank == 0 else True
    e2e_trace = eng.last_trace()
    e2e_last_kernel_end = max((p.t_end_ms for p in e2e_trace.packages), default=0.0)

    # --- native single-kernel baseline (overhead denominator) ---
    barrier()
    native_k, native_host, native_e2e, native_split = [], [], [], []
    if wl.steps_per_run == 1:
        n0, n1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        for _ in range(args.warmup + args.steps):
            flush_l2()  # same L2 state as the timed engine steps
            # kernel-only time, and the native program's host call bracketed
            # exactly like an engine step (launch + completion wait included)
            n0.record(stream)
            native_k.append(eng.native_run(None, None)[0])
            n1.record(stream)
            n1.synchronize()
            native_host.append(n0.elapsed_time(n1))
            # the best plain-CUDA program: the same kernel as sub-launches of
            # the engine's piece size over two streams, no scheduler
            flush_l2()
            native_split.append(eng.native_run_split(copy_split))
        native_split = native_split[args.warmup:]
        for _ in range(max(1, args.steps)):
            native_e2e.append(eng.native_run(in_arrays, out_arrays)[1])
        native_k = native_k[args.warmup:]
        native_host = native_host[args.warmup:]
    barrier()
    k_single = sorted(native_k)[len(native_k) // 2] if native_k else None
    k_split = sorted(native_split)[len(native_split) // 2] if native_split else None
    k_native = min(k_single, k_split) if k_single and k_split else k_single
    h_native = sorted(native_host)[len(native_host) // 2] if native_host else None
    t_native_e2e = sorted(native_e2e)[len(native_e2e) // 2] if native_e2e else None

    # --- roofline: vector peaks measured on this device ---
    f64, add, f32 = ctypes.c_double(), ctypes.c_double(), ctypes.c_double()
    N.lib.ecl_probe_vector_peaks(my_gpu, ctypes.byref(f64), ctypes.byref(add), ctypes.byref(f32))
    mix = ctypes.c_double(0.0)
    if wl.name == "mandelbrot":
        N.lib.ecl_probe_mandel_mix(my_gpu, ctypes.byref(mix))
    elif wl.name == "mandelbrot_f32":
        N.lib.ecl_probe_mandel_mix_f32(my_gpu, ctypes.byref(mix))
    peak = (f64.value if wl.bound == "fp64" else f32.value) * n  # whole job: N GPUs
    achieved = wl.flops() / (ms_kernel * 1e-3) / 1e12
    achieved_step = wl.flops() / (ms_dev * 1e-3) / 1e12
    eng.close()
    h2d = sum(a.nbytes for a in in_arrays)
    d2h = sum(a.nbytes for a in out_arrays)
    del in_arrays, out_arrays
    for pb in pinned_in + pinned_out:
        pb.free()

    cpu = None
    if n == 1 and rank == 0 and not args.no_cpu_baseline:
        try:
            h = cpu_threads()
            ref, _ = reference_runner(np)
            secs, units_s, sample = wl.cpu_run(ref, host_in, h, full=True)
            cpu = {"value": units_s / secs, "unit": "work-items/s", "cores": h, "kind": "reference",
                   "sample": sample + f"; reference engine wall mode, {h} NativePool devices x 1 worker, "
                                      f"{describe_doc(wl.sched_doc(1))}"}
        except Exception as exc:  # noqa: BLE001 — report it, keep the GPU line
            cpu = {"value": None, "unit": "work-items/s", "cores": cpu_threads(), "kind": "reference",
                   "sample": f"unavailable: {exc}"}

    traffic, traffic_basis = ncu_traffic(wl.name)
    units = wl.units()
    cfg = wl.config(n, sched.to_json())
    # NVLink peer access between the GPUs this process drives (replication
    # and exchange copies use it when enabled)
    p2p = None
    if len(my_gpus) > 1:
        pairs = {}
        for a in my_gpus:
            for b in my_gpus:
                if a != b:
                    can, en = ctypes.c_int(0), ctypes.c_int(0)
                    N.lib.ecl_peer_access(a, b, ctypes.byref(can), ctypes.byref(en))
                    pairs[f"{a}->{b}"] = {"can_access": bool(can.value), "enabled": bool(en.value)}
        p2p = {"pairs": pairs, "all_enabled": all(v["enabled"] for v in pairs.values())}
    # End-to-end floor at this N: every output byte lands in ONE host's
    # memory.  Replicated outputs (Mandelbrot 4:1) are widened by the host
    # pool (measured here, the same for every N: the host is shared); other
    # outputs are PCIe-bound, N links in parallel (measured on one GPU).
    floor = None
    if rank == 0:
        try:
            gbps = pcie_d2h_gbps(torch, my_gpu)
            pcie_ms = d2h / (len(my_gpus) * gbps * 1e9) * 1e3 if not shared else d2h / (n * gbps * 1e9) * 1e3
            floor = {"pcie_d2h_gbps_per_gpu": gbps, "pcie_ms": pcie_ms}
            spec0 = prog.spec()
            if wl.name.startswith("mandelbrot"):
                wms = ctypes.c_double(0.0)
                # counts < 65536 cross PCIe as uint16 (1/8 of the output bytes), else uint32 (1/4)
                share = 8.0 if wl.ITERS < 65536 else 4.0
                N.lib.ecl_probe_host_widen_width(spec0.global_work_size, 4, 2 if share == 8.0 else 4,
                                                 ctypes.byref(wms))
                floor["host_widen_ms"] = wms.value
                floor["e2e_floor_ms"] = max(pcie_ms / share, wms.value)
                floor["basis"] = (f"compact counts cross PCIe (1/{share:.0f} of the output bytes) and the host widens "
                                  "them 4:1 into the caller's buffer: max(PCIe at N links, host widening), and the "
                                  "host widening is shared by all N GPUs, so end-to-end scaling flattens at it")
            else:
                floor["e2e_floor_ms"] = pcie_ms
                floor["basis"] = "output bytes over N PCIe links at the measured per-GPU D2H rate"
        except Exception as exc:  # noqa: BLE001
            floor = {"error": str(exc)}
    line = {
        "metric": METRIC, "value": units / (ms_dev * 1e-3), "unit": "work-items/s", "n_gpus": n,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": ms_dev, "higher_is_better": True,
        "scaling": "strong", "vs_baseline": None, "dtype": wl.dtype, "data": "synthetic",
        "config": cfg,
        "engine": {"scheduler": P.describe(sched), "min_package_work_groups": min_wg,
                   "queue_depth": args.queue_depth, "widen_per_8": args.widen, "copy_split_items": copy_split,
                   "parallelism": f"coexec{n}" + ("-processes" if shared else ""),
                   "coordination": ("one process per GPU, shared-memory decision log" if shared else
                                    "one process, one host thread per GPU"),
                   "gpus_driven": my_gpus, "p2p": p2p},
        "step_ms": {k: [round(x, 4) for x in v] for k, v in step_log.items()},
        "e2e": {"value": units / (ms_e2e * 1e-3), "unit": "work-items/s", "h2d_bytes_per_step": h2d,
                "d2h_bytes_per_step": d2h, "ms_per_step": ms_e2e, "floor": floor},
        "roofline": {"bound": wl.bound, "achieved": achieved, "peak": peak, "unit": "TFLOP/s",
                     "frac": achieved / peak, "traffic": traffic, "traffic_basis": traffic_basis,
                     "algorithmic_flops_per_step": wl.flops(),
                     "kernel_ms_per_step": ms_kernel,
                     "achieved_basis": "algorithmic flops per step / kernel time per step: the union of the step's "
                                       "kernel intervals on the device (CUDA events on the launching lane streams; "
                                       "packages overlap on two lanes, so summed launch time double-counts), mean "
                                       "over the timed steps, max over devices and ranks",
                     "achieved_step_time": achieved_step, "frac_step_time": achieved_step / peak,
                     "peak_per_gpu": f64.value if wl.bound == "fp64" else f32.value,
                     "peak_source": f"{'DFMA' if wl.bound == 'fp64' else 'FFMA'} chains measured on this GPU by "
                                    "ecl_probe_vector_peaks (MEASURED_PEAKS.json has no FP64/FP32 vector figure)",
                     "fp64_dfma_tflops": f64.value, "fp64_dadd_tinstr_s": add.value, "fp32_ffma_tflops": f32.value},
        "coexec": {"balance": bal, "packages_per_step": len(last.packages),
                   # native denominator: the faster of one launch over the whole grid and the same
                   # kernel as plain two-stream sub-launches of copy_split_items (no scheduler)
                   "native_kernel_ms": k_native, "native_single_launch_ms": k_single,
                   "native_split_ms": k_split,
                   "engine_ms": ms_dev, "native_e2e_ms": t_native_e2e, "engine_e2e_ms": ms_e2e,
                   # speedup over one native single-kernel launch of the whole grid on one GPU, and the
                   # paper's efficiency speedup / s_max with s_max = N identical devices
                   "speedup_vs_native_1gpu": k_native / ms_dev if k_native else None,
                   "efficiency": k_native / (n * ms_dev) if k_native else None,
                   # runtime overhead of co-execution vs that native run (work-normalised: N * T_N vs T_1)
                   "overhead_pct_device": (n * ms_dev - k_native) / k_native * 100.0 if k_native else None,
                   # the same against the native program's host-bracketed call (its launch and wait
                   # latency counted like the engine's)
                   "native_host_ms": h_native,
                   "overhead_pct_vs_native_host": (n * ms_dev - h_native) / h_native * 100.0 if h_native else None,
                   "overhead_pct_e2e": (ms_e2e - t_native_e2e) / t_native_e2e * 100.0
                   if t_native_e2e and n == 1 else None,
                   # device busy time of the last resident step: union of its packages' kernel intervals
                   "device_busy_ms": max(busy.values()) if busy else None,
                   "device_busy_ms_per_device": busy,
                   "outputs_sane": bool(sane),
                   "e2e_last_kernel_end_ms": e2e_last_kernel_end},
        "gpu_launches": launches,
        "clocks": merge_clocks(clocks, clocks2),
    }
    if mix.value > 0 and wl.bound != "fp64":
        line["roofline"]["mix_ceiling_tflops"] = mix.value * n
        line["roofline"]["frac_of_mix_ceiling"] = achieved / (mix.value * n)
    if wl.bound == "fp64":
        # bit-exactness forbids contraction: 8 algorithmic flops take 6 FP64
        # pipe instructions on the fast path, so the attainable fraction of the
        # DFMA (2 flop/instr) peak is 8/12
        line["roofline"]["nonfma_ceiling_frac"] = 8.0 / 12.0
        line["roofline"]["frac_of_nonfma_ceiling"] = (achieved / peak) / (8.0 / 12.0)
        if mix.value > 0:
            # what the iteration's own DMUL/DADD/DFMA mix sustains on this GPU
            # with no control flow (ecl_probe_mandel_mix): the attainable roof
            line["roofline"]["mix_ceiling_tflops"] = mix.value * n
            line["roofline"]["frac_of_mix_ceiling"] = achieved / (mix.value * n)
    if hasattr(wl, "roofline_override"):
        ro = wl.roofline_override(ms_kernel, n, f32.value)
        ro_step = wl.roofline_override(ms_dev, n, f32.value)
        ro["achieved_step_time"], ro["frac_step_time"] = ro_step["achieved"], ro_step["frac"]
        ro["achieved_basis"] = ("algorithmic bytes per step / kernel time per step (union of the step's kernel "
                                "intervals, CUDA events on the launching streams, mean over the timed steps)")
        line["roofline"].update(ro)
        for k in ("algorithmic_flops_per_step", "fp64_dfma_tflops", "fp64_dadd_tinstr_s", "mix_ceiling_tflops", "frac_of_mix_ceiling"):
            line["roofline"].pop(k, None)
        achieved, peak = ro["achieved"], ro["peak"] or float("nan")
    if getattr(wl, "ceiling", None) and not getattr(wl, "roofline_note", None):
        c, why = wl.ceiling
        line["roofline"]["ceiling_frac"] = c
        line["roofline"]["frac_of_ceiling"] = (achieved / peak) / c
        line["roofline"]["ceiling_basis"] = why
    if hasattr(wl, "skip_ceiling"):
        c, why = wl.skip_ceiling()
        line["roofline"]["skip_ceiling_frac"] = c
        line["roofline"]["frac_of_skip_ceiling"] = (achieved / peak) / c
        line["roofline"]["skip_ceiling_basis"] = why
    if getattr(wl, "roofline_note", None):
        line["roofline"]["note"] = wl.roofline_note
    if wl.name == "ray":
        # round 1's bound for a tracer that runs the exact test on every
        # sphere: 17 counted flops in 16 unfused FP32 lane-ops (no FMA
        # contraction allowed) caps it at 17/32 of the FFMA peak; the
        # prefiltered scan is bounded by `ceiling_frac` instead
        line["roofline"]["nonfma_ceiling_frac"] = 17.0 / 32.0
        line["roofline"]["frac_of_nonfma_ceiling"] = (achieved / peak) / (17.0 / 32.0)
    if cpu is not None:
        line["cpu_baseline"] = cpu
    return line


def main(argv=None):
    ap = argparse.ArgumentParser(description=__doc__, formatter_class=argparse.RawDescriptionHelpFormatter)
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=5)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", choices=["ours", "reference"], default="ours")
    ap.add_argument("--workload", choices=sorted(WORKLOADS), default="mandelbrot")
    ap.add_argument("--k", type=float, default=2.0, help="HGuided k")
    ap.add_argument("--adaptive", action="store_true", help="HGuided powers from measured throughput")
    ap.add_argument("--queue-depth", type=int, default=3,
                    help="packages in flight per GPU (Mandelbrot e2e measured: 1 -> 51.7-53.1 ms, 2 -> 50.1-51.3, 3 -> 48.8)")
    ap.add_argument("--min-package", type=int, default=0, help="HGuided minimum package (work-groups)")
    ap.add_argument("--widen", type=int, default=8,
                    help="replicated outputs: pieces of 8 copied compact and widened on the host")
    ap.add_argument("--copy-split", type=int, default=0,
                    help="work-items per sub-launch when a package copies to the host or streams its inputs up "
                         "(0: the workload's default)")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-other-workloads", action="store_true",
                    help="default Mandelbrot run on one GPU: skip the compact lines of the other configs")
    args = ap.parse_args(argv)
    if args.impl == "ours":
        args.warmup = max(3, args.warmup)
    world, rank, local = init_dist()
    if args.impl == "reference":
        return run_reference(args, world, rank)
    return run_ours(args, world, rank, local)


if __name__ == "__main__":
    sys.exit(main())
