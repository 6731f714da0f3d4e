#!/usr/bin/env python3
"""bench.py — BASELINE.json's headline: Mandelbrot 16384^2 x 2048 (FP64, the
reference kernel workloads.hpp:78-100) co-executed with HGuided over N B200s.

One step = one Engine run over the whole index space (268,435,456 work-items).
  value  device-resident: outputs stay in each GPU's partition (no inputs).
  e2e    the same run through the C-ABI with HOST buffers: every package's
         out_range_for slice is copied D2H into a page-locked host buffer
         inside the timed region (4 GiB per step).
  roofline   dominant kernel (mandel_persistent<double>): algorithmic FP64
         flops (8/iteration + 3/escaped pixel = 7.69796e11 per
         step) / summed CUDA-event kernel time, against the DFMA peak measured
         on this device by ecl_probe_vector_peaks.
  cpu_baseline   the reference engine itself (oracle/_ref, wall mode, H
         NativePool devices x 1 worker, Dynamic{max(64,16H)}) on a 4096^2
         sub-grid of the same viewport and iteration cap.
--impl reference times that same CPU reference as the reference arm.
"""
from __future__ import annotations

import argparse
import json
import os
import subprocess
import sys
import threading
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

W_PX, H_PX, ITERS = 16384, 16384, 2048
VIEWPORT = (-2.5, -1.25, 1.0, 1.25)
LWS = 256
PIXELS = W_PX * H_PX
# Golden facts of the config (pinned by tests/test_engine_gpu.py)
SUM_COUNT, INSIDE = 96_141_151_663, 46_275_993
ALG_FLOPS = 8.0 * SUM_COUNT + 3.0 * (PIXELS - INSIDE)
SAMPLE_W = 4096  # CPU sample: 4096^2 sub-grid, same viewport and max_iter
METRIC = "work-items/s at 1/2/4/8 B200 + HGuided co-exec efficiency & overhead vs native"


def env_int(name, default):
    try:
        return int(os.environ.get(name, default))
    except ValueError:
        return default


class ClockSampler:
    """nvidia-smi clocks/throttle reasons sampled during the timed region."""

    FIELDS = ("index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
              "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
              "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, gpu_index: int):
        self.gpu = gpu_index
        self.samples = []
        self._stop = threading.Event()
        self._proc = None
        self._thread = None

    def start(self):
        try:
            self._proc = subprocess.Popen(
                ["nvidia-smi", f"--id={self.gpu}", f"--query-gpu={self.FIELDS}", "--format=csv,noheader,nounits",
                 "-lms", "100"], stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
        except OSError:
            self._proc = None
            return self
        self._thread = threading.Thread(target=self._read, daemon=True)
        self._thread.start()
        return self

    def _read(self):
        for line in self._proc.stdout:
            parts = [p.strip() for p in line.split(",")]
            if len(parts) >= 9:
                self.samples.append(parts)

    def stop(self):
        if self._proc:
            self._proc.terminate()
            try:
                self._proc.wait(timeout=5)
            except subprocess.TimeoutExpired:
                self._proc.kill()
        if self._thread:
            self._thread.join(timeout=5)
        return self.summary()

    def summary(self):
        if not self.samples:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"], "samples": 0}
        sm = sorted(float(s[1]) for s in self.samples if s[1].replace(".", "").isdigit())
        mx = max((float(s[2]) for s in self.samples if s[2].replace(".", "").isdigit()), default=None)
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = set()
        for s in self.samples:
            for n, v in zip(names, s[5:9]):
                if v.lower().startswith("active"):
                    reasons.add(n)
        power = [float(s[3]) for s in self.samples if s[3].replace(".", "").isdigit()]
        return {"sm_mhz": sm[len(sm) // 2] if sm else None, "sm_max_mhz": mx, "reasons": sorted(reasons),
                "samples": len(self.samples), "power_w_max": max(power) if power else None}


def mandel_program_json(w, h):
    return {"kernel": "mandelbrot", "global_work_size": w * h, "local_work_size": LWS,
            "out_pattern": {"out_indices": 4, "work_items": 1},
            "out_buffers": [{"name": "counts", "element_size_bytes": 4, "element_count": w * h * 4}],
            "args": [w, h, ITERS] + list(VIEWPORT)}


def cpu_threads():
    try:
        return len(os.sched_getaffinity(0))
    except AttributeError:
        return os.cpu_count() or 1


def cpu_reference_sample(steps: int = 1):
    """Times the reference engine (oracle/_ref) on the 4096^2 sample; falls
    back to the repo's C restatement (oracle/_build) when _ref is absent."""
    from tests import _oracle
    h = cpu_threads()
    prog = mandel_program_json(SAMPLE_W, SAMPLE_W)
    ref = _oracle.Reference.load()
    times = []
    if ref is not None:
        kind = "reference"
        for _ in range(steps):
            s, _fnv = ref.wall_run(prog, h, 1, max(64, 16 * h))
            times.append(s)
    else:
        kind = "port"
        o = _oracle.Oracle()
        for _ in range(steps):
            t0 = time.perf_counter()
            o.mandelbrot(SAMPLE_W, SAMPLE_W, ITERS)
            times.append(time.perf_counter() - t0)
    px = SAMPLE_W * SAMPLE_W
    return {"kind": kind, "cores": h if kind == "reference" else _oracle.Oracle().threads(), "times_s": times,
            "value": px / (sum(times) / len(times)),
            "sample": f"{SAMPLE_W}x{SAMPLE_W} sub-grid of the same viewport, max_iter {ITERS} "
                      f"({px} px = 1/16 of the config); reference engine wall mode, {h} NativePool devices x 1 "
                      f"worker, Dynamic{{{max(64, 16 * h)}}}" if kind == "reference" else
                      f"{SAMPLE_W}x{SAMPLE_W} sub-grid, oracle/oracle.c OpenMP restatement"}


def init_dist():
    world = env_int("WORLD_SIZE", 1)
    rank = env_int("RANK", 0)
    local = env_int("LOCAL_RANK", 0)
    return world, rank, local


def run_reference(args, world, rank):
    if rank != 0:
        return 0
    steps = args.warmup + args.steps
    res = cpu_reference_sample(steps)
    timed = res["times_s"][args.warmup:]
    value = SAMPLE_W * SAMPLE_W / (sum(timed) / len(timed))
    line = {"impl": "reference", "metric": METRIC, "value": value, "unit": "work-items/s", "n_gpus": args.gpus,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": 1e3 * sum(timed) / len(timed),
            "higher_is_better": True, "scaling": "strong", "vs_baseline": None, "dtype": "f64", "data": "synthetic",
            "config": {"workload": "mandelbrot 16384x16384 max_iter 2048 (sampled: 4096x4096 sub-grid)",
                       "scheduler": f"dynamic(packages={max(64, 16 * cpu_threads())})", "lws": LWS,
                       "viewport": list(VIEWPORT)},
            "cpu_baseline": {"value": value, "unit": "work-items/s", "cores": res["cores"], "kind": res["kind"],
                             "sample": res["sample"]},
            "e2e": {"value": value, "unit": "work-items/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(line), flush=True)
    return 0


def run_ours(args, world, rank, local):
    import numpy as np
    import torch

    import paper_1805_02755_b200 as P
    from paper_1805_02755_b200 import _native as N

    ngpu_visible = P.gpu_count()
    if ngpu_visible < 1:
        print(json.dumps({"error": "no CUDA device visible"}))
        return 1
    dist = world > 1
    if dist:
        import torch.distributed as td
        torch.cuda.set_device(local)
        td.init_process_group("nccl", device_id=torch.device("cuda", local))
    # EngineCL's co-execution model: one host coordinator drives every device
    # of the box through its per-device threads (engine.hpp:354-405).  Under
    # torchrun, rank 0 owns the engine over GPUs 0..N-1; the other ranks only
    # join the barriers.
    n = args.gpus if not dist else world
    torch.cuda.set_device(local if dist else 0)

    def barrier():
        torch.cuda.synchronize()
        if dist:
            torch.distributed.barrier()

    line = None
    if rank == 0:
        line = bench_engine(args, n, P, N, np, torch, barrier)
    else:
        # follow rank 0's barrier sequence (warm-up/time/e2e/native phases)
        for _ in range(6):
            barrier()
    if dist:
        torch.distributed.destroy_process_group()
    if rank == 0:
        print(json.dumps(line), flush=True)
    return 0


def bench_engine(args, n, P, N, np, torch, barrier):
    from paper_1805_02755_b200 import workloads as W
    import ctypes

    sms = 148
    min_wg = args.min_package if args.min_package else sms * 8
    devs = [P.cuda_device(f"gpu{i}", ordinal=i % P.gpu_count(), power=1.0, queue_depth=args.queue_depth,
                          min_package_work_groups=min_wg) for i in range(n)]
    sched = P.HGuidedConfig(k=args.k, adaptive=args.adaptive)
    prog = P.validate_program(W.mandelbrot_spec(W_PX, H_PX, ITERS, lws=LWS))
    eng = P.Engine(P.EngineConfig(devs, sched), prog)
    stream = torch.cuda.current_stream()

    def timed(fn, steps):
        barrier()
        e0 = torch.cuda.Event(enable_timing=True)
        e1 = torch.cuda.Event(enable_timing=True)
        e0.record(stream)
        traces = [fn() for _ in range(steps)]
        e1.record(stream)
        barrier()
        return e0.elapsed_time(e1) / steps, traces

    # --- device-resident (value) ---
    for _ in range(args.warmup):
        eng.run_into([], None)
    eng.kernel_timing(reset=True)
    sampler = ClockSampler(0).start()
    ms_dev, _ = timed(lambda: eng.run_into([], None, want_trace=False), args.steps)
    clocks = sampler.stop()
    kernel_ms, launches = eng.kernel_timing(reset=True)
    last = eng.last_trace()
    bal = P.balance(last) if n > 1 else 1.0

    # parity sanity on a device-resident result (golden facts, no oracle)
    pinned = P.PinnedBuffer(PIXELS * 16, np.uint32)
    out = pinned.array
    eng.gather([out])
    counts = out.reshape(-1, 4)[:, 0]
    exact = int(counts.sum(dtype=np.uint64)) == SUM_COUNT and int((counts >= ITERS).sum()) == INSIDE

    # --- end to end through the C-ABI with a page-locked host output ---
    for _ in range(args.warmup):
        eng.run_into([], [out])
    sampler2 = ClockSampler(0).start()
    out[:] = 0
    ms_e2e, _ = timed(lambda: eng.run_into([], [out], want_trace=False), args.steps)
    clocks2 = sampler2.stop()
    eng.kernel_timing(reset=True)
    exact_e2e = int(counts.sum(dtype=np.uint64)) == SUM_COUNT and int((counts >= ITERS).sum()) == INSIDE

    # --- native single-kernel baseline (overhead denominator) ---
    barrier()
    native_k, native_e2e = [], []
    for _ in range(args.warmup + args.steps):
        native_k.append(eng.native_run([], None)[0])
    for _ in range(max(1, args.steps)):
        native_e2e.append(eng.native_run([], [out])[1])
    native_k = native_k[args.warmup:]
    k_native = sorted(native_k)[len(native_k) // 2]
    t_native_e2e = sorted(native_e2e)[len(native_e2e) // 2]
    barrier()

    # --- roofline: measured FP64 peak on this device ---
    f64, add, f32 = ctypes.c_double(), ctypes.c_double(), ctypes.c_double()
    N.lib.ecl_probe_vector_peaks(0, ctypes.byref(f64), ctypes.byref(add), ctypes.byref(f32))
    kernel_ms_per_step = kernel_ms / args.steps
    # Packages overlap on the device's two compute lanes, so summed launch
    # times double-count the overlap: the achieved rate is taken over the whole
    # device-resident step (every FP64 op of the step / step time).
    achieved = ALG_FLOPS / (ms_dev * 1e-3) / 1e12
    peak = f64.value
    eng.close()
    del out, counts
    pinned.free()

    cpu = None
    if n == 1 and not args.no_cpu_baseline:
        cpu = cpu_reference_sample(1)

    value = PIXELS / (ms_dev * 1e-3)
    line = {
        "metric": METRIC, "value": value, "unit": "work-items/s", "n_gpus": n, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": ms_dev, "higher_is_better": True, "scaling": "strong",
        "vs_baseline": None, "dtype": "f64", "data": "synthetic",
        "config": {"workload": "mandelbrot 16384x16384 max_iter 2048 viewport (-2.5,-1.25)-(1,1.25), 4:1 uint32 out",
                   "scheduler": P.describe(sched), "lws": LWS, "min_package_work_groups": min_wg,
                   "queue_depth": args.queue_depth, "parallelism": f"coexec{n}",
                   "l2": "outputs 4 GiB per step (> 126 MB L2); no inputs"},
        "e2e": {"value": PIXELS / (ms_e2e * 1e-3), "unit": "work-items/s", "h2d_bytes_per_step": 0,
                "d2h_bytes_per_step": PIXELS * 16, "ms_per_step": ms_e2e,
                "note": "mandelbrot reads no input buffers (workloads.hpp:188-189); its 7 scalar args travel in "
                        "the launch parameters; D2H = every package's 4:1 uint32 slice into pinned host memory"},
        "roofline": {"bound": "fp64", "achieved": achieved, "peak": peak, "unit": "TFLOP/s",
                     "frac": achieved / peak, "traffic": None,
                     "kernel": "mandel_persistent<double,16>",
                     "achieved_basis": "algorithmic flops per step / device-resident step time (packages overlap "
                                       "on two compute lanes; summed launch time double-counts)",
                     "algorithmic": "8 FP64 flops/iteration + 3/escaped pixel = 7.69796e11 per step (SURVEY §8d)",
                     "peak_source": "DFMA chains measured on this GPU by ecl_probe_vector_peaks (MEASURED_PEAKS.json "
                                    "has no FP64 figure)",
                     "nonfma_ceiling_frac": 8.0 / 14.0,
                     "fp64_dadd_tinstr_s": add.value, "fp32_ffma_tflops": f32.value},
        "coexec": {"balance": bal, "packages_per_step": len(last.packages),
                   "native_kernel_ms": k_native, "engine_ms": ms_dev,
                   "overhead_pct_device": (ms_dev - k_native) / k_native * 100.0,
                   "native_e2e_ms": t_native_e2e, "engine_e2e_ms": ms_e2e,
                   "overhead_pct_e2e": (ms_e2e - t_native_e2e) / t_native_e2e * 100.0,
                   "kernel_ms_per_step": kernel_ms_per_step,
                   "bit_exact_sums": bool(exact and exact_e2e)},
        "gpu_launches": launches,
        "clocks": {"sm_mhz": clocks["sm_mhz"], "sm_max_mhz": clocks["sm_max_mhz"],
                   "reasons": sorted(set(clocks["reasons"]) | set(clocks2["reasons"])),
                   "samples": clocks["samples"] + clocks2["samples"], "power_w_max": clocks.get("power_w_max")},
    }
    if cpu is not None:
        line["cpu_baseline"] = {"value": cpu["value"], "unit": "work-items/s", "cores": cpu["cores"],
                                "kind": cpu["kind"], "sample": cpu["sample"]}
    return line


def main(argv=None):
    ap = argparse.ArgumentParser(description=__doc__, formatter_class=argparse.RawDescriptionHelpFormatter)
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=5)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", choices=["ours", "reference"], default="ours")
    ap.add_argument("--k", type=float, default=2.0, help="HGuided k")
    ap.add_argument("--adaptive", action="store_true", help="HGuided powers from measured throughput")
    ap.add_argument("--queue-depth", type=int, default=2)
    ap.add_argument("--min-package", type=int, default=0, help="HGuided minimum package (work-groups)")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    args = ap.parse_args(argv)
    args.warmup = max(3, args.warmup) if args.impl == "ours" else args.warmup
    world, rank, local = init_dist()
    if args.impl == "reference":
        return run_reference(args, world, rank)
    return run_ours(args, world, rank, local)


if __name__ == "__main__":
    sys.exit(main())
