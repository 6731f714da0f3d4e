#!/usr/bin/env python3
"""Predicted multi-GPU co-execution of the Ray benchmark (8192^2, 64 spheres,
depth 4) from one B200: the reference's virtual-clock model (drive_virtual,
engine.hpp:306-352) replays each scheduler over N simulated B200s whose
per-pixel costs come from the image this GPU rendered.

Cost per pixel = 1 + 4 * bounces (w channel of the output): every surface
hit traces one reflection scan plus up to three shadow-ray scans, a miss one
primary scan.  A proxy (the sphere-test count per pixel is not an output),
calibrated so that one simulated device takes the measured single-GPU step
time.  Package dispatch costs 3 us; minimum package as in bench.py.

  python tools/virtual_scaling_ray.py [--out profiles/r1/experiments/virtual-scaling-ray.json]
"""
import argparse
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402

import bench  # noqa: E402
import paper_1805_02755_b200 as P  # noqa: E402
from paper_1805_02755_b200 import workloads as W  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--out", default=os.path.join(ROOT, "profiles", "r1", "experiments", "virtual-scaling-ray.json"))
    ap.add_argument("--min-package", type=int, default=0, help="work-groups (0: bench.py's)")
    args = ap.parse_args()
    wl = bench.WORKLOADS["ray"](P, W, np)
    prog = P.validate_program(wl.spec())
    dev = [P.cuda_device("gpu0", 0, min_package_work_groups=wl.min_package(1))]
    with P.Engine(P.EngineConfig(dev, wl.scheduler(1)), prog) as e:
        e.run_into(wl.host_inputs(), None, want_trace=False)
        times = []
        for _ in range(5):
            t = e.run_into(None, None)
            times.append(t.t_total_ms)
        out = np.empty(wl.units() * 4, np.float32)
        e.gather([out])
    t1 = float(np.median(times))
    bounces = out.reshape(-1, 4)[:, 3]
    cost = 1.0 + 4.0 * bounces.astype(np.float64)
    power = float(cost.sum()) / t1  # cost units per ms of one B200

    result = {"workload": wl.workload, "t1_ms_measured": t1, "cost_model": "1 + 4*bounces per pixel",
              "cost_total": float(cost.sum()), "power_per_gpu": power, "dispatch_ms": 0.003,
              "min_package_work_groups": args.min_package or wl.min_package(1), "runs": []}
    for n in (1, 2, 4, 8):
        for name, sched in (("hguided", P.HGuidedConfig(2.0)), (f"dynamic({64 * n})", P.DynamicConfig(64 * n)),
                            ("static", P.StaticConfig())):
            devs = [P.simulated_device(f"b200_{i}", power, overhead_ms=0.003, bandwidth=1e15,
                                       min_wg=args.min_package or wl.min_package(n)) for i in range(n)]
            cfg = P.EngineConfig(devs, sched, clock_mode=P.ClockMode.Virtual)
            with P.Engine(cfg, prog) as e:
                tr = e.run_virtual(cost)
            rep = P.make_report(tr, [t1] * n)
            eff = t1 / (n * tr.t_total_ms)
            result["runs"].append({"gpus": n, "scheduler": name, "t_total_ms": tr.t_total_ms,
                                   "packages": len(tr.packages), "balance": rep.balance, "efficiency": eff})
            print(f"N={n} {name:14s} t={tr.t_total_ms:8.3f} ms  packages {len(tr.packages):5d}  "
                  f"balance {rep.balance:.3f}  efficiency {eff:.3f}")
    os.makedirs(os.path.dirname(args.out), exist_ok=True)
    with open(args.out, "w") as f:
        json.dump(result, f, indent=2)


if __name__ == "__main__":
    main()
