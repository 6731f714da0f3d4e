#!/usr/bin/env python3
"""Measured-throughput HGuided on heterogeneous devices (one B200).

Two logical devices share one GPU but run different code for the same
counts: device 0 the periodic-orbit Mandelbrot variant (mandelbrot@14,
~2.6x fewer iterations at the config), device 1 the default kernel.  Seeds
say the devices are equal (powers 1:1).  For each scheduler the engine runs
the 16384^2 x 2048 config `--runs` times (device-resident, one Engine, so
adaptive HGuided carries its learned rates from run to run) and reports the
time, balance, package count and learned powers per run.

  python tools/adaptive_hetero.py [--runs 6] [--out profiles/r2/adaptive_hetero.json]
"""
import argparse
import json
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402

import paper_1805_02755_b200 as P  # noqa: E402
from paper_1805_02755_b200 import workloads as W  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--runs", type=int, default=6)
    ap.add_argument("--size", type=int, default=16384)
    ap.add_argument("--out", default="")
    args = ap.parse_args()
    prog = P.validate_program(W.mandelbrot_spec(args.size, args.size, 2048))
    result = {"workload": f"mandelbrot {args.size}^2 x 2048, two logical devices on one B200: "
                          "gpu0 runs mandelbrot@14, gpu1 mandelbrot; seeds 1:1", "schedulers": {}}
    for name, sched in (("hguided(k=2) static seeds", P.HGuidedConfig(2.0)),
                        ("hguided(k=2) adaptive", P.HGuidedConfig(2.0, adaptive=True, ema_alpha=0.5)),
                        ("dynamic(64)", P.DynamicConfig(64))):
        devs = [P.cuda_device("gpu0", 0, kernel="mandelbrot@14", min_package_work_groups=148),
                P.cuda_device("gpu1", 0, min_package_work_groups=148)]
        rows = []
        with P.Engine(P.EngineConfig(devs, sched), prog) as e:
            e.run_into([], None, want_trace=False)  # warm-up (init charged here)
            for _ in range(args.runs):
                t0 = time.perf_counter()
                e.run_into([], None, want_trace=False)
                wall = (time.perf_counter() - t0) * 1e3
                t = e.last_trace()
                share = {}
                for p in t.packages:
                    share[p.device_id] = share.get(p.device_id, 0) + p.size_wg
                rows.append({"wall_ms": wall, "t_total_ms": t.t_total_ms, "balance": P.balance(t),
                             "packages": len(t.packages),
                             "work_share_gpu0": share.get("gpu0", 0) / prog.total_work_groups(),
                             "learned_powers": e.learned_powers()})
        result["schedulers"][name] = rows
        med = float(np.median([r["wall_ms"] for r in rows[1:]] or [rows[0]["wall_ms"]]))
        print(f"{name:28s} median wall {med:7.2f} ms  balance {rows[-1]['balance']:.3f}  "
              f"packages {rows[-1]['packages']}  gpu0 share {rows[-1]['work_share_gpu0']:.3f}  "
              f"powers {rows[-1]['learned_powers']}")
    if args.out:
        os.makedirs(os.path.dirname(os.path.abspath(args.out)), exist_ok=True)
        with open(args.out, "w") as f:
            json.dump(result, f, indent=1)


if __name__ == "__main__":
    main()
