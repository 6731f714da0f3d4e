#!/usr/bin/env python3
"""One warm-up run plus one measured run of a bench workload on one GPU —
the short command ncu profiles (never a multi-rank command).

  python tools/profile_run.py --workload gaussian [--e2e]
"""
import argparse
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
    ap.add_argument("--workload", default="mandelbrot", choices=sorted(bench.WORKLOADS))
    ap.add_argument("--steps-override", type=int, default=0, help="NBody timesteps (default: the workload's)")
    ap.add_argument("--e2e", action="store_true", help="host outputs (D2H inside the run)")
    args = ap.parse_args()
    wl = bench.WORKLOADS[args.workload](P, W, np)
    prog = P.validate_program(wl.spec())
    devs = [P.cuda_device("gpu0", 0, min_package_work_groups=wl.min_package(1))]
    inputs = wl.host_inputs()
    outs = None
    if args.e2e:
        outs = [np.zeros(b.size_bytes(), np.uint8) for b in prog.spec().out_buffers]
    steps = args.steps_override or wl.steps_per_run
    with P.Engine(P.EngineConfig(devs, wl.scheduler(1)), prog) as e:
        for _ in range(2):
            if steps > 1:
                e.run_steps(inputs, outs, steps, wl.swaps, want_trace=False)
            else:
                e.run_into(inputs, outs, want_trace=False)
        t = e.last_trace()
    print(f"{args.workload}: {len(t.packages)} packages, t_total {t.t_total_ms:.3f} ms")


if __name__ == "__main__":
    main()
