#!/usr/bin/env python3
"""Kernel-only A/B timing of a bench workload's kernel variants on one GPU:
one native launch over the whole grid per repetition (an L2 flush before
each), median of the repetitions.  Diagnostic only; the bench numbers come
from bench.py.

  python tools/kernel_time.py --workload binomial --variants 0,3,1 --reps 7
"""
import argparse
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402
import torch  # noqa: E402

import bench  # noqa: E402
import paper_1805_02755_b200 as P  # noqa: E402
from paper_1805_02755_b200 import workloads as W  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--workload", default="binomial", choices=sorted(bench.WORKLOADS))
    ap.add_argument("--variants", default="0")
    ap.add_argument("--reps", type=int, default=7)
    args = ap.parse_args()
    wl = bench.WORKLOADS[args.workload](P, W, np)
    spec = wl.spec()
    inputs = wl.host_inputs()
    flush = torch.empty(512 << 20, dtype=torch.uint8, device="cuda:0")
    for v in args.variants.split(","):
        kern = f"{spec.kernel}@{v}" if v != "-" else ""
        prog = P.validate_program(spec)
        devs = [P.cuda_device("gpu0", 0, kernel=kern)]
        ks = []
        with P.Engine(P.EngineConfig(devs, wl.scheduler(1)), prog) as e:
            e.run_into(inputs, None, want_trace=False)  # upload + warm-up
            for _ in range(args.reps + 1):
                flush.fill_(1)
                torch.cuda.synchronize()
                ks.append(e.native_run(None, None)[0])
        ks = sorted(ks[1:])
        print(f"{args.workload} {kern or spec.kernel}: median {ks[len(ks) // 2]:.3f} ms "
              f"(min {ks[0]:.3f}, max {ks[-1]:.3f})", flush=True)


if __name__ == "__main__":
    main()
