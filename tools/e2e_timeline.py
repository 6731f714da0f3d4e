#!/usr/bin/env python3
"""Per-package timeline of a Mandelbrot run with and without host outputs
(diagnostic: where the end-to-end step loses time against the resident one).

  python tools/e2e_timeline.py [--copy-split N] [--queue-depth D] [--k K]
"""
import argparse
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402

import bench  # noqa: E402
import paper_1805_02755_b200 as P  # noqa: E402
from paper_1805_02755_b200 import workloads as W  # noqa: E402


def show(tag, t, wall):
    pk = sorted(t.packages, key=lambda p: p.t_start_ms)
    t0 = min(p.t_enqueue_ms for p in pk)
    busy = sum(p.t_end_ms - p.t_start_ms for p in pk)
    print(f"{tag}: wall {wall:.2f} ms  t_total {t.t_total_ms:.2f}  packages {len(pk)}  sum(pkg) {busy:.2f}")
    for p in pk:
        print(f"   seq {p.seq:3d} off {p.offset_wg:8d} size {p.size_wg:8d}  enq {p.t_enqueue_ms - t0:8.3f}"
              f"  start {p.t_start_ms - t0:8.3f}  end {p.t_end_ms - t0:8.3f}  dur {p.t_end_ms - p.t_start_ms:7.3f}")


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--copy-split", type=int, default=1 << 23)
    ap.add_argument("--queue-depth", type=int, default=2)
    ap.add_argument("--widen", type=int, default=8)
    ap.add_argument("--k", type=float, default=2.0)
    ap.add_argument("--min-package", type=int, default=0)
    args = ap.parse_args()
    wl = bench.WORKLOADS["mandelbrot"](P, W, np)
    prog = P.validate_program(wl.spec())
    devs = [P.cuda_device("gpu0", 0, queue_depth=args.queue_depth,
                          min_package_work_groups=args.min_package or wl.min_package(1),
                          widen_per_8=args.widen, copy_split_items=args.copy_split)]
    sched = wl.scheduler(1)
    if hasattr(sched, "k"):
        sched.k = args.k
    outs = [P.PinnedBuffer(b.size_bytes(), np.uint8) for b in prog.spec().out_buffers]
    out_arrays = [b.array for b in outs]
    with P.Engine(P.EngineConfig(devs, sched), prog) as e:
        for mode, o in (("resident", None), ("e2e", out_arrays)):
            for _ in range(3):
                e.run_into([], o, want_trace=False)
            t0 = time.perf_counter()
            e.run_into([], o, want_trace=False)
            wall = (time.perf_counter() - t0) * 1e3
            show(mode, e.last_trace(), wall)


if __name__ == "__main__":
    main()
