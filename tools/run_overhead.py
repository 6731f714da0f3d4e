#!/usr/bin/env python3
"""Where a short run's fixed cost goes: host wall time of run_into vs the
kernel's own start/end inside the trace (device-resident Gaussian)."""
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402

import bench  # noqa: E402
import paper_1805_02755_b200 as P  # noqa: E402
from paper_1805_02755_b200 import workloads as W  # noqa: E402


def main():
    name = sys.argv[1] if len(sys.argv) > 1 else "gaussian"
    wl = bench.WORKLOADS[name](P, W, np)
    prog = P.validate_program(wl.spec())
    devs = [P.cuda_device("gpu0", 0, min_package_work_groups=wl.min_package(1))]
    with P.Engine(P.EngineConfig(devs, wl.scheduler(1)), prog) as e:
        e.run_into(wl.host_inputs(), None, want_trace=False)
        walls, starts, ends = [], [], []
        for _ in range(50):
            t0 = time.perf_counter()
            e.run_into(None, None, want_trace=False)
            walls.append((time.perf_counter() - t0) * 1e3)
            t = e.last_trace()
            starts.append(min(p.t_start_ms for p in t.packages))
            ends.append(max(p.t_end_ms for p in t.packages))
        kt = e.kernel_timing(reset=True)
    m = lambda v: float(np.median(v))  # noqa: E731
    print(f"{name}: wall {m(walls):.4f} ms  first kernel start {m(starts):.4f} ms  last kernel end {m(ends):.4f} ms"
          f"  -> before {m(starts):.4f}, after {m(walls) - m(ends):.4f} ms; kernel timing {kt}")


if __name__ == "__main__":
    main()
