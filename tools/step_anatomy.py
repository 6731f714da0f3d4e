#!/usr/bin/env python3
"""Where a short device-resident step's time goes in the bench harness:
the same engine run timed (a) by host wall clock, (b) between CUDA events on
torch's stream, (c) as (b) after an L2 flush, (d) as (c) with the NVML clock
sampler running — medians over the repetitions.  Diagnostic only.

  python tools/step_anatomy.py [workload] [reps]
"""
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402
import torch  # noqa: E402

import bench  # noqa: E402
import paper_1805_02755_b200 as P  # noqa: E402
from paper_1805_02755_b200 import workloads as W  # noqa: E402


def main():
    name = sys.argv[1] if len(sys.argv) > 1 else "gaussian"
    reps = int(sys.argv[2]) if len(sys.argv) > 2 else 50
    wl = bench.WORKLOADS[name](P, W, np)
    prog = P.validate_program(wl.spec())
    devs = [P.cuda_device("gpu0", 0, queue_depth=3, min_package_work_groups=wl.min_package(1))]
    flush = torch.empty(bench.L2_FLUSH_BYTES, dtype=torch.uint8, device="cuda:0")
    stream = torch.cuda.current_stream()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    med = lambda v: float(np.median(v))  # noqa: E731
    with P.Engine(P.EngineConfig(devs, wl.scheduler(1)), prog) as e:
        e.run_into(wl.host_inputs(), None, want_trace=False)
        for _ in range(5):
            e.run_into(None, None, want_trace=False)
        walls = []
        for _ in range(reps):
            t0 = time.perf_counter()
            e.run_into(None, None, want_trace=False)
            walls.append((time.perf_counter() - t0) * 1e3)

        def evented(do_flush):
            out, busy = [], []
            for _ in range(reps):
                if do_flush:
                    flush.zero_()
                torch.cuda.synchronize()
                e0.record(stream)
                e.run_into(None, None, want_trace=False)
                e1.record(stream)
                e1.synchronize()
                out.append(e0.elapsed_time(e1))
                t = e.last_trace()
                busy.append(max(p.t_end_ms for p in t.packages) - min(p.t_start_ms for p in t.packages))
            return out, busy

        b, kb = evented(False)
        c, kc = evented(True)
        s = bench.ClockSampler(0).start()
        d, kd = evented(True)
        s.stop()
    print(f"{name}: (a) wall {med(walls):.4f} ms  (b) events {med(b):.4f} (kernel {med(kb):.4f})  "
          f"(c) +L2 flush {med(c):.4f} (kernel {med(kc):.4f})  (d) +NVML sampler {med(d):.4f} (kernel {med(kd):.4f})",
          flush=True)


if __name__ == "__main__":
    main()
