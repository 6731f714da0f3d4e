#!/usr/bin/env python3
"""Per-kernel totals of an ncu launch list (--metrics gpu__time_duration.sum
--csv --log-file X.csv): launches, summed time, share of GPU time.

  python tools/launch_summary.py gpurun_out/launches.csv > profiles/r1/launches.md
"""
import collections
import csv
import sys

SCALE = {"ns": 1e-6, "nsecond": 1e-6, "us": 1e-3, "usecond": 1e-3, "ms": 1.0, "msecond": 1.0, "s": 1e3, "second": 1e3}


def main(path):
    rows = [r for r in csv.reader(open(path)) if len(r) > 10]
    hdr = rows[0]
    ki, ui, vi = hdr.index("Kernel Name"), hdr.index("Metric Unit"), hdr.index("Metric Value")
    agg = collections.defaultdict(lambda: [0, 0.0])
    for r in rows[1:]:
        ms = float(r[vi].replace(",", "")) * SCALE.get(r[ui], 1.0)
        name = r[ki].split("(")[0]
        agg[name][0] += 1
        agg[name][1] += ms
    total = sum(t for _, t in agg.values())
    print(f"ncu launch list `{path.split('/')[-1]}` (cold-cache, serialised replay; compare shares, not absolutes)\n")
    print("| kernel | launches | total ms | mean ms | share of GPU time |")
    print("|---|---:|---:|---:|---:|")
    for name, (n, t) in sorted(agg.items(), key=lambda x: -x[1][1]):
        print(f"| `{name}` | {n} | {t:.3f} | {t / n:.3f} | {100 * t / total:.2f}% |")


if __name__ == "__main__":
    main(sys.argv[1])
