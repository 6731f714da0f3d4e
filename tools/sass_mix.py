#!/usr/bin/env python3
"""Executed-instruction mix by opcode (and the hottest stall lines) from an
ncu report's SASS source page.

  python tools/sass_mix.py gpurun_out/ncu_x.ncu-rep [--top 14]
"""
import argparse
import collections
import csv
import io
import subprocess


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("report")
    ap.add_argument("--top", type=int, default=14)
    a = ap.parse_args()
    out = subprocess.run(["ncu", "-i", a.report, "--page", "source", "--csv", "--print-source", "sass"],
                         capture_output=True, text=True, check=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    hi = next(i for i, r in enumerate(rows) if "Address" in r and "Source" in r)
    h = rows[hi]
    ci, si, st = h.index("Instructions Executed"), h.index("Source"), h.index("Warp Stall Sampling (All Samples)")
    mix, stall = collections.Counter(), collections.Counter()
    for r in rows[hi + 1:]:
        try:
            n = float(r[ci])
            s = float(r[st])
        except (ValueError, IndexError):
            continue
        toks = r[si].split()
        if not toks:
            continue
        op = toks[1] if toks[0].startswith("@") and len(toks) > 1 else toks[0]
        mix[op.split(".")[0]] += n
        stall[op.split(".")[0]] += s
    tot, stot = sum(mix.values()), sum(stall.values())
    print(f"{'opcode':10s} {'executed':>10s} {'share':>6s} {'stall-smpl':>10s}")
    for k, n in mix.most_common(a.top):
        print(f"{k:10s} {n / 1e6:9.1f}M {n / tot:6.3f} {stall[k] / max(stot, 1):10.3f}")
    print(f"total {tot / 1e6:.1f}M warp instructions")


if __name__ == "__main__":
    main()
