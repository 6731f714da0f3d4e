#!/usr/bin/env python3
"""Markdown results table from the committed bench lines (profiles/<round>/bench_*.json).

  python tools/results_table.py profiles/r1
"""
import json
import os
import sys

ROWS = [
    ("mandelbrot", "Mandelbrot 16384²×2048 FP64, HGuided", "px/s"),
    ("mandelbrot_periodic", "Mandelbrot FP64 @14 (opt-in periodic-orbit exit, same counts)", "px/s"),
    ("mandelbrot_f32", "Mandelbrot FP32 variant", "px/s"),
    ("gaussian", "Gaussian 4096², 31×31, Static", "px/s"),
    ("binomial", "Binomial 8M × 254, HGuided", "opt/s"),
    ("nbody", "NBody 1M × 10 steps, Dynamic", "body-steps/s"),
    ("ray", "Ray 8192², HGuided", "px/s"),
]


def main(d):
    print("| Workload | device-resident | e2e (host buffers) | frac of peak | overhead vs native | CPU reference |")
    print("|---|---|---|---|---|---|")
    for key, name, unit in ROWS:
        path = os.path.join(d, f"bench_{key}.json")
        if not os.path.exists(path):
            continue
        b = json.loads(open(path).read().strip().splitlines()[-1])
        r, e, c, co = b["roofline"], b["e2e"], b.get("cpu_baseline") or {}, b.get("coexec") or {}
        ms = b["ms_per_step"]
        t = f"{ms / 1e3:.2f} s" if ms > 1000 else f"{ms:.3g} ms"
        ovh = co.get("overhead_pct_device")
        cpu = f"{c['value']:.3g} {unit} ({c.get('cores')} threads)" if c.get("value") else "—"
        frac = (f"— (effective {r['frac']:.2f})" if r.get("note") else f"{r['frac']:.3f} {r['bound'].upper()}")
        print(f"| {name} | {b['value']:.3g} {unit} ({t}) | {e['value']:.3g} {unit} ({e['ms_per_step']:.3g} ms) | "
              f"{frac} | {'—' if ovh is None else f'{ovh:.1f} %'} | {cpu} |")


if __name__ == "__main__":
    main(sys.argv[1] if len(sys.argv) > 1 else "profiles/r1")
