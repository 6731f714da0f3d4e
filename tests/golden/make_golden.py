#!/usr/bin/env python3
"""Regenerates the committed golden fixtures from the reference itself.

Runs where /root/reference exists (this container): oracle/Makefile compiles
the reference headers in place into oracle/_ref/libcoexec_ref.so, and this
script calls the reference's own schedulers (through the drain emulator of
test_schedulers.cpp:27-49) and its virtual-clock engine (engine.hpp:306-338)
to write:

  scheduler_drains.json   package sequences for a grid of (scheduler,
                          device powers/minimums, total work-groups)
  virtual_traces.json     reference traces (schema 1) of the
                          experiments/mandelbrot-{batel,remo}.json matrices,
                          statics resolved like load_experiment (config.hpp:192)
  mandelbrot_counts.json  FNV-1a/sum/inside of reference Mandelbrot counts

Usage: python tests/golden/make_golden.py
"""
import json
import os
import sys

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(os.path.dirname(HERE))
sys.path.insert(0, ROOT)

from tests._oracle import Oracle, Reference  # noqa: E402

REF = "/root/reference/proj"


def splitmix(seed):
    state = seed

    def nxt():
        nonlocal state
        state = (state + 0x9E3779B97F4A7C15) & (2 ** 64 - 1)
        z = state
        z = ((z ^ (z >> 30)) * 0xBF58476D1CE4E5B9) & (2 ** 64 - 1)
        z = ((z ^ (z >> 27)) * 0x94D049BB133111EB) & (2 ** 64 - 1)
        return z ^ (z >> 31)

    return nxt


def sim(id, power, min_wg=1):
    return {"id": id, "name": id, "computing_power": power, "launch_overhead_ms": 0.0,
            "bandwidth_bytes_per_ms": float(1 << 20), "backend": {"kind": "simulated"},
            "min_package_work_groups": min_wg}


def scheduler_grid():
    rng = splitmix(20261018)
    cases = []
    for trial in range(120):
        n = 1 + rng() % 8
        powers = [1.0 + (rng() >> 11) * 2.0 ** -53 * 9.0 for _ in range(n)]
        mins = [1 + rng() % 5 if rng() % 3 == 0 else 1 for _ in range(n)]
        total = n + rng() % 20000
        devices = [sim(f"d{i}", p, m) for i, (p, m) in enumerate(zip(powers, mins))]
        kind = trial % 4
        if kind == 0:
            sched = {"type": "static"}
        elif kind == 1:
            props = [1.0 + rng() % 7 for _ in range(n)]
            sched = {"type": "static", "proportions": props,
                     "device_order": [f"d{i}" for i in reversed(range(n))]}
        elif kind == 2:
            sched = {"type": "dynamic", "num_packages": n + rng() % 300}
        else:
            sched = {"type": "hguided", "k": 0.5 + (rng() >> 11) * 2.0 ** -53 * 4.0,
                     "include_device_count": bool(rng() % 4)}
        cases.append({"scheduler": sched, "devices": devices, "total_work_groups": total})
    # the paper-scale case: 8 equal B200s on the Mandelbrot config
    for mn in (1, 1184):
        cases.append({"scheduler": {"type": "hguided", "k": 2.0},
                      "devices": [sim(f"gpu{i}", 1.0, mn) for i in range(8)], "total_work_groups": 1048576})
    return cases


def main():
    ref = Reference.load()
    if ref is None:
        sys.exit("oracle/_ref not built (needs /root/reference): make -C oracle")
    drains = []
    for c in scheduler_grid():
        c = dict(c)
        c["packages"] = ref.drain(c["scheduler"], c["devices"], c["total_work_groups"])
        drains.append(c)
    with open(os.path.join(HERE, "scheduler_drains.json"), "w") as f:
        json.dump(drains, f, separators=(",", ":"))

    traces = {}
    for exp_name in ("mandelbrot-batel", "mandelbrot-remo"):
        exp = json.load(open(os.path.join(REF, "experiments", exp_name + ".json")))
        prof = json.load(open(os.path.join(REF, "experiments", exp["devices_file"])))
        for i, s in enumerate(exp["schedulers"]):
            cfg = {"program": exp["program"], "devices": prof["devices"], "scheduler": s,
                   "clock_mode": "virtual", "seed": exp["seed"]}
            trace, fnv = ref.run_json(cfg)
            traces[f"{exp_name}/s{i}"] = {"config": cfg, "trace": trace, "outputs_fnv": fnv}
    with open(os.path.join(HERE, "virtual_traces.json"), "w") as f:
        json.dump(traces, f, separators=(",", ":"))

    o = Oracle()
    counts = {}
    for w, it in ((64, 100), (256, 256), (512, 512), (1024, 2048)):
        c = ref.mandelbrot(w, w, it)
        counts[f"{w}x{w}x{it}"] = {"fnv1a64": o.fnv1a64(c), "sum": int(c.sum()), "inside": int((c >= it).sum())}
    with open(os.path.join(HERE, "mandelbrot_counts.json"), "w") as f:
        json.dump(counts, f, indent=1)
    print(f"{len(drains)} scheduler drains, {len(traces)} virtual traces, {len(counts)} mandelbrot checksums")


if __name__ == "__main__":
    main()
