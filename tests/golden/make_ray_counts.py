#!/usr/bin/env python3
"""Algorithmic operation counts and image checksums of the Ray config
(8192^2, 64 spheres, depth 4, seed 42) from the CPU oracle (oracle.c:orc_ray
instruments sphere tests, plane tests and shading evaluations).  bench.py
reads the committed numbers as the Ray roofline's algorithmic work (SURVEY
§8d: "instrumented flop count from the CPU oracle"); the config-size parity
test (tests/test_config_parity_gpu.py) compares the device image's FNV-1a
with `fnv1a64` bit for bit.  The GPU never runs the oracle.

Usage: python tests/golden/make_ray_counts.py
"""
import json
import os
import sys

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, os.path.dirname(os.path.dirname(HERE)))

from paper_1805_02755_b200 import workloads as W  # noqa: E402
from tests._oracle import Oracle  # noqa: E402


def main():
    o = Oracle()
    out = {}
    for w, h in ((8192, 8192), (1024, 1024)):
        scene = W.ray_scene(64, seed=42)
        img, (st, pt, sh) = o.ray(scene, 64, w, h, 4)
        out[f"{w}x{h}"] = {"sphere_tests": st, "plane_tests": pt, "shades": sh,
                           "flops": W.ray_flops(st, pt, sh),
                           "bounce_histogram": [int(x) for x in
                                                __import__("numpy").bincount(img[:, 3].astype(int), minlength=5)],
                           "rgb_sum": [float(x) for x in img[:, :3].astype("float64").sum(axis=0)],
                           "fnv1a64": hex(o.fnv1a64(img))}
    with open(os.path.join(HERE, "ray_counts.json"), "w") as f:
        json.dump(out, f, indent=1)
    print(json.dumps(out, indent=1))


if __name__ == "__main__":
    main()
