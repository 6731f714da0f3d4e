#!/usr/bin/env python3
"""Regenerates tests/golden/experiments/ from the reference's own harness.

For each virtual-clock experiment file of the reference
(proj/experiments/{mandelbrot-batel,mandelbrot-remo,vecscale-batel}.json)
this copies the experiment and its device profile as fixtures and runs the
reference's run_experiment (experiment.hpp:67-181, compiled in place into
oracle/_ref by oracle/Makefile) to record what it writes: summary.json, the
per-scheduler median charts (*.svg) and the rep-0 traces.  Virtual-clock
repetitions are identical, so rep 0 stands for every repetition.

Runs only where /root/reference exists (this container).
Usage: python tests/golden/make_experiments.py
"""
import ctypes
import json
import os
import shutil
import sys
import tempfile

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(os.path.dirname(HERE))
REF = "/root/reference/proj"
REF_SO = os.path.join(ROOT, "oracle", "_ref", "libcoexec_ref.so")
NAMES = ["mandelbrot-batel", "mandelbrot-remo", "vecscale-batel"]


def main():
    lib = ctypes.CDLL(REF_SO)
    lib.ref_run_experiment.restype = ctypes.c_int
    lib.ref_run_experiment.argtypes = [ctypes.c_char_p, ctypes.c_char_p, ctypes.c_char_p, ctypes.c_uint64]
    for name in NAMES:
        dst = os.path.join(HERE, "experiments", name)
        shutil.rmtree(dst, ignore_errors=True)
        os.makedirs(dst)
        with open(os.path.join(REF, "experiments", name + ".json")) as f:
            cfg = json.load(f)
        prof = cfg["devices_file"]
        shutil.copyfile(os.path.normpath(os.path.join(REF, "experiments", prof)), os.path.join(dst, "profile.json"))
        cfg["devices_file"] = "profile.json"
        cfg["output_dir"] = "out"
        with open(os.path.join(dst, "experiment.json"), "w") as f:
            json.dump(cfg, f, indent=2)
            f.write("\n")
        with tempfile.TemporaryDirectory() as tmp:
            err = ctypes.create_string_buffer(1024)
            rc = lib.ref_run_experiment(os.path.join(dst, "experiment.json").encode(), tmp.encode(), err, 1024)
            if rc != 0:
                raise SystemExit(f"{name}: {err.value.decode()}")
            for fn in sorted(os.listdir(tmp)):
                if fn == "summary.json" or fn.endswith(".svg") or fn.endswith("-rep0.trace.json"):
                    shutil.copyfile(os.path.join(tmp, fn), os.path.join(dst, fn))
        print(name, sorted(os.listdir(dst)))


if __name__ == "__main__":
    sys.exit(main())
