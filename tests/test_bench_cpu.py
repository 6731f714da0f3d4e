"""bench.py's host-side logic that runs without a GPU: the workload table
(metric, units, ceilings), and where multi-rank runs put their shared
output buffer."""
import argparse
import os
from types import SimpleNamespace

import numpy as np
import pytest

import bench
import paper_1805_02755_b200 as P
from paper_1805_02755_b200 import workloads as W


def test_workloads_have_units_flops_and_ceilings():
    for name, cls in bench.WORKLOADS.items():
        wl = cls(P, W, np)
        assert wl.units() > 0 and wl.flops() > 0, name
        c = getattr(wl, "ceiling", None)
        assert c is not None and 0.0 < c[0] <= 1.5 and c[1], name
        assert wl.min_package(1) >= 1 and wl.min_package(8) >= wl.min_package(1), name


def test_binomial_ceiling_counts_the_lattice_slots():
    # 3 counted flops per node in one FMA lane-op; the phases of 32 levels
    # (binomial.cu) execute 1143 packed FMAs per lane for a 254-step pair
    slots, j = 0, 254
    for nl in range(8, 0, -1):
        stop = 32 * (nl - 1) - 1 if nl > 1 else 0
        if j > stop:
            slots += (j - stop) * nl
            j = stop
    assert slots == 1143
    live = 2 * sum(range(1, 255))
    assert bench.WORKLOADS["binomial"].ceiling[0] == pytest.approx(1.5 * live / (slots * 64))


@pytest.mark.parametrize("shm_free,expect", [(1 << 40, "/dev/shm"), (64 << 20, "/tmp")])
def test_shared_output_dir_falls_back_when_dev_shm_is_small(monkeypatch, shm_free, expect):
    real = os.statvfs

    def fake(path):
        if path == "/dev/shm":
            return SimpleNamespace(f_bavail=shm_free // 4096, f_frsize=4096)
        if path == "/tmp":
            return SimpleNamespace(f_bavail=(1 << 40) // 4096, f_frsize=4096)
        return real(path)

    monkeypatch.setattr(os, "statvfs", fake)
    monkeypatch.setattr(os.path, "isdir", lambda d: d in ("/dev/shm", "/tmp"))
    monkeypatch.delenv("TMPDIR", raising=False)
    assert bench.shared_out_dir(argparse.Namespace(workload="mandelbrot")) == expect
