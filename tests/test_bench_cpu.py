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


def test_reference_inputs_are_the_product_inputs_byte_for_byte(oracle):
    """The reference arm makes its inputs with oracle.c (OracleInputs); they
    must be the very bytes workloads.py gives the B200 arm."""
    synth = bench.OracleInputs(oracle, np)
    for name, cls in bench.WORKLOADS.items():
        ours = cls(P, W, np).host_inputs()
        theirs = cls(None, synth, np).host_inputs()
        assert len(ours) == len(theirs), name
        for a, b in zip(ours, theirs):
            assert np.ascontiguousarray(a).tobytes() == np.ascontiguousarray(b).tobytes(), name


@pytest.mark.parametrize("name", sorted(bench.WORKLOADS))
@pytest.mark.parametrize("n", [1, 2, 8])
def test_both_arms_print_the_same_config(oracle, name, n):
    cls = bench.WORKLOADS[name]
    ours = cls(P, W, np)
    sched = ours.scheduler(n)
    theirs = cls(None, bench.OracleInputs(oracle, np), np)
    assert ours.config(n, sched.to_json()) == theirs.config(n)
    assert bench.describe_doc(sched.to_json()) == P.describe(sched)


def test_describe_doc_matches_the_engine():
    for cfg in (P.StaticConfig(), P.DynamicConfig(12), P.HGuidedConfig(k=3.0), P.HGuidedConfig(adaptive=True)):
        assert bench.describe_doc(cfg.to_json()) == P.describe(cfg)


def test_reference_arm_loads_no_product_code(tmp_path):
    """--impl reference runs the reference (oracle/_ref) only: the product
    package is never imported and none of its libraries is mapped."""
    import json
    import subprocess
    import sys
    from tests._oracle import REF_SO
    if not os.path.exists(REF_SO):
        pytest.skip("oracle/_ref not built")
    code = ("import sys, json, bench\n"
            "rc = bench.main(['--impl', 'reference', '--workload', 'gaussian', '--steps', '1', '--warmup', '0'])\n"
            "maps = open('/proc/self/maps').read()\n"
            "print(json.dumps({'rc': rc, 'imported': [m for m in sys.modules if m.startswith('paper_1805')],\n"
            "                  'libs': [l for l in ('libcoexec.so', 'libecl_cuda.so') if l in maps]}))\n")
    r = subprocess.run([sys.executable, "-c", code], cwd=bench.ROOT, capture_output=True, text=True, timeout=600)
    assert r.returncode == 0, r.stderr
    lines = [json.loads(x) for x in r.stdout.splitlines() if x.startswith("{")]
    line, probe = lines[0], lines[-1]
    assert probe == {"rc": 0, "imported": [], "libs": []}
    assert line["impl"] == "reference" and line["value"] > 0
    assert line["config"]["work_items_per_step"] == 4096 * 4096


def test_binomial_zero_skip_ceiling_matches_a_brute_force_count():
    # the closed form steps(steps+1)/2 - t0(t0-1)/2 of nonzero node updates
    # against a direct count on the lattice of a few options
    wl = bench.WORKLOADS["binomial"](P, W, np)
    n = wl.STEPS
    rv = W.binomial_inputs(64, seed=3)[0].astype(np.float64)
    S, K, T = 5 * (1 - rv) + 30 * rv, 1 * (1 - rv) + 100 * rv, 0.25 * (1 - rv) + 10 * rv
    v = 0.30 * np.sqrt(T / n)
    t = np.arange(n + 1)
    for o in range(len(rv)):
        leaf = S[o] * np.exp(v[o] * (2 * t - n)) - K[o]
        nz = (leaf > 0).astype(int)
        count = 0
        for j in range(n, 0, -1):  # level j-1 computed from level j: nodes 0..j-1
            nz = np.maximum(nz[:-1], nz[1:])
            count += int(nz.sum())
        t0 = int((leaf <= 0).sum())
        assert count == n * (n + 1) // 2 - t0 * (t0 - 1) // 2
    c, why = wl.skip_ceiling()
    assert 1.33 < c < 3.0 and "nonzero" in why.lower()


def test_gaussian_roofline_is_hbm_with_both_flop_counts():
    wl = bench.WORKLOADS["gaussian"](P, W, np)
    ro = wl.roofline_override(0.1, 1, 70.0)
    px = wl.WIDTH * wl.HEIGHT
    assert ro["bound"] == "hbm" and ro["unit"] == "GB/s"
    assert ro["achieved"] == pytest.approx(8.0 * px / 1e-4 / 1e9)
    assert ro["frac"] == pytest.approx(ro["achieved"] / ro["peak"])
    assert ro["separable_fp32"]["flops_per_step"] == 4.0 * wl.F * px
    assert ro["direct_form"]["flops_per_step"] == wl.flops() == 2.0 * wl.F ** 2 * px
