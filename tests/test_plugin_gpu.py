"""The device kernel plugin seam: user kernels compiled out of tree
(tests/plugins/plugins.cu, include/ecl_plugin.h ABI) registered at run time
and co-executed like the built-in kernels — the B200 form of the reference's
Engine::run(inputs, KernelFn, CostFn) (engine.hpp:223, workloads.hpp:44-47,
kernel_for at workloads.hpp:203) and of the paper's per-device binary kernels
(PAPER.md:395-421)."""
import os
import subprocess

import numpy as np
import pytest

import paper_1805_02755_b200 as P
from paper_1805_02755_b200 import workloads as W

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
PLUG = os.path.join(ROOT, "tests", "plugins")
BUILD = os.path.join(PLUG, "_build")


def image(kind="cubin"):
    path = os.path.join(BUILD, f"plugins.{kind}")
    if not os.path.exists(path):
        r = subprocess.run(["make", "-s", "-C", PLUG], capture_output=True, text=True, timeout=300)
        assert r.returncode == 0, r.stdout + r.stderr
    return path


def devices(n, **kw):
    ng = P.gpu_count()
    return [P.cuda_device(f"gpu{i}", ordinal=i % ng, **kw) for i in range(n)]


@pytest.fixture
def registered(gpu_available):
    ids = []

    def reg(kid, entry, kind="cubin"):
        P.register_kernel(kid, image(kind), entry)
        ids.append(kid)
        return kid

    yield reg
    for kid in ids:
        if P.is_registered_kernel(kid):
            P.unregister_kernel(kid)


def vecscale_program(kernel, gws=1 << 20, lws=128):
    spec = W.vecscale_spec(gws, lws, 2.5, -1.0)
    spec.kernel = kernel
    return spec


def test_registration_needs_a_gpu_and_rejects_bad_ids():
    # no GPU here: registering reports ConfigError instead of crashing; with a
    # GPU, built-in ids are refused (checked in the gpu tests below)
    if P.gpu_count() > 0:
        pytest.skip("covered by the gpu tests")
    with pytest.raises(P.Error) as ei:
        P.register_kernel("my_kernel", b"not an image", "entry")
    assert ei.value.code == P.ErrorCode.ConfigError
    assert not P.is_registered_kernel("my_kernel")


@pytest.mark.gpu
@pytest.mark.parametrize("kind", ["cubin", "fatbin", "ptx"])
@pytest.mark.parametrize("n_dev,sched", [(1, P.StaticConfig()), (2, P.DynamicConfig(37)), (3, P.HGuidedConfig())])
def test_plugin_program_co_executes_bit_exact(registered, oracle, kind, n_dev, sched):
    kid = registered(f"my_vecscale_{kind}", "vecscale_plugin", kind)
    spec = vecscale_program(kid)
    x = W.fill_default_inputs(spec, 7)[0]
    prog = P.validate_program(spec)
    with P.Engine(P.EngineConfig(devices(n_dev), sched, tally=True), prog) as e:
        res = e.run([x])
    assert P.tiles_exactly(res.trace.packages, prog.total_work_groups())
    assert np.array_equal(res.outputs[0].view(np.float64), oracle.vecscale(2.5, -1.0, x.view(np.float64)))


@pytest.mark.gpu
def test_run_with_kernel_overrides_the_program_kernel_for_one_run(registered, oracle):
    """Engine.run(inputs, kernel, cost): the built-in vecscale program runs the
    plugin for one run, then its own kernel again; inputs stay resident."""
    kid = registered("vs_override", "vecscale_plugin")
    spec = vecscale_program("vecscale")
    x = W.fill_default_inputs(spec, 3)[0]
    exp = oracle.vecscale(2.5, -1.0, x.view(np.float64))
    prog = P.validate_program(spec)
    with P.Engine(P.EngineConfig(devices(2), P.DynamicConfig(9)), prog) as e:
        a = e.run([x], kernel=kid, cost=lambda i: 1.0)
        assert np.array_equal(a.outputs[0].view(np.float64), exp)
        out = np.zeros(spec.global_work_size, np.float64)
        e.run_into(None, [out], kernel=kid)  # resident inputs, plugin again
        assert np.array_equal(out, exp)
        b = e.run([x])  # the program's own kernel
        assert np.array_equal(b.outputs[0].view(np.float64), exp)


@pytest.mark.gpu
def test_plugin_per_device_binary_kernel(registered, oracle):
    """Device(platform, device, kernel): device 1 runs a registered binary
    kernel while device 0 runs the program's built-in kernel."""
    kid = registered("vs_binary", "vecscale_plugin")
    spec = vecscale_program("vecscale", 1 << 18)
    x = W.fill_default_inputs(spec, 5)[0]
    devs = devices(2)
    devs[1].kernel = kid
    prog = P.validate_program(spec)
    with P.Engine(P.EngineConfig(devs, P.DynamicConfig(32), tally=True), prog) as e:
        res = e.run([x])
    assert {p.device_id for p in res.trace.packages} == {"gpu0", "gpu1"}
    assert np.array_equal(res.outputs[0].view(np.float64), oracle.vecscale(2.5, -1.0, x.view(np.float64)))


@pytest.mark.gpu
def test_plugin_sees_every_item_once(registered):
    kid = registered("whoami", "whoami_plugin")
    gws = 1 << 16
    spec = P.ProgramSpec(gws, 256, [], [P.BufferDesc("out", 8, gws)], P.OutPattern(1, 1), kid, [])
    prog = P.validate_program(spec)
    with P.Engine(P.EngineConfig(devices(3), P.HGuidedConfig(), tally=True), prog) as e:
        res = e.run([])
    v = res.outputs[0].view(np.uint64)
    assert np.array_equal(v >> np.uint64(8), np.arange(gws, dtype=np.uint64))
    assert set((v & np.uint64(0xFF)).tolist()) <= set(range(P.gpu_count()))


@pytest.mark.gpu
def test_indivisible_package_fails_the_run(registered):
    """test_engine.cpp:256-278: an out pattern 1:256 with 128-item packages
    passes validation and fails at run time with IndivisiblePackage."""
    kid = registered("group_sum", "group_sum_plugin")
    spec = P.ProgramSpec(1024, 128, [], [P.BufferDesc("out", 8, 4)], P.OutPattern(1, 256), kid, [])
    prog = P.validate_program(spec)
    with P.Engine(P.EngineConfig(devices(1), P.DynamicConfig(8)), prog) as e:
        with pytest.raises(P.EngineFailure) as ei:
            e.run([])
    assert ei.value.has(P.ErrorCode.IndivisiblePackage)
    # the same program with whole 256-item packages runs and sums correctly
    with P.Engine(P.EngineConfig(devices(2), P.DynamicConfig(4)), prog) as e:
        res = e.run([])
    got = res.outputs[0].view(np.float64)
    exp = np.arange(1024, dtype=np.float64).reshape(4, 256).sum(axis=1)
    assert np.array_equal(got, exp)


@pytest.mark.gpu
def test_register_errors(registered):
    with pytest.raises(P.Error) as ei:
        P.register_kernel("mandelbrot", image(), "vecscale_plugin")
    assert ei.value.code == P.ErrorCode.ConfigError
    with pytest.raises(P.Error) as ei:
        P.register_kernel("no_entry", image(), "not_there")
    assert ei.value.code == P.ErrorCode.UnknownKernel
    with pytest.raises(P.Error) as ei:
        P.register_kernel("garbage", b"\x7fELF garbage", "vecscale_plugin")
    assert ei.value.code == P.ErrorCode.UnknownKernel
    registered("twice", "vecscale_plugin")
    with pytest.raises(P.Error):
        P.register_kernel("twice", image(), "vecscale_plugin")
    # lws above one CTA
    kid = registered("wide", "vecscale_plugin")
    with pytest.raises(P.Error) as ei:
        P.Engine(P.EngineConfig(devices(1), P.StaticConfig()), P.validate_program(vecscale_program(kid, 4096, 2048)))
    assert ei.value.code == P.ErrorCode.BadKernelArgs


@pytest.mark.gpu
def test_kernel_outlives_unregister(registered, oracle):
    kid = registered("transient", "vecscale_plugin")
    spec = vecscale_program(kid, 1 << 14)
    x = W.fill_default_inputs(spec, 1)[0]
    with P.Engine(P.EngineConfig(devices(1), P.StaticConfig()), P.validate_program(spec)) as e:
        P.unregister_kernel(kid)
        assert not P.is_registered_kernel(kid)
        res = e.run([x])
    assert np.array_equal(res.outputs[0].view(np.float64), oracle.vecscale(2.5, -1.0, x.view(np.float64)))
