"""GPU parity of the co-execution path against the CPU oracle.

Ports the reference's wall-mode checks (test_engine.cpp:210-297,
acceptance.cpp:112-168) to CUDA devices, and pins Mandelbrot against the
golden FNV-1a checksums of SURVEY.md §8c, up to the 16384^2 x 2048 config.
Several logical devices may share one physical GPU (each has its own
streams): that exercises co-execution on a one-GPU box.
"""
import numpy as np
import pytest

import paper_1805_02755_b200 as P
from paper_1805_02755_b200 import workloads as W
from tests._oracle import expand_4to1

pytestmark = pytest.mark.gpu

VIEW = (-2.5, -1.25, 1.0, 1.25)


def devices(n, depth=2, powers=(4.0, 2.0, 1.0, 1.0, 1.0, 1.0, 1.0, 1.0)):
    ng = P.gpu_count()
    return [P.cuda_device(f"gpu{i}", ordinal=i % ng, power=powers[i], queue_depth=depth) for i in range(n)]


def run_engine(spec, sched, n_dev=1, inputs=(), depth=2, tally=False):
    prog = P.validate_program(spec)
    with P.Engine(P.EngineConfig(devices(n_dev, depth), sched, tally=tally), prog) as e:
        res = e.run(list(inputs))
    return prog, res


def test_mandelbrot_native_equals_sequential(gpu_available, oracle):
    # test_engine.cpp:210-220: 64x32, 80 iterations, lws 32, Dynamic{8}, 2 devices
    prog, res = run_engine(W.mandelbrot_spec(64, 32, 80, lws=32), P.DynamicConfig(8), n_dev=2)
    got = res.outputs[0].view(np.uint32)
    assert np.array_equal(got, expand_4to1(oracle.mandelbrot(64, 32, 80)))
    assert P.tiles_exactly(res.trace.packages, prog.total_work_groups())


@pytest.mark.parametrize("n_dev", [1, 2, 3])
@pytest.mark.parametrize("sched", [P.StaticConfig(), P.DynamicConfig(50), P.HGuidedConfig()],
                         ids=["static", "dynamic50", "hguided"])
def test_acceptance_c1_mandelbrot(gpu_available, oracle, sched, n_dev):
    # acceptance.cpp:112-168 criterion 1 (mandelbrot 256^2 x 256), tally on
    prog, res = run_engine(W.mandelbrot_spec(256, 256, 256, lws=256), sched, n_dev=n_dev, tally=True)
    assert np.array_equal(res.outputs[0].view(np.uint32), expand_4to1(oracle.mandelbrot(256, 256, 256)))
    assert P.tiles_exactly(res.trace.packages, prog.total_work_groups())


@pytest.mark.parametrize("n_dev", [1, 2, 3])
@pytest.mark.parametrize("sched", [P.StaticConfig(), P.DynamicConfig(50), P.HGuidedConfig()],
                         ids=["static", "dynamic50", "hguided"])
def test_acceptance_c1_vecscale(gpu_available, oracle, sched, n_dev):
    spec = W.vecscale_spec(1 << 16, 128, 2.0, 1.0)
    inputs = W.fill_default_inputs(spec, 2024)
    prog, res = run_engine(spec, sched, n_dev=n_dev, inputs=inputs, tally=True)
    x = inputs[0].view(np.float64)
    assert np.array_equal(res.outputs[0].view(np.float64), oracle.vecscale(2.0, 1.0, x))
    assert P.tiles_exactly(res.trace.packages, prog.total_work_groups())


@pytest.mark.parametrize("w,it,fnv,total,inside", [
    (64, 100, 0xf2542a73f41ccde5, 88510, 731),
    (512, 512, 0x303b77894ff2aeaf, 24432502, 45427),
    (1024, 2048, 0xba7913ec187cbc5f, 375815484, 180918),
    (4096, 2048, 0xb928fb12dcaf9ffa, 6009619671, 2892623),
])
@pytest.mark.parametrize("kernel", ["mandelbrot", "mandelbrot@14"])
def test_mandelbrot_golden_checksums(gpu_available, oracle, w, it, fnv, total, inside, kernel):
    _, res = run_engine(W.mandelbrot_spec(w, w, it, kernel=kernel), P.HGuidedConfig(), n_dev=1)
    quad = res.outputs[0].view(np.uint32).reshape(-1, 4)
    assert (quad == quad[:, :1]).all(), "4:1 pattern: four identical counts per pixel"
    counts = np.ascontiguousarray(quad[:, 0])
    assert int(counts.sum(dtype=np.uint64)) == total
    assert int((counts >= it).sum()) == inside
    assert oracle.fnv1a64(counts) == fnv


@pytest.mark.parametrize("kernel", ["mandelbrot", "mandelbrot@14"])
def test_mandelbrot_config_checksum(gpu_available, oracle, kernel):
    """16384^2 x 2048, HGuided: the BASELINE config, bit-exact,
    also for the periodic-orbit early exit (mandelbrot@14)."""
    w, it = 16384, 2048
    spec = W.mandelbrot_spec(w, w, it, kernel=kernel)
    prog = P.validate_program(spec)
    with P.Engine(P.EngineConfig(devices(1), P.HGuidedConfig()), prog) as e:
        e.run_into([], None)  # device-resident
        out = np.empty(w * w * 4, np.uint32)
        e.gather([out])
    counts = np.ascontiguousarray(out.reshape(-1, 4)[:, 0])
    assert int(counts.sum(dtype=np.uint64)) == 96141151663
    assert int((counts >= it).sum()) == 46275993
    assert oracle.fnv1a64(counts) == 0xc19e9aef35d040ac


def test_mandelbrot_f32_config_checksum(gpu_available):
    """16384^2 x 2048 FP32 variant: the sum of counts of the FP32 restatement
    measured in SURVEY.md §8c (96,141,248,575)."""
    w, it = 16384, 2048
    prog = P.validate_program(W.mandelbrot_spec(w, w, it, kernel="mandelbrot_f32"))
    with P.Engine(P.EngineConfig(devices(1), P.HGuidedConfig()), prog) as e:
        e.run_into([], None)
        out = np.empty(w * w * 4, np.uint32)
        e.gather([out])
    counts = out.reshape(-1, 4)
    assert (counts == counts[:, :1]).all()
    assert int(counts[:, 0].sum(dtype=np.uint64)) == 96141248575


def test_mandelbrot_f32_bit_exact(gpu_available, oracle):
    _, res = run_engine(W.mandelbrot_spec(1024, 1024, 2048, kernel="mandelbrot_f32"), P.HGuidedConfig(), n_dev=2)
    got = res.outputs[0].view(np.uint32)
    assert np.array_equal(got, expand_4to1(oracle.mandelbrot(1024, 1024, 2048, f32=True)))


@pytest.mark.parametrize("profile,pid,args", [("constant", 0, ()), ("constant", 0, (3.5,)), ("ramp", 1, ()),
                                               ("step", 2, ()), ("step", 2, (7.0,))])
def test_synthetic_profiles(gpu_available, oracle, profile, pid, args):
    _, res = run_engine(W.synthetic_spec(1000, 10, profile, args), P.DynamicConfig(7), n_dev=2)
    exp = oracle.synthetic(pid, 1000, args[0] if args else None)
    assert np.array_equal(res.outputs[0].view(np.float64), exp)


def test_vecscale_odd_offsets(gpu_available, oracle):
    # packages starting on odd elements exercise the vector-peel path
    spec = W.vecscale_spec(999 * 3, 3, 1.5, -0.25)
    inputs = W.fill_default_inputs(spec, 7)
    _, res = run_engine(spec, P.DynamicConfig(97), n_dev=2, inputs=inputs)
    assert np.array_equal(res.outputs[0].view(np.float64), oracle.vecscale(1.5, -0.25, inputs[0].view(np.float64)))


def test_device_resident_then_gather(gpu_available, oracle):
    spec = W.mandelbrot_spec(512, 256, 300, lws=64)
    prog = P.validate_program(spec)
    with P.Engine(P.EngineConfig(devices(3), P.HGuidedConfig()), prog) as e:
        e.run_into([], None)
        out = np.zeros(512 * 256 * 4, np.uint32)
        e.gather([out])
    assert np.array_equal(out, expand_4to1(oracle.mandelbrot(512, 256, 300)))


def test_queue_depth_one_matches_two(gpu_available):
    spec = W.mandelbrot_spec(256, 256, 500)
    a = run_engine(spec, P.DynamicConfig(64), n_dev=2, depth=1)[1].outputs[0]
    b = run_engine(spec, P.DynamicConfig(64), n_dev=2, depth=4)[1].outputs[0]
    assert np.array_equal(a, b)


def test_native_run_matches_engine(gpu_available, oracle):
    spec = W.mandelbrot_spec(512, 512, 512)
    prog = P.validate_program(spec)
    with P.Engine(P.EngineConfig(devices(1), P.HGuidedConfig()), prog) as e:
        out = e.allocate_outputs()
        kms, tms = e.native_run([], out)
    assert kms > 0 and tms >= kms * 0.5
    assert np.array_equal(out[0].view(np.uint32), expand_4to1(oracle.mandelbrot(512, 512, 512)))


@pytest.mark.parametrize("depth,max_concurrent", [(1, 1), (2, 2), (4, 2)])
def test_per_device_package_concurrency(gpu_available, depth, max_concurrent):
    # test_engine.cpp:193-208: with queue depth 1 (reference semantics) a
    # device's packages never overlap; with depth >= 2 consecutive packages
    # alternate between the device's two compute lanes, so at most two
    # kernels of one device overlap (a drain tail with the next ramp).
    _, res = run_engine(W.mandelbrot_spec(256, 256, 1000), P.HGuidedConfig(), n_dev=3, depth=depth)
    by_dev = {}
    for p in res.trace.packages:
        by_dev.setdefault(p.device_id, []).append((p.t_start_ms, p.t_end_ms))
        assert p.t_enqueue_ms <= p.t_start_ms + 1e-3 and p.t_start_ms <= p.t_end_ms
    for iv in by_dev.values():
        events = sorted([(a, 1) for a, _ in iv] + [(b - 1e-3, -1) for _, b in iv])
        live = peak = 0
        for _, d in events:
            live += d
            peak = max(peak, live)
        assert peak <= max_concurrent


def test_indivisible_package_fails_mid_run(gpu_available):
    # test_engine.cpp:256-278: 1:256 pattern with 128-item packages
    spec = P.ProgramSpec(1024, 128, [], [P.BufferDesc("out", 8, 4)], P.OutPattern(1, 256), "synthetic:constant", [])
    prog = P.validate_program(spec)
    with pytest.raises(P.Error) as ei:
        # the kernel registry already refuses a non-1:1 synthetic program
        P.Engine(P.EngineConfig(devices(1), P.DynamicConfig(8)), prog)
    assert ei.value.code == P.ErrorCode.BadKernelArgs


def test_engine_rejects_bad_configs(gpu_available):
    prog = P.validate_program(W.synthetic_spec(100, 10))
    with pytest.raises(P.Error):
        P.Engine(P.EngineConfig([], P.DynamicConfig(2)), prog)
    with pytest.raises(P.Error):
        P.Engine(P.EngineConfig([P.simulated_device("s", 1.0)], P.DynamicConfig(2), P.ClockMode.Wall), prog)
    with pytest.raises(P.Error):
        P.Engine(P.EngineConfig([P.cuda_device("d"), P.cuda_device("d")], P.DynamicConfig(2)), prog)
    with pytest.raises(P.Error) as ei:
        P.Engine(P.EngineConfig([P.cuda_device("d", ordinal=999)], P.DynamicConfig(2)), prog)
    assert ei.value.code == P.ErrorCode.ConfigError


def test_engine_rejects_mismatched_inputs(gpu_available):
    prog = P.validate_program(W.vecscale_spec(128, 64))
    with P.Engine(P.EngineConfig(devices(1), P.DynamicConfig(2)), prog) as e:
        with pytest.raises(P.Error) as ei:
            e.run([])
        assert ei.value.code == P.ErrorCode.InputSizeMismatch
        with pytest.raises(P.Error):
            e.run([np.zeros(100, np.uint8)])


def test_repeated_runs_reuse_engine(gpu_available, oracle):
    spec = W.mandelbrot_spec(256, 128, 200, lws=128)
    prog = P.validate_program(spec)
    exp = expand_4to1(oracle.mandelbrot(256, 128, 200))
    with P.Engine(P.EngineConfig(devices(2), P.HGuidedConfig(adaptive=True)), prog) as e:
        for _ in range(5):
            r = e.run([])
            assert np.array_equal(r.outputs[0].view(np.uint32), exp)
            assert P.tiles_exactly(r.trace.packages, prog.total_work_groups())


_FAULT_SCRIPT = """
import paper_1805_02755_b200 as P
spec = P.ProgramSpec(1 << 16, 256, out_buffers=[P.BufferDesc("out", 8, 1 << 16)], kernel="fault", args=[40000])
prog = P.validate_program(spec)
devs = [P.cuda_device("gpu0", 0)]
try:
    with P.Engine(P.EngineConfig(devs, P.DynamicConfig(8)), prog) as e:
        e.run()
    print("NO-ERROR")
except P.EngineFailure as f:
    print("FAILURE", [x.code.name for x in f.errors])
except P.Error as x:
    print("ERROR", x.code.name)
"""


def test_device_fault_becomes_kernel_panic(gpu_available):
    # reference test_engine.cpp:236-254 (a throwing kernel -> KernelPanic):
    # a work-item traps on the device; the run must fail with KernelPanic
    # instead of hanging on the faulted context.  Subprocess: a device trap
    # poisons the CUDA context for the rest of its process.
    import os
    import subprocess
    import sys
    env = dict(os.environ, ECL_FAULT_INJECTION="1")
    r = subprocess.run([sys.executable, "-c", _FAULT_SCRIPT], env=env, capture_output=True, text=True, timeout=120)
    out = r.stdout + r.stderr
    assert "FAILURE" in r.stdout or "ERROR" in r.stdout, out
    assert "KernelPanic" in r.stdout, out


def test_fault_kernel_is_not_registered_by_default(gpu_available):
    spec = P.ProgramSpec(1 << 10, 256, out_buffers=[P.BufferDesc("out", 8, 1 << 10)], kernel="fault", args=[1])
    with pytest.raises(P.Error) as e:
        with P.Engine(P.EngineConfig([P.cuda_device("gpu0", 0)], P.StaticConfig()), P.validate_program(spec)) as eng:
            eng.run()
    assert e.value.code == P.ErrorCode.UnknownKernel


@pytest.mark.parametrize("variants", [("mandelbrot", "mandelbrot@5"), ("mandelbrot@3", "mandelbrot@6")])
def test_per_device_kernel_specialization_is_bit_exact(gpu_available, oracle, variants):
    # SURVEY §8f row 4 / PAPER.md:395-421: each device runs its own variant of
    # the program's kernel; the co-executed image is still the reference's
    w, h, it = 512, 384, 512
    ng = P.gpu_count()
    devs = [P.cuda_device(f"gpu{i}", i % ng, kernel=k) for i, k in enumerate(variants)]
    prog = P.validate_program(W.mandelbrot_spec(w, h, it))
    with P.Engine(P.EngineConfig(devs, P.HGuidedConfig()), prog) as e:
        res = e.run()
    assert P.tiles_exactly(res.trace.packages, prog.total_work_groups())
    assert len({p.device_id for p in res.trace.packages}) == 2
    assert np.array_equal(res.outputs[0].view(np.uint32), expand_4to1(oracle.mandelbrot(w, h, it)))
    assert res.trace.raw["devices"][1]["kernel"] == variants[1]


def test_specialization_must_be_a_variant_of_the_program_kernel(gpu_available):
    devs = [P.cuda_device("gpu0", 0), P.cuda_device("gpu1", 0, kernel="vecscale")]
    prog = P.validate_program(W.mandelbrot_spec(64, 64, 16))
    with pytest.raises(P.Error) as e:
        P.Engine(P.EngineConfig(devs, P.StaticConfig()), prog).close()
    assert e.value.code == P.ErrorCode.ConfigError


@pytest.mark.parametrize("kernel", [f"mandelbrot@{v}" for v in range(16)] + ["mandelbrot_f32@0", "mandelbrot_f32@1", "mandelbrot_f32@2"])
def test_every_mandelbrot_variant_is_bit_exact(gpu_available, oracle, kernel):
    # tuning variants selectable per device must all reproduce the reference
    w, h, it = 640, 480, 1000
    spec = W.mandelbrot_spec(w, h, it)
    spec.kernel = kernel
    _, res = run_engine(spec, P.HGuidedConfig(), n_dev=2)
    exp = oracle.mandelbrot(w, h, it, f32=kernel.startswith("mandelbrot_f32"))
    assert np.array_equal(res.outputs[0].view(np.uint32), expand_4to1(exp))


_RING_SCRIPT = """
import sys, numpy as np
import paper_1805_02755_b200 as P
from paper_1805_02755_b200 import workloads as W
prog = P.validate_program(W.mandelbrot_spec(512, 256, 300))
devs = [P.cuda_device(f"gpu{i}", 0, copy_split_items=8192) for i in range(2)]
with P.Engine(P.EngineConfig(devs, P.DynamicConfig(9)), prog) as e:
    for _ in range(2):
        out = e.run([]).outputs[0]
np.save(sys.argv[1], out.view(np.uint32))
"""


@pytest.mark.parametrize("slots", ["1", "2", "5"])
def test_staging_ring_wraps_and_matches_oracle(gpu_available, oracle, tmp_path, slots):
    # The compact copies land in a ring of page-locked slots that the widen
    # workers release (device.cu ring_setup); with 1 KiB-item slots a 512x256
    # image cycles a 1-, 2- or 5-slot ring dozens of times per run, across
    # two logical devices with their own rings and two runs.
    import os
    import subprocess
    import sys
    f = tmp_path / "out.npy"
    env = dict(os.environ, ECL_WIDEN_RING_SLOTS=slots, ECL_WIDEN_RING_SLOT_KB="4")
    r = subprocess.run([sys.executable, "-c", _RING_SCRIPT, str(f)], env=env, capture_output=True, text=True,
                       timeout=300)
    assert r.returncode == 0, r.stderr
    assert np.array_equal(np.load(f), expand_4to1(oracle.mandelbrot(512, 256, 300)))


@pytest.mark.parametrize("kernel", ["mandelbrot", "mandelbrot@14"])
def test_mandelbrot_random_viewports(gpu_available, oracle, kernel):
    # seeded random windows: zooms into the cardioid, the period-2 bulb, the
    # boundary and the exterior, odd sizes and iteration limits (1..3000),
    # against the oracle's FP64 restatement (SURVEY §8c op order)
    rng = np.random.default_rng(2024)
    for _ in range(12):
        w, h = int(rng.integers(16, 220)), int(rng.integers(8, 160))
        it = int(rng.choice([1, 2, 31, 32, 33, 100, 777, 2048, 3000]))
        centers = [(-0.1, 0.0), (-1.0, 0.0), (-0.75, 0.1), (0.3, 0.5), (-1.8, 0.0), (0.26, 0.0)]
        cx, cy = centers[int(rng.integers(len(centers)))]
        span = float(10.0 ** rng.uniform(-6, 0.5))
        vp = (cx - span, cy - span * h / w, cx + span, cy + span * h / w)
        spec = W.mandelbrot_spec(w, h, it, viewport=vp, lws=1, kernel=kernel)
        _, res = run_engine(spec, P.HGuidedConfig(), n_dev=2)
        exp = oracle.mandelbrot(w, h, it, viewport=vp)
        assert np.array_equal(res.outputs[0].view(np.uint32), expand_4to1(exp)), (w, h, it, vp)


@pytest.mark.parametrize("center", [(0.25, 0.0), (-0.75, 0.0), (-1.25, 0.0)])
def test_periodic_exit_near_parabolic_points(gpu_available, oracle, center):
    # orbits near the cusp (c = 1/4) and the bulb junctions converge
    # slowly and may become periodic only after tens of thousands of
    # iterations or never: the early exit must still give the reference
    # counts at a 50000-iteration limit
    cx, cy = center
    w = h = 64
    span = 1e-3
    vp = (cx - span, cy - span, cx + span, cy + span)
    spec = W.mandelbrot_spec(w, h, 50000, viewport=vp, lws=64, kernel="mandelbrot@14")
    _, res = run_engine(spec, P.DynamicConfig(5), n_dev=1)
    assert np.array_equal(res.outputs[0].view(np.uint32), expand_4to1(oracle.mandelbrot(w, h, 50000, viewport=vp)))


def test_adaptive_hguided_learns_and_carries_powers(gpu_available, oracle):
    """Measured-throughput HGuided: a run measures every device's
    work-items/ms over non-overlapping busy time; the next run starts from
    those rates.  Device 0 runs the periodic-orbit variant (mandelbrot@14,
    same counts, fewer iterations) so the two logical devices differ.  The
    viewport lies inside the main cardioid, so every pixel costs the same
    (max_iter iterations, or an early periodic exit): the measured rates do
    not depend on which rows a device happened to draw."""
    w, it = 1024, 2048
    vp = (-0.5, -0.3, 0.1, 0.3)
    spec = W.mandelbrot_spec(w, w, it, viewport=vp)
    prog = P.validate_program(spec)
    devs = devices(2)
    devs[0].kernel = "mandelbrot@14"
    exp = expand_4to1(oracle.mandelbrot(w, w, it, viewport=vp))
    assert (exp == it).all()  # all interior
    with P.Engine(P.EngineConfig(devs, P.HGuidedConfig(adaptive=True)), prog) as e:
        assert e.learned_powers() == []
        first = e.run([])
        lp = e.learned_powers()
        assert len(lp) == 2 and all(p > 1e3 for p in lp), lp  # work-items/ms, not the unit seeds
        second = e.run([])
        lp2 = e.learned_powers()
    print("learned powers", lp, lp2)
    for r in (first, second):
        assert np.array_equal(r.outputs[0].view(np.uint32), exp)
        assert P.tiles_exactly(r.trace.packages, prog.total_work_groups())
    assert lp2[0] > lp2[1]  # the variant that skips periodic orbits is faster


@pytest.mark.parametrize("kernel", ["mandelbrot", "mandelbrot_f32"])
@pytest.mark.parametrize("max_iter", [65535, 65536, 70001])
def test_compact_count_width_at_16_bit_boundary(gpu_available, oracle, max_iter, kernel):
    # Host-bound counts cross PCIe as uint16 when max_iter < 65536 (every
    # count fits) and as uint32 otherwise; interior pixels of this window
    # reach max_iter itself, so a truncated count would show.
    vp = (-0.9, -0.2, 0.5, 0.6)  # the main cardioid and its boundary: counts from 5 to max_iter
    w, h = 48, 32
    prog = P.validate_program(W.mandelbrot_spec(w, h, max_iter, lws=32, viewport=vp, kernel=kernel))
    devs = [P.cuda_device(f"gpu{i}", 0, copy_split_items=256) for i in range(2)]
    with P.Engine(P.EngineConfig(devs, P.DynamicConfig(5)), prog) as e:
        got = e.run([]).outputs[0].view(np.uint32)
    exp = oracle.mandelbrot(w, h, max_iter, viewport=vp, f32=kernel == "mandelbrot_f32")
    assert int(exp.max()) == max_iter
    assert np.array_equal(got, expand_4to1(exp))
