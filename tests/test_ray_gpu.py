"""Ray tracer parity: the device renders the oracle's pixels bit for bit
(IEEE-rounded ops in the same order on both sides)."""
import numpy as np
import pytest

import paper_1805_02755_b200 as P
from paper_1805_02755_b200 import workloads as W

pytestmark = pytest.mark.gpu


def devices(n):
    ng = P.gpu_count()
    return [P.cuda_device(f"gpu{i}", ordinal=i % ng) for i in range(n)]


@pytest.mark.parametrize("w,h,ns,depth,n_dev,sched", [
    (256, 192, 64, 4, 1, P.StaticConfig()),
    (320, 200, 64, 4, 3, P.HGuidedConfig()),
    (128, 96, 17, 2, 2, P.DynamicConfig(23)),
    (160, 120, 64, 0, 1, P.StaticConfig()),
    # more than one 32-pair candidate-scan chunk: a full chunk + a 16-pair
    # group + an odd sphere; three chunks + 4 single pairs; the maximum
    (96, 64, 97, 3, 1, P.StaticConfig()),
    (96, 64, 200, 2, 2, P.HGuidedConfig()),
    (64, 48, 256, 4, 1, P.DynamicConfig(5)),
])
def test_ray_bit_exact(gpu_available, oracle, w, h, ns, depth, n_dev, sched):
    scene = W.ray_scene(ns, seed=42)
    prog = P.validate_program(W.ray_spec(w, h, ns, depth, lws=64))
    with P.Engine(P.EngineConfig(devices(n_dev), sched, tally=True), prog) as e:
        res = e.run([scene])
    got = res.outputs[0].view(np.float32).reshape(-1, 4)
    exp, _ = oracle.ray(scene, ns, w, h, depth)
    assert P.tiles_exactly(res.trace.packages, prog.total_work_groups())
    mism = np.flatnonzero(np.any(got != exp, axis=1))
    assert mism.size == 0, f"{mism.size} pixels differ, first {mism[:5]}: {got[mism[:2]]} vs {exp[mism[:2]]}"


def test_ray_irregular_depths(oracle):
    # the scene exercises every bounce count 0..4 (divergence the kernel must absorb)
    scene = W.ray_scene(64)
    out, counts = oracle.ray(scene, 64, 192, 144, 4)
    depths = np.bincount(out[:, 3].astype(int), minlength=5)
    assert (depths > 0).all()
    assert counts[0] > 0 and counts[2] > 0


@pytest.mark.parametrize("kernel", ["ray@0", "ray@1", "ray@2"])
def test_ray_variants_bit_exact(gpu_available, oracle, kernel):
    w, h, ns = 96, 64, 17
    scene = W.ray_scene(ns, seed=4)
    spec = W.ray_spec(w, h, ns, 4, lws=64)
    spec.kernel = kernel
    prog = P.validate_program(spec)
    with P.Engine(P.EngineConfig([P.cuda_device("gpu0", 0)], P.HGuidedConfig()), prog) as e:
        res = e.run([scene])
    exp, _ = oracle.ray(scene, ns, w, h, 4)
    assert np.array_equal(res.outputs[0].view(np.float32).reshape(-1, 4), exp)


@pytest.mark.parametrize("w,h,n_dev,sched", [
    (1600, 1400, 1, P.StaticConfig()),        # 2.24M pixels: three 2^20-pixel two-lane pieces
    (2048, 1536, 2, P.HGuidedConfig()),       # pieces inside co-executed packages
])
def test_ray_resident_two_lane_pieces(gpu_available, oracle, w, h, n_dev, sched):
    """Device-resident runs cut Ray's packages into 2^20-pixel launches that
    alternate over the device's two compute lanes (compute_split_items);
    the gathered image is still the oracle's, bit for bit."""
    ns, depth = 64, 4
    scene = W.ray_scene(ns, seed=9)
    prog = P.validate_program(W.ray_spec(w, h, ns, depth))
    out = np.empty((w * h, 4), np.float32)
    with P.Engine(P.EngineConfig(devices(n_dev), sched), prog) as e:
        e.kernel_timing(reset=True)
        t = e.run_into([scene], None)
        _, launches = e.kernel_timing(reset=True)
        e.gather([out])
    assert P.tiles_exactly(t.packages, prog.total_work_groups())
    # every piece is counted as a launch: at least one per 2^20 pixels
    assert launches >= max(len(t.packages), -(-w * h // (1 << 20)))
    exp, _ = oracle.ray(scene, ns, w, h, depth)
    assert np.array_equal(out.view(np.uint32), exp.view(np.uint32))
