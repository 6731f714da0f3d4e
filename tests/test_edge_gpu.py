"""Edge cases of the kernels and the package machinery at the extremes of
their shapes (the reference tests its path on degenerate and ragged sizes,
SURVEY.md §4): single work-item / single work-group programs, images
smaller than a tile or a filter, one body, one option group, ragged
packages over several logical devices, the maximum Binomial depth."""
import numpy as np
import pytest

import paper_1805_02755_b200 as P
from paper_1805_02755_b200 import workloads as W
from tests._oracle import expand_4to1

pytestmark = pytest.mark.gpu


def run(spec, inputs=(), n_dev=1, sched=None, split=1 << 23):
    ng = P.gpu_count()
    devs = [P.cuda_device(f"gpu{i}", i % ng, copy_split_items=split) for i in range(n_dev)]
    prog = P.validate_program(spec)
    with P.Engine(P.EngineConfig(devs, sched or P.StaticConfig(), tally=True), prog) as e:
        res = e.run(list(inputs))
    assert P.tiles_exactly(res.trace.packages, prog.total_work_groups())
    return res


def rel_ok(got, exp, rtol, atol=0.0):
    got, exp = got.astype(np.float64), exp.astype(np.float64)
    return bool(np.all(np.abs(got - exp) <= rtol * np.abs(exp) + atol))


@pytest.mark.parametrize("w,h,lws", [(1, 1, 1), (3, 5, 1), (256, 1, 256), (1, 256, 16), (17, 13, 13)])
def test_mandelbrot_tiny_and_ragged(gpu_available, oracle, w, h, lws):
    for n_dev, sched in ((1, P.StaticConfig()), (3, P.DynamicConfig(7)), (2, P.HGuidedConfig())):
        res = run(W.mandelbrot_spec(w, h, 300, lws=lws), n_dev=n_dev, sched=sched)
        assert np.array_equal(res.outputs[0].view(np.uint32), expand_4to1(oracle.mandelbrot(w, h, 300)))


def test_mandelbrot_single_iteration_and_degenerate_viewport(gpu_available, oracle):
    # max_iter 1 (every pixel stops at once) and a zero-span viewport (all
    # pixels share one c: the origin, inside the set)
    res = run(W.mandelbrot_spec(64, 32, 1))
    assert np.array_equal(res.outputs[0].view(np.uint32), expand_4to1(oracle.mandelbrot(64, 32, 1)))
    vp = (0.0, 0.0, 0.0, 0.0)
    res = run(W.mandelbrot_spec(32, 8, 777, viewport=vp))
    got = res.outputs[0].view(np.uint32)
    assert np.array_equal(got, expand_4to1(oracle.mandelbrot(32, 8, 777, viewport=vp)))
    assert (got == 777).all()


def test_vecscale_single_item(gpu_available, oracle):
    x = np.array([0.3125], np.float64)
    res = run(W.vecscale_spec(1, 1, 3.0, -1.0), [x])
    assert np.array_equal(res.outputs[0].view(np.float64), oracle.vecscale(3.0, -1.0, x))


@pytest.mark.parametrize("w,h,f", [(1, 1, 31), (5, 3, 31), (31, 2, 31), (2, 40, 3), (1, 1, 1)])
def test_gaussian_smaller_than_filter_and_tile(gpu_available, oracle, w, h, f):
    import math
    img, filt = W.gaussian_inputs(w, h, f, seed=5)
    lws = math.gcd(w * h, 128)
    for split in (1 << 23, 1):  # whole inputs, and one-work-group streamed pieces
        res = run(W.gaussian_spec(w, h, f, lws=lws), [img, filt], split=split, sched=P.DynamicConfig(3))
        assert rel_ok(res.outputs[0].view(np.float32), oracle.gaussian(img, filt, w, h, f), 1e-5)


def test_nbody_one_and_two_bodies(gpu_available, oracle):
    for n in (1, 2):
        pos, vel = W.nbody_inputs(n, seed=3)
        res = run(W.nbody_spec(n, lws=1), [pos, vel])
        npos, nvel = oracle.nbody_step(pos, vel, 0.005, 500.0)
        assert rel_ok(res.outputs[0].view(np.float32).reshape(-1, 4), npos, 1e-4)
        assert rel_ok(res.outputs[1].view(np.float32).reshape(-1, 4), nvel, 1e-4, atol=1e-6)


@pytest.mark.parametrize("kernel", ["binomial", "binomial@1", "binomial@2", "binomial@3", "binomial@4", "binomial@5"])
@pytest.mark.parametrize("steps", [1, 2, 15, 16, 17, 31, 32, 33, 63, 64, 127, 128, 129, 255])
def test_binomial_depth_edges(gpu_available, oracle, steps, kernel):
    # phase boundaries of the lattices (multiples of 32 levels for the warp
    # kernels, 16 for the half-warp kernels), the 128-node limit of the
    # default kernel's half-warp window and the maximum depth; 4 options =
    # one work-group, one of them deep in the money (a window from node 0)
    rand = W.binomial_inputs(4, seed=steps)[0]
    rand[1] = 1e-6
    spec = W.binomial_spec(4, steps)
    spec.kernel = kernel
    res = run(spec, [rand])
    assert rel_ok(res.outputs[0].view(np.float32), oracle.binomial(rand, steps), 1e-5, atol=1e-6)


def test_ray_single_pixel_and_odd_sphere_count(gpu_available, oracle):
    for w, h, ns in ((1, 1, 64), (7, 3, 5), (33, 9, 1)):
        scene = W.ray_scene(ns, seed=ns)
        res = run(W.ray_spec(w, h, ns, 4, lws=1), [scene])
        exp, _ = oracle.ray(scene, ns, w, h, 4)
        assert np.array_equal(res.outputs[0].view(np.float32).reshape(-1, 4), exp)
