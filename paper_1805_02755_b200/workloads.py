"""Program builders and deterministic synthetic inputs for the benchmarks.

Program shapes follow the reference's tests/experiments for vecscale,
mandelbrot and synthetic (test_engine.cpp:16-48, experiments/*.json) and
PAPER.md Table 2 / Listings 1-2 for the paper's other benchmarks
(SURVEY.md §8d, Appendix B).  Inputs come from the reference's splitmix64
recipe (fill_default_inputs, workloads.hpp:261-283), vectorized.
"""
from __future__ import annotations

import math

import numpy as np

from .coexec import BufferDesc, OutPattern, ProgramSpec

_GOLDEN = np.uint64(0x9E3779B97F4A7C15)
_M1 = np.uint64(0xBF58476D1CE4E5B9)
_M2 = np.uint64(0x94D049BB133111EB)


def splitmix64(seed: int, start: int, n: int) -> np.ndarray:
    """Draws start+1 .. start+n of the splitmix64 stream seeded with `seed`."""
    with np.errstate(over="ignore"):
        i = np.arange(start + 1, start + n + 1, dtype=np.uint64)
        z = np.uint64(seed) + i * _GOLDEN
        z = (z ^ (z >> np.uint64(30))) * _M1
        z = (z ^ (z >> np.uint64(27))) * _M2
        return z ^ (z >> np.uint64(31))


def unit_doubles(seed: int, start: int, n: int) -> np.ndarray:
    """(z >> 11) * 2^-53 in [0,1) (workloads.hpp:272-274)."""
    return (splitmix64(seed, start, n) >> np.uint64(11)).astype(np.float64) * (2.0 ** -53)


def fill_default_inputs(spec: ProgramSpec, seed: int):
    """One generator state across all input buffers, in order; 8-byte
    elements are doubles in [0,1), anything else gets one byte per draw."""
    out, drawn = [], 0
    for b in spec.in_buffers:
        if b.element_size_bytes == 8:
            v = unit_doubles(seed, drawn, b.element_count)
            drawn += b.element_count
            out.append(np.ascontiguousarray(v).view(np.uint8))
        else:
            n = b.size_bytes()
            v = (splitmix64(seed, drawn, n) & np.uint64(0xFF)).astype(np.uint8)
            drawn += n
            out.append(v)
    return out


# ---- reference kernels ------------------------------------------------------

def vecscale_spec(gws: int, lws: int, a: float = 2.0, b: float = 1.0) -> ProgramSpec:
    return ProgramSpec(gws, lws, [BufferDesc("in", 8, gws)], [BufferDesc("out", 8, gws)], OutPattern(1, 1),
                       "vecscale", [float(a), float(b)])


def mandelbrot_spec(width: int, height: int, max_iter: int, lws: int = 256, viewport=(-2.5, -1.25, 1.0, 1.25),
                    kernel: str = "mandelbrot") -> ProgramSpec:
    return ProgramSpec(width * height, lws, [], [BufferDesc("counts", 4, width * height * 4)], OutPattern(4, 1),
                       kernel, [int(width), int(height), int(max_iter)] + [float(v) for v in viewport])


def synthetic_spec(gws: int, lws: int, profile: str = "constant", args=()) -> ProgramSpec:
    return ProgramSpec(gws, lws, [], [BufferDesc("out", 8, gws)], OutPattern(1, 1), "synthetic:" + profile,
                       list(args))


# ---- paper benchmarks -------------------------------

def gaussian_spec(width: int, height: int, filt: int = 31, lws: int = 128) -> ProgramSpec:
    return ProgramSpec(width * height, lws, [BufferDesc("image", 4, width * height), BufferDesc("filter", 4, filt * filt)],
                       [BufferDesc("blurred", 4, width * height)], OutPattern(1, 1), "gaussian",
                       [int(width), int(height), int(filt)])


def gaussian_filter(filt: int = 31, sigma: float = 5.0) -> np.ndarray:
    r = filt // 2
    i = np.arange(filt, dtype=np.float64) - r
    w = np.exp(-(i[:, None] ** 2 + i[None, :] ** 2) / (2.0 * sigma * sigma))
    return (w / w.sum()).astype(np.float32)


def gaussian_inputs(width: int, height: int, filt: int = 31, seed: int = 42):
    img = unit_doubles(seed, 0, width * height).astype(np.float32)
    return [img, gaussian_filter(filt).ravel()]


def nbody_spec(bodies: int, dt: float = 0.005, eps2: float = 500.0, lws: int = 64) -> ProgramSpec:
    return ProgramSpec(bodies, lws, [BufferDesc("pos", 16, bodies), BufferDesc("vel", 16, bodies)],
                       [BufferDesc("new_pos", 16, bodies), BufferDesc("new_vel", 16, bodies)], OutPattern(1, 1),
                       "nbody", [int(bodies), float(dt), float(eps2)])


def nbody_inputs(bodies: int, seed: int = 42):
    u = unit_doubles(seed, 0, 4 * bodies).reshape(bodies, 4)
    pos = np.empty((bodies, 4), np.float32)
    pos[:, :3] = (3.0 + 47.0 * u[:, :3]).astype(np.float32)
    pos[:, 3] = (1.0 + 999.0 * u[:, 3]).astype(np.float32)
    vel = np.zeros((bodies, 4), np.float32)
    return [pos, vel]


def binomial_spec(options: int, steps: int = 254) -> ProgramSpec:
    groups = options // 4
    lws = steps + 1
    return ProgramSpec(lws * groups, lws, [BufferDesc("rand", 16, groups)], [BufferDesc("call", 16, groups)],
                       OutPattern(1, lws), "binomial", [int(steps)])


def binomial_inputs(options: int, seed: int = 42):
    return [unit_doubles(seed, 0, options).astype(np.float32)]


def ray_spec(width: int, height: int, spheres: int = 64, max_depth: int = 4, lws: int = 128) -> ProgramSpec:
    return ProgramSpec(width * height, lws, [BufferDesc("scene", 16, 2 * spheres + 8)],
                       [BufferDesc("rgba", 16, width * height)], OutPattern(1, 1), "ray",
                       [int(width), int(height), int(spheres), int(max_depth)])


def ray_scene(spheres: int = 64, seed: int = 42) -> np.ndarray:
    """Seeded fixed scene (float4 records, layout in oracle.c:orc_ray):
    spheres resting above a checkered mirror-ish floor, every third sphere a
    mirror, three point lights."""
    u = unit_doubles(seed, 0, 8 * spheres).reshape(spheres, 8)
    s = np.zeros((2 * spheres + 8, 4), np.float64)
    r = 0.3 + 1.2 * u[:, 2]
    s[:spheres, 0] = -8.0 + 16.0 * u[:, 0]
    s[:spheres, 1] = r + 2.0 * u[:, 3]
    s[:spheres, 2] = 2.0 + 16.0 * u[:, 1]
    s[:spheres, 3] = r
    s[spheres:2 * spheres, 0:3] = 0.2 + 0.8 * u[:, 4:7]
    mirror = (np.arange(spheres) % 3) == 0
    s[spheres:2 * spheres, 3] = np.where(mirror, 0.6 + 0.3 * u[:, 7], 0.15 * u[:, 7])
    c = 2 * spheres
    s[c + 0] = (0.0, 2.5, -12.0, 0.6)        # camera (x, y, z, tan(fov/2))
    s[c + 1] = (-10.0, 12.0, -6.0, 0.7)      # lights (x, y, z, intensity)
    s[c + 2] = (8.0, 15.0, 0.0, 0.5)
    s[c + 3] = (0.0, 20.0, 10.0, 0.4)
    s[c + 4] = (0.9, 0.9, 0.9, 0.3)          # floor material (r, g, b, reflectivity)
    s[c + 5] = (0.08, 0.5, 0.0, 0.0)         # ambient, specular k
    s[c + 6] = (0.25, 0.35, 0.55, 0.0)       # sky
    return s.astype(np.float32)


# ---- algorithmic work ---------------------------------------

RAY_FLOPS_PER_SPHERE_TEST = 17  # oc (3), b (5), |oc|^2 - r^2 (7), disc (2); sqrt/roots excluded
RAY_FLOPS_PER_PLANE_TEST = 2
RAY_FLOPS_PER_SHADE = 30


def ray_flops(sphere_tests: int, plane_tests: int, shades: int) -> float:
    return float(RAY_FLOPS_PER_SPHERE_TEST * sphere_tests + RAY_FLOPS_PER_PLANE_TEST * plane_tests +
                 RAY_FLOPS_PER_SHADE * shades)

def mandelbrot_flops(counts: np.ndarray, max_iter: int) -> float:
    """8 FP ops per iteration + 3 for the final (failed) escape test."""
    inside = int(np.count_nonzero(counts >= max_iter))
    return 8.0 * float(counts.sum(dtype=np.uint64)) + 3.0 * (counts.size - inside)


def gaussian_flops(width: int, height: int, filt: int) -> float:
    return float(width * height) * (2 * filt * filt)


def nbody_flops(bodies: int, steps: int = 1) -> float:
    return 20.0 * float(bodies) * float(bodies) * steps


def binomial_flops(options: int, steps: int = 254) -> float:
    return 3.0 * (steps * (steps + 1) / 2) * options


def ceil_div(a: int, b: int) -> int:
    return -(-a // b)


__all__ = [n for n in dir() if not n.startswith("_") and n not in ("math", "np")]
