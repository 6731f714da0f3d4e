"""ctypes access to the CPU checkers (test infrastructure only).

Oracle     — oracle/_build/liboracle.so, this repo's C restatement
Reference  — oracle/_ref/libcoexec_ref.so, the reference headers compiled
             in place by oracle/Makefile (present where it was built)
"""
from __future__ import annotations

import ctypes
import json
import os
import subprocess

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
ORACLE_SO = os.path.join(ROOT, "oracle", "_build", "liboracle.so")
REF_SO = os.path.join(ROOT, "oracle", "_ref", "libcoexec_ref.so")

U64, U32, D, F, VP = ctypes.c_uint64, ctypes.c_uint32, ctypes.c_double, ctypes.c_float, ctypes.c_void_p


def _build_oracle():
    subprocess.run(["make", "-s", "-C", os.path.join(ROOT, "oracle"), "_build/liboracle.so"], check=True)


class Oracle:
    def __init__(self):
        if not os.path.exists(ORACLE_SO):
            _build_oracle()
        lib = ctypes.CDLL(ORACLE_SO)
        self.lib = lib
        lib.orc_fnv1a64.restype = U64
        lib.orc_fnv1a64.argtypes = [VP, U64, U64]
        for name in ("orc_mandelbrot_f64", "orc_mandelbrot_f32"):
            getattr(lib, name).argtypes = [U64, U64, U32, D, D, D, D, U64, U64, VP]
        lib.orc_mandel_count_f64.restype = U32
        lib.orc_mandel_count_f64.argtypes = [U64, U64, U64, U32, D, D, D, D]
        lib.orc_vecscale.argtypes = [D, D, VP, VP, U64, U64]
        lib.orc_synthetic.argtypes = [ctypes.c_int, D, ctypes.c_int, U64, VP, U64, U64]
        lib.orc_fill_f64.argtypes = [ctypes.POINTER(U64), U64, VP]
        lib.orc_gaussian.argtypes = [VP, VP, VP, U32, U32, U32, U64, U64]
        lib.orc_gaussian_filter.argtypes = [U32, D, VP]
        lib.orc_nbody_step.argtypes = [VP, VP, U64, F, F, VP, VP, U64, U64]
        lib.orc_nbody_init.argtypes = [U64, U64, VP, VP]
        lib.orc_binomial.argtypes = [VP, VP, U32, U64, U64]
        lib.orc_binomial_init.argtypes = [U64, U64, VP]
        lib.orc_ray_scene.argtypes = [U64, U32, VP]
        lib.orc_num_threads.restype = ctypes.c_int
        lib.orc_ray.argtypes = [VP, U32, U32, U32, U32, VP, U64, U64, VP]

    def ray(self, scene, spheres, w, h, max_depth=4, first=0, count=None):
        """Returns (rgba float32[w*h,4], (sphere_tests, plane_tests, shades))."""
        count = w * h - first if count is None else count
        out = np.zeros((w * h, 4), np.float32)
        cnt = np.zeros(3, np.uint64)
        self.lib.orc_ray(np.ascontiguousarray(scene).ctypes.data, spheres, w, h, max_depth, out.ctypes.data, first,
                         count, cnt.ctypes.data)
        return out, tuple(int(c) for c in cnt)

    def fnv1a64(self, a: np.ndarray) -> int:
        a = np.ascontiguousarray(a)
        return self.lib.orc_fnv1a64(a.ctypes.data, a.nbytes, 0)

    def mandelbrot(self, w, h, it, viewport=(-2.5, -1.25, 1.0, 1.25), first=0, count=None, f32=False):
        count = w * h - first if count is None else count
        out = np.zeros(count, np.uint32)
        fn = self.lib.orc_mandelbrot_f32 if f32 else self.lib.orc_mandelbrot_f64
        fn(w, h, it, *viewport, first, count, out.ctypes.data)
        return out

    def vecscale(self, a, b, x: np.ndarray) -> np.ndarray:
        out = np.zeros_like(x)
        self.lib.orc_vecscale(a, b, x.ctypes.data, out.ctypes.data, 0, x.size)
        return out

    def synthetic(self, profile: int, gws: int, param=None) -> np.ndarray:
        out = np.zeros(gws, np.float64)
        self.lib.orc_synthetic(profile, 0.0 if param is None else param, 0 if param is None else 1, gws,
                               out.ctypes.data, 0, gws)
        return out

    def fill_f64(self, seed: int, n: int) -> np.ndarray:
        st = U64(seed)
        out = np.zeros(n, np.float64)
        self.lib.orc_fill_f64(ctypes.byref(st), n, out.ctypes.data)
        return out

    def gaussian_filter(self, f=31, sigma=5.0):
        out = np.zeros(f * f, np.float32)
        self.lib.orc_gaussian_filter(f, sigma, out.ctypes.data)
        return out

    def gaussian(self, img, filt, w, h, f, first=0, count=None):
        count = w * h - first if count is None else count
        out = np.zeros(w * h, np.float32)
        self.lib.orc_gaussian(img.ctypes.data, filt.ctypes.data, out.ctypes.data, w, h, f, first, count)
        return out

    def nbody_init(self, seed, n):
        pos = np.zeros((n, 4), np.float32)
        vel = np.zeros((n, 4), np.float32)
        self.lib.orc_nbody_init(seed, n, pos.ctypes.data, vel.ctypes.data)
        return pos, vel

    def nbody_step(self, pos, vel, dt, eps2, first=0, count=None):
        n = pos.shape[0]
        count = n - first if count is None else count
        npos = np.zeros_like(pos)
        nvel = np.zeros_like(vel)
        self.lib.orc_nbody_step(pos.ctypes.data, vel.ctypes.data, n, dt, eps2, npos.ctypes.data, nvel.ctypes.data,
                                first, count)
        return npos, nvel

    def binomial(self, rand: np.ndarray, steps=254, first=0, count=None):
        count = rand.size - first if count is None else count
        out = np.zeros(rand.size, np.float32)
        self.lib.orc_binomial(rand.ctypes.data, out.ctypes.data, steps, first, count)
        return out

    def binomial_init(self, seed, n):
        out = np.zeros(n, np.float32)
        self.lib.orc_binomial_init(seed, n, out.ctypes.data)
        return out

    def ray_scene(self, seed, spheres):
        out = np.zeros((2 * spheres + 8, 4), np.float32)
        self.lib.orc_ray_scene(seed, spheres, out.ctypes.data)
        return out

    def threads(self) -> int:
        return self.lib.orc_num_threads()


class Reference:
    """The reference's own code, compiled in place (oracle/Makefile)."""

    @staticmethod
    def load():
        if not os.path.exists(REF_SO):
            return None
        return Reference()

    def __init__(self):
        lib = ctypes.CDLL(REF_SO)
        self.lib = lib
        lib.ref_last_error.restype = ctypes.c_char_p
        lib.ref_mandelbrot_counts.argtypes = [U64, U64, U32, D, D, D, D, U64, U64, VP]
        lib.ref_drain.restype = ctypes.c_int64
        lib.ref_drain.argtypes = [ctypes.c_char_p, ctypes.c_char_p, U64, ctypes.POINTER(U64), U64]
        lib.ref_run_json.restype = ctypes.c_int64
        lib.ref_run_json.argtypes = [ctypes.c_char_p, ctypes.c_char_p, U64, ctypes.POINTER(U64)]
        lib.ref_wall_run.restype = D
        lib.ref_wall_run.argtypes = [ctypes.c_char_p, U32, U32, U64, U64, ctypes.POINTER(U64)]

    def wall_run_restated(self, kind, inputs, out, sample, stride, params, devices, scheduler=None):
        """Reference engine (wall mode) driving oracle.c's restated kernel;
        scheduler: a schema-1 scheduler dict (None = Dynamic{max(64,16H)})."""
        f = self.lib.ref_wall_run_restated
        f.restype = D
        f.argtypes = [ctypes.c_char_p, VP, VP, VP, U64, U64, ctypes.POINTER(D), U32, ctypes.c_char_p]
        ins = [np.ascontiguousarray(a) for a in inputs] + [None, None]
        p = (D * len(params))(*params)
        s = f(kind.encode(), ins[0].ctypes.data if ins[0] is not None else None,
              ins[1].ctypes.data if ins[1] is not None else None, out.ctypes.data, sample, stride, p, devices,
              json.dumps(scheduler).encode() if scheduler else None)
        if s < 0:
            raise RuntimeError(self.lib.ref_last_error().decode())
        return s

    def mandelbrot(self, w, h, it, viewport=(-2.5, -1.25, 1.0, 1.25)):
        out = np.zeros(w * h, np.uint32)
        self.lib.ref_mandelbrot_counts(w, h, it, *viewport, 0, w * h, out.ctypes.data)
        return out

    def drain(self, sched: dict, devices: list, total_wg: int):
        cap = 3 * (total_wg + 16)
        buf = (U64 * cap)()
        n = self.lib.ref_drain(json.dumps(sched).encode(), json.dumps(devices).encode(), total_wg, buf, cap)
        if n < 0:
            raise RuntimeError(self.lib.ref_last_error().decode())
        return [(int(buf[3 * i]), int(buf[3 * i + 1]), int(buf[3 * i + 2])) for i in range(n)]

    def run_json(self, config: dict):
        fnv = U64(0)
        n = self.lib.ref_run_json(json.dumps(config).encode(), None, 0, ctypes.byref(fnv))
        if n < 0:
            raise RuntimeError(self.lib.ref_last_error().decode())
        buf = ctypes.create_string_buffer(n + 1)
        self.lib.ref_run_json(json.dumps(config).encode(), buf, n + 1, ctypes.byref(fnv))
        return json.loads(buf.value.decode()), fnv.value

    def wall_run_sched(self, program: dict, scheduler: dict, devices: int, workers: int, seed: int = 0):
        """Reference Engine::run in wall mode with any scheduler (schema-1 dict)."""
        f = self.lib.ref_wall_run_sched
        f.restype = D
        f.argtypes = [ctypes.c_char_p, ctypes.c_char_p, U32, U32, U64, ctypes.POINTER(U64)]
        fnv = U64(0)
        s = f(json.dumps(program).encode(), json.dumps(scheduler).encode(), devices, workers, seed, ctypes.byref(fnv))
        if s < 0:
            raise RuntimeError(self.lib.ref_last_error().decode())
        return s, fnv.value

    def wall_run(self, program: dict, devices: int, workers: int, packages: int, seed: int = 0):
        fnv = U64(0)
        s = self.lib.ref_wall_run(json.dumps(program).encode(), devices, workers, packages, seed, ctypes.byref(fnv))
        if s < 0:
            raise RuntimeError(self.lib.ref_last_error().decode())
        return s, fnv.value


def expand_4to1(counts: np.ndarray) -> np.ndarray:
    """The reference's 4:1 layout: each count written 4 times."""
    return np.repeat(counts.astype(np.uint32), 4)
