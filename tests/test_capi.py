"""The drop-in boundary: both native libraries load without a GPU and export
every function include/*.h declares; without a device, compute entry points
fail loudly (no CPU fallback)."""
import ctypes
import os
import re

import pytest

import paper_1805_02755_b200 as P
from paper_1805_02755_b200 import _native as N
from paper_1805_02755_b200 import workloads as W

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def declared(header):
    text = open(os.path.join(ROOT, "include", header)).read()
    text = re.sub(r"/\*.*?\*/", "", text, flags=re.S)
    return sorted(set(re.findall(r"\b(ecl_[a-z0-9_]+)\s*\(", text)) - {"ecl_done_fn"})


@pytest.mark.parametrize("header,lib", [("ecl_cuda.h", N.CUDA_LIB_PATH), ("ecl_engine.h", N.LIB_PATH)])
def test_every_declared_symbol_is_exported(header, lib):
    names = declared(header)
    assert len(names) > 10
    so = ctypes.CDLL(lib)
    missing = [n for n in names if not hasattr(so, n)]
    assert not missing, missing


def test_libraries_are_sm100a_builds():
    import subprocess
    out = subprocess.run(["cuobjdump", "--list-elf", N.CUDA_LIB_PATH], capture_output=True, text=True).stdout
    assert "sm_100a" in out


def test_status_codes_follow_error_order():
    # include/ecl_cuda.h: status = -(ErrorCode + 1), error.hpp order
    assert N.code_name(-1) == "NonDivisibleWorkSize"
    assert N.code_name(-9) == "KernelPanic"
    assert N.code_name(-21) == "IoError"


def test_no_cpu_fallback_without_device():
    if P.gpu_count() > 0:
        pytest.skip("a CUDA device is visible")
    prog = P.validate_program(W.mandelbrot_spec(64, 64, 16, lws=64))
    with pytest.raises(P.Error) as e:
        P.Engine(P.EngineConfig([P.cuda_device("gpu0")], P.HGuidedConfig()), prog)
    assert e.value.code == P.ErrorCode.ConfigError
    assert "CUDA" in str(e.value)


def test_native_pool_backend_is_rejected():
    import json
    cfg = {"program": W.synthetic_spec(100, 10).to_json(),
           "devices": [{"id": "p", "backend": {"kind": "native_pool", "worker_count": 2}}],
           "scheduler": {"type": "dynamic", "num_packages": 2}, "clock_mode": "wall"}
    h = ctypes.c_void_p()
    rc = N.lib.ecl_engine_create(json.dumps(cfg).encode(), ctypes.byref(h))
    assert N.code_name(rc) == "ConfigError" and "native_pool" in N.last_error()


def test_kernel_registry_validates_shapes():
    # workloads.hpp:154-199 semantics, checked by the device layer even without a GPU
    lib = ctypes.CDLL(N.CUDA_LIB_PATH)
    lib.ecl_kernel_create.restype = ctypes.c_int

    class Geom(ctypes.Structure):
        _fields_ = [("element_size_bytes", ctypes.c_uint64), ("element_count", ctypes.c_uint64)]

    class Arg(ctypes.Structure):
        _fields_ = [("is_double", ctypes.c_int32), ("reserved", ctypes.c_int32), ("i", ctypes.c_int64),
                    ("d", ctypes.c_double)]

    def create(kid, gws, lws, args, ins, outs, oi=1, wi=1):
        a = (Arg * max(1, len(args)))(*[Arg(int(isinstance(x, float)), 0, int(x) if isinstance(x, int) else 0,
                                              float(x)) for x in args])
        gi = (Geom * max(1, len(ins)))(*[Geom(*g) for g in ins])
        go = (Geom * max(1, len(outs)))(*[Geom(*g) for g in outs])
        k = ctypes.c_void_p()
        rc = lib.ecl_kernel_create(kid.encode(), ctypes.c_uint64(gws), ctypes.c_uint64(lws), a, len(args), gi,
                                   len(ins), go, len(outs), ctypes.c_uint64(oi), ctypes.c_uint64(wi), ctypes.byref(k))
        if rc == 0:
            lib.ecl_kernel_destroy(k)
        return rc

    assert create("vecscale", 128, 64, [2.0, 1.0], [(8, 128)], [(8, 128)]) == 0
    assert N.code_name(create("warp-drive", 128, 64, [], [], [(8, 128)])) == "UnknownKernel"
    assert N.code_name(create("synthetic:spiky", 128, 64, [], [], [(8, 128)])) == "UnknownProfile"
    assert N.code_name(create("vecscale", 128, 64, [2.0, 1.0], [], [(8, 128)])) == "BadKernelArgs"
    assert N.code_name(create("mandelbrot", 256, 64, [16, 16, 10], [], [(4, 1024)], 1, 1)) == "BadKernelArgs"
    assert create("mandelbrot", 256, 64, [16, 16, 10], [], [(4, 1024)], 4, 1) == 0
    assert N.code_name(create("mandelbrot", 256, 64, [16, 8, 10], [], [(4, 1024)], 4, 1)) == "BadKernelArgs"
    assert create("binomial", 255 * 8, 255, [254], [(16, 8)], [(16, 8)], 1, 255) == 0
    assert create("gaussian", 64 * 32, 128, [64, 32, 31], [(4, 64 * 32), (4, 31 * 31)], [(4, 64 * 32)]) == 0
    assert create("nbody", 1024, 64, [1024, 0.005, 500.0], [(16, 1024)] * 2, [(16, 1024)] * 2) == 0


def test_kernel_variant_ids():
    # per-device specialization ids "<kernel>@<n>", resolved
    # by the device layer without a GPU
    lib = ctypes.CDLL(N.CUDA_LIB_PATH)
    lib.ecl_kernel_create.restype = ctypes.c_int

    class Geom(ctypes.Structure):
        _fields_ = [("element_size_bytes", ctypes.c_uint64), ("element_count", ctypes.c_uint64)]

    class Arg(ctypes.Structure):
        _fields_ = [("is_double", ctypes.c_int32), ("reserved", ctypes.c_int32), ("i", ctypes.c_int64),
                    ("d", ctypes.c_double)]

    def create(kid):
        vals = [64, 64, 16, -2.5, -1.25, 1.0, 1.25]
        a = (Arg * 7)(*[Arg(int(isinstance(x, float)), 0, int(x) if isinstance(x, int) else 0, float(x))
                        for x in vals])
        go = (Geom * 1)(Geom(4, 64 * 64 * 4))
        k = ctypes.c_void_p()
        rc = lib.ecl_kernel_create(kid.encode(), ctypes.c_uint64(64 * 64), ctypes.c_uint64(256), a, 7, None, 0,
                                   go, 1, ctypes.c_uint64(4), ctypes.c_uint64(1), ctypes.byref(k))
        if rc == 0:
            lib.ecl_kernel_destroy(k)
        return rc

    for ok in ("mandelbrot", "mandelbrot@0", "mandelbrot@5", "mandelbrot@13", "mandelbrot@14", "mandelbrot@15"):
        assert create(ok) == 0, ok
    for bad in ("mandelbrot@16", "mandelbrot@", "mandelbrot@x", "mandelbrot@-1"):
        assert N.code_name(create(bad)) == "UnknownKernel", bad
