"""The device layer used directly as the reference's executor seam
(include/ecl_cuda.h): open a B200, bind a kernel, move
raw bytes, launch packages by work-item range and wait on their events —
the calls a coexec maintainer substitutes for NativePool::execute_package
(engine.hpp:120-136).  Checked against the oracle."""
import ctypes

import numpy as np
import pytest

from paper_1805_02755_b200 import _native as N

pytestmark = pytest.mark.gpu

c_int, c_u32, c_u64, c_vp, c_sz = ctypes.c_int, ctypes.c_uint32, ctypes.c_uint64, ctypes.c_void_p, ctypes.c_size_t


class Arg(ctypes.Structure):
    _fields_ = [("is_double", ctypes.c_int32), ("reserved", ctypes.c_int32), ("i", ctypes.c_int64),
                ("d", ctypes.c_double)]


class Geom(ctypes.Structure):
    _fields_ = [("element_size_bytes", c_u64), ("element_count", c_u64)]


@pytest.fixture(scope="module")
def lib():
    so = ctypes.CDLL(N.CUDA_LIB_PATH)
    sig = {
        "ecl_gpu_open": (c_int, [c_int, c_u32, ctypes.POINTER(c_vp)]),
        "ecl_gpu_close": (c_int, [c_vp]),
        "ecl_kernel_create": (c_int, [ctypes.c_char_p, c_u64, c_u64, ctypes.POINTER(Arg), c_u32, ctypes.POINTER(Geom),
                                      c_u32, ctypes.POINTER(Geom), c_u32, c_u64, c_u64, ctypes.POINTER(c_vp)]),
        "ecl_kernel_destroy": (None, [c_vp]),
        "ecl_gpu_bind": (c_int, [c_vp, c_vp]),
        "ecl_gpu_buffer": (c_int, [c_vp, c_int, c_u32, ctypes.POINTER(c_vp)]),
        "ecl_gpu_alloc": (c_int, [c_vp, c_sz, ctypes.POINTER(c_vp)]),
        "ecl_gpu_free": (c_int, [c_vp, c_vp]),
        "ecl_gpu_upload": (c_int, [c_vp, c_vp, c_vp, c_sz]),
        "ecl_gpu_download": (c_int, [c_vp, c_vp, c_vp, c_sz]),
        "ecl_gpu_launch": (c_int, [c_vp, c_vp, c_u64, c_u64, c_u64, c_vp, c_vp]),
        "ecl_gpu_wait": (c_int, [c_vp, c_u64]),
        "ecl_gpu_sync": (c_int, [c_vp]),
    }
    for name, (res, args) in sig.items():
        f = getattr(so, name)
        f.restype, f.argtypes = res, args
    return so


def test_raw_executor_vecscale(gpu_available, lib, oracle):
    g = c_vp()
    assert lib.ecl_gpu_open(0, 2, ctypes.byref(g)) == 0
    try:
        # raw device memory round trip
        d = c_vp()
        assert lib.ecl_gpu_alloc(g, 4096, ctypes.byref(d)) == 0
        src = np.arange(1024, dtype=np.uint32)
        dst = np.zeros_like(src)
        assert lib.ecl_gpu_upload(g, d, src.ctypes.data, src.nbytes) == 0
        assert lib.ecl_gpu_download(g, dst.ctypes.data, d, dst.nbytes) == 0
        assert np.array_equal(src, dst)
        assert lib.ecl_gpu_free(g, d) == 0

        # vecscale: the bound input replica is filled with raw bytes, packages
        # launched by work-item range in a scrambled order
        n, lws = 1 << 14, 128
        args = (Arg * 2)(Arg(1, 0, 0, 2.5), Arg(1, 0, 0, -1.0))
        geom = (Geom * 1)(Geom(8, n))
        k = c_vp()
        assert lib.ecl_kernel_create(b"vecscale", n, lws, args, 2, geom, 1, geom, 1, 1, 1, ctypes.byref(k)) == 0
        assert lib.ecl_gpu_bind(g, k) == 0
        din, dout = c_vp(), c_vp()
        assert lib.ecl_gpu_buffer(g, 0, 0, ctypes.byref(din)) == 0
        assert lib.ecl_gpu_buffer(g, 1, 0, ctypes.byref(dout)) == 0
        x = np.linspace(-3, 3, n)
        assert lib.ecl_gpu_upload(g, din, x.ctypes.data, x.nbytes) == 0
        ranges = [(8192, 4096), (0, 1024), (12288, 4096), (1024, 7168)]
        for seq, (first, count) in enumerate(ranges):
            assert lib.ecl_gpu_launch(g, k, first, count, seq, None, None) == 0
        for seq in range(len(ranges)):
            assert lib.ecl_gpu_wait(g, seq) == 0
        y = np.zeros(n)
        assert lib.ecl_gpu_download(g, y.ctypes.data, dout, y.nbytes) == 0
        assert np.array_equal(y, oracle.vecscale(2.5, -1.0, x))
        # a range that is not whole work-groups is refused before any launch
        assert N.code_name(lib.ecl_gpu_launch(g, k, 100, 128, 99, None, None)) == "IndivisiblePackage"
        lib.ecl_kernel_destroy(k)
    finally:
        lib.ecl_gpu_close(g)


def test_native_run_split_covers_the_grid(gpu_available, lib, oracle):
    # the best-native denominator (ecl_gpu_native_run_split): the same grid
    # as plain sub-launches over the two compute lanes, any piece size
    so = lib
    so.ecl_gpu_native_run_split.restype = c_int
    so.ecl_gpu_native_run_split.argtypes = [c_vp, c_u64, ctypes.POINTER(ctypes.c_float)]
    g = c_vp()
    assert so.ecl_gpu_open(0, 2, ctypes.byref(g)) == 0
    try:
        n, lws = 3 * 4096 + 128, 128
        args = (Arg * 2)(Arg(1, 0, 0, -0.5), Arg(1, 0, 0, 3.0))
        geom = (Geom * 1)(Geom(8, n))
        k = c_vp()
        assert so.ecl_kernel_create(b"vecscale", n, lws, args, 2, geom, 1, geom, 1, 1, 1, ctypes.byref(k)) == 0
        assert so.ecl_gpu_bind(g, k) == 0
        din, dout = c_vp(), c_vp()
        assert so.ecl_gpu_buffer(g, 0, 0, ctypes.byref(din)) == 0
        assert so.ecl_gpu_buffer(g, 1, 0, ctypes.byref(dout)) == 0
        x = np.linspace(-7, 5, n)
        assert so.ecl_gpu_upload(g, din, x.ctypes.data, x.nbytes) == 0
        ms = ctypes.c_float(0)
        for items in (1000, 0, 4096, 1 << 30):  # 1000 -> 896 (whole work-groups), 0 -> one work-group
            zero = np.zeros(n)
            assert so.ecl_gpu_upload(g, dout, zero.ctypes.data, zero.nbytes) == 0
            assert so.ecl_gpu_native_run_split(g, items, ctypes.byref(ms)) == 0
            assert ms.value > 0
            y = np.zeros(n)
            assert so.ecl_gpu_download(g, y.ctypes.data, dout, y.nbytes) == 0
            assert np.array_equal(y, oracle.vecscale(-0.5, 3.0, x)), items
        so.ecl_kernel_destroy(k)
    finally:
        so.ecl_gpu_close(g)


def test_peer_outputs_refused_for_kernels_without_peer_writes(gpu_available, lib):
    # ecl_gpu_set_peer_outputs: only kernels that store into peer buffers
    # (NBody) accept targets; host memory is refused as a target
    so = lib
    so.ecl_gpu_set_peer_outputs.restype = c_int
    so.ecl_gpu_set_peer_outputs.argtypes = [c_vp, ctypes.POINTER(c_vp), c_u32]
    so.ecl_gpu_peer_writes.restype = c_int
    so.ecl_gpu_peer_writes.argtypes = [c_vp, ctypes.POINTER(c_int)]
    g = c_vp()
    assert so.ecl_gpu_open(0, 2, ctypes.byref(g)) == 0
    try:
        n, lws = 4096, 128
        args = (Arg * 2)(Arg(1, 0, 0, 1.0), Arg(1, 0, 0, 0.0))
        geom = (Geom * 1)(Geom(8, n))
        k = c_vp()
        assert so.ecl_kernel_create(b"vecscale", n, lws, args, 2, geom, 1, geom, 1, 1, 1, ctypes.byref(k)) == 0
        assert so.ecl_gpu_bind(g, k) == 0
        ok = c_int(-1)
        assert so.ecl_gpu_peer_writes(g, ctypes.byref(ok)) == 0 and ok.value == 0
        dout = c_vp()
        assert so.ecl_gpu_buffer(g, 1, 0, ctypes.byref(dout)) == 0
        ptrs = (c_vp * 1)(dout)
        assert N.code_name(so.ecl_gpu_set_peer_outputs(g, ptrs, 1)) == "ConfigError"
        assert so.ecl_gpu_set_peer_outputs(g, None, 0) == 0  # clearing is always fine
        so.ecl_kernel_destroy(k)

        # NBody accepts device targets and refuses host memory
        nb = 1024
        args = (Arg * 2)(Arg(1, 0, 0, 0.005), Arg(1, 0, 0, 500.0))
        geom4 = (Geom * 2)(Geom(16, nb), Geom(16, nb))
        nargs = (Arg * 3)(Arg(0, 0, nb, 0.0), Arg(1, 0, 0, 0.005), Arg(1, 0, 0, 500.0))
        assert so.ecl_kernel_create(b"nbody", nb, 64, nargs, 3, geom4, 2, geom4, 2, 1, 1, ctypes.byref(k)) == 0
        assert so.ecl_gpu_bind(g, k) == 0
        assert so.ecl_gpu_peer_writes(g, ctypes.byref(ok)) == 0 and ok.value == 1
        d0, d1 = c_vp(), c_vp()
        assert so.ecl_gpu_buffer(g, 0, 0, ctypes.byref(d0)) == 0 and so.ecl_gpu_buffer(g, 0, 1, ctypes.byref(d1)) == 0
        assert so.ecl_gpu_set_peer_outputs(g, (c_vp * 2)(d0, d1), 1) == 0
        host = np.zeros(64)
        bad = (c_vp * 2)(host.ctypes.data, d1)
        assert N.code_name(so.ecl_gpu_set_peer_outputs(g, bad, 1)) == "ConfigError"
        assert so.ecl_gpu_set_peer_outputs(g, None, 0) == 0
        so.ecl_kernel_destroy(k)
    finally:
        so.ecl_gpu_close(g)
