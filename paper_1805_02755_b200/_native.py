"""ctypes binding of the in-tree native libraries (include/ecl_engine.h,
include/ecl_cuda.h).

There is no Python or CPU fallback: if ``_lib/libcoexec.so`` is missing the
import fails loudly, and compute calls fail with the device layer's error
when no CUDA device is visible.
"""
from __future__ import annotations

import ctypes
import os

LIB_DIR = os.path.join(os.path.dirname(os.path.abspath(__file__)), "_lib")
LIB_PATH = os.path.join(LIB_DIR, "libcoexec.so")
CUDA_LIB_PATH = os.path.join(LIB_DIR, "libecl_cuda.so")

if not os.path.exists(LIB_PATH):
    raise ImportError(
        f"{LIB_PATH} is not built; run `python -c 'import __graft_entry__ as g; g.build()'` "
        "(make -C paper_1805_02755_b200/csrc)")

lib = ctypes.CDLL(LIB_PATH)

c_u64 = ctypes.c_uint64
c_i64 = ctypes.c_int64
c_u32 = ctypes.c_uint32
c_int = ctypes.c_int
c_dbl = ctypes.c_double
c_char_p = ctypes.c_char_p
c_void_p = ctypes.c_void_p
PVOID = ctypes.POINTER(c_void_p)


def _sig(name, res, *args):
    f = getattr(lib, name)
    f.restype = res
    f.argtypes = list(args)
    return f


# engine
_sig("ecl_engine_create", c_int, c_char_p, ctypes.POINTER(c_void_p))
_sig("ecl_engine_destroy", None, c_void_p)
_sig("ecl_engine_run", c_int, c_void_p, PVOID, c_u32, PVOID, c_u32)
_sig("ecl_engine_run_virtual", c_int, c_void_p, ctypes.POINTER(c_dbl), c_u64)
_sig("ecl_engine_run_steps", c_int, c_void_p, PVOID, c_u32, PVOID, c_u32, c_u32, ctypes.POINTER(c_u32),
     ctypes.POINTER(c_u32), c_u32)
_sig("ecl_engine_gather", c_int, c_void_p, PVOID, c_u32)
_sig("ecl_engine_trace_json", c_i64, c_void_p, c_char_p, c_u64)
_sig("ecl_engine_native_run", c_int, c_void_p, PVOID, c_u32, PVOID, c_u32, ctypes.POINTER(c_dbl),
     ctypes.POINTER(c_dbl))
_sig("ecl_engine_native_run_split", c_int, c_void_p, c_u64, ctypes.POINTER(c_dbl))
_sig("ecl_engine_kernel_time", c_int, c_void_p, ctypes.POINTER(c_dbl), ctypes.POINTER(c_u64), c_int)
_sig("ecl_engine_init_ms", c_dbl, c_void_p)
_sig("ecl_engine_learned_powers", c_int, c_void_p, ctypes.POINTER(c_dbl), c_u32, ctypes.POINTER(c_u32))
_sig("ecl_engine_error_count", c_u32, c_void_p)
_sig("ecl_engine_error", c_i64, c_void_p, c_u32, ctypes.POINTER(c_int), c_char_p, c_u64)
# scheduler seam
_sig("ecl_scheduler_create", c_int, c_char_p, ctypes.POINTER(c_void_p))
_sig("ecl_scheduler_destroy", None, c_void_p)
_sig("ecl_scheduler_next", c_int, c_void_p, c_u32, ctypes.POINTER(c_u64), ctypes.POINTER(c_u64))
_sig("ecl_scheduler_remaining", c_u64, c_void_p)
_sig("ecl_scheduler_observe", c_int, c_void_p, c_u32, c_u64, c_dbl)
_sig("ecl_scheduler_unclamped", c_i64, c_void_p, c_u64, c_u32)
_sig("ecl_describe_scheduler", c_i64, c_char_p, c_char_p, c_u64)
_sig("ecl_resolve_static", c_i64, c_char_p, c_char_p, c_char_p, c_u64)
_sig("ecl_apply_default_min_package", c_i64, c_char_p, c_char_p, c_u64)
# core
_sig("ecl_validate_program", c_int, c_char_p, ctypes.POINTER(c_u64))
_sig("ecl_out_range_for", c_int, c_char_p, c_u64, c_u64, ctypes.POINTER(c_u64), ctypes.POINTER(c_u64))
_sig("ecl_tiles_exactly", c_int, ctypes.POINTER(c_u64), ctypes.POINTER(c_u64), c_u64, c_u64)
_sig("ecl_metrics_report", c_i64, c_char_p, ctypes.POINTER(c_dbl), c_u32, c_dbl, c_char_p, c_u64)
_sig("ecl_trace_csv", c_i64, c_char_p, c_char_p, c_u64)
_sig("ecl_chart_svg", c_i64, c_char_p, c_char_p, c_u64)
_sig("ecl_experiment_run", c_int, c_char_p, c_char_p, c_char_p, c_u64)
_sig("ecl_experiment_validate", c_i64, c_char_p, c_char_p, c_u64)
_sig("ecl_engine_last_error", c_char_p)
# device layer (subset used from Python)
_sig("ecl_gpu_count", c_int, ctypes.POINTER(c_int))
_sig("ecl_probe_mandel_mix", c_int, c_int, ctypes.POINTER(c_dbl))
_sig("ecl_probe_mandel_mix_f32", c_int, c_int, ctypes.POINTER(c_dbl))
_sig("ecl_host_register", c_int, c_void_p, ctypes.c_size_t)
_sig("ecl_host_unregister", c_int, c_void_p)
_sig("ecl_host_alloc", c_int, ctypes.c_size_t, ctypes.POINTER(c_void_p))
_sig("ecl_host_free", c_int, c_void_p)
_sig("ecl_last_error", c_char_p)
_sig("ecl_kernel_register", c_int, c_char_p, c_void_p, ctypes.c_size_t, c_char_p)
_sig("ecl_kernel_unregister", c_int, c_char_p)
_sig("ecl_kernel_is_plugin", c_int, c_char_p)
_sig("ecl_engine_run_kernel", c_int, c_void_p, c_char_p, PVOID, c_u32, PVOID, c_u32)
_sig("ecl_peer_access", c_int, c_int, c_int, ctypes.POINTER(c_int), ctypes.POINTER(c_int))
_sig("ecl_probe_host_widen", c_int, c_u64, c_u32, ctypes.POINTER(c_dbl))
_sig("ecl_probe_host_widen_width", c_int, c_u64, c_u32, c_u32, ctypes.POINTER(c_dbl))
_sig("ecl_probe_vector_peaks", c_int, c_int, ctypes.POINTER(c_dbl), ctypes.POINTER(c_dbl), ctypes.POINTER(c_dbl))

ERROR_NAMES = [
    "NonDivisibleWorkSize", "BadOutPattern", "EmptyProgram", "IndivisiblePackage", "TooFewWorkGroups",
    "BadSchedulerConfig", "SchedulerError", "InputSizeMismatch", "KernelPanic", "EmptyQueueWithPendingWork",
    "TallyViolation", "EmptyTrace", "NonPositiveTime", "MissingBaseline", "NonPositiveReference", "UnknownKernel",
    "UnknownProfile", "BadKernelArgs", "MalformedTrace", "ConfigError", "IoError",
]


def code_name(status: int) -> str:
    i = -status - 1
    return ERROR_NAMES[i] if 0 <= i < len(ERROR_NAMES) else "KernelPanic"


def last_error() -> str:
    msg = lib.ecl_engine_last_error()
    return msg.decode() if msg else ""


def device_last_error() -> str:
    msg = lib.ecl_last_error()
    return msg.decode() if msg else ""


def read_string(fn, *args) -> str:
    """Calls an int64-returning string API twice: size, then fill."""
    n = fn(*args, None, 0)
    if n < 0:
        return n  # type: ignore[return-value]
    buf = ctypes.create_string_buffer(n + 1)
    m = fn(*args, buf, n + 1)
    if m < 0:
        return m  # type: ignore[return-value]
    return buf.value.decode()


def pointer_array(ptrs):
    arr = (c_void_p * max(1, len(ptrs)))()
    for i, p in enumerate(ptrs):
        arr[i] = p
    return arr


def gpu_count() -> int:
    n = c_int(0)
    rc = lib.ecl_gpu_count(ctypes.byref(n))
    return n.value if rc == 0 else 0
