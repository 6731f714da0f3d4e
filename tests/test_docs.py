"""The C-ABI names the integration guide and DESIGN.md tell a maintainer to
call exist in include/*.h and are exported by the built libraries."""
import ctypes
import os
import re

from paper_1805_02755_b200 import _native as N

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _headers():
    return "".join(open(os.path.join(ROOT, "include", h)).read() for h in ("ecl_cuda.h", "ecl_engine.h"))


def _declared():
    return set(re.findall(r"\b(ecl_[a-z0-9_]+)\s*\(", _headers()))


def _types():
    return set(re.findall(r"\b(ecl_[a-z0-9_]+)\s*;", _headers())) | set(re.findall(r"struct\s+(ecl_[a-z0-9_]+)", _headers()))


def _mentioned(doc):
    text = open(os.path.join(ROOT, doc)).read()
    return set(re.findall(r"\b(ecl_[a-z0-9_]+)\s*\(", text)) | set(re.findall(r"`(ecl_[a-z0-9_]+)`", text))


def _plugin_helpers():
    """Device-side inline helpers of the plugin launch ABI (include/ecl_plugin.h):
    compiled into the user's kernel, not exported by a library."""
    text = open(os.path.join(ROOT, "include", "ecl_plugin.h")).read()
    return set(re.findall(r"\b(ecl_plugin_[a-z0-9_]+)\s*\(", text)) | set(re.findall(r"\b(ecl_[a-z0-9_]+)\s*;", text))


def test_documented_entry_points_are_declared_and_exported():
    declared, types, helpers = _declared(), _types(), _plugin_helpers()
    libs = [ctypes.CDLL(N.CUDA_LIB_PATH), ctypes.CDLL(N.LIB_PATH)]
    for doc in ("INTEGRATION.md", "DESIGN.md"):
        for name in sorted(_mentioned(doc) - types - helpers):
            assert name in declared, f"{doc} mentions {name}, not declared in include/*.h"
            assert any(hasattr(lib, name) for lib in libs), f"{name} not exported"
