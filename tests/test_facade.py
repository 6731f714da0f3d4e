"""The C++ drop-in surface (csrc/coexec/ecl.hpp): the paper's Listings 1-2
 compiled as a user program against the product headers
and libraries, checked against the oracle (tests/cpp/test_facade.cpp)."""
import os
import subprocess

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
CPP = os.path.join(ROOT, "tests", "cpp")
EXE = os.path.join(CPP, "build", "test_facade")


def build():
    r = subprocess.run(["make", "-s", "-C", CPP], capture_output=True, text=True, timeout=300)
    assert r.returncode == 0, r.stdout + r.stderr
    return EXE


def run(*args):
    r = subprocess.run([build(), *args], capture_output=True, text=True, timeout=300)
    assert r.returncode == 0 and "OK" in r.stdout, r.stdout + r.stderr
    return r.stdout


def test_facade_compiles_and_reports_errors_without_running_kernels():
    # No kernel launches: an unknown kernel id is reported through
    # has_errors()/get_errors() rather than thrown.
    run("--no-gpu")


@pytest.mark.gpu
def test_facade_listings_match_oracle(gpu_available):
    run()


@pytest.mark.gpu
def test_cpp_engine_run_with_a_plugin_kernel(gpu_available):
    """coexec::Engine::run(inputs, DeviceKernel, CostFn) from C++ with a cubin
    registered by coexec::register_device_kernel_file."""
    plug = os.path.join(ROOT, "tests", "plugins")
    r = subprocess.run(["make", "-s", "-C", plug], capture_output=True, text=True, timeout=300)
    assert r.returncode == 0, r.stdout + r.stderr
    run("--plugin", os.path.join(plug, "_build", "plugins.cubin"))
