"""The drop-in C++ API (include/tbsim/*.hpp, libtbsim_cpp.so) through a C++
test binary that mirrors the reference's own suites (tests/cpp/test_api.cpp)."""
import os
import subprocess

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
BIN = os.path.join(ROOT, "tests", "cpp", "test_api")


def _build():
    subprocess.check_call(["make", "-s", "-C", os.path.join(ROOT, "tests", "cpp")])


def _run(args):
    r = subprocess.run([BIN] + args, capture_output=True, text=True, timeout=600)
    assert r.returncode == 0, r.stdout[-3000:] + r.stderr[-3000:]
    return r.stdout


def test_cpp_api_host_side():
    _build()
    out = _run(["--cpu-only"])
    assert " 0 failed" in out


@pytest.mark.gpu
def test_cpp_api_on_device():
    _build()
    out = _run([])
    assert " 0 failed" in out
