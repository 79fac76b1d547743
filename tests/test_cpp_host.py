"""The C++ host API (include/mersenne_b200/mersenne_b200.hpp) runs the
reference's own unit-test cases on the GPU (tests/cpp/test_host_api.cpp)."""
import os
import subprocess

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
BIN = os.path.join(ROOT, "tests", "cpp", "test_host_api")


def _build():
    subprocess.check_call(["make", "-C", ROOT, "cpptest"], stdout=subprocess.DEVNULL)


def test_cpp_host_api_builds():
    _build()
    assert os.path.exists(BIN)


@pytest.mark.gpu
def test_cpp_host_api_on_gpu(cuda):
    if not os.path.exists(BIN):
        _build()
    r = subprocess.run([BIN], capture_output=True, text=True, timeout=600)
    assert r.returncode == 0, r.stdout + r.stderr
    assert "0 failed" in r.stdout
