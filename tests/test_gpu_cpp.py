"""Runs the C++ drop-in API test (tests/cpp/test_dropin.cpp) on the GPU (-m gpu)."""
import os
import subprocess

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
BIN = os.path.join(ROOT, "build", "cpptest", "test_dropin")


@pytest.mark.gpu
def test_cpp_dropin_api():
    if not os.path.exists(BIN):
        subprocess.run(["make", "-C", ROOT, "cpptest"], check=True)
    r = subprocess.run([BIN], capture_output=True, text=True, timeout=600)
    assert r.returncode == 0, r.stdout + r.stderr
    assert "all checks passed" in r.stdout
