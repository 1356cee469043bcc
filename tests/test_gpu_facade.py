"""-m gpu: the C++ facade (adamas::gpu) driver re-running the reference's
hot-path doctest cases on the device (tests/cpp/facade_tests.cpp)."""
import os
import subprocess

import pytest

pytestmark = pytest.mark.gpu
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def test_facade_driver(gpu):
    import __graft_entry__
    __graft_entry__._build_module().build()
    exe = os.path.join(ROOT, "tests", "cpp", "facade_tests")
    r = subprocess.run([exe], capture_output=True, text=True, timeout=300)
    print(r.stdout, r.stderr)
    assert r.returncode == 0, r.stdout + r.stderr
    assert "0 failed" in r.stdout
