"""Runs the reference's own tracking tests re-targeted at the GPU through the
C++ drop-in adapter (tests/cpp/test_adapter.cpp, include/l1rx_gpu.hpp),
compiled against the unmodified reference headers."""
import os
import subprocess

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
BIN = os.path.join(ROOT, "tests", "cpp", "_build", "test_adapter")


@pytest.mark.gpu
def test_reference_tests_through_cpp_adapter(native_lib):
    if not os.path.exists(BIN):
        if os.path.isdir("/root/reference/proj/include"):
            subprocess.run(["make", "-s", "-C", os.path.join(ROOT, "tests", "cpp")], check=True)
        else:
            pytest.fail("tests/cpp/_build/test_adapter not built (build it where the reference exists)")
    r = subprocess.run([BIN], capture_output=True, text=True, timeout=600)
    print(r.stdout[-2000:])
    assert r.returncode == 0, r.stdout[-2000:] + r.stderr[-2000:]
    assert "OK:" in r.stdout
