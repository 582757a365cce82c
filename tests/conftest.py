"""Shared test plumbing.

Markers: ``gpu`` -- needs a B200 (run with ``-m gpu`` via gpurun); every other
test runs on CPU (``-m "not gpu"``).  The oracle (oracle/) is the checker in
both; the product under test is libl1rxg.so through the C ABI.
"""
import os
import sys

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: requires a CUDA device (B200)")


def _gpu_ok():
    try:
        import torch
        return torch.cuda.is_available()
    except Exception:
        return False


@pytest.fixture(scope="session")
def oracle_mod():
    import oracle
    oracle.build()
    return oracle


@pytest.fixture(scope="session")
def native_lib():
    from paper_1907_00463_b200 import build
    build.build()
    from paper_1907_00463_b200 import _native
    return _native.lib()


@pytest.fixture(scope="session")
def ctx(native_lib):
    if not _gpu_ok():
        pytest.fail("GPU test selected but no CUDA device is visible")
    from paper_1907_00463_b200.tracking import Context
    c = Context(0)
    yield c
    c.close()


def rel_err(got, want, scale=None):
    got = np.asarray(got, np.float64)
    want = np.asarray(want, np.float64)
    s = np.abs(want).max() if scale is None else scale
    return float(np.abs(got - want).max() / max(s, 1e-300))
