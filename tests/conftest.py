"""Shared fixtures.  `-m gpu` tests need a B200 (run through gpurun); everything else runs on CPU."""
import os
import sys

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)
GOLDEN = os.path.join(ROOT, "tests", "golden")


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA B200 device and the built libsliceeig_cuda.so")
    config.addinivalue_line("markers", "slow: long-running parity case")


@pytest.fixture(scope="session")
def golden():
    """Loader for committed golden fixtures (tests/golden/*.npz, made by make_golden.py)."""
    def load(name):
        return dict(np.load(os.path.join(GOLDEN, name + ".npz"), allow_pickle=False))
    return load


@pytest.fixture(scope="session")
def gpu_ctx():
    from paper_1802_05215_b200 import api
    if api.device_count() < 1:
        pytest.fail("no CUDA device visible for a -m gpu test")
    return api.default_context(0)
