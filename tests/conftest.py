import os
import sys

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)

GOLDEN = os.path.join(ROOT, "tests", "golden")


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA device (B200, sm_100a) and the built librwb.so")


@pytest.fixture
def rng():
    # the reference suite's fixture seed (pkg/tests/conftest.py:8-10)
    return np.random.default_rng(0xC0FFEE)


def load_golden(name):
    return np.load(os.path.join(GOLDEN, name))
