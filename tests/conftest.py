import os
import sys

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)
GOLDEN = os.path.join(ROOT, "tests", "golden")


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a B200 (run with -m gpu)")
    config.addinivalue_line("markers", "slow: multi-second CPU oracle runs")


def golden(name):
    return np.load(os.path.join(GOLDEN, f"{name}.npz"))


@pytest.fixture(scope="session")
def small_golden():
    return golden("small")


@pytest.fixture(scope="session")
def overflow_golden():
    return golden("overflow")


@pytest.fixture(scope="session")
def cfg1_golden():
    return golden("cfg1")


@pytest.fixture(scope="session")
def rng_golden():
    return golden("rng")
