import os
import sys

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)
GOLDEN = os.path.join(ROOT, "tests", "golden")


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA device (B200); run with -m gpu")
    config.addinivalue_line("markers", "slow: CPU test taking more than ~10 s")


@pytest.fixture(scope="session")
def golden_small():
    return dict(np.load(os.path.join(GOLDEN, "golden_small.npz")))


@pytest.fixture(scope="session")
def golden_c1():
    return dict(np.load(os.path.join(GOLDEN, "golden_config1.npz")))


@pytest.fixture(scope="session")
def golden_pipeline():
    return dict(np.load(os.path.join(GOLDEN, "golden_pipeline.npz")))


@pytest.fixture(scope="session")
def golden_rotation():
    return dict(np.load(os.path.join(GOLDEN, "golden_rotation.npz")))
