import os
import sys

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
GOLDEN = os.path.join(ROOT, "tests", "golden")


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA B200 (sm_100a)")
    config.addinivalue_line("markers", "slow: long CPU-oracle run (minutes)")


def load_golden(name):
    path = os.path.join(GOLDEN, f"golden_{name}.npz")
    if not os.path.exists(path):
        pytest.skip(f"golden fixture {name} not generated")
    return dict(np.load(path, allow_pickle=False))


@pytest.fixture(scope="session")
def golden_A():
    return load_golden("A")


@pytest.fixture(scope="session")
def golden_A2():
    return load_golden("A2")
