import os
import sys

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
for _p in (ROOT, os.path.join(ROOT, "tests")):
    if _p not in sys.path:
        sys.path.insert(0, _p)

from pmpd_testutil import load_golden, rel_l2  # noqa: E402,F401


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a B200 (runs through the CUDA C-ABI library)")
    config.addinivalue_line("markers", "slow: long-running parity case")


@pytest.fixture(scope="session")
def gold_quant():
    return load_golden("quant.npz")


@pytest.fixture(scope="session")
def gold_model():
    return load_golden("model.npz")


@pytest.fixture(scope="session")
def gold_layer():
    return load_golden("layer.npz")


@pytest.fixture(scope="session")
def gold_sched():
    return load_golden("schedule.npz")


@pytest.fixture(scope="session")
def gold_learn():
    return load_golden("learnsched.npz")

