"""Shared test setup.

Markers: ``gpu`` -- needs a CUDA device (run on the B200 box with
``pytest -m gpu``); everything else runs on the CPU container.
"""

import os
import sys

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
for _p in (ROOT, os.path.join(ROOT, "tests")):
    if _p not in sys.path:
        sys.path.insert(0, _p)

from mrs_testutil import load_golden, have_cuda  # noqa: E402,F401


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA device (B200)")
    config.addinivalue_line("markers", "slow: long-running")


@pytest.fixture(scope="session")
def golden_kernels():
    return load_golden("kernels.npz")


@pytest.fixture(scope="session")
def golden_solves():
    return load_golden("solves.npz")


@pytest.fixture(scope="session")
def golden_hier():
    return load_golden("hierarchies.npz")


@pytest.fixture(scope="session")
def rng():
    return np.random.default_rng(20240817)
