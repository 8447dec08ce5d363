"""Shared pytest setup: the `gpu` marker and fixture loading.

`-m "not gpu"` (the CPU suite run in the build container) covers the oracle
against the reference's golden vectors, the host logic and the C-ABI's
exports; `-m gpu` (on a B200) runs the parity tests through the C-ABI.
"""

import sys
from pathlib import Path

import numpy as np
import pytest

ROOT = Path(__file__).resolve().parents[1]
GOLDEN = ROOT / "tests" / "golden"
if str(ROOT) not in sys.path:
    sys.path.insert(0, str(ROOT))


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA device (B200) and libpndose_b200.so")


def golden(name):
    return np.load(GOLDEN / name, allow_pickle=False)


@pytest.fixture(scope="session")
def kernels_npz():
    return golden("kernels.npz")


@pytest.fixture(scope="session")
def steps_npz():
    return golden("steps.npz")


@pytest.fixture(scope="session")
def traverse_npz():
    return golden("traverse.npz")
