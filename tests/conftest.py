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


# Measured GPU-vs-reference deviations, collected by the parity tests and
# written at session end to $PND_PARITY_OUT (the round's profiles/parity_rNN.json
# is a copy of that file from the GPU box): every deviation next to its bound.
PARITY_RECORDS = []


@pytest.fixture(scope="session")
def parity_log():
    return PARITY_RECORDS


def pytest_sessionfinish(session, exitstatus):
    import json
    import os

    path = os.environ.get("PND_PARITY_OUT")
    if not path or not PARITY_RECORDS:
        return
    Path(path).parent.mkdir(parents=True, exist_ok=True)
    Path(path).write_text(json.dumps({"records": PARITY_RECORDS}, indent=1) + "\n")
