"""Shared fixtures.  GPU tests carry @pytest.mark.gpu; everything else runs on
the CPU (oracle vs golden fixtures, host logic, C-ABI exports, gloo ranks)."""

import sys
from pathlib import Path

import numpy as np
import pytest

ROOT = Path(__file__).resolve().parents[1]
if str(ROOT) not in sys.path:
    sys.path.insert(0, str(ROOT))

GOLDEN = Path(__file__).resolve().parent / "golden"


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a B200 (run with -m gpu)")


@pytest.fixture(scope="session")
def golden_cfg1():
    return dict(np.load(GOLDEN / "cfg1_reference.npz"))


@pytest.fixture(scope="session")
def golden_small():
    return dict(np.load(GOLDEN / "small_reference.npz"))


@pytest.fixture(scope="session")
def golden_dense():
    return dict(np.load(GOLDEN / "dense_reference.npz"))


@pytest.fixture(scope="session")
def cfg1_workload():
    from paper_1709_04794_b200.workloads import make_workload

    return make_workload("cfg1")


@pytest.fixture
def rng():
    return np.random.default_rng(12345)
