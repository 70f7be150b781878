"""BASELINE configs[2] shape (cfg3: 1.5M x 500k, 75M nnz, Zipf 1.05, 30
shifts) on the device: bitwise equal to the C oracle over the first Krylov
iterations (the oracle needs ~1 s per iteration at this size on the host)."""

import numpy as np
import pytest

import paper_1709_04794_b200 as fb
from oracle import c_oracle
from paper_1709_04794_b200.workloads import make_workload

from helpers import problem_from_workload

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def cfg3():
    return make_workload("cfg3")


def test_cfg3_sweep_bitwise_vs_oracle(cfg3):
    k = 6
    rep = fb.fsda_solve(problem_from_workload(cfg3, max_iter=k))
    ref = c_oracle.fsda_solve_workload(cfg3, max_iter=k)
    dirs = np.stack([rep.directions[float(b)] for b in cfg3.betas])
    np.testing.assert_array_equal(dirs, ref["directions"])
    np.testing.assert_array_equal(rep.regression.residuals, ref["residuals"])
    assert rep.regression.operator_applications == k
