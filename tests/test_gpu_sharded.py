"""The row-sharded path on the device (world size 1 over NCCL on the one
GPU this run has): the orchestrator + C-ABI building blocks must reproduce
the single-context solve bit for bit (same trees, trivial collectives)."""

import os
import socket

import numpy as np
import pytest

import paper_1709_04794_b200 as fb
from paper_1709_04794_b200.workloads import make_workload

from helpers import problem_from_workload

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def nccl_world1():
    import torch
    import torch.distributed as dist

    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        port = s.getsockname()[1]
    os.environ.setdefault("MASTER_ADDR", "127.0.0.1")
    os.environ["MASTER_PORT"] = str(port)
    torch.cuda.set_device(0)
    dist.init_process_group("nccl", rank=0, world_size=1, device_id=torch.device("cuda", 0))
    yield dist
    dist.destroy_process_group()


@pytest.mark.parametrize("k", [20, 50])
def test_sharded_world1_equals_single_solve(nccl_world1, k):
    from paper_1709_04794_b200.sharded import solve_sharded

    w = make_workload("cfg1")
    out = solve_sharded(w.x_offsets, w.x_cols, w.d, w.l_offsets, w.l_cols, w.l_vals, w.labels,
                        w.alpha, w.betas, w.tol, k, seed=w.seed, device=0)
    rep = fb.fsda_solve(problem_from_workload(w, max_iter=k))
    dirs = np.stack([rep.directions[float(b)] for b in w.betas])
    scores = np.stack([rep.ratings[float(b)].scores for b in w.betas])
    np.testing.assert_array_equal(out["directions"], dirs)
    np.testing.assert_array_equal(out["scores"], scores)
    np.testing.assert_array_equal(out["iterations"], rep.regression.iterations)
    np.testing.assert_array_equal(out["residuals"], rep.regression.residuals)
    assert out["n_applies"] == rep.regression.operator_applications == k
