"""The row-sharded solve on the device (csrc/fsda_shard.cuh).

This run has one GPU, so the multi-rank path is exercised as a *local group*:
world 2 and 4 contexts on the same B200 driven by one process, exchanges as
device copies ordered by events (no kernel waits on another rank).  The NCCL
path (one process per GPU, collectives captured in the iteration graph) runs
at world 1.  Tolerances:
* world 1 (local and NCCL): bit for bit equal to fsda_solve;
* world 2 / 4: bit for bit equal to the oracle's partitioned mode
  (oracle_fsda_solve_sharded: rank-ordered partial sums), and within 1e-9 of
  the reference's arithmetic (oracle/ref_numpy.py) at the stable K.
The old Python orchestrator over NCCL is kept for world 1 as well."""

import os
import socket

import numpy as np
import pytest

import paper_1709_04794_b200 as fb
from oracle import c_oracle, ref_numpy
from paper_1709_04794_b200.sharded import partition_rows, solve_row_sharded_local
from paper_1709_04794_b200.workloads import make_workload

from helpers import labeled_aucs, problem_from_workload, rel_rows

pytestmark = pytest.mark.gpu


def _single(w, k, storage=64):
    rep = fb.fsda_solve(problem_from_workload(w, max_iter=k), storage=storage)
    dirs = np.stack([rep.directions[float(b)] for b in w.betas])
    scores = np.stack([rep.ratings[float(b)].scores for b in w.betas])
    return rep, dirs, scores


def _local(w, k, world, storage=64, bounds=None):
    return solve_row_sharded_local(w.x_offsets, w.x_cols, w.d, w.l_offsets, w.l_cols, w.l_vals,
                                   w.labels, w.alpha, w.betas, w.tol, k, seed=w.seed, world=world,
                                   storage=storage, bounds=bounds)


def test_local_world1_equals_single_solve():
    w = make_workload("cfg1")
    rep, dirs, scores = _single(w, 50)
    out = _local(w, 50, 1)
    np.testing.assert_array_equal(out["directions"], dirs)
    np.testing.assert_array_equal(out["scores"], scores)
    np.testing.assert_array_equal(out["residuals"], rep.regression.residuals)
    np.testing.assert_array_equal(out["iterations"], rep.regression.iterations)
    assert out["n_applies"] == 50


@pytest.mark.parametrize("world", [2, 4])
@pytest.mark.parametrize("cfg,k", [("cfg1", 50), ("cfg2", 30)])
def test_local_group_bitwise_vs_partitioned_oracle(cfg, k, world):
    w = make_workload(cfg)
    out = _local(w, k, world)
    b = out["row_bounds"]
    assert b.size == world + 1 and np.all(np.diff(b) > 0)
    ref = c_oracle.fsda_solve_sharded(w.x_offsets, w.x_cols, w.d, w.l_offsets, w.l_cols, w.l_vals,
                                      w.labels, w.alpha, w.betas, w.tol, k, w.probe(), b)
    np.testing.assert_array_equal(out["directions"], ref["directions"])
    np.testing.assert_array_equal(out["scores"], ref["scores"])
    np.testing.assert_array_equal(out["residuals"], ref["residuals"])
    assert out["n_applies"] == ref["n_applies"] == k


@pytest.mark.parametrize("world", [2, 4])
def test_local_group_vs_reference_order_stable_k(world):
    """Against the reference's own arithmetic at cfg1's stable K = 20."""
    w = make_workload("cfg1")
    out = _local(w, 20, world)
    ref = ref_numpy.fsda_solve_workload(w, max_iter=20)
    assert rel_rows(out["directions"], ref["directions"]) <= 1e-9
    np.testing.assert_array_equal(labeled_aucs(out["scores"], w.labels),
                                  labeled_aucs(ref["scores"], w.labels))


def test_local_group_uneven_bounds_and_fp32_storage():
    """Hand-picked uneven row blocks (one rank holding no labeled row) in the
    fp32-storage mode: bitwise vs the partitioned oracle in fp32."""
    w = make_workload("cfg1")
    b = np.array([0, 700, 4100, 10000])
    out = _local(w, 30, 3, storage=32, bounds=b)
    c_oracle.set_storage(32)
    try:
        ref = c_oracle.fsda_solve_sharded(w.x_offsets, w.x_cols, w.d, w.l_offsets, w.l_cols, w.l_vals,
                                          w.labels, w.alpha, w.betas, w.tol, 30, w.probe(), b)
    finally:
        c_oracle.set_storage(64)
    np.testing.assert_array_equal(out["directions"], ref["directions"])
    np.testing.assert_array_equal(out["scores"], ref["scores"])


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
def test_nccl_world1_equals_single_solve(nccl_world1, k):
    """The NCCL backend: ncclUniqueId through torch.distributed, collectives
    captured with the kernels in the iteration graph, launched K times."""
    from paper_1709_04794_b200.sharded import solve_row_sharded

    w = make_workload("cfg1")
    rep, dirs, scores = _single(w, k)
    for _ in range(2):      # the second call replays the cached graph
        out = solve_row_sharded(w.x_offsets, w.x_cols, w.d, w.l_offsets, w.l_cols, w.l_vals, w.labels,
                                w.alpha, w.betas, w.tol, k, seed=w.seed, device=0)
        np.testing.assert_array_equal(out["directions"], dirs)
        np.testing.assert_array_equal(out["scores"], scores)
        np.testing.assert_array_equal(out["residuals"], rep.regression.residuals)
        assert out["n_applies"] == k


def test_python_orchestrator_world1_equals_single_solve(nccl_world1):
    from paper_1709_04794_b200.sharded import solve_sharded

    w = make_workload("cfg1")
    rep, dirs, scores = _single(w, 20)
    out = solve_sharded(w.x_offsets, w.x_cols, w.d, w.l_offsets, w.l_cols, w.l_vals, w.labels,
                        w.alpha, w.betas, w.tol, 20, seed=w.seed, device=0)
    np.testing.assert_array_equal(out["directions"], dirs)
    np.testing.assert_array_equal(out["scores"], scores)
