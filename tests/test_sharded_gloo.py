"""The row-sharded sweep (paper_1709_04794_b200/sharded.py) on CPU ranks.

World size 2 over gloo: each rank runs the product orchestrator
(sharded_fsda_solve + TorchComm) with a numpy implementation of the local
products on its row block (reference arithmetic: scipy products, numpy sums,
the krylov.py recurrence stepwise).  The result must match the single-process
reference-order oracle at a stable Krylov dimension, and every rank must hold
identical directions."""

import os
import socket

import numpy as np
import pytest
import scipy.sparse as sp
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from paper_1709_04794_b200.sharded import (TorchComm, partition_rows, sharded_fsda_solve,
                                           take_shard)
from paper_1709_04794_b200.workloads import make_workload


class StepCG:
    """krylov.py:168-281 one iteration at a time (the state every rank replicates)."""

    def __init__(self, b, betas, tol, max_iter):
        self.betas = np.asarray(betas, dtype=np.float64)
        ns, dim = self.betas.size, b.size
        self.ns, self.max_iter = ns, max_iter
        self.b_norm = float(np.linalg.norm(b))
        self.sols = np.zeros((ns, dim))
        self.iters = np.full(ns, max_iter, dtype=np.int64)
        self.resid = np.full(ns, self.b_norm)
        self.conv = np.zeros(ns, dtype=bool)
        self.it = 0
        if self.b_norm == 0.0:
            self.finished, self.iters[:], self.resid[:], self.conv[:] = True, 0, 0.0, True
            self.active = np.zeros(ns, dtype=bool)
            return
        self.thresh = tol * self.b_norm
        self.r, self.p = b.copy(), b.copy()
        self.P = np.tile(b, (ns, 1))
        self.rr, self.gp, self.al = self.b_norm * self.b_norm, 1.0, 0.0
        self.zp, self.z = np.ones(ns), np.ones(ns)
        self.active = np.ones(ns, dtype=bool)
        self.finished = max_iter <= 0

    def step(self, q):
        if self.finished:
            return
        i = self.it
        pq = float(self.p @ q)
        gamma = -self.rr / pq
        zn, gs, good = np.zeros(self.ns), np.zeros(self.ns), np.zeros(self.ns, bool)
        for s in np.flatnonzero(self.active):
            denom = gamma * self.al * (self.zp[s] - self.z[s]) + \
                self.zp[s] * self.gp * (1.0 - self.betas[s] * gamma)
            with np.errstate(all="ignore"):
                v = np.float64(self.zp[s] * self.z[s] * self.gp) / np.float64(denom)
            if np.isfinite(v) and abs(v) >= 1e-290:
                good[s], zn[s], gs[s] = True, v, gamma * v / self.z[s]
        for s in np.flatnonzero(good):
            self.sols[s] -= self.P[s] * gs[s]
        self.r = self.r + gamma * q
        rr_new = float(self.r @ self.r)
        r_norm = np.sqrt(rr_new)
        a_new = rr_new / self.rr
        self.p = self.r + a_new * self.p
        for s in np.flatnonzero(good):
            a_s = a_new * (zn[s] * gs[s]) / (self.z[s] * gamma)
            self.P[s] = zn[s] * self.r + a_s * self.P[s]
        for s in np.flatnonzero(self.active):
            if not good[s]:
                self.iters[s], self.resid[s], self.active[s] = i + 1, np.inf, False
                continue
            res = abs(zn[s]) * r_norm
            if res < self.thresh:
                self.iters[s], self.resid[s], self.conv[s], self.active[s] = i + 1, res, True, False
            else:
                self.zp[s], self.z[s] = self.z[s], zn[s]
        self.gp, self.al, self.rr = gamma, a_new, rr_new
        self.it = i + 1
        if not self.active.any() or self.it >= self.max_iter:
            self.finished = True


class NumpyShardOps:
    """Local products of one row block, in the reference's arithmetic."""

    def __init__(self, shard):
        self.s = shard
        ones = np.ones(shard.x_cols.size)
        self.x = sp.csr_matrix((ones, shard.x_cols, shard.x_offsets), shape=(shard.n_local, shard.d))
        self.xt = sp.csc_matrix((ones, shard.x_cols, shard.x_offsets), shape=(shard.d, shard.n_local))
        self.lap = sp.csr_matrix((shard.l_vals, shard.l_cols, shard.l_offsets),
                                 shape=(shard.n_local, shard.n_global))
        self.lab = shard.labels

    t = staticmethod(lambda a: torch.from_numpy(np.ascontiguousarray(a, dtype=np.float64)))

    def indicator(self):
        return self.t((self.lab != 0).astype(np.float64))

    def new_d1(self):
        return torch.zeros(self.s.d + 1, dtype=torch.float64)

    def upload_d(self, host):
        return self.t(host)

    def alloc_n_global(self):
        return torch.zeros(self.s.n_global, dtype=torch.float64)

    def to_host(self, x):
        return x.numpy().copy()

    def xrows(self, v):
        return self.t(self.x.dot(v.numpy()))

    def smoother(self, alpha, y_full):
        y = y_full.numpy()
        own = y[self.s.row_base:self.s.row_base + self.s.n_local]
        masked = np.where(self.lab != 0, own, 0.0)
        if alpha == 0.0:
            return self.t(masked)
        sm = alpha * self.lap.dot(y)
        return self.t(sm if alpha == 1.0 else (1.0 - alpha) * masked + sm)

    def xt_partial(self, z, out):
        zz = z.numpy()
        out[: self.s.d] = self.t(self.xt.dot(zz))
        out[self.s.d] = float(np.sum(zz))
        return out

    def class_sums(self, t):
        tt = t.numpy()
        return self.t([tt[self.lab == 1].sum(), tt[self.lab == -1].sum()])

    def apply_w(self, c1, c2):
        return self.t(np.where(self.lab == 1, c1, np.where(self.lab == -1, c2, 0.0)))

    def center(self, mu, q, scale):
        d = self.s.d
        if mu is None:
            q[:d] = q[:d] / scale
        else:
            q[:d] = q[:d] - mu[:d] * q[d]

    def cg_begin(self, betas, tol, max_iter, b):
        self.cg = StepCG(b[: self.s.d].numpy().copy(), betas, tol, max_iter)

    def direction(self):
        return self.t(self.cg.p if not self.cg.finished or self.cg.it else self.cg.p)

    def cg_step(self, q):
        self.cg.step(q[: self.s.d].numpy().copy())

    def status(self):
        return self.cg.finished, self.cg.it, 0

    def project(self):
        sc = np.stack([self.x.dot(w) for w in self.cg.sols]) if self.s.n_local else \
            np.zeros((self.cg.ns, 0))
        orient = self.t([float(self.lab.astype(np.float64) @ row) for row in sc])
        return sc, orient

    def finish(self, flip, scores):
        dirs = self.cg.sols.copy()
        for s in np.flatnonzero(flip):
            dirs[s] = -dirs[s]
            scores[s] = -scores[s]
        active = self.cg.active
        res = self.cg.resid.copy()
        if active.any():
            res[active] = np.abs(self.cg.z[active]) * np.sqrt(self.cg.rr)
        return dict(directions=dirs, scores=scores, residuals=res, iterations=self.cg.iters.copy(),
                    converged=self.cg.conv.copy(), n_applies=self.cg.it)


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _worker(rank, world, port, w, max_iter, out_q):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        bounds = partition_rows(w.x_offsets, world, w.l_offsets)
        shard = take_shard(w.x_offsets, w.x_cols, w.d, w.l_offsets, w.l_cols, w.l_vals, w.labels,
                           bounds, rank)
        lab = w.labels
        res = sharded_fsda_solve(NumpyShardOps(shard), TorchComm(np.diff(bounds)), w.alpha, w.betas,
                                 w.tol, max_iter, w.probe(), int((lab == 1).sum()),
                                 int((lab == -1).sum()), check_every=1)
        out_q.put((rank, bounds, res))
    finally:
        dist.destroy_process_group()


def _run(world, w, max_iter):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, w, max_iter, q)) for r in range(world)]
    for p in procs:
        p.start()
    outs = [q.get(timeout=300) for _ in range(world)]
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    return sorted(outs, key=lambda o: o[0])


@pytest.fixture(scope="module")
def small():
    return make_workload("cfg1", n=3000, d=1200, ell=300, n_pos=60, lam=12.0, k=6, n_shifts=6,
                         max_iter=15)


def test_partition_rows_balances_work():
    w = make_workload("cfg1", n=5000, d=800, ell=100, n_pos=20, lam=10.0, k=5)
    b = partition_rows(w.x_offsets, 4, w.l_offsets)
    assert b[0] == 0 and b[-1] == w.n and np.all(np.diff(b) > 0)
    work = np.diff(w.x_offsets) + np.diff(w.l_offsets) + 1
    per = np.array([work[b[i]:b[i + 1]].sum() for i in range(4)])
    assert per.max() / per.min() < 1.05
    assert np.array_equal(partition_rows(w.x_offsets, 1), [0, w.n])


def test_two_rank_sweep_matches_single_process(small):
    from oracle import ref_numpy

    from helpers import labeled_aucs, rel_rows

    outs = _run(2, small, small.max_iter)
    (_, b0, r0), (_, b1, r1) = outs
    np.testing.assert_array_equal(b0, b1)
    np.testing.assert_array_equal(r0["directions"], r1["directions"])    # replicated state
    np.testing.assert_array_equal(r0["iterations"], r1["iterations"])
    scores = np.concatenate([r0["scores"], r1["scores"]], axis=1)
    ref = ref_numpy.fsda_solve_workload(small)
    assert rel_rows(r0["directions"], ref["directions"]) <= 1e-9
    assert rel_rows(scores, ref["scores"]) <= 1e-9
    np.testing.assert_array_equal(labeled_aucs(scores, small.labels),
                                  labeled_aucs(ref["scores"], small.labels))
    np.testing.assert_array_equal(r0["iterations"], ref["iterations"])
    assert r0["n_applies"] == ref["n_applies"] == small.max_iter
