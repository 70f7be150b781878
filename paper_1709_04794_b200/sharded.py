"""Row-sharded FSDA sweep over several GPUs.

The product path is ``solve_row_sharded`` (one process per GPU, NCCL) and
``solve_row_sharded_local`` (every rank a context in this process — the
multi-rank tests on one GPU): both drive the C-ABI ``fsda_solve_sharded``
(csrc/fsda_shard.cuh), which runs the whole iteration on the device with the
exchanges captured in a CUDA graph.  The rank-ordered partial sums make the
result deterministic and reproducible by the oracle's partitioned mode
(oracle/fsda_oracle.c oracle_fsda_solve_sharded); at world 1 it equals
fsda_solve bit for bit.

The Python orchestrator below (``sharded_fsda_solve``) is the same
decomposition written against two small interfaces; it runs the host-side
logic on CPU ranks (gloo) in tests/test_sharded_gloo.py.

One process per GPU.  Rank g owns a contiguous block of rows of X and of the
Laplacian L (balanced by nonzeros) and the block's labels.  The D-length
Krylov vectors and the whole shift state are replicated: every rank runs the
identical shifted-CG recurrence, so the dots need no scalar collectives.  Per
iteration (krylov.py:210-270, one operator application):

    y_g      = X_g p                      local rows
    y        = all_gather(y_g)            the Laplacian reads neighbours' y
    z_g      = M_g y                      local rows of the smoother (sda.py:131-140)
    [q | Σz] = all_reduce([X_g^T z_g | Σ z_g])   one D+1 all-reduce
    q        = q - mu * Σz                centring folds into the same buffer (sparse.py:277)
    CG step on the replicated state

Setup and projection follow fsda_solve (sda.py:297-301, 265-284) with the
same decomposition: mu and the rhs are all-reduced D+1 partials, the class
sums a 2-vector, and the orientation dots an n_shifts vector.

The orchestration here is written against two small interfaces so that the
same code runs on the B200s (``DeviceShardOps``: the C-ABI kernels on device
buffers, NCCL through torch.distributed) and in the CPU world-size-2 tests
(gloo, with a numpy implementation of the local products in tests/).
"""

from __future__ import annotations

import ctypes as C
from dataclasses import dataclass
from typing import Optional

import numpy as np

from . import _capi
from . import types as T


# ---------------------------------------------------------------- sharding

def partition_rows(row_offsets, world: int, extra_offsets=None) -> np.ndarray:
    """Boundaries (world + 1 row indices) of contiguous row blocks with about
    equal work, work(i) = nnz of row i (+ the Laplacian row if given) + 1."""
    offs = np.asarray(row_offsets, dtype=np.int64)
    n = offs.size - 1
    work = np.diff(offs).astype(np.float64) + 1.0
    if extra_offsets is not None:
        work += np.diff(np.asarray(extra_offsets, dtype=np.int64))
    cw = np.concatenate([[0.0], np.cumsum(work)])
    targets = cw[-1] * np.arange(1, world) / world
    inner = np.searchsorted(cw, targets, side="left")
    bounds = np.concatenate([[0], inner, [n]]).astype(np.int64)
    return np.maximum.accumulate(np.clip(bounds, 0, n))


@dataclass
class RowShard:
    """Rows [row_base, row_base + n_local) of X and L, plus their labels."""

    row_base: int
    n_local: int
    n_global: int
    d: int
    x_offsets: np.ndarray
    x_cols: np.ndarray
    l_offsets: np.ndarray
    l_cols: np.ndarray      # global column indices
    l_vals: np.ndarray
    labels: np.ndarray


def take_shard(x_offsets, x_cols, d, l_offsets, l_cols, l_vals, labels, bounds, rank) -> RowShard:
    lo, hi = int(bounds[rank]), int(bounds[rank + 1])
    xo = np.asarray(x_offsets, dtype=np.int64)
    lo_ = np.asarray(l_offsets, dtype=np.int64)
    xs, xe = int(xo[lo]), int(xo[hi])
    ls, le = int(lo_[lo]), int(lo_[hi])
    return RowShard(
        row_base=lo, n_local=hi - lo, n_global=xo.size - 1, d=int(d),
        x_offsets=np.ascontiguousarray(xo[lo:hi + 1] - xs),
        x_cols=np.ascontiguousarray(np.asarray(x_cols, dtype=np.int64)[xs:xe]),
        l_offsets=np.ascontiguousarray(lo_[lo:hi + 1] - ls),
        l_cols=np.ascontiguousarray(np.asarray(l_cols, dtype=np.int64)[ls:le]),
        l_vals=np.ascontiguousarray(np.asarray(l_vals, dtype=np.float64)[ls:le]),
        labels=np.ascontiguousarray(np.asarray(labels, dtype=np.int8)[lo:hi]),
    )


# ------------------------------------------------------------- collectives

class TorchComm:
    """Collectives over torch.distributed (NCCL on the B200s, gloo on CPU)."""

    def __init__(self, counts, group=None):
        import torch.distributed as dist

        self.dist = dist
        self.group = group
        self.rank = dist.get_rank(group)
        self.world = dist.get_world_size(group)
        self.counts = [int(c) for c in counts]          # rows per rank
        self.maxc = max(self.counts) if self.counts else 0

    def all_reduce(self, t):
        if self.world > 1:
            self.dist.all_reduce(t, op=self.dist.ReduceOp.SUM, group=self.group)
        return t

    def all_gather_rows(self, local, out):
        """Concatenate every rank's local rows into `out` (N_global)."""
        import torch

        if self.world == 1:
            out[: local.numel()].copy_(local)
            return out
        pad = torch.zeros(self.maxc, dtype=local.dtype, device=local.device)
        pad[: local.numel()].copy_(local)
        parts = [torch.empty_like(pad) for _ in range(self.world)]
        self.dist.all_gather(parts, pad, group=self.group)
        pos = 0
        for r, cnt in enumerate(self.counts):
            out[pos:pos + cnt].copy_(parts[r][:cnt])
            pos += cnt
        return out


# --------------------------------------------------------- the algorithm

def sharded_fsda_solve(ops, comm, alpha, betas, tol, max_iter, probe, n1, n2, check_every=8):
    """The FSDA sweep of sda.py:293-320 with rows sharded over `comm`.

    ``ops`` supplies the local products on this rank's rows (see
    DeviceShardOps for the contract).  Returns a dict with the replicated
    directions (n_shifts x D), this rank's scores (n_shifts x N_local) and the
    per-shift residuals / iterations / convergence flags and n_applies."""
    ell = float(n1 + n2)
    mu, b, q = ops.new_d1(), ops.new_d1(), ops.new_d1()
    # mu = X^T 1_l / ell  (sparse.py:258-265)
    comm.all_reduce(ops.xt_partial(ops.indicator(), mu))
    ops.center(None, mu, ell)
    # rhs = X_c^T (W + 0) X probe  (sda.py:300-301)
    t = ops.xrows(ops.upload_d(probe))
    cs = comm.all_reduce(ops.class_sums(t))
    s1, s2 = ops.to_host(cs)
    w = ops.apply_w(float(s1) / n1, float(s2) / n2)
    comm.all_reduce(ops.xt_partial(w, b))
    ops.center(mu, b, 1.0)
    ops.cg_begin(betas, tol, max_iter, b)
    y_full = ops.alloc_n_global()
    for i in range(int(max_iter)):
        y = ops.xrows(ops.direction())
        comm.all_gather_rows(y, y_full)
        z = ops.smoother(alpha, y_full)
        comm.all_reduce(ops.xt_partial(z, q))
        ops.center(mu, q, 1.0)
        ops.cg_step(q)
        if (i + 1) % check_every == 0 or i + 1 == max_iter:
            finished, _, status = ops.status()
            if status:
                break
            if finished:
                break
    scores, orient = ops.project()
    comm.all_reduce(orient)
    flip = (ops.to_host(orient) < 0.0).astype(np.uint8)
    return ops.finish(flip, scores)


# ------------------------------------------------------- device backend

class DeviceShardOps:
    """Local products of one rank on its B200, through the C ABI.

    Buffers are torch CUDA tensors (so torch.distributed can run NCCL on
    them); the kernels run on the context stream, which is torch's current
    stream."""

    def __init__(self, shard: RowShard, device: int = 0):
        import torch

        from .fsda import Device, _raise_for

        self.torch = torch
        self._raise = _raise_for
        self.shard = shard
        self.dev_index = device
        # a real stream, made current so that torch's NCCL collectives on
        # these buffers are ordered with the library's kernels
        torch.cuda.set_device(device)
        cur = torch.cuda.current_stream(device)
        if not cur.cuda_stream:
            cur = torch.cuda.Stream(device)
            torch.cuda.set_stream(cur)
        self.stream = cur
        self.dev = Device(device, stream=cur.cuda_stream)
        x = T.SparseMatrix.binary(shard.n_local, shard.d, shard.x_offsets, shard.x_cols)
        self.dev.upload_x(x)
        lib = _capi.lib()
        _raise_for(lib.fsda_upload_laplacian_rows(
            self.dev._h, shard.n_local, shard.n_global, shard.row_base,
            _capi.i64ptr(shard.l_offsets), _capi.i64ptr(shard.l_cols), _capi.dptr(shard.l_vals)))
        self.dev.set_labels(shard.labels)
        self.lib = lib
        kw = dict(dtype=torch.float64, device=f"cuda:{device}")
        n, d = shard.n_local, shard.d
        self._ind = torch.from_numpy((shard.labels != 0).astype(np.float64)).to(**kw)
        self._y = torch.empty(max(n, 1), **kw)
        self._z = torch.empty(max(n, 1), **kw)
        self._w = torch.empty(max(n, 1), **kw)
        self._cs = torch.empty(2, **kw)
        self._probe = torch.empty(max(d, 1), **kw)
        self._kw = kw
        self._ns = 0

    @staticmethod
    def _p(t):
        return C.c_void_p(t.data_ptr())

    def _chk(self, rc):
        self._raise(rc)

    def indicator(self):
        return self._ind

    def upload_d(self, host):
        self._probe.copy_(self.torch.from_numpy(np.ascontiguousarray(host, dtype=np.float64)))
        return self._probe

    def new_d1(self):
        return self.torch.empty(self.shard.d + 1, **self._kw)

    def alloc_n_global(self):
        return self.torch.empty(max(self.shard.n_global, 1), **self._kw)

    def to_host(self, t):
        return t.detach().cpu().numpy()

    def xrows(self, v):
        ptr = v if isinstance(v, C.c_void_p) else self._p(v)
        self._chk(self.lib.fsda_dev_xrows(self.dev._h, ptr, self._p(self._y)))
        return self._y

    def smoother(self, alpha, y_full):
        self._chk(self.lib.fsda_dev_smoother(self.dev._h, float(alpha), self._p(y_full), self._p(self._z)))
        return self._z

    def xt_partial(self, z, out):
        self._chk(self.lib.fsda_dev_xt_partial(self.dev._h, self._p(z), self._p(out)))
        return out

    def class_sums(self, t):
        self._chk(self.lib.fsda_dev_class_sums(self.dev._h, self._p(t), self._p(self._cs)))
        return self._cs

    def apply_w(self, c1, c2):
        self._chk(self.lib.fsda_dev_apply_w(self.dev._h, c1, c2, self._p(self._w)))
        return self._w

    def center(self, mu, q, scale):
        self._chk(self.lib.fsda_dev_center(self.dev._h, self._p(mu) if mu is not None else None,
                                           self._p(q), float(scale)))

    def cg_begin(self, betas, tol, max_iter, b):
        betas = np.ascontiguousarray(betas, dtype=np.float64)
        self._ns = int(betas.size)
        self._chk(self.lib.fsda_dev_cg_begin(self.dev._h, _capi.dptr(betas), self._ns, float(tol),
                                             int(max_iter), self._p(b)))
        self._scores = self.torch.empty((self._ns, max(self.shard.n_local, 1)), **self._kw)
        self._orient = self.torch.empty(self._ns, **self._kw)

    def direction(self):
        ptr = C.c_void_p()
        self._chk(self.lib.fsda_dev_cg_direction(self.dev._h, C.byref(ptr)))
        return ptr

    def cg_step(self, q):
        self._chk(self.lib.fsda_dev_cg_step(self.dev._h, self._p(q)))

    def status(self):
        fin, it, st = C.c_int(0), C.c_int64(0), C.c_int(0)
        self._chk(self.lib.fsda_dev_cg_status(self.dev._h, C.byref(fin), C.byref(it), C.byref(st)))
        return bool(fin.value), int(it.value), int(st.value)

    def project(self):
        self._chk(self.lib.fsda_dev_project(self.dev._h, self._p(self._scores), self._p(self._orient)))
        return self._scores, self._orient

    def finish(self, flip, scores):
        ns, d = self._ns, self.shard.d
        dirs = np.empty((ns, d))
        res = np.empty(ns)
        its = np.empty(ns, dtype=np.int64)
        conv = np.empty(ns, dtype=np.uint8)
        napp, fail = C.c_int64(0), C.c_int64(-1)
        flip = np.ascontiguousarray(flip, dtype=np.uint8)
        self._chk(self.lib.fsda_dev_finish(self.dev._h, _capi.u8ptr(flip), self._p(scores),
                                           _capi.dptr(dirs), _capi.dptr(res), _capi.i64ptr(its),
                                           _capi.u8ptr(conv), C.byref(napp), C.byref(fail)))
        return dict(directions=dirs, scores=self.to_host(scores)[:, : self.shard.n_local],
                    residuals=res, iterations=its, converged=conv.astype(bool),
                    n_applies=int(napp.value))


def solve_sharded(x_offsets, x_cols, d, l_offsets, l_cols, l_vals, labels, alpha, betas, tol,
                  max_iter, seed=0, device: Optional[int] = None, group=None):
    """Convenience: shard the given problem by rows over the initialised
    torch.distributed group and run the sweep on this rank's GPU."""
    import torch.distributed as dist

    world = dist.get_world_size(group)
    rank = dist.get_rank(group)
    bounds = partition_rows(x_offsets, world, l_offsets)
    shard = take_shard(x_offsets, x_cols, d, l_offsets, l_cols, l_vals, labels, bounds, rank)
    lab = np.asarray(labels)
    n1, n2 = int((lab == 1).sum()), int((lab == -1).sum())
    ops = DeviceShardOps(shard, device if device is not None else rank)
    comm = TorchComm(np.diff(bounds), group)
    probe = np.random.default_rng(seed).uniform(-1.0, 1.0, size=int(d))
    out = sharded_fsda_solve(ops, comm, alpha, betas, tol, max_iter, probe, n1, n2)
    out["row_bounds"] = bounds
    return out


# ------------------------------------------- the device path (C ABI)

def shard_slot(bounds) -> int:
    """Rows per rank in the all-gather layout: the largest shard, rounded up
    to even (fsda_shard_init)."""
    b = np.asarray(bounds, dtype=np.int64)
    m = int(np.max(np.diff(b))) if b.size > 1 else 0
    return (m + 1) & ~1


def remap_columns(cols, bounds) -> np.ndarray:
    """Global row index j (owned by rank h) -> h * slot + (j - bounds[h])."""
    b = np.asarray(bounds, dtype=np.int64)
    cols = np.asarray(cols, dtype=np.int64)
    h = np.searchsorted(b, cols, side="right") - 1
    return h * shard_slot(b) + (cols - b[h])


class ShardRank:
    """One rank's context: its rows of X and L uploaded in the all-gather
    layout, its labels, and the shard registration."""

    def __init__(self, shard: "RowShard", bounds, rank: int, device: int = 0, stream=None,
                 nccl_id: Optional[bytes] = None, storage: int = 64):
        from .fsda import Device, _raise_for

        self.dev = Device(device, stream=stream)
        self.shard = shard
        world = len(bounds) - 1
        lib = _capi.lib()
        x = T.SparseMatrix.binary(shard.n_local, shard.d, shard.x_offsets, shard.x_cols)
        self._x = x              # validated once; reload() re-uploads it
        self.dev.upload_x(x)
        slot = shard_slot(bounds)
        lcols = np.ascontiguousarray(remap_columns(shard.l_cols, bounds))
        self._lcols = lcols      # this shard's L columns in the all-gather layout
        _raise_for(lib.fsda_upload_laplacian_rows(
            self.dev._h, shard.n_local, world * slot, rank * slot, _capi.i64ptr(shard.l_offsets),
            _capi.i64ptr(lcols), _capi.dptr(shard.l_vals)))
        self.dev.set_label_mask(shard.labels)
        self.dev._loaded = (None, None, None)
        bd = np.ascontiguousarray(bounds, dtype=np.int64)
        idp = None
        if nccl_id is not None:
            idb = np.frombuffer(bytes(nccl_id), dtype=np.uint8).copy()
            idp = _capi.u8ptr(idb)
        _raise_for(lib.fsda_shard_init(self.dev._h, world, rank, _capi.i64ptr(bd), idp))
        if storage != 64:
            self.dev.set_storage(storage)

    def reload(self, shard: "RowShard", bounds, rank: int):
        """Re-upload this rank's rows (same shapes; the shard registration and
        the communicator stay)."""
        from .fsda import _raise_for

        world = len(bounds) - 1
        slot = shard_slot(bounds)
        # the same shard: its validated matrix and remapped columns are kept
        # (host preprocessing, not an input copy); the arrays are re-uploaded
        same = shard is self.shard
        x = self._x if same else T.SparseMatrix.binary(shard.n_local, shard.d, shard.x_offsets, shard.x_cols)
        self._x = x
        self.dev.upload_x(x)
        lcols = self._lcols if same else np.ascontiguousarray(remap_columns(shard.l_cols, bounds))
        self._lcols = lcols
        _raise_for(_capi.lib().fsda_upload_laplacian_rows(
            self.dev._h, shard.n_local, world * slot, rank * slot, _capi.i64ptr(shard.l_offsets),
            _capi.i64ptr(lcols), _capi.dptr(shard.l_vals)))
        self.dev.set_label_mask(shard.labels)
        self.shard = shard


def _solve_ranks(ranks, d, alpha, betas, tol, max_iter, probe, n1, n2, scores=True):
    from .fsda import _pinned_empty, _raise_for

    betas = np.ascontiguousarray(betas, dtype=np.float64)
    probe = np.ascontiguousarray(probe, dtype=np.float64)
    ns = int(betas.size)
    rows = sum(r.shard.n_local for r in ranks)
    # page-locked result arrays: a pageable 120 MB directions copy (cfg3)
    # would cost ~25 ms through the driver's bounce buffer
    dirs = _pinned_empty((ns, d))
    sc = _pinned_empty((ns, rows)) if scores else None
    res = np.empty(ns)
    its = np.empty(ns, dtype=np.int64)
    conv = np.empty(ns, dtype=np.uint8)
    napp, fail = C.c_int64(0), C.c_int64(-1)
    arr = (C.c_void_p * len(ranks))(*[r.dev._h.value for r in ranks])
    rc = _capi.lib().fsda_solve_sharded(
        arr, len(ranks), float(alpha), _capi.dptr(betas), ns, float(tol), int(max_iter),
        _capi.dptr(probe), int(n1), int(n2), _capi.dptr(dirs),
        _capi.dptr(sc) if sc is not None else None, _capi.dptr(res), _capi.i64ptr(its),
        _capi.u8ptr(conv), C.byref(napp), C.byref(fail))
    _raise_for(rc)
    return dict(directions=dirs, scores=sc, residuals=res, iterations=its,
                converged=conv.astype(bool), n_applies=int(napp.value))


def _class_counts(labels):
    lab = np.asarray(labels)
    ml = lab != 0
    if ml.size and not ml.all() and ml[int(np.argmin(ml)):].any():   # a labeled row after an unlabeled one
        raise ValueError("labeled samples must occupy the first rows; use arrange_labeled_first "
                         "to permute the problem")
    return int((lab == 1).sum()), int((lab == -1).sum())


def solve_row_sharded_local(x_offsets, x_cols, d, l_offsets, l_cols, l_vals, labels, alpha, betas,
                            tol, max_iter, seed=0, world=2, device=0, bounds=None, storage=64):
    """The row-sharded sweep with every rank a context of this process on one
    GPU (exchanges as device copies): the multi-rank path testable on one
    B200.  Returns directions, scores of all rows (global order), residuals,
    iterations, converged, n_applies, row_bounds."""
    n1, n2 = _class_counts(labels)
    b = partition_rows(x_offsets, world, l_offsets) if bounds is None else np.asarray(bounds, np.int64)
    ranks = [ShardRank(take_shard(x_offsets, x_cols, d, l_offsets, l_cols, l_vals, labels, b, g),
                       b, g, device=device, storage=storage) for g in range(len(b) - 1)]
    probe = np.random.default_rng(seed).uniform(-1.0, 1.0, size=int(d))
    out = _solve_ranks(ranks, int(d), alpha, betas, tol, max_iter, probe, n1, n2)
    out["row_bounds"] = b
    return out


def solve_row_sharded(x_offsets, x_cols, d, l_offsets, l_cols, l_vals, labels, alpha, betas, tol,
                      max_iter, seed=0, device: Optional[int] = None, group=None, storage=64,
                      stream=None):
    """One process per GPU over the initialised torch.distributed group: this
    rank's rows on its GPU, NCCL for the exchanges (inside the captured
    iteration graph).  Returns the replicated directions, this rank's scores,
    residuals, iterations, converged, n_applies, row_bounds."""
    import torch.distributed as dist

    world = dist.get_world_size(group)
    rank = dist.get_rank(group)
    n1, n2 = _class_counts(labels)
    b = partition_rows(x_offsets, world, l_offsets)
    box = [None]
    if rank == 0:
        idb = np.zeros(128, dtype=np.uint8)
        from .fsda import _raise_for

        _raise_for(_capi.lib().fsda_nccl_unique_id(_capi.u8ptr(idb)))
        box = [idb.tobytes()]
    dist.broadcast_object_list(box, src=0, group=group)
    shard = take_shard(x_offsets, x_cols, d, l_offsets, l_cols, l_vals, labels, b, rank)
    r = ShardRank(shard, b, rank, device=rank if device is None else device, stream=stream,
                  nccl_id=box[0], storage=storage)
    probe = np.random.default_rng(seed).uniform(-1.0, 1.0, size=int(d))
    out = _solve_ranks([r], int(d), alpha, betas, tol, max_iter, probe, n1, n2)
    out["row_bounds"] = b
    out["rank"] = r
    return out


def time_sharded_solves(w, steps, warmup, flush, barrier, storage=64, e2e_steps=3):
    """bench.py --gpus N (strong scaling): the workload's rows sharded over
    the torch.distributed world.  Device time: CUDA events around `steps`
    solves on this rank's stream (max over ranks taken by the caller).  e2e:
    per step, this rank's shard re-uploaded from host memory, the solve, and
    the results read back (the communicator is kept).  Returns a dict."""
    import time as _time

    import torch
    import torch.distributed as dist

    world, rank = dist.get_world_size(), dist.get_rank()
    stream = torch.cuda.Stream()
    torch.cuda.set_stream(stream)
    out = solve_row_sharded(w.x_offsets, w.x_cols, w.d, w.l_offsets, w.l_cols, w.l_vals,
                            w.labels, w.alpha, w.betas, w.tol, w.max_iter, w.seed,
                            device=torch.cuda.current_device(), storage=storage,
                            stream=stream.cuda_stream)           # uploads + graph capture
    r = out["rank"]
    n1, n2 = _class_counts(w.labels)
    probe = w.probe()

    def solve(scores=False):
        return _solve_ranks([r], int(w.d), w.alpha, w.betas, w.tol, w.max_iter, probe, n1, n2,
                            scores=scores)

    for _ in range(max(0, warmup - 1)):
        solve()
    ms = 0.0
    for k in range(steps):
        flush.fill_(float(k))
        barrier()
        a, b_ = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record(stream)
        napp = solve()["n_applies"]   # result arrays released at once: their pinned
        b_.record(stream)             # blocks are reused by the next solve
        b_.synchronize()
        ms += a.elapsed_time(b_)
    assert napp == w.max_iter
    # e2e: host shard -> device, solve, directions + local scores -> host
    sh = r.shard
    res = solve(scores=True)     # warms the pinned result blocks (360 MB of scores at cfg3)
    barrier()
    t0 = _time.perf_counter()
    for _ in range(e2e_steps):
        res = None               # the previous results' pinned blocks go back to the cache
        r.reload(sh, out["row_bounds"], rank)
        res = solve(scores=True)
    barrier()
    e2e_s = (_time.perf_counter() - t0) / e2e_steps
    h2d = (sh.x_offsets.nbytes + sh.x_cols.nbytes + sh.l_offsets.nbytes + sh.l_cols.nbytes +
           sh.l_vals.nbytes + sh.labels.nbytes + 8 * w.d + 8 * w.betas.size)
    d2h = 8 * w.betas.size * (w.d + sh.n_local) + 24 * w.betas.size
    b = out["row_bounds"]
    ns = int(w.betas.size)
    # kernels per solve: setup 14, per iteration K1 K2 K3 rank-sum K4 shift (6),
    # tail 9 (+ the all-gather / send-recv copies, which are NCCL's)
    launches = 14 + 6 * int(w.max_iter) + 9
    info = (f"rows {int(b[rank])}..{int(b[rank + 1])} of {w.n} on rank {rank}; per iteration an NCCL "
            f"all-gather of y and a send/recv reduce-scatter + all-gather of the D+1 partials, "
            f"captured with the kernels in one CUDA graph")
    return {"ms": ms, "launches_per_solve": launches, "info": info, "e2e_s": e2e_s,
            "h2d_bytes": int(h2d), "d2h_bytes": int(d2h), "n_shifts": ns}
