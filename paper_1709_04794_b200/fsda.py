"""Drop-in FSDA solver on the B200: the host side of the hot path.

``fsda_solve(p)`` has the signature and result of the reference's
``sdakit.sda.fsda_solve`` (/root/reference/pkg/src/sdakit/sda.py:293-320) and
can be registered as its ``_SOLVERS["fsda"]`` entry (sda.py:465-486).  The
whole computation — labeled mean, rhs, the shifted-CG sweep over every beta
and the per-shift projections — runs on the device through the C ABI in
include/fsda_b200.h; this module only validates, uploads, and builds the
report.  It accepts the reference's own objects (duck-typed) and, when the
problem comes from sdakit, returns sdakit's report / exception classes.
"""

from __future__ import annotations

import ctypes as C
import importlib
import threading
import time
import types as _pytypes
from dataclasses import dataclass
from typing import Optional

import numpy as np

from . import _capi
from . import types as T

ALGORITHMS = ("fsda", "lda", "sa-sda")


# ------------------------------------------------------------ API families

def _family(obj) -> _pytypes.SimpleNamespace:
    """Classes to build results / raise errors with: sdakit's when the
    problem object comes from sdakit, else this package's."""
    mod = type(obj).__module__ or ""
    root = mod.split(".")[0]
    if root == "sdakit":
        sda = importlib.import_module("sdakit.sda")
        kry = importlib.import_module("sdakit.krylov")
        spm = importlib.import_module("sdakit.sparse")
        return _pytypes.SimpleNamespace(
            SolveReport=sda.SolveReport, PhaseStats=sda.PhaseStats,
            RatingVector=sda.RatingVector, ShiftedSolveResult=kry.ShiftedSolveResult,
            SolverBreakdownError=kry.SolverBreakdownError,
            NumericalFailureError=kry.NumericalFailureError, LabelError=spm.LabelError,
            CenteringVector=spm.CenteringVector)
    return _pytypes.SimpleNamespace(
        SolveReport=T.SolveReport, PhaseStats=T.PhaseStats, RatingVector=T.RatingVector,
        ShiftedSolveResult=T.ShiftedSolveResult, SolverBreakdownError=T.SolverBreakdownError,
        NumericalFailureError=T.NumericalFailureError, LabelError=T.LabelError,
        CenteringVector=T.CenteringVector)


_OWN = _family(None)


def _raise_for(rc: int, fam=_OWN):
    if rc == _capi.FSDA_OK:
        return
    msg = _capi.last_error()
    if rc == _capi.FSDA_EINVAL:
        raise ValueError(msg)
    if rc == _capi.FSDA_ELABEL:
        raise fam.LabelError(msg)
    if rc == _capi.FSDA_EBREAKDOWN:
        raise fam.SolverBreakdownError(msg)
    if rc == _capi.FSDA_ENONFINITE:
        raise fam.NumericalFailureError(msg)
    raise RuntimeError(f"fsda_b200: {msg}")


def _f64(a) -> np.ndarray:
    return np.ascontiguousarray(a, dtype=np.float64)


def _i64(a) -> np.ndarray:
    return np.ascontiguousarray(a, dtype=np.int64)


# ------------------------------------------------------------------ device

@dataclass
class SweepResult:
    """Raw device outputs of one solve (rows are shifts)."""

    directions: np.ndarray   # n_shifts x D
    scores: Optional[np.ndarray]  # n_shifts x N
    residuals: np.ndarray
    iterations: np.ndarray
    converged: np.ndarray
    n_applies: int
    launches: int = 0


_ONES_CACHE: dict = {}   # id(values array) -> (weakref, all-ones?) for read-only arrays


def _all_ones(values) -> bool:
    """Every stored value of X equals 1 (the reference's SparseMatrix keeps
    explicit float64 values, sparse.py:43-58, and has no binary flag): checked
    by all host threads in C, and remembered per read-only array — the
    reference freezes its arrays, so the answer cannot change."""
    v = np.ascontiguousarray(values, dtype=np.float64)
    frozen = v is values and not v.flags.writeable
    if frozen:
        hit = _ONES_CACHE.get(id(v))
        if hit is not None and hit[0]() is v:
            return hit[1]
    ok = bool(_capi.lib().fsda_values_all_ones(_capi.dptr(v), int(v.size)))
    if frozen:
        import weakref

        key = id(v)
        _ONES_CACHE[key] = (weakref.ref(v, lambda _r, k=key: _ONES_CACHE.pop(k, None)), ok)
    return ok


def _pinned_empty(shape) -> np.ndarray:
    """A float64 host array in page-locked memory, from torch's caching host
    allocator, so the result copies (directions, scores) run at link speed
    instead of through a pageable bounce buffer.  It is an ordinary ndarray
    to the caller and is recycled when the caller drops it.  Plain numpy
    memory when torch is absent (this changes where results land, not how
    they are computed)."""
    try:
        import torch
    except ImportError:  # pragma: no cover - torch ships with this image
        return np.empty(shape)
    return torch.empty(shape, dtype=torch.float64, pin_memory=True).numpy()


class Device:
    """One fsda context (device buffers, stream, cached solve graph)."""

    def __init__(self, device: int = 0, stream: Optional[int] = None):
        h = C.c_void_p()
        rc = _capi.lib().fsda_ctx_create(C.byref(h), int(device), C.c_void_p(stream) if stream else None)
        _raise_for(rc)
        self._h = h
        self.device = device
        self.n = self.d = 0
        self._loaded = (None, None, None)

    def close(self):
        if getattr(self, "_h", None) is not None and self._h.value:
            _capi.lib().fsda_ctx_destroy(self._h)
            self._h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    def set_shift_update_mode(self, mode: int):
        """0 auto (deferred basis when it fits), 1 per-iteration shift
        updates, 2 deferred basis (include/fsda_b200.h)."""
        _raise_for(_capi.lib().fsda_set_shift_update_mode(self._h, int(mode)))

    def set_eager(self, eager: bool = True):
        """Launch solves kernel by kernel instead of through the cached CUDA
        graph (same kernels, same results; for profilers)."""
        _raise_for(_capi.lib().fsda_set_eager(self._h, int(bool(eager))))

    def set_storage(self, bits: int):
        """64 (default) or 32: fp32 storage of the solve's vectors with fp64
        reductions (BASELINE cfg5; include/fsda_b200.h)."""
        _raise_for(_capi.lib().fsda_set_storage(self._h, int(bits)))
        self.storage_bits = int(bits)

    @property
    def last_shift_update_mode(self) -> int:
        return int(_capi.lib().fsda_last_shift_update_mode(self._h))

    def set_stream(self, stream: Optional[int]):
        _raise_for(_capi.lib().fsda_ctx_set_stream(self._h, C.c_void_p(stream) if stream else None))

    # ---- uploads
    def upload_x(self, x, fam=_OWN):
        binary = x.is_binary if hasattr(x, "is_binary") else _all_ones(x.values)
        if not binary:
            raise ValueError("the B200 FSDA path needs a binary X (every stored value 1)")
        offs, cols = _i64(x.row_offsets), _i64(x.col_indices)
        _raise_for(_capi.lib().fsda_upload_x(self._h, int(x.n_rows), int(x.n_cols),
                                             _capi.i64ptr(offs), _capi.i64ptr(cols)), fam)
        self.n, self.d = int(x.n_rows), int(x.n_cols)

    def upload_laplacian(self, lap, fam=_OWN):
        m = lap.matrix if hasattr(lap, "matrix") else lap
        offs, cols, vals = _i64(m.row_offsets), _i64(m.col_indices), _f64(m.values)
        _raise_for(_capi.lib().fsda_upload_laplacian(self._h, int(m.n_rows), _capi.i64ptr(offs),
                                                     _capi.i64ptr(cols), _capi.dptr(vals)), fam)

    def set_labels(self, labels, fam=_OWN):
        lab = np.ascontiguousarray(getattr(labels, "labels", labels), dtype=np.int8)
        if lab.size != self.n:
            raise ValueError(f"labels cover {lab.size} samples but x has {self.n} rows")
        _raise_for(_capi.lib().fsda_set_labels(self._h, _capi.i8ptr(lab)), fam)

    def set_label_mask(self, labels, fam=_OWN):
        """Labels in any row order (the nested-CV mask form, no labeled-first
        requirement)."""
        lab = np.ascontiguousarray(getattr(labels, "labels", labels), dtype=np.int8)
        if lab.size != self.n:
            raise ValueError(f"labels cover {lab.size} samples but x has {self.n} rows")
        _raise_for(_capi.lib().fsda_set_label_mask(self._h, _capi.i8ptr(lab)), fam)
        self._loaded = (self._loaded[0], self._loaded[1], None)

    def load_problem(self, p, fam=_OWN, reuse: bool = False):
        """Upload p.x, p.lap and p.labels.  With reuse=True, objects already
        resident (same immutable objects as the last load) are not re-sent."""
        last_x, last_l, last_lab = self._loaded
        # a failed upload leaves the device state unknown: nothing counts as
        # resident until this load succeeds
        self._loaded = (None, None, None)
        if not (reuse and (p.x is last_x or p.lap is last_l)):
            # all three travel: one call, L's copies overlapped with X's processing
            x, m = p.x, (p.lap.matrix if hasattr(p.lap, "matrix") else p.lap)
            binary = x.is_binary if hasattr(x, "is_binary") else _all_ones(x.values)
            if not binary:
                raise ValueError("the B200 FSDA path needs a binary X (every stored value 1)")
            if int(m.n_rows) != int(x.n_rows):
                raise ValueError("laplacian must be square with one row per sample")
            lab = np.ascontiguousarray(getattr(p.labels, "labels", p.labels), dtype=np.int8)
            if lab.size != int(x.n_rows):
                raise ValueError(f"labels cover {lab.size} samples but x has {int(x.n_rows)} rows")
            xo, xc = _i64(x.row_offsets), _i64(x.col_indices)
            lo, lc, lv = _i64(m.row_offsets), _i64(m.col_indices), _f64(m.values)
            _raise_for(_capi.lib().fsda_upload_problem(
                self._h, int(x.n_rows), int(x.n_cols), _capi.i64ptr(xo), _capi.i64ptr(xc),
                _capi.i64ptr(lo), _capi.i64ptr(lc), _capi.dptr(lv), _capi.i8ptr(lab)), fam)
            self.n, self.d = int(x.n_rows), int(x.n_cols)
            self._loaded = (p.x, p.lap, p.labels)
            return
        if not (reuse and p.x is last_x):
            self.upload_x(p.x, fam)
            last_l = last_lab = None
        if not (reuse and p.lap is last_l):
            self.upload_laplacian(p.lap, fam)
        if not (reuse and p.labels is last_lab):
            self.set_labels(p.labels, fam)
        self._loaded = (p.x, p.lap, p.labels)

    # ---- single products (parity probes)
    def matvec(self, v) -> np.ndarray:
        v = _f64(v)
        if v.shape != (self.d,):
            raise ValueError(f"matvec expects a vector of length {self.d}, got {v.shape}")
        out = np.empty(self.n)
        _raise_for(_capi.lib().fsda_matvec(self._h, _capi.dptr(v), _capi.dptr(out)))
        return out

    def matvec_transpose(self, w) -> np.ndarray:
        w = _f64(w)
        if w.shape != (self.n,):
            raise ValueError(f"matvec_transpose expects a vector of length {self.n}, got {w.shape}")
        out = np.empty(self.d)
        _raise_for(_capi.lib().fsda_matvec_transpose(self._h, _capi.dptr(w), _capi.dptr(out)))
        return out

    def labeled_mean(self, fam=_OWN) -> np.ndarray:
        out = np.empty(self.d)
        _raise_for(_capi.lib().fsda_labeled_mean(self._h, _capi.dptr(out)), fam)
        return out

    def centered_matvec_transpose(self, mu, w) -> np.ndarray:
        mu, w = _f64(mu), _f64(w)
        out = np.empty(self.d)
        _raise_for(_capi.lib().fsda_centered_matvec_transpose(self._h, _capi.dptr(mu), _capi.dptr(w),
                                                              _capi.dptr(out)))
        return out

    def apply_smoother(self, alpha: float, z) -> np.ndarray:
        z = _f64(z)
        out = np.empty(self.n)
        _raise_for(_capi.lib().fsda_apply_smoother(self._h, float(alpha), _capi.dptr(z), _capi.dptr(out)))
        return out

    def operator_apply(self, alpha: float, w) -> np.ndarray:
        w = _f64(w)
        out = np.empty(self.d)
        _raise_for(_capi.lib().fsda_operator_apply(self._h, float(alpha), _capi.dptr(w), _capi.dptr(out)))
        return out

    # ---- the sweep
    def solve_fsda(self, alpha, betas, tol, max_iter, probe, *, scores=True, fam=_OWN) -> SweepResult:
        betas = _f64(betas)
        ns = int(betas.size)
        probe = _f64(probe)
        if probe.shape != (self.d,):
            raise ValueError("probe must have one entry per feature")
        dirs = _pinned_empty((ns, self.d))
        sc = _pinned_empty((ns, self.n)) if scores else None
        res = np.empty(ns)
        its = np.empty(ns, dtype=np.int64)
        conv = np.empty(ns, dtype=np.uint8)
        napp = C.c_int64(0)
        fail = C.c_int64(-1)
        rc = _capi.lib().fsda_solve(
            self._h, float(alpha), _capi.dptr(betas), ns, float(tol), int(max_iter), _capi.dptr(probe),
            _capi.dptr(dirs), _capi.dptr(sc), _capi.dptr(res), _capi.i64ptr(its), _capi.u8ptr(conv),
            C.byref(napp), C.byref(fail))
        _raise_for(rc, fam)
        return SweepResult(dirs, sc, res, its, conv.astype(bool), int(napp.value))

    def solve_batch(self, label_sets, alpha, betas, tol, max_iter, probes, *, scores=True,
                    fam=_OWN) -> list:
        """T sweeps in one batched pass (fsda_solve_batch): task t uses label
        mask label_sets[t] (any row order) and probe probes[t].  Each result
        equals set_label_mask + solve_fsda for that task, bit for bit."""
        lab = np.ascontiguousarray(np.asarray(label_sets, dtype=np.int8))
        probes = _f64(probes)
        if lab.ndim != 2 or lab.shape[1] != self.n:
            raise ValueError("label_sets must be n_tasks x N")
        T = lab.shape[0]
        if probes.shape != (T, self.d):
            raise ValueError("probes must be n_tasks x D")
        betas = _f64(betas)
        ns = int(betas.size)
        dirs = _pinned_empty((T, ns, self.d))
        sc = _pinned_empty((T, ns, self.n)) if scores else None
        res = np.empty((T, ns))
        its = np.empty((T, ns), dtype=np.int64)
        conv = np.empty((T, ns), dtype=np.uint8)
        napp = np.empty(T, dtype=np.int64)
        fail = np.empty(T, dtype=np.int64)
        status = np.empty(T, dtype=np.int32)
        rc = _capi.lib().fsda_solve_batch(
            self._h, T, _capi.i8ptr(lab), float(alpha), _capi.dptr(betas), ns, float(tol),
            int(max_iter), _capi.dptr(probes), _capi.dptr(dirs), _capi.dptr(sc), _capi.dptr(res),
            _capi.i64ptr(its), _capi.u8ptr(conv), _capi.i64ptr(napp), _capi.i64ptr(fail),
            status.ctypes.data_as(C.POINTER(C.c_int)))
        _raise_for(rc, fam)
        for t in range(T):
            if status[t] == _capi.FSDA_EBREAKDOWN:
                raise fam.SolverBreakdownError(
                    f"task {t}: singular direction: <p, Bp> = 0 at iteration {fail[t]}")
            if status[t] == _capi.FSDA_ENONFINITE:
                raise fam.NumericalFailureError(
                    f"task {t}: non-finite <p, Bp> or residual at iteration {fail[t]}")
        return [SweepResult(dirs[t], None if sc is None else sc[t], res[t], its[t],
                            conv[t].astype(bool), int(napp[t])) for t in range(T)]

    def prepare_resident(self, alpha, betas, tol, max_iter, probe):
        betas, probe = _f64(betas), _f64(probe)
        self._res_ns = int(betas.size)
        _raise_for(_capi.lib().fsda_prepare_resident(self._h, float(alpha), _capi.dptr(betas),
                                                     self._res_ns, float(tol), int(max_iter),
                                                     _capi.dptr(probe)))

    def solve_async(self):
        _raise_for(_capi.lib().fsda_solve_async(self._h))

    def fetch(self, *, directions=True, scores=True) -> SweepResult:
        ns = self._res_ns
        dirs = _pinned_empty((ns, self.d)) if directions else None
        sc = _pinned_empty((ns, self.n)) if scores else None
        res = np.empty(ns)
        its = np.empty(ns, dtype=np.int64)
        conv = np.empty(ns, dtype=np.uint8)
        napp, fail, launches = C.c_int64(0), C.c_int64(-1), C.c_int64(0)
        _raise_for(_capi.lib().fsda_fetch_results(
            self._h, _capi.dptr(dirs), _capi.dptr(sc), _capi.dptr(res), _capi.i64ptr(its),
            _capi.u8ptr(conv), C.byref(napp), C.byref(fail), C.byref(launches)))
        return SweepResult(dirs, sc, res, its, conv.astype(bool), int(napp.value), int(launches.value))

    def profile_kernels(self, max_kernels: int = 64) -> list[dict]:
        n = C.c_int(0)
        names = (C.c_char_p * max_kernels)()
        ms = np.zeros(max_kernels)
        by = np.zeros(max_kernels)
        cnt = np.zeros(max_kernels, dtype=np.int64)
        _raise_for(_capi.lib().fsda_profile_kernels(self._h, max_kernels, C.byref(n), names,
                                                    _capi.dptr(ms), _capi.dptr(by), _capi.i64ptr(cnt)))
        return [dict(name=names[k].decode(), ms=float(ms[k]), bytes=float(by[k]),
                     launches=int(cnt[k])) for k in range(n.value)]

    def shifted_cg_dense(self, a, b, betas, tol=1e-8, max_iter=1000, absolute_tol=False, fam=_OWN):
        a = _f64(a)
        b = _f64(b)
        betas = _f64(betas)
        dim, ns = int(b.size), int(betas.size)
        sols = np.empty((ns, dim))
        res = np.empty(ns)
        its = np.empty(ns, dtype=np.int64)
        conv = np.empty(ns, dtype=np.uint8)
        napp, fail = C.c_int64(0), C.c_int64(-1)
        rc = _capi.lib().fsda_shifted_cg_dense(
            self._h, dim, _capi.dptr(a), _capi.dptr(b), _capi.dptr(betas), ns, float(tol),
            int(max_iter), int(bool(absolute_tol)), _capi.dptr(sols), _capi.dptr(res),
            _capi.i64ptr(its), _capi.u8ptr(conv), C.byref(napp), C.byref(fail))
        _raise_for(rc, fam)
        return sols, res, its, conv.astype(bool), int(napp.value)


_devices: dict[int, Device] = {}


def default_device(index: Optional[int] = None) -> Device:
    """The process-wide context of device `index` (default: LOCAL_RANK or 0)."""
    import os

    if index is None:
        index = int(os.environ.get("FSDA_B200_DEVICE", os.environ.get("LOCAL_RANK", "0")))
    dev = _devices.get(index)
    if dev is None:
        dev = Device(index)
        _devices[index] = dev
    return dev


# ------------------------------------------------------------ drop-in API

def _report(p, res: SweepResult, fam, t0: float, algorithm: str = "fsda"):
    betas = np.asarray(p.betas.betas)
    ratings, directions = {}, {}
    for s, beta in enumerate(betas):
        ratings[float(beta)] = fam.RatingVector(scores=res.scores[s], source="projection")
        directions[float(beta)] = res.directions[s]
    return fam.SolveReport(
        algorithm=algorithm, alpha=p.alpha, betas=betas, ratings=ratings, directions=directions,
        spectral=None,
        regression=fam.PhaseStats(dimension=int(p.x.n_cols), iterations=res.iterations,
                                  operator_applications=res.n_applies, residuals=res.residuals,
                                  converged=res.converged),
        wall_time_s=time.perf_counter() - t0)


def fsda_solve(p, *, device: Optional[Device] = None, storage: Optional[int] = None) -> "T.SolveReport":
    """One shifted Krylov solve of the centred rating operator in feature
    space for every beta of p.betas, rating s = X w per shift — on the GPU.

    Drop-in for sdakit.sda.fsda_solve (sda.py:293-320): same probe draw
    (default_rng(p.seed).uniform(-1, 1, D), sda.py:297-300), same report
    fields, same exceptions.  storage=32 runs the fp32-storage mode (fp64
    reductions; BASELINE cfg5) for this call; the default keeps the device's
    setting (fp64 unless Device.set_storage(32))."""
    t0 = time.perf_counter()
    fam = _family(p)
    dev = device or default_device()
    # the probe draw (a few ms of one core at D ~ 10^5..10^6) runs beside the
    # upload, which spends its time in C with the GIL released
    drawn = {}

    def _draw(quiet=True):
        try:
            drawn["probe"] = np.random.default_rng(p.seed).uniform(-1.0, 1.0, size=int(p.x.n_cols))
        except Exception:
            if not quiet:
                raise

    th = threading.Thread(target=_draw)
    th.start()
    try:
        dev.load_problem(p, fam)
    finally:
        th.join()
    if "probe" not in drawn:   # the draw failed (e.g. a bad seed): raise it here, as the reference does
        _draw(quiet=False)
    probe = drawn["probe"]
    prev = getattr(dev, "storage_bits", 64)
    if storage is not None and int(storage) != prev:
        dev.set_storage(int(storage))
    try:
        res = dev.solve_fsda(p.alpha, p.betas.betas, p.tol, p.max_iter_d, probe, fam=fam)
    finally:
        if storage is not None and int(storage) != prev:
            dev.set_storage(prev)
    return _report(p, res, fam, t0)


def orthogonalized_probe(p) -> np.ndarray:
    """The reference's sample-space probe (sda.py:287-290): r ~ U(-1, 1)^N
    from default_rng(p.seed), minus its labeled mean."""
    lab = np.asarray(p.labels.labels)
    mask = lab != 0
    r = np.random.default_rng(p.seed).uniform(-1.0, 1.0, size=lab.size)
    return r - r[mask].sum() / int(mask.sum())


def sa_sda_solve(p, *, device: Optional[Device] = None) -> "T.SolveReport":
    """SA-SDA on the device (sda.py:360-396): one shifted CG in sample
    space on the centred spectral operator for every beta; the oriented
    solutions are the ratings (source "spectral")."""
    fam = _family(p)
    if p.alpha == 0.0:
        raise ValueError("sa-sda requires alpha != 0: without the Laplacian term the "
                         "spectral system never propagates ratings to unlabeled samples")
    t0 = time.perf_counter()
    dev = device or default_device()
    dev.load_problem(p, fam)
    betas = _f64(p.betas.betas)
    ns, n = int(betas.size), int(p.x.n_rows)
    probe = _f64(orthogonalized_probe(p))
    sols = np.empty((ns, n))
    res = np.empty(ns)
    its = np.empty(ns, dtype=np.int64)
    conv = np.empty(ns, dtype=np.uint8)
    napp, fail = C.c_int64(0), C.c_int64(-1)
    tol = p.tol if getattr(p, "tol_spectral", None) is None else p.tol_spectral
    rc = _capi.lib().fsda_sa_solve(dev._h, float(p.alpha), _capi.dptr(betas), ns, float(tol),
                                   int(p.max_iter_n), _capi.dptr(probe), _capi.dptr(sols),
                                   _capi.dptr(res), _capi.i64ptr(its), _capi.u8ptr(conv),
                                   C.byref(napp), C.byref(fail))
    _raise_for(rc, fam)
    ratings = {float(b): fam.RatingVector(scores=sols[s], source="spectral")
               for s, b in enumerate(betas)}
    return fam.SolveReport(
        algorithm="sa-sda", alpha=p.alpha, betas=np.asarray(p.betas.betas), ratings=ratings,
        spectral=fam.PhaseStats(dimension=n, iterations=its, operator_applications=int(napp.value),
                                residuals=res, converged=conv.astype(bool)),
        regression=None, wall_time_s=time.perf_counter() - t0,
        spectral_vectors=np.ascontiguousarray(sols.T))


def solve(p, algorithm: str = "fsda") -> "T.SolveReport":
    """Dispatch like sdakit.sda.solve (sda.py:473-486) for the algorithms on
    the B200 path: 'fsda', and 'lda' = fsda constrained to alpha = 0."""
    if algorithm == "lda":
        if p.alpha != 0.0:
            raise ValueError(f"algorithm 'lda' is fsda at alpha = 0, but alpha = {p.alpha}; "
                             "drop the alpha setting or use fsda")
        rep = fsda_solve(p)
        rep.algorithm = "lda"
        return rep
    if algorithm == "fsda":
        return fsda_solve(p)
    if algorithm == "sa-sda":
        return sa_sda_solve(p)
    raise ValueError(f"unknown algorithm {algorithm!r} for the B200 path; choose from {ALGORITHMS}")


def install_into_sdakit(sda_module=None, algorithms=("fsda", "sa-sda")):
    """Register the device solvers in the reference's table
    (sdakit.sda._SOLVERS, sda.py:465-470).  'lda' follows 'fsda'
    automatically because the reference's solve() calls the module-level
    fsda_solve name."""
    sda = sda_module or importlib.import_module("sdakit.sda")
    if "fsda" in algorithms:
        sda._SOLVERS["fsda"] = fsda_solve
        sda.fsda_solve = fsda_solve
    if "sa-sda" in algorithms:
        sda._SOLVERS["sa-sda"] = sa_sda_solve
        sda.sa_sda_solve = sa_sda_solve
    return sda


class DeviceProblem:
    """A problem kept resident on the device across solves (X, L, labels
    uploaded once), e.g. for beta/alpha sweeps on one dataset."""

    def __init__(self, p, device: Optional[Device] = None):
        self.p = p
        self.fam = _family(p)
        self.dev = device or default_device()
        self.dev.load_problem(p, self.fam)

    def solve(self, *, alpha=None, betas=None, tol=None, max_iter=None, seed=None):
        t0 = time.perf_counter()
        p = self.p
        alpha = p.alpha if alpha is None else alpha
        grid = p.betas if betas is None else T.as_shift_grid(betas)
        seed = p.seed if seed is None else seed
        probe = np.random.default_rng(seed).uniform(-1.0, 1.0, size=int(p.x.n_cols))
        self.dev.load_problem(p, self.fam, reuse=True)
        res = self.dev.solve_fsda(alpha, grid.betas, p.tol if tol is None else tol,
                                  p.max_iter_d if max_iter is None else max_iter, probe, fam=self.fam)
        q = _pytypes.SimpleNamespace(betas=grid, alpha=alpha, x=p.x)
        return _report(q, res, self.fam, t0)


def solve_label_sets(x, lap, label_sets, alpha, betas, tol: float = 1e-8, max_iter: int = 1000,
                     seeds=0, *, device: Optional[Device] = None, scores: bool = True,
                     batched: bool = True):
    """Many FSDA sweeps on one dataset: X and L are uploaded once and every
    label set (any row order — a mask, as the folds of nested CV) is solved
    against them.  Each result is what fsda_solve returns for that task after
    the reference's arrange_labeled_first permutation and its undo
    (evaluation.py:110-123), up to the summation order of the permuted rows.

    batched=True solves all label sets in one pass (fsda_solve_batch: every
    operator product serves all tasks); batched=False solves them one after
    the other.  The results are identical.

    Returns a list of SweepResult (directions n_shifts x D, scores n_shifts x N
    in the original row order)."""
    grid = T.as_shift_grid(betas)
    sets = [np.asarray(getattr(l, "labels", l), dtype=np.int8) for l in label_sets]
    seed_list = list(seeds) if np.ndim(seeds) else [int(seeds)] * len(sets)
    if len(seed_list) != len(sets):
        raise ValueError("one seed per label set")
    for lab in sets:
        if lab.shape != (int(x.n_rows),):
            raise ValueError("every label set needs one entry per sample")
        if not (np.any(lab == 1) and np.any(lab == -1)):
            raise ValueError("both classes need at least one labeled sample")
    dev = device or default_device()
    dev.upload_x(x)
    dev.upload_laplacian(lap)
    probes = [np.random.default_rng(seed).uniform(-1.0, 1.0, size=int(x.n_cols)) for seed in seed_list]
    if batched and sets:
        out = dev.solve_batch(np.stack(sets), alpha, grid.betas, tol, max_iter, np.stack(probes),
                              scores=scores)
    else:
        out = []
        for lab, probe in zip(sets, probes):
            dev.set_label_mask(lab)
            out.append(dev.solve_fsda(alpha, grid.betas, tol, max_iter, probe, scores=scores))
    dev._loaded = (None, None, None)
    return out


# ----------------------------------------------- device parity primitives

def _dev_with_x(x, labels=None, lap=None) -> Device:
    dev = default_device()
    dev.upload_x(x)
    if lap is not None:
        dev.upload_laplacian(lap)
    if labels is not None:
        dev.set_labels(labels)
    dev._loaded = (None, None, None)
    return dev


def matvec(x, v) -> np.ndarray:
    """X v on the device (SparseMatrix.matvec, sparse.py:116-121)."""
    return _dev_with_x(x).matvec(v)


def matvec_transpose(x, w) -> np.ndarray:
    """X^T w on the device (SparseMatrix.matvec_transpose, sparse.py:123-134)."""
    return _dev_with_x(x).matvec_transpose(w)


def labeled_mean(x, labels):
    """mu = X^T 1_l / l on the device (labeled_mean, sparse.py:258-265)."""
    fam = _family(labels)
    lab = getattr(labels, "labels", labels)
    if int(np.count_nonzero(np.asarray(lab))) == 0:
        raise fam.LabelError("centering requires at least one labeled sample")
    dev = _dev_with_x(x, labels)
    return fam.CenteringVector(mu=dev.labeled_mean(fam), n_labeled=int(np.count_nonzero(lab)))


def centered_matvec_transpose(x, c, w) -> np.ndarray:
    """X^T w - mu sum(w) on the device (sparse.py:274-277)."""
    return _dev_with_x(x).centered_matvec_transpose(c.mu, w)


def apply_smoother(labels, lap, alpha, z) -> np.ndarray:
    """[(1-alpha)(I_l + 0) + alpha L] z on the device (sda.py:131-140)."""
    m = lap.matrix
    dev = default_device()
    n = int(m.n_rows)
    # The smoother needs only L and the labels; a zero-column X of matching height
    # satisfies the context's shape checks.
    dev.upload_x(T.SparseMatrix(n, 1, np.zeros(n + 1, dtype=np.int64), np.zeros(0, np.int64),
                                np.zeros(0)))
    dev.upload_laplacian(lap)
    dev.set_labels(labels)
    dev._loaded = (None, None, None)
    return dev.apply_smoother(alpha, z)


def fsda_operator_apply(p, w) -> np.ndarray:
    """w -> (X - 1 mu^T)^T M X w on the device (fsda_operator, sda.py:162-174)."""
    dev = default_device()
    dev.load_problem(p, _family(p))
    return dev.operator_apply(p.alpha, w)


class LinearOperator:
    """Counting operator wrapper (krylov.py:44-66).  Only dense operators
    (from_dense) can run on the device shifted CG."""

    def __init__(self, dim: int, apply_fn=None, *, dense: Optional[np.ndarray] = None):
        if dim <= 0:
            raise ValueError("operator dimension must be positive")
        self.dim = int(dim)
        self._apply = apply_fn
        self.dense = dense
        self.n_applies = 0

    def __call__(self, v):
        self.n_applies += 1
        if self._apply is not None:
            return self._apply(v)
        return self.dense @ v

    def reset_count(self):
        self.n_applies = 0

    @classmethod
    def from_dense(cls, a) -> "LinearOperator":
        a = np.asarray(a, dtype=np.float64)
        if a.ndim != 2 or a.shape[0] != a.shape[1]:
            raise ValueError("from_dense expects a square matrix")
        return cls(a.shape[0], dense=a)


class RegressionOperator:
    """w -> X^T X w (regression_operator, sda.py:177-179) held on the device;
    shifted_cg on it runs the whole grid in one device solve (the regression
    phase of CSR-SDA / SR-SDA and bench_shifted, evaluation.py:288-291)."""

    def __init__(self, x, device: Optional[Device] = None):
        self.x = x
        self.dim = int(x.n_cols)
        self.dev = device or default_device()
        self.n_applies = 0

    def _load(self):
        self.dev.upload_x(self.x)
        self.dev._loaded = (None, None, None)

    def __call__(self, w):
        self._load()
        self.n_applies += 1
        return self.dev.matvec_transpose(self.dev.matvec(w))

    def reset_count(self):
        self.n_applies = 0

    def solve(self, b, betas, tol, max_iter, absolute_tol=False, fam=_OWN):
        self._load()
        b = _f64(b)
        betas = _f64(betas)
        ns = int(betas.size)
        sols = np.empty((ns, self.dim))
        res = np.empty(ns)
        its = np.empty(ns, dtype=np.int64)
        conv = np.empty(ns, dtype=np.uint8)
        napp, fail = C.c_int64(0), C.c_int64(-1)
        rc = _capi.lib().fsda_regression_shifted_cg(
            self.dev._h, _capi.dptr(b), _capi.dptr(betas), ns, float(tol), int(max_iter),
            int(bool(absolute_tol)), _capi.dptr(sols), _capi.dptr(res), _capi.i64ptr(its),
            _capi.u8ptr(conv), C.byref(napp), C.byref(fail))
        _raise_for(rc, fam)
        self.n_applies += int(napp.value)
        return sols, res, its, conv.astype(bool), int(napp.value)


def regression_operator(p_or_x, device: Optional[Device] = None) -> RegressionOperator:
    """The regression operator X^T X of a problem (or of a SparseMatrix)."""
    x = getattr(p_or_x, "x", p_or_x)
    return RegressionOperator(x, device)


def shifted_cg(op, b, shifts, tol: float = 1e-8, max_iter: int = 1000, *,
               absolute_tol: bool = False) -> T.ShiftedSolveResult:
    """Device shifted CG (krylov.py:168-281) for a dense operator: same
    recurrences, freezing rules and result fields; op.n_applies advances by
    the number of base iterations run."""
    grid = T.as_shift_grid(shifts)
    b = _f64(b)
    if b.shape != (op.dim,):
        raise ValueError(f"rhs must have shape ({op.dim},)")
    if tol <= 0:
        raise ValueError("tol must be positive")
    if isinstance(op, RegressionOperator):
        sols, res, its, conv, napp = op.solve(b, grid.betas, tol, max_iter, absolute_tol)
    else:
        dense = getattr(op, "dense", None)
        if dense is None:
            raise TypeError("device shifted_cg needs a device operator: LinearOperator.from_dense "
                            "or regression_operator (or use fsda_solve)")
        sols, res, its, conv, napp = default_device().shifted_cg_dense(
            dense, b, grid.betas, tol, max_iter, absolute_tol)
        op.n_applies += napp
    return T.ShiftedSolveResult(solutions=np.ascontiguousarray(sols.T), residual_norms=res,
                                iterations=its, converged=conv)
