"""ctypes wrapper of oracle/fsda_oracle.c (CPU ORACLE — test infrastructure).

See oracle/__init__.py for who may import this.  ``build()`` compiles the
library in-tree (oracle/build/, git-ignored, travels to the GPU box).
"""

from __future__ import annotations

import ctypes as C
import subprocess
from pathlib import Path

import numpy as np

HERE = Path(__file__).resolve().parent
SRC = HERE / "fsda_oracle.c"
LIB = HERE / "build" / "libfsda_oracle.so"

_PD = C.POINTER(C.c_double)
_PI64 = C.POINTER(C.c_int64)
_PI8 = C.POINTER(C.c_int8)
_PU8 = C.POINTER(C.c_uint8)
_I64 = C.c_int64

_lib = None


def build(force: bool = False) -> Path:
    if LIB.exists() and not force and LIB.stat().st_mtime >= SRC.stat().st_mtime:
        return LIB
    LIB.parent.mkdir(parents=True, exist_ok=True)
    subprocess.run(["gcc", "-O2", "-fopenmp", "-ffp-contract=off", "-fPIC", "-shared", "-o",
                    str(LIB), str(SRC), "-lm"], check=True)
    return LIB


def lib():
    global _lib
    if _lib is None:
        if not LIB.exists():
            build()
        h = C.CDLL(str(LIB))
        h.oracle_r256.restype = C.c_double
        h.oracle_r256.argtypes = [_PD, _I64]
        h.oracle_dot.restype = C.c_double
        h.oracle_dot.argtypes = [_PD, _PD, _I64]
        h.oracle_matvec.restype = None
        h.oracle_matvec.argtypes = [_I64, _PI64, _PI64, _PD, _PD]
        h.oracle_matvec_r256.restype = None
        h.oracle_matvec_r256.argtypes = [_I64, _PI64, _PI64, _PD, _PD]
        h.oracle_matvec_transpose.restype = None
        h.oracle_matvec_transpose.argtypes = [_I64, _I64, _PI64, _PI64, _PD, _PD]
        h.oracle_centered_matvec_transpose.restype = None
        h.oracle_centered_matvec_transpose.argtypes = [_I64, _I64, _PI64, _PI64, _PD, _PD, _PD]
        h.oracle_labeled_mean.restype = None
        h.oracle_labeled_mean.argtypes = [_I64, _I64, _PI64, _PI64, _PI8, _PD]
        h.oracle_apply_smoother.restype = C.c_double
        h.oracle_apply_smoother.argtypes = [_I64, _PI64, _PI64, _PD, _PI8, C.c_double, _PD, _PD]
        h.oracle_operator_apply.restype = None
        h.oracle_operator_apply.argtypes = [_I64, _I64, _PI64, _PI64, _PI64, _PI64, _PD, _PI8,
                                            C.c_double, _PD, _PD]
        h.oracle_shifted_cg_dense.restype = C.c_int
        h.oracle_shifted_cg_dense.argtypes = [_I64, _PD, _PD, _PD, C.c_int, C.c_double, _I64, C.c_int,
                                              _PD, _PD, _PI64, _PU8, _PI64, _PI64]
        h.oracle_regression_shifted_cg.restype = C.c_int
        h.oracle_regression_shifted_cg.argtypes = [_I64, _I64, _PI64, _PI64, _PD, _PD, C.c_int, C.c_double,
                                                   _I64, C.c_int, _PD, _PD, _PI64, _PU8, _PI64, _PI64]
        h.oracle_sa_solve.restype = C.c_int
        h.oracle_sa_solve.argtypes = [_I64, _PI64, _PI64, _PD, _PI8, C.c_double, _PD, C.c_int, C.c_double,
                                      _I64, _PD, _PD, _PD, _PI64, _PU8, _PI64, _PI64]
        h.oracle_fsda_solve.restype = C.c_int
        h.oracle_fsda_solve.argtypes = [_I64, _I64, _PI64, _PI64, _PI64, _PI64, _PD, _PI8, C.c_double,
                                        _PD, C.c_int, C.c_double, _I64, _PD, C.c_int, _PD, _PD, _PD,
                                        _PI64, _PU8, _PI64, _PI64]
        h.oracle_max_threads.restype = C.c_int
        h.oracle_max_threads.argtypes = []
        h.oracle_fsda_solve_sharded.restype = C.c_int
        h.oracle_fsda_solve_sharded.argtypes = [_I64, _I64, _PI64, _PI64, _PI64, _PI64, _PD, _PI8, C.c_double,
                                                _PD, C.c_int, C.c_double, _I64, _PD, C.c_int, C.c_int,
                                                _PI64, _PD, _PD, _PD, _PI64, _PU8, _PI64, _PI64]
        h.oracle_set_deferred.restype = None
        h.oracle_set_deferred.argtypes = [C.c_int]
        h.oracle_set_deferred(1 if _shift_mode == 2 else 0)
        h.oracle_set_storage.restype = None
        h.oracle_set_storage.argtypes = [C.c_int]
        h.oracle_set_storage(_storage_bits)
        _lib = h
    return _lib


# Shift-update mode mirrored from the device (fsda_set_shift_update_mode):
# 1 per-iteration sols / P updates, 2 deferred basis (the device default
# whenever the basis fits; tests force the device's mode to match).
_shift_mode = 2


def set_shift_mode(mode: int) -> None:
    global _shift_mode
    if mode not in (1, 2):
        raise ValueError("shift mode must be 1 or 2")
    _shift_mode = mode
    if _lib is not None:
        _lib.oracle_set_deferred(1 if mode == 2 else 0)


def shift_mode() -> int:
    return _shift_mode


# Storage precision of the FSDA vectors mirrored from the device
# (fsda_set_storage): 64, or 32 = fp32 storage with fp64 reductions.
_storage_bits = 64


def set_storage(bits: int) -> None:
    global _storage_bits
    if bits not in (32, 64):
        raise ValueError("storage must be 32 or 64 bits")
    _storage_bits = bits
    if _lib is not None:
        _lib.oracle_set_storage(bits)


def _d(a):
    a = np.ascontiguousarray(a, dtype=np.float64)
    return a, a.ctypes.data_as(_PD)


def _i(a):
    a = np.ascontiguousarray(a, dtype=np.int64)
    return a, a.ctypes.data_as(_PI64)


def _b(a):
    a = np.ascontiguousarray(a, dtype=np.int8)
    return a, a.ctypes.data_as(_PI8)


def r256(v) -> float:
    v, pv = _d(v)
    return lib().oracle_r256(pv, v.size)


def dot(x, y) -> float:
    x, px = _d(x)
    y, py = _d(y)
    return lib().oracle_dot(px, py, x.size)


def matvec(offs, cols, v):
    offs, po = _i(offs)
    cols, pc = _i(cols)
    v, pv = _d(v)
    n = offs.size - 1
    out = np.empty(n)
    lib().oracle_matvec(n, po, pc, pv, out.ctypes.data_as(_PD))
    return out


def matvec_r256(offs, cols, v):
    """X v with every row summed by the canonical R256 tree (the device's K1)."""
    offs, po = _i(offs)
    cols, pc = _i(cols)
    v, pv = _d(v)
    n = offs.size - 1
    out = np.empty(n)
    lib().oracle_matvec_r256(n, po, pc, pv, out.ctypes.data_as(_PD))
    return out


def matvec_transpose(offs, cols, d, w):
    offs, po = _i(offs)
    cols, pc = _i(cols)
    w, pw = _d(w)
    out = np.empty(d)
    lib().oracle_matvec_transpose(offs.size - 1, d, po, pc, pw, out.ctypes.data_as(_PD))
    return out


def centered_matvec_transpose(offs, cols, d, mu, w):
    offs, po = _i(offs)
    cols, pc = _i(cols)
    mu, pm = _d(mu)
    w, pw = _d(w)
    out = np.empty(d)
    lib().oracle_centered_matvec_transpose(offs.size - 1, d, po, pc, pm, pw, out.ctypes.data_as(_PD))
    return out


def labeled_mean(offs, cols, d, labels):
    offs, po = _i(offs)
    cols, pc = _i(cols)
    lab, pl = _b(labels)
    out = np.empty(d)
    lib().oracle_labeled_mean(offs.size - 1, d, po, pc, pl, out.ctypes.data_as(_PD))
    return out


def apply_smoother(loffs, lcols, lvals, labels, alpha, y):
    loffs, po = _i(loffs)
    lcols, pc = _i(lcols)
    lvals, pv = _d(lvals)
    lab, pl = _b(labels)
    y, py = _d(y)
    out = np.empty(y.size)
    lib().oracle_apply_smoother(y.size, po, pc, pv, pl, float(alpha), py, out.ctypes.data_as(_PD))
    return out


def operator_apply(xoffs, xcols, d, loffs, lcols, lvals, labels, alpha, w):
    xo, pxo = _i(xoffs)
    xc, pxc = _i(xcols)
    lo, plo = _i(loffs)
    lc, plc = _i(lcols)
    lv, plv = _d(lvals)
    lab, pl = _b(labels)
    w, pw = _d(w)
    out = np.empty(d)
    lib().oracle_operator_apply(xo.size - 1, d, pxo, pxc, plo, plc, plv, pl, float(alpha), pw,
                                out.ctypes.data_as(_PD))
    return out


class OracleFailure(RuntimeError):
    def __init__(self, status, fail_iter):
        super().__init__(f"oracle status {status} at iteration {fail_iter}")
        self.status = status
        self.fail_iter = fail_iter


def shifted_cg_dense(a, b, betas, tol=1e-8, max_iter=1000, absolute_tol=False):
    a, pa = _d(a)
    b, pb = _d(b)
    betas, pbe = _d(betas)
    ns, dim = betas.size, b.size
    sols = np.empty((ns, dim))
    res = np.empty(ns)
    its = np.empty(ns, dtype=np.int64)
    conv = np.empty(ns, dtype=np.uint8)
    napp, fail = C.c_int64(0), C.c_int64(-1)
    st = lib().oracle_shifted_cg_dense(dim, pa, pb, pbe, ns, float(tol), int(max_iter),
                                       int(bool(absolute_tol)), sols.ctypes.data_as(_PD),
                                       res.ctypes.data_as(_PD), its.ctypes.data_as(_PI64),
                                       conv.ctypes.data_as(_PU8), C.byref(napp), C.byref(fail))
    if st:
        raise OracleFailure(st, fail.value)
    return sols, res, its, conv.astype(bool), napp.value


def regression_shifted_cg(xoffs, xcols, d, b, betas, tol=1e-8, max_iter=1000, absolute_tol=False):
    """shifted_cg on X^T X (the regression phase) in the device's summation order."""
    xo, pxo = _i(xoffs)
    xc, pxc = _i(xcols)
    b, pb = _d(b)
    betas, pbe = _d(betas)
    ns = betas.size
    sols = np.empty((ns, d))
    res = np.empty(ns)
    its = np.empty(ns, dtype=np.int64)
    conv = np.empty(ns, dtype=np.uint8)
    napp, fail = C.c_int64(0), C.c_int64(-1)
    st = lib().oracle_regression_shifted_cg(xo.size - 1, d, pxo, pxc, pb, pbe, ns, float(tol),
                                            int(max_iter), int(bool(absolute_tol)),
                                            sols.ctypes.data_as(_PD), res.ctypes.data_as(_PD),
                                            its.ctypes.data_as(_PI64), conv.ctypes.data_as(_PU8),
                                            C.byref(napp), C.byref(fail))
    if st:
        raise OracleFailure(st, fail.value)
    return sols, res, its, conv.astype(bool), napp.value


def sa_solve(loffs, lcols, lvals, labels, alpha, betas, tol, max_iter, probe):
    """SA-SDA in the device's summation order; returns (solutions ns x N, residuals,
    iterations, converged, n_applies)."""
    lo, plo = _i(loffs)
    lc, plc = _i(lcols)
    lv, plv = _d(lvals)
    lab, pl = _b(labels)
    betas, pbe = _d(betas)
    probe, ppr = _d(probe)
    n, ns = lo.size - 1, betas.size
    sols = np.empty((ns, n))
    res = np.empty(ns)
    its = np.empty(ns, dtype=np.int64)
    conv = np.empty(ns, dtype=np.uint8)
    napp, fail = C.c_int64(0), C.c_int64(-1)
    st = lib().oracle_sa_solve(n, plo, plc, plv, pl, float(alpha), pbe, ns, float(tol), int(max_iter),
                               ppr, sols.ctypes.data_as(_PD), res.ctypes.data_as(_PD),
                               its.ctypes.data_as(_PI64), conv.ctypes.data_as(_PU8), C.byref(napp),
                               C.byref(fail))
    if st:
        raise OracleFailure(st, fail.value)
    return sols, res, its, conv.astype(bool), napp.value


def fsda_solve(xoffs, xcols, d, loffs, lcols, lvals, labels, alpha, betas, tol, max_iter, probe,
               n_threads=0, scores=True):
    """Full sweep; returns dict(directions ns x D, scores ns x N, residuals,
    iterations, converged, n_applies)."""
    xo, pxo = _i(xoffs)
    xc, pxc = _i(xcols)
    lo, plo = _i(loffs)
    lc, plc = _i(lcols)
    lv, plv = _d(lvals)
    lab, pl = _b(labels)
    betas, pbe = _d(betas)
    probe, ppr = _d(probe)
    n, ns = xo.size - 1, betas.size
    dirs = np.empty((ns, d))
    sc = np.empty((ns, n)) if scores else None
    res = np.empty(ns)
    its = np.empty(ns, dtype=np.int64)
    conv = np.empty(ns, dtype=np.uint8)
    napp, fail = C.c_int64(0), C.c_int64(-1)
    st = lib().oracle_fsda_solve(n, d, pxo, pxc, plo, plc, plv, pl, float(alpha), pbe, ns,
                                 float(tol), int(max_iter), ppr, int(n_threads),
                                 dirs.ctypes.data_as(_PD),
                                 sc.ctypes.data_as(_PD) if sc is not None else None,
                                 res.ctypes.data_as(_PD), its.ctypes.data_as(_PI64),
                                 conv.ctypes.data_as(_PU8), C.byref(napp), C.byref(fail))
    if st:
        raise OracleFailure(st, fail.value)
    return dict(directions=dirs, scores=sc, residuals=res, iterations=its,
                converged=conv.astype(bool), n_applies=napp.value)


def fsda_solve_workload(w, n_threads=0, scores=True, max_iter=None):
    """Convenience over paper_1709_04794_b200.workloads.Workload."""
    return fsda_solve(w.x_offsets, w.x_cols, w.d, w.l_offsets, w.l_cols, w.l_vals, w.labels,
                      w.alpha, w.betas, w.tol, w.max_iter if max_iter is None else max_iter,
                      w.probe(), n_threads=n_threads, scores=scores)


def max_threads() -> int:
    return lib().oracle_max_threads()


def fsda_solve_sharded(xoffs, xcols, d, loffs, lcols, lvals, labels, alpha, betas, tol, max_iter,
                       probe, bounds, n_threads=0, scores=True):
    """The row-sharded sweep's arithmetic (device fsda_solve_sharded): rows
    split at `bounds`; column sums, sum(z), class sums and orientation dots
    are rank-ordered sums of per-rank canonical trees."""
    xo, pxo = _i(xoffs)
    xc, pxc = _i(xcols)
    lo, plo = _i(loffs)
    lc, plc = _i(lcols)
    lv, plv = _d(lvals)
    lab, pl = _b(labels)
    betas, pbe = _d(betas)
    probe, ppr = _d(probe)
    bd, pbd = _i(bounds)
    n, ns = xo.size - 1, betas.size
    dirs = np.empty((ns, d))
    sc = np.empty((ns, n)) if scores else None
    res = np.empty(ns)
    its = np.empty(ns, dtype=np.int64)
    conv = np.empty(ns, dtype=np.uint8)
    napp, fail = C.c_int64(0), C.c_int64(-1)
    st = lib().oracle_fsda_solve_sharded(n, d, pxo, pxc, plo, plc, plv, pl, float(alpha), pbe, ns,
                                         float(tol), int(max_iter), ppr, int(n_threads), int(bd.size - 1),
                                         pbd, dirs.ctypes.data_as(_PD),
                                         sc.ctypes.data_as(_PD) if sc is not None else None,
                                         res.ctypes.data_as(_PD), its.ctypes.data_as(_PI64),
                                         conv.ctypes.data_as(_PU8), C.byref(napp), C.byref(fail))
    if st:
        raise OracleFailure(st, fail.value)
    return dict(directions=dirs, scores=sc, residuals=res, iterations=its,
                converged=conv.astype(bool), n_applies=napp.value)
