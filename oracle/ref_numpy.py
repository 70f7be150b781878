"""Reference-order restatement of the FSDA path in numpy/scipy.

CPU ORACLE — test infrastructure only (see oracle/__init__.py).

It performs the reference's arithmetic with the reference's own library
calls — scipy csr/csc matvec for every sparse product, BLAS dots for
``p @ q`` / ``r @ r`` / ``y @ s``, ``np.linalg.norm`` for ||b|| and numpy's
pairwise sums for class means and ``sum(w)`` — on raw arrays, so it can run
on the GPU box where /root/reference is absent.  Each step cites the
reference line it restates (paths under /root/reference/pkg/src/sdakit).
It is pinned bit-for-bit against the reference's own outputs by
tests/test_oracle_golden.py.
"""

from __future__ import annotations

import numpy as np
import scipy.sparse as sp


class Problem:
    """Raw arrays of one FSDA problem in sdakit's storage conventions."""

    def __init__(self, xoffs, xcols, d, loffs, lcols, lvals, labels):
        self.n = int(len(xoffs) - 1)
        self.d = int(d)
        ones = np.ones(len(xcols))
        xoffs = np.asarray(xoffs, dtype=np.int64)
        xcols = np.asarray(xcols, dtype=np.int64)
        # X as scipy sees it (sparse.py:108-114) and X^T as the csc view of
        # the same arrays (sparse.py:131-134).
        self.x = sp.csr_matrix((ones, xcols, xoffs), shape=(self.n, self.d))
        self.xt = sp.csc_matrix((ones, xcols, xoffs), shape=(self.d, self.n))
        self.lap = sp.csr_matrix((np.asarray(lvals, dtype=np.float64),
                                  np.asarray(lcols, dtype=np.int64),
                                  np.asarray(loffs, dtype=np.int64)), shape=(self.n, self.n))
        self.labels = np.asarray(labels, dtype=np.int8)
        self.m1 = self.labels == 1
        self.m2 = self.labels == -1
        self.ml = self.labels != 0

    @classmethod
    def from_workload(cls, w):
        return cls(w.x_offsets, w.x_cols, w.d, w.l_offsets, w.l_cols, w.l_vals, w.labels)

    # sparse.py:258-265
    def labeled_mean(self) -> np.ndarray:
        return self.xt.dot(self.ml.astype(np.float64)) / int(self.ml.sum())

    # sparse.py:274-277
    def centered_t(self, mu, w) -> np.ndarray:
        return self.xt.dot(w) - mu * float(np.sum(w))

    # sda.py:120-128
    def apply_w(self, z) -> np.ndarray:
        out = np.zeros_like(z)
        out[self.m1] = z[self.m1].sum() / int(self.m1.sum())
        out[self.m2] = z[self.m2].sum() / int(self.m2.sum())
        return out

    # sda.py:131-140
    def smoother(self, alpha, z) -> np.ndarray:
        masked = np.where(self.ml, z, 0.0)
        if alpha == 0.0:
            return masked
        smoothed = alpha * self.lap.dot(z)
        if alpha == 1.0:
            return smoothed
        return (1.0 - alpha) * masked + smoothed

    # sda.py:169-172
    def operator(self, alpha, mu, w) -> np.ndarray:
        return self.centered_t(mu, self.smoother(alpha, self.x.dot(w)))


def shifted_cg(apply, b, betas, tol, max_iter, absolute_tol=False, on_iter=None):
    """Multi-shift CG, krylov.py:168-281, per-shift columns kept as rows of
    (n_shifts, dim) arrays; every update rounds as the reference's does.
    ``on_iter(i, sols)`` (optional, the noise-floor tool) sees the solutions
    after iteration i — what a run with max_iter = i + 1 returns."""
    betas = np.asarray(betas, dtype=np.float64)
    ns, dim = betas.size, b.size
    b_norm = float(np.linalg.norm(b))                              # krylov.py:185
    sols = np.zeros((ns, dim))
    if b_norm == 0.0:                                              # krylov.py:188-194
        return dict(directions=sols, residuals=np.zeros(ns),
                    iterations=np.zeros(ns, dtype=np.int64), converged=np.ones(ns, bool),
                    n_applies=0)
    thresh = tol if absolute_tol else tol * b_norm                 # krylov.py:117-120
    r, p = b.copy(), b.copy()
    big_p = np.tile(b, (ns, 1))
    rr, gamma_prev, alpha = b_norm * b_norm, 1.0, 0.0              # krylov.py:200-203
    zeta_prev, zeta = np.ones(ns), np.ones(ns)
    active = np.ones(ns, dtype=bool)
    iters = np.full(ns, max_iter, dtype=np.int64)
    resid = np.full(ns, b_norm)
    conv = np.zeros(ns, dtype=bool)
    n_applies = 0
    for i in range(max_iter):
        q = apply(p)
        n_applies += 1
        pq = float(p @ q)                                          # krylov.py:212
        if not np.isfinite(pq):
            raise FloatingPointError(f"non-finite <p, Bp> at iteration {i}")
        if pq == 0.0:
            raise ZeroDivisionError(f"singular direction at iteration {i}")
        gamma = -rr / pq
        zn = np.zeros(ns)
        gs = np.zeros(ns)
        good = np.zeros(ns, dtype=bool)
        for s in np.flatnonzero(active):                           # krylov.py:219-229
            denom = gamma * alpha * (zeta_prev[s] - zeta[s]) + \
                zeta_prev[s] * gamma_prev * (1.0 - betas[s] * gamma)
            with np.errstate(divide="ignore", invalid="ignore", over="ignore"):
                v = np.float64(zeta_prev[s] * zeta[s] * gamma_prev) / np.float64(denom)
            if np.isfinite(v) and abs(v) >= 1e-290:
                good[s] = True
                zn[s] = v
                gs[s] = gamma * v / zeta[s]
        for s in np.flatnonzero(good):                             # krylov.py:230
            sols[s] -= big_p[s] * gs[s]
        r = r + gamma * q                                          # krylov.py:232
        rr_new = float(r @ r)
        if not np.isfinite(rr_new):
            raise FloatingPointError(f"non-finite residual at iteration {i}")
        r_norm = np.sqrt(rr_new)
        alpha_new = rr_new / rr
        p = r + alpha_new * p                                      # krylov.py:239
        for s in np.flatnonzero(good):                             # krylov.py:240-241
            a_s = alpha_new * (zn[s] * gs[s]) / (zeta[s] * gamma)
            big_p[s] = zn[s] * r + a_s * big_p[s]
        for s in np.flatnonzero(active):                           # krylov.py:250-268
            if not good[s]:
                iters[s], resid[s], active[s] = i + 1, np.inf, False
                continue
            shift_res = abs(zn[s]) * r_norm
            if shift_res < thresh:
                iters[s], resid[s], conv[s], active[s] = i + 1, shift_res, True, False
            else:
                zeta_prev[s], zeta[s] = zeta[s], zn[s]
        gamma_prev, alpha, rr = gamma, alpha_new, rr_new
        if on_iter is not None:
            on_iter(i, sols)
        if not active.any():
            break
    for s in np.flatnonzero(active):                               # krylov.py:272-275
        iters[s] = max_iter
        resid[s] = abs(zeta[s]) * np.sqrt(rr)
    return dict(directions=sols, residuals=resid, iterations=iters, converged=conv,
                n_applies=n_applies)


def fsda_solve(prob: Problem, alpha, betas, tol, max_iter, seed=0, on_iter=None, operator=None):
    """sda.py:293-320 on raw arrays; directions/scores rows are shifts.
    ``operator(alpha, mu, w)`` replaces prob.operator (the noise-floor tool
    perturbs it)."""
    rng = np.random.default_rng(seed)                              # sda.py:297
    mu = prob.labeled_mean()                                       # sda.py:298
    r = rng.uniform(-1.0, 1.0, size=prob.d)                        # sda.py:300
    rhs = prob.centered_t(mu, prob.apply_w(prob.x.dot(r)))         # sda.py:301
    op = operator or prob.operator
    out = shifted_cg(lambda w: op(alpha, mu, w), rhs, betas, tol, max_iter, on_iter=on_iter)
    y = prob.labels.astype(np.float64)
    scores = np.empty((len(betas), prob.n))
    for s in range(len(betas)):                                    # sda.py:277-283
        sv = prob.x.dot(out["directions"][s])
        if float(y @ sv) < 0.0:
            sv = -sv
            out["directions"][s] = -out["directions"][s]
        scores[s] = sv
    out["scores"] = scores
    return out


def orient(prob: Problem, directions):
    """The sign rule of sda.py:277-283 applied to a stack of directions."""
    y = prob.labels.astype(np.float64)
    out = np.array(directions, copy=True)
    for s in range(out.shape[0]):
        if float(y @ prob.x.dot(out[s])) < 0.0:
            out[s] = -out[s]
    return out


def fsda_solve_workload(w, max_iter=None):
    return fsda_solve(Problem.from_workload(w), w.alpha, w.betas, w.tol,
                      w.max_iter if max_iter is None else max_iter, w.seed)
