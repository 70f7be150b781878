"""Load the reference's FSDA acceptance cases (tests/golden/acceptance_reference.npz,
made by tests/golden/make_golden_acceptance.py from the unmodified reference)
as this package's SdaProblem objects, and a stand-in for the reference's
solver table so the cases run through fb.install_into_sdakit exactly as a
sdakit user would call solve(p, "fsda") (sda.py:465-486)."""

from __future__ import annotations

import types
from pathlib import Path

import numpy as np

import paper_1709_04794_b200 as fb

FIXTURE = Path(__file__).resolve().parent / "golden" / "acceptance_reference.npz"


def load():
    return dict(np.load(FIXTURE))


def keys(g, prefix):
    return sorted({k.split("__")[0] for k in g if k.startswith(prefix)},
                  key=lambda s: int(s.rsplit("_", 1)[1]) if s.rsplit("_", 1)[1].isdigit() else 0)


def problem(g, key):
    n, d = (int(v) for v in g[f"{key}__shape"])
    x = fb.SparseMatrix.binary(n, d, g[f"{key}__x_offsets"].astype(np.int64),
                               g[f"{key}__x_cols"].astype(np.int64))
    lap = fb.Laplacian(fb.SparseMatrix(n, n, g[f"{key}__l_offsets"].astype(np.int64),
                                       g[f"{key}__l_cols"].astype(np.int64), g[f"{key}__l_vals"]),
                       g[f"{key}__degrees"])
    alpha, tol, max_iter, seed = g[f"{key}__knobs"]
    return fb.SdaProblem(x=x, labels=fb.LabelVector(g[f"{key}__labels"].astype(np.int64)), lap=lap,
                         alpha=float(alpha), betas=g[f"{key}__betas"], tol=float(tol),
                         max_iter_d=int(max_iter), seed=int(seed))


def dense(m) -> np.ndarray:
    out = np.zeros((int(m.n_rows), int(m.n_cols)))
    offs = np.asarray(m.row_offsets)
    for i in range(int(m.n_rows)):
        out[i, np.asarray(m.col_indices)[offs[i]:offs[i + 1]]] = np.asarray(m.values)[offs[i]:offs[i + 1]]
    return out


def sdakit_stub():
    """A module with sdakit.sda's plugin surface: the _SOLVERS table and a
    solve(p, algorithm) that dispatches through it (sda.py:465-486)."""
    mod = types.ModuleType("sdakit_sda_stub")

    def _unreachable(p):
        raise AssertionError("the reference solver ran instead of the plugin")

    mod._SOLVERS = {"fsda": _unreachable, "sa-sda": _unreachable}
    mod.fsda_solve = _unreachable
    mod.sa_sda_solve = _unreachable
    mod.solve = lambda p, algorithm="fsda": mod._SOLVERS[algorithm](p)
    return mod
