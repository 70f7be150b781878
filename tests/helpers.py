"""Test helpers: problem construction from workloads / golden cases and the
parity metrics (per-shift relative error, labeled-row AUC, rankings)."""

from __future__ import annotations

import numpy as np

import paper_1709_04794_b200 as fb
from paper_1709_04794_b200.workloads import Workload


def problem_from_workload(w: Workload, max_iter=None, **kw) -> fb.SdaProblem:
    x = fb.SparseMatrix.binary(w.n, w.d, w.x_offsets, w.x_cols)
    lap = fb.Laplacian(fb.SparseMatrix(w.n, w.n, w.l_offsets, w.l_cols, w.l_vals), w.degrees)
    args = dict(alpha=w.alpha, betas=w.betas, tol=w.tol,
                max_iter_d=w.max_iter if max_iter is None else max_iter, seed=w.seed)
    args.update(kw)
    return fb.SdaProblem(x=x, labels=fb.LabelVector(w.labels), lap=lap, **args)


def small_case(g: dict, idx: int) -> dict:
    pre = f"c{idx}_"
    return {k[len(pre):]: v for k, v in g.items() if k.startswith(pre)}


def problem_from_case(c: dict, **kw) -> fb.SdaProblem:
    n, d = int(c["n"]), int(c["d"])
    x = fb.SparseMatrix.binary(n, d, c["x_offsets"], c["x_cols"])
    lap = fb.Laplacian(fb.SparseMatrix(n, n, c["l_offsets"], c["l_cols"], c["l_vals"]),
                       c["degrees"])
    args = dict(alpha=float(c["alpha"]), betas=c["betas"], tol=float(c["tol"]),
                max_iter_d=int(c["max_iter"]), seed=int(c["seed"]))
    args.update(kw)
    return fb.SdaProblem(x=x, labels=fb.LabelVector(c["labels"]), lap=lap, **args)


def dense_case(g: dict, idx: int) -> dict:
    pre = f"d{idx}_"
    return {k[len(pre):]: v for k, v in g.items() if k.startswith(pre)}


def rel_rows(a: np.ndarray, b: np.ndarray) -> float:
    """max over shifts of ||a_s - b_s|| / ||b_s||."""
    num = np.linalg.norm(np.asarray(a) - np.asarray(b), axis=1)
    den = np.maximum(np.linalg.norm(np.asarray(b), axis=1), 1e-300)
    return float(np.max(num / den))


def auc(scores, truth) -> float:
    """Rank-sum AUC with average ranks (the reference's auc_roc,
    evaluation.py:45-63), restated with scipy.stats.rankdata."""
    from scipy.stats import rankdata

    scores = np.asarray(scores, dtype=np.float64)
    truth = np.asarray(truth)
    pos = truth == 1
    n_pos = int(pos.sum())
    n_neg = truth.size - n_pos
    ranks = rankdata(scores)
    return float((ranks[pos].sum() - n_pos * (n_pos + 1) / 2.0) / (n_pos * n_neg))


def labeled_aucs(scores: np.ndarray, labels: np.ndarray) -> np.ndarray:
    m = np.asarray(labels) != 0
    return np.array([auc(s[m], np.asarray(labels)[m]) for s in scores])


def same_ranking(a: np.ndarray, b: np.ndarray) -> bool:
    """Identical induced ordering (ties broken by index) for every shift."""
    return all(np.array_equal(np.argsort(x, kind="stable"), np.argsort(y, kind="stable"))
               for x, y in zip(a, b))


def ranking_violations(a: np.ndarray, b: np.ndarray, rel_gap: float = 1e-9):
    """Per shift: rows whose order under `a` contradicts the order under the
    reference scores `b`, outside near-ties of b — consecutive sorted values
    closer than max(rel_gap * max|b|, 4 max_i |a_i - b_i|): two rows whose
    reference scores differ by less than the scores' own discrepancy may swap
    under any reordered sum.  Returns (violations per shift, fraction of rows
    inside near-tie groups)."""
    viol, tied = [], []
    for x, y in zip(np.asarray(a), np.asarray(b)):
        ob = np.argsort(y, kind="stable")
        sy = y[ob]
        gap = max(rel_gap * max(float(np.max(np.abs(y))), 1e-300), 4.0 * float(np.max(np.abs(x - y))))
        new = np.concatenate([[True], np.diff(sy) > gap])
        cluster = np.empty(y.size, dtype=np.int64)
        cluster[ob] = np.cumsum(new) - 1
        seq = cluster[np.argsort(x, kind="stable")]
        viol.append(int(np.count_nonzero(np.diff(seq) < 0)))
        sizes = np.bincount(cluster)
        tied.append(float(np.sum(sizes[sizes > 1])) / y.size)
    return np.array(viol), np.array(tied)
