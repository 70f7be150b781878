"""Seeded synthetic FSDA problems with the shapes of BASELINE.json's configs.

The reference publishes no dataset for this path (its ChEMBL corpus is not
shipped), so every measurement and parity case runs on generated inputs with
the stated shapes and value distributions:

* X: row i draws ``n_i ~ Poisson(lam)`` nonzeros, then ``n_i`` *distinct*
  columns by successive weighted sampling without replacement from
  ``P(j) ∝ (j+1)^-s`` (low index = popular; the convention of the reference's
  ``random_sparse_binary``, /root/reference/pkg/src/sdakit/synthetic.py:49).
* Graph: every node picks ``k`` distinct uniform neighbours other than
  itself; the edge set is union-symmetrized (graph.py:141-149) and
  ``L = diag(deg) - S`` (graph.py:191-195), stored exactly as sdakit stores it.
* Labels: rows ``0 .. ell-1`` are labeled (rows are i.i.d., so this equals a
  random selection and needs no ``arrange_labeled_first``); ``n_pos`` of them,
  a seeded random subset, are +1, the rest -1.

Everything is plain numpy; the arrays plug straight into either the
reference's ``SdaProblem`` or ours.
"""

from __future__ import annotations

from dataclasses import dataclass, field

import numpy as np

# (name, N, D, Poisson mean, Zipf s, k, ell, n_pos, n_shifts, beta_lo, beta_hi, K)
CONFIGS = {
    "cfg1": dict(n=10_000, d=5_000, lam=25.0, s=1.1, k=10, ell=1_000, n_pos=200,
                 n_shifts=10, beta_lo=1e-4, beta_hi=1e2, max_iter=50),
    "cfg2": dict(n=200_000, d=100_000, lam=50.0, s=1.1, k=10, ell=10_000, n_pos=3_000,
                 n_shifts=20, beta_lo=1e-5, beta_hi=1e3, max_iter=100),
    "cfg3": dict(n=1_500_000, d=500_000, lam=50.0, s=1.05, k=10, ell=30_000, n_pos=3_000,
                 n_shifts=30, beta_lo=1e-6, beta_hi=1e3, max_iter=150),
    # cfg4: the cfg3 matrix and graph shared by 64 binary tasks, each labeling a
    # random 1% of rows with 10% positives; 20 shifts per task
    "cfg4": dict(n=1_500_000, d=500_000, lam=50.0, s=1.05, k=10, ell=30_000, n_pos=3_000,
                 n_shifts=20, beta_lo=1e-6, beta_hi=1e3, max_iter=150, tasks=64,
                 task_frac=0.01, task_pos=0.10),
    # cfg5: scale-out stress case (8M x 2M, Poisson 80, Zipf 1.05, 15-NN, 1% labeled with 5%
    # positives, 30 shifts, K=200).  BASELINE allows fp32 storage; this build keeps fp64 — the
    # whole problem needs < 15 GB of one B200's 180 GB.  Generated row-chunked (make_workload_chunked).
    "cfg5": dict(n=8_000_000, d=2_000_000, lam=80.0, s=1.05, k=15, ell=80_000, n_pos=4_000,
                 n_shifts=30, beta_lo=1e-6, beta_hi=1e3, max_iter=200),
}

ALPHA = 0.5      # reference default, config.py:36
TOL = 1e-8       # reference default, sda.py:78


@dataclass
class Workload:
    """Raw arrays of one FSDA problem (reference storage conventions)."""

    name: str
    n: int
    d: int
    x_offsets: np.ndarray   # int64, N+1
    x_cols: np.ndarray      # int64, nnz (strictly increasing per row)
    l_offsets: np.ndarray   # int64, N+1
    l_cols: np.ndarray      # int64
    l_vals: np.ndarray      # float64 (-1 off the diagonal, degree on it)
    degrees: np.ndarray     # int64
    labels: np.ndarray      # int8, labeled first
    betas: np.ndarray       # ascending
    alpha: float = ALPHA
    tol: float = TOL
    max_iter: int = 100
    seed: int = 0
    meta: dict = field(default_factory=dict)

    @property
    def nnz(self) -> int:
        return int(self.x_cols.size)

    def probe(self) -> np.ndarray:
        """The reference's probe draw: default_rng(seed).uniform(-1, 1, D)
        (sda.py:297,300)."""
        return np.random.default_rng(self.seed).uniform(-1.0, 1.0, size=self.d)


def _first_distinct(row: np.ndarray, cand: np.ndarray, width: int, want: np.ndarray):
    """For candidate draws grouped by row (draw order), keep the first
    ``want[r]`` distinct values of each row.  Returns (rows, values, short)
    with ``short`` the rows that ran out of distinct candidates."""
    n = want.size
    key = row.astype(np.int64) * width + cand
    order = np.argsort(key, kind="stable")
    ks = key[order]
    first = np.ones(ks.size, dtype=bool)
    first[1:] = ks[1:] != ks[:-1]
    pos = np.sort(order[first])            # first occurrences, back in draw order
    r = row[pos]
    start = np.searchsorted(r, np.arange(n))
    rank = np.arange(r.size) - start[r]
    keep = rank < want[r]
    got = np.bincount(r[keep], minlength=n)
    return r[keep], cand[pos][keep], np.flatnonzero(got < want)


def _searchsorted_threads(cdf: np.ndarray, u: np.ndarray) -> np.ndarray:
    """np.searchsorted(cdf, u, side="right") over host threads (numpy
    releases the GIL there); identical output, the draws stay sequential."""
    if u.size < 4_000_000:
        return np.searchsorted(cdf, u, side="right")
    from concurrent.futures import ThreadPoolExecutor
    import os

    parts = np.array_split(u, min(32, os.cpu_count() or 1) * 2)
    out = np.empty(u.size, dtype=np.int64)
    bounds = np.cumsum([0] + [a.size for a in parts])

    def one(k):
        out[bounds[k]:bounds[k + 1]] = np.searchsorted(cdf, parts[k], side="right")

    with ThreadPoolExecutor(min(32, os.cpu_count() or 1)) as ex:
        list(ex.map(one, range(len(parts))))
    return out


def zipf_binary_rows(n: int, d: int, lam: float, s: float, seed: int):
    """CSR (offsets, cols) of the binary X described in the module docstring."""
    rng = np.random.default_rng(seed)
    counts = np.minimum(rng.poisson(lam, size=n), d).astype(np.int64)
    cdf = np.cumsum((np.arange(d, dtype=np.float64) + 1.0) ** (-s))
    cdf /= cdf[-1]
    m = 2 * counts + 8
    row = np.repeat(np.arange(n, dtype=np.int64), m)
    cand = np.minimum(_searchsorted_threads(cdf, rng.random(row.size)), d - 1)
    rows, cols, short = _first_distinct(row, cand.astype(np.int64), d, counts)
    if short.size:  # rare: successive sampling row by row for the leftovers
        extra_r, extra_c = [], []
        keep_mask = ~np.isin(rows, short)
        rows, cols = rows[keep_mask], cols[keep_mask]
        for i in short:
            chosen: list[int] = []
            seen = set()
            while len(chosen) < counts[i]:
                c = int(min(np.searchsorted(cdf, rng.random(), side="right"), d - 1))
                if c not in seen:
                    seen.add(c)
                    chosen.append(c)
            extra_r.append(np.full(len(chosen), i, dtype=np.int64))
            extra_c.append(np.asarray(chosen, dtype=np.int64))
        rows = np.concatenate([rows] + extra_r)
        cols = np.concatenate([cols] + extra_c)
    key = np.sort(rows * d + cols)
    rows, cols = key // d, key % d
    offsets = np.zeros(n + 1, dtype=np.int64)
    np.cumsum(np.bincount(rows, minlength=n), out=offsets[1:])
    return offsets, cols.astype(np.int64)


def random_knn_laplacian(n: int, k: int, seed: int):
    """Union-symmetrized random k-NN graph, returned as the Laplacian CSR
    (offsets, cols, vals) plus the degree vector."""
    rng = np.random.default_rng(seed)
    m = k + 4
    row = np.repeat(np.arange(n, dtype=np.int64), m)
    cand = rng.integers(0, n - 1, size=row.size)
    cand = cand + (cand >= row)                      # skip self
    want = np.full(n, k, dtype=np.int64)
    src, dst, short = _first_distinct(row, cand, n, want)
    if short.size:
        keep_mask = ~np.isin(src, short)
        src, dst = src[keep_mask], dst[keep_mask]
        er, ec = [], []
        for i in short:
            pick = rng.choice(np.delete(np.arange(n), i), size=k, replace=False)
            er.append(np.full(k, i, dtype=np.int64))
            ec.append(pick.astype(np.int64))
        src = np.concatenate([src] + er)
        dst = np.concatenate([dst] + ec)
    keys = np.sort(np.concatenate([src * n + dst, dst * n + src]))
    keep = np.ones(keys.size, dtype=bool)
    keep[1:] = keys[1:] != keys[:-1]
    keys = keys[keep]                                # np.unique, without its slow path
    a_rows, a_cols = keys // n, keys % n
    deg = np.bincount(a_rows, minlength=n).astype(np.int64)
    # L = D - S with the diagonal at its sorted position; isolated vertices store nothing.
    has_d = deg > 0
    d_idx = np.flatnonzero(has_d)
    # every (row, col) key is unique, so one sort of the keys is the
    # (row, col) lexicographic order
    all_keys = np.sort(np.concatenate([keys, d_idx * n + d_idx]))
    l_rows, l_cols = all_keys // n, all_keys % n
    diag = l_rows == l_cols
    l_vals = np.full(all_keys.size, -1.0)
    l_vals[diag] = deg[l_rows[diag]].astype(np.float64)
    offsets = np.zeros(n + 1, dtype=np.int64)
    np.cumsum(np.bincount(l_rows, minlength=n), out=offsets[1:])
    return offsets, l_cols.astype(np.int64), l_vals, deg


def labels_first(n: int, ell: int, n_pos: int, seed: int) -> np.ndarray:
    rng = np.random.default_rng(seed)
    lab = np.zeros(n, dtype=np.int8)
    lab[:ell] = -1
    lab[rng.choice(ell, size=n_pos, replace=False)] = 1
    return lab


def make_workload(name: str = "cfg2", *, max_iter: int | None = None, seed: int = 2024,
                  **overrides) -> Workload:
    """Generate config ``name`` (see CONFIGS) deterministically."""
    cfg = dict(CONFIGS[name])
    cfg.update(overrides)
    n, d = cfg["n"], cfg["d"]
    xo, xc = zipf_binary_rows(n, d, cfg["lam"], cfg["s"], seed)
    lo, lc, lv, deg = random_knn_laplacian(n, cfg["k"], seed + 1)
    lab = labels_first(n, cfg["ell"], cfg["n_pos"], seed + 2)
    betas = np.geomspace(cfg["beta_lo"], cfg["beta_hi"], cfg["n_shifts"])
    return Workload(
        name=name, n=n, d=d, x_offsets=xo, x_cols=xc, l_offsets=lo, l_cols=lc, l_vals=lv,
        degrees=deg, labels=lab, betas=betas,
        max_iter=int(cfg["max_iter"] if max_iter is None else max_iter),
        meta={k: v for k, v in cfg.items()},
    )


def task_masks(n: int, n_tasks: int, frac: float, pos_frac: float, seed: int) -> np.ndarray:
    """n_tasks x n label masks (cfg4): each task labels a random frac of the
    rows, pos_frac of them positive, the rest negative; any row order."""
    rng = np.random.default_rng(seed)
    n_lab = max(2, int(round(frac * n)))
    n_pos = min(n_lab - 1, max(1, int(round(pos_frac * n_lab))))
    out = np.zeros((n_tasks, n), dtype=np.int8)
    for t in range(n_tasks):
        idx = rng.choice(n, size=n_lab, replace=False)
        out[t, idx] = -1
        out[t, idx[:n_pos]] = 1
    return out


def make_workload_chunked(name: str = "cfg5", *, max_iter: int | None = None, seed: int = 2024,
                          chunk: int = 1_000_000, **overrides) -> Workload:
    """Like make_workload, but X is drawn in independent row chunks (each
    chunk its own seeded stream) so the largest configs fit in host memory;
    the distribution is the same, the exact draw differs from make_workload."""
    cfg = dict(CONFIGS[name])
    cfg.update(overrides)
    n, d = cfg["n"], cfg["d"]
    offs, cols = [np.zeros(1, dtype=np.int64)], []
    base = 0
    for c, r0 in enumerate(range(0, n, chunk)):
        m = min(chunk, n - r0)
        o, cc = zipf_binary_rows(m, d, cfg["lam"], cfg["s"], seed * 1000 + c)
        offs.append(o[1:] + base)
        cols.append(cc)
        base += int(o[-1])
    xo = np.concatenate(offs)
    xc = np.concatenate(cols)
    del cols
    lo, lc, lv, deg = random_knn_laplacian(n, cfg["k"], seed + 1)
    lab = labels_first(n, cfg["ell"], cfg["n_pos"], seed + 2)
    betas = np.geomspace(cfg["beta_lo"], cfg["beta_hi"], cfg["n_shifts"])
    return Workload(
        name=name, n=n, d=d, x_offsets=xo, x_cols=xc, l_offsets=lo, l_cols=lc, l_vals=lv,
        degrees=deg, labels=lab, betas=betas,
        max_iter=int(cfg["max_iter"] if max_iter is None else max_iter),
        meta={k: v for k, v in cfg.items()},
    )


def workload_digest(w: Workload) -> str:
    """sha256 over the raw input arrays (pins fixtures to generator output)."""
    import hashlib

    h = hashlib.sha256()
    for a in (w.x_offsets, w.x_cols, w.l_offsets, w.l_cols, w.l_vals, w.labels, w.betas):
        h.update(np.ascontiguousarray(a).tobytes())
    return h.hexdigest()
