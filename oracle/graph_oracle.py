"""CPU ORACLE for the Tanimoto k-NN and threshold graphs — test
infrastructure only.

Imported only by tests/ and bench.py's CPU baseline, as the checker; the
product path is libfsda_b200.so (graph_knn.cuh).

Restates the reference construction (/root/reference/pkg/src/sdakit/graph.py):
  * similarity of rows a, b = |a & b| / (|a| + |b| - |a & b|) in float64
    (graph.py:91-93; the reference divides float64 counts by float64 unions);
  * row i ranks the rows j != i that share at least one feature by
    (similarity descending, index ascending) and keeps k (graph.py:94-95);
  * rows with fewer than k such candidates are padded with the lowest
    indices not yet taken and != i (graph.py:96-109);
  * the edge set is the union of both directions, stored as a CSR adjacency
    with ascending columns and unit values (graph.py:141-149, 163-166).
Pinned to the reference's own outputs by tests/golden/graph_reference.npz
(tests/golden/make_golden_graph.py).

Counts come from an integer sparse product per row block, so it runs in
seconds at the parity sizes (a few thousand rows).
"""

from __future__ import annotations

import numpy as np
import scipy.sparse as sp


def _pattern(n_rows, n_cols, row_offsets, col_indices):
    offs = np.asarray(row_offsets, dtype=np.int64)
    cols = np.asarray(col_indices, dtype=np.int64)
    return sp.csr_matrix((np.ones(cols.size, dtype=np.int32), cols, offs), shape=(n_rows, n_cols))


def knn_neighbours(n_rows, n_cols, row_offsets, col_indices, k, block=512, rows=None):
    """k neighbour indices per row (n_rows x k, or len(rows) x k for a
    subset of rows), in rank order."""
    pat = _pattern(n_rows, n_cols, row_offsets, col_indices)
    pt = pat.T.tocsr()
    size = np.diff(np.asarray(row_offsets, dtype=np.int64))
    sel = np.arange(n_rows) if rows is None else np.asarray(rows, dtype=np.int64)
    out = np.empty((sel.size, k), dtype=np.int64)
    for r0 in range(0, sel.size, block):
        r1 = min(sel.size, r0 + block)
        counts = (pat[sel[r0:r1]] @ pt).tocsr()
        for b in range(r1 - r0):
            i = int(sel[r0 + b])
            js = counts.indices[counts.indptr[b]:counts.indptr[b + 1]].astype(np.int64)
            cs = counts.data[counts.indptr[b]:counts.indptr[b + 1]].astype(np.float64)
            keep = (js != i) & (cs > 0)
            js, cs = js[keep], cs[keep]
            sims = cs / ((size[i] + size[js]).astype(np.float64) - cs)
            rank = np.lexsort((js, -sims))[:k]
            chosen = list(js[rank])
            if len(chosen) < k:
                taken = set(chosen) | {i}
                j = 0
                while len(chosen) < k:
                    if j not in taken:
                        chosen.append(j)
                    j += 1
            out[r0 + b] = chosen
    return out


def knn_adjacency(n_rows, n_cols, row_offsets, col_indices, k):
    """(row_offsets, col_indices) of the union-symmetrized k-NN adjacency."""
    nb = knn_neighbours(n_rows, n_cols, row_offsets, col_indices, k)
    src = np.repeat(np.arange(n_rows, dtype=np.int64), k)
    dst = nb.ravel()
    keys = np.unique(np.concatenate([src * n_rows + dst, dst * n_rows + src]))
    rows, cols = keys // n_rows, keys % n_rows
    offs = np.zeros(n_rows + 1, dtype=np.int64)
    np.cumsum(np.bincount(rows, minlength=n_rows), out=offs[1:])
    return offs, cols


def threshold_adjacency(n_rows, n_cols, row_offsets, col_indices, theta, block=512):
    """(row_offsets, col_indices) of the threshold graph: every pair of
    distinct rows sharing a feature with similarity >= theta (graph.py:114-133,
    169-188; theta > 0, so pairs sharing nothing never qualify)."""
    pat = _pattern(n_rows, n_cols, row_offsets, col_indices)
    pt = pat.T.tocsr()
    size = np.diff(np.asarray(row_offsets, dtype=np.int64))
    src, dst = [], []
    for r0 in range(0, n_rows, block):
        r1 = min(n_rows, r0 + block)
        counts = (pat[r0:r1] @ pt).tocoo()
        i = counts.row.astype(np.int64) + r0
        j = counts.col.astype(np.int64)
        c = counts.data.astype(np.float64)
        keep = (i != j) & (c > 0)
        i, j, c = i[keep], j[keep], c[keep]
        hit = c / ((size[i] + size[j]).astype(np.float64) - c) >= theta
        src.append(i[hit])
        dst.append(j[hit])
    s = np.concatenate(src) if src else np.empty(0, np.int64)
    d = np.concatenate(dst) if dst else np.empty(0, np.int64)
    keys = np.unique(np.concatenate([s * n_rows + d, d * n_rows + s]))
    rows, cols = keys // n_rows, keys % n_rows
    offs = np.zeros(n_rows + 1, dtype=np.int64)
    np.cumsum(np.bincount(rows, minlength=n_rows), out=offs[1:])
    return offs, cols
