"""Device k-NN / threshold graphs (graph_knn.cuh via fsda_graph_knn /
fsda_graph_threshold) against the
reference's own graphs (tests/golden/graph_reference.npz) and the oracle
(oracle/graph_oracle.py).  Integer/index work: the adjacency must be
identical, entry for entry."""

import numpy as np
import pytest

import paper_1709_04794_b200.graph as G
from oracle import graph_oracle
from paper_1709_04794_b200 import types as T
from paper_1709_04794_b200.workloads import make_workload

from conftest import GOLDEN

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def gold():
    return dict(np.load(GOLDEN / "graph_reference.npz"))


def _x(n, d, offs, cols):
    return T.SparseMatrix.binary(n, d, offs, np.asarray(cols, dtype=np.int64))


def _check(g, offs, cols):
    assert np.array_equal(g.adjacency.row_offsets, offs)
    assert np.array_equal(g.adjacency.col_indices, cols)
    assert np.array_equal(g.degrees, np.diff(offs))


def test_device_matches_reference_graphs(gold):
    for name in gold["names"]:
        n, d, k = (int(v) for v in gold[f"{name}__x_shape"])
        x = _x(n, d, gold[f"{name}__x_offsets"], gold[f"{name}__x_cols"])
        g = G.knn_graph(x, k)
        _check(g, gold[f"{name}__g_offsets"], gold[f"{name}__g_cols"].astype(np.int64))


def test_device_matches_reference_cfg1(gold):
    w = make_workload("cfg1")
    x = T.SparseMatrix.binary(w.n, w.d, w.x_offsets, w.x_cols)
    _check(G.knn_graph(x, 10), gold["cfg1__g_offsets"], gold["cfg1__g_cols"].astype(np.int64))
    _check(G.threshold_graph(x, 0.3), gold["cfg1__t030_offsets"], gold["cfg1__t030_cols"].astype(np.int64))


def test_device_threshold_matches_reference_graphs(gold):
    for name in gold["names"]:
        n, d, _ = (int(v) for v in gold[f"{name}__x_shape"])
        x = _x(n, d, gold[f"{name}__x_offsets"], gold[f"{name}__x_cols"])
        for theta in gold["thetas"]:
            tag = f"{name}__t{int(round(theta * 100)):03d}"
            _check(G.threshold_graph(x, float(theta)), gold[f"{tag}_offsets"],
                   gold[f"{tag}_cols"].astype(np.int64))


@pytest.mark.parametrize("n,d,nnz,power,theta,dup,empty", [
    (333, 5000, 4000, 1.1, 0.2, 20, 10),
    (1000, 9000, 30000, 1.05, 0.1, 40, 5),
    (3000, 8000, 450000, 0.0, 0.05, 0, 0),   # > 2048 tail occurrences per row
    (200, 50, 2000, 0.0, 0.3333333333333333, 0, 0),
    (50, 30, 0, 0.0, 0.5, 0, 0),             # empty X: no edges
])
def test_device_threshold_matches_oracle(n, d, nnz, power, theta, dup, empty):
    rng = np.random.default_rng(n + int(theta * 1000))
    n, d, offs, cols = _random_x(rng, n, d, nnz, power, dup, empty)
    g = G.threshold_graph(_x(n, d, offs, cols), theta)
    go, gc = graph_oracle.threshold_adjacency(n, d, offs, cols, theta)
    _check(g, go, gc)


def _random_x(rng, n, d, nnz, power=0.0, dup_rows=0, empty_rows=0):
    p = (np.arange(d) + 1.0) ** -power
    p /= p.sum()
    keys = np.unique(rng.integers(0, n, nnz) * d + rng.choice(d, nnz, p=p))
    rows, cols = keys // d, keys % d
    if dup_rows:         # copies of earlier rows: exact similarity ties (1.0) with different indices
        src = rng.choice(n // 2, dup_rows, replace=False)
        dst = n // 2 + rng.choice(n - n // 2, dup_rows, replace=False)
        keep = ~np.isin(rows, dst)
        rows, cols = rows[keep], cols[keep]
        extra = [(t, c) for s, t in zip(src, dst) for c in cols[rows == s]]
        if extra:
            er, ec = np.array(extra).T
            rows, cols = np.concatenate([rows, er]), np.concatenate([cols, ec])
    if empty_rows:
        drop = rng.choice(n, empty_rows, replace=False)
        keep = ~np.isin(rows, drop)
        rows, cols = rows[keep], cols[keep]
    order = np.lexsort((cols, rows))
    rows, cols = rows[order], cols[order]
    offs = np.zeros(n + 1, dtype=np.int64)
    np.cumsum(np.bincount(rows, minlength=n), out=offs[1:])
    return n, d, offs, cols.astype(np.int64)


@pytest.mark.parametrize("n,d,nnz,power,k,dup,empty", [
    (97, 13, 300, 0.0, 5, 0, 0),           # every column is a head column
    (333, 5000, 4000, 1.1, 10, 20, 10),    # wide: head + tail, ties, empty rows
    (1000, 9000, 30000, 1.05, 15, 40, 5),  # head capped at 4096 columns, tail re-ranking
    (515, 300, 2000, 0.5, 64, 0, 3),       # k at the device limit
    (64, 40, 40, 0.0, 7, 0, 20),           # mostly padding
    (50, 30, 0, 0.0, 3, 0, 0),             # empty X: every row padded
    (3000, 8000, 450000, 0.0, 10, 0, 0),   # > 2048 tail occurrences per row: direct intersections
])
def test_device_matches_oracle(n, d, nnz, power, k, dup, empty):
    rng = np.random.default_rng(n * 7 + k)
    n, d, offs, cols = _random_x(rng, n, d, nnz, power, dup, empty)
    g = G.knn_graph(_x(n, d, offs, cols), k)
    go, gc = graph_oracle.knn_adjacency(n, d, offs, cols, k)
    _check(g, go, gc)


def test_device_graph_invariants_and_laplacian():
    rng = np.random.default_rng(3)
    n, d, offs, cols = _random_x(rng, 400, 700, 6000, 1.1)
    g = G.knn_graph(_x(n, d, offs, cols), 6)
    a = g.adjacency
    rows = np.repeat(np.arange(n), np.diff(a.row_offsets))
    assert not np.any(rows == a.col_indices)                      # zero diagonal
    pairs = set(zip(rows.tolist(), a.col_indices.tolist()))
    assert all((j, i) in pairs for i, j in pairs)                 # symmetric
    assert np.all(g.degrees >= 6)                                 # every row kept k neighbours
    lap = G.laplacian(g)
    lr = np.repeat(np.arange(n), np.diff(lap.matrix.row_offsets))
    assert np.all(np.bincount(lr, weights=lap.matrix.values, minlength=n) == 0.0)


def test_hand_cases_on_device():
    def rows_x(supports, d):
        offs = np.zeros(len(supports) + 1, dtype=np.int64)
        np.cumsum([len(s) for s in supports], out=offs[1:])
        return _x(len(supports), d, offs, np.concatenate([np.asarray(s) for s in supports]))

    def edges(g):
        a = g.adjacency
        r = np.repeat(np.arange(a.n_rows), np.diff(a.row_offsets))
        return {(int(i), int(j)) for i, j in zip(r, a.col_indices) if i < j}

    assert edges(G.knn_graph(rows_x([[0, 1], [0, 1], [5, 6], [5, 6]], 8), 1)) == {(0, 1), (2, 3)}
    g = G.knn_graph(rows_x([[0, 1, 2, 3], [0, 1, 2, 4], [0, 1, 4, 5]], 6), 1)
    assert edges(g) == {(0, 1), (1, 2)} and g.degrees.tolist() == [1, 2, 1]
    assert edges(G.knn_graph(rows_x([[0], [1], [2]], 3), 1)) == {(0, 1), (0, 2)}


def test_device_rejects_k_above_limit():
    x = T.SparseMatrix.binary(100, 5, np.arange(101), np.arange(100) % 5)
    with pytest.raises(G.GraphError):
        G.knn_graph(x, 65)


def test_cfg2_rows_contain_their_oracle_neighbours():
    """cfg2 scale (200k x 100k, 10M nnz): every sampled row's oracle k-NN list
    is inside its row of the device adjacency (the oracle ranks only the
    sampled rows; the full reference build would take hours)."""
    w = make_workload("cfg2")
    g = G.knn_graph(T.SparseMatrix.binary(w.n, w.d, w.x_offsets, w.x_cols), 10)
    rows = np.random.default_rng(11).choice(w.n, 150, replace=False)
    nb = graph_oracle.knn_neighbours(w.n, w.d, w.x_offsets, w.x_cols, 10, rows=rows)
    a = g.adjacency
    for i, expect in zip(rows, nb):
        have = set(a.col_indices[a.row_offsets[i]:a.row_offsets[i + 1]].tolist())
        assert set(expect.tolist()) <= have, int(i)
    assert g.n_edges >= 10 * w.n // 2


@pytest.mark.parametrize("n,h,r0,nb,density", [
    (1000, 300, 0, 1000, 0.05),      # one 128-deep K step after padding, ragged N tile
    (777, 129, 13, 500, 0.3),        # N, r0 and nb off every tile / 16 boundary
    (4096, 4096, 1024, 2048, 0.02),  # the cfg2 head width: 32 K steps, many tiles per CTA
    (300, 1, 0, 300, 0.5),           # one head column
    (3000, 640, 2900, 100, 1.0),     # all ones: counts = h (largest values)
])
@pytest.mark.parametrize("kernel", ["pairs", "1sm"])
def test_head_count_gemm_exact(n, h, r0, nb, density, kernel, monkeypatch):
    """The hand-written tcgen05 int8 GEMMs (k_head_gemm2 on CTA pairs, the
    product path, and the single-CTA k_head_gemm) against numpy's integer
    product: exact counts, every entry."""
    if kernel == "1sm":
        monkeypatch.setenv("FSDA_B200_HEAD_GEMM", "1sm")
    rng = np.random.default_rng(n + h)
    a = (rng.random((n, h)) < density).astype(np.int8)
    got = G.head_counts(a, r0, nb)
    ai = a.astype(np.int32)
    want = ai[r0:r0 + nb] @ ai.T
    assert np.array_equal(got, want)


def test_head_count_gemm_zipf_rows():
    """Rows of a Zipf-headed binary X (the graph builds' real operand)."""
    w = make_workload("cfg1", n=2500, d=1200)
    a = np.zeros((w.n, 512), dtype=np.int8)
    for i in range(w.n):
        c = w.x_cols[w.x_offsets[i]:w.x_offsets[i + 1]]
        a[i, c[c < 512]] = 1
    got = G.head_counts(a, 640, 1500)
    ai = a.astype(np.int32)
    assert np.array_equal(got, ai[640:2140] @ ai.T)


@pytest.mark.parametrize("rows", ["16", "1008", "4000"])
def test_device_graphs_in_many_blocks(gold, rows, monkeypatch):
    """The builds cut the rows into blocks sized by a memory budget (one block
    at these sizes); forcing small blocks — including a last, ragged one —
    must give the reference's graphs entry for entry."""
    monkeypatch.setenv("FSDA_B200_GRAPH_BLOCK_ROWS", rows)
    w = make_workload("cfg1")
    x = T.SparseMatrix.binary(w.n, w.d, w.x_offsets, w.x_cols)
    _check(G.knn_graph(x, 10), gold["cfg1__g_offsets"], gold["cfg1__g_cols"].astype(np.int64))
    _check(G.threshold_graph(x, 0.3), gold["cfg1__t030_offsets"], gold["cfg1__t030_cols"].astype(np.int64))
