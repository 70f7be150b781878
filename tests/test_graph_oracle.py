"""Graph oracles (oracle/graph_oracle.py) pinned to the reference's own
graphs (tests/golden/graph_reference.npz, made by make_golden_graph.py from
sdakit.graph.knn_graph / threshold_graph), plus the host-side graph logic: argument
validation, Tanimoto, Laplacian assembly (graph.py:58-66, 152-160, 191-195).
CPU only."""

import numpy as np
import pytest

import paper_1709_04794_b200.graph as G
from oracle import graph_oracle
from paper_1709_04794_b200 import types as T
from paper_1709_04794_b200.workloads import make_workload, workload_digest

from conftest import GOLDEN


@pytest.fixture(scope="module")
def gold():
    return dict(np.load(GOLDEN / "graph_reference.npz"))


def _case(gold, name):
    n, d, k = (int(v) for v in gold[f"{name}__x_shape"])
    return n, d, k, gold[f"{name}__x_offsets"], gold[f"{name}__x_cols"].astype(np.int64)


def test_oracle_matches_reference_graphs(gold):
    for name in gold["names"]:
        n, d, k, offs, cols = _case(gold, str(name))
        g_offs, g_cols = graph_oracle.knn_adjacency(n, d, offs, cols, k)
        assert np.array_equal(g_offs, gold[f"{name}__g_offsets"]), name
        assert np.array_equal(g_cols, gold[f"{name}__g_cols"]), name


def test_threshold_oracle_matches_reference_graphs(gold):
    for name in gold["names"]:
        n, d, _, offs, cols = _case(gold, str(name))
        for theta in gold["thetas"]:
            tag = f"{name}__t{int(round(theta * 100)):03d}"
            g_offs, g_cols = graph_oracle.threshold_adjacency(n, d, offs, cols, float(theta))
            assert np.array_equal(g_offs, gold[f"{tag}_offsets"]), tag
            assert np.array_equal(g_cols, gold[f"{tag}_cols"]), tag


def test_threshold_oracle_hand_case():
    # supports {0,1}, {0,1,2,3}, {0}: pairwise 2/4, 1/2, 1/4
    d, offs, cols = _rows([[0, 1], [0, 1, 2, 3], [0]], 4)
    assert _edges(*graph_oracle.threshold_adjacency(3, d, offs, cols, 0.4)) == {(0, 1), (0, 2)}
    assert _edges(*graph_oracle.threshold_adjacency(3, d, offs, cols, 0.2)) == {(0, 1), (0, 2), (1, 2)}


def test_threshold_validates_theta_before_the_device():
    x = T.SparseMatrix.binary(2, 2, [0, 1, 2], [0, 1])
    for bad in (0.0, 1.5, -0.1):
        with pytest.raises(G.GraphError):
            G.threshold_graph(x, bad)


def test_oracle_matches_reference_cfg1(gold):
    w = make_workload("cfg1")
    assert workload_digest(w) == str(gold["cfg1__digest"][0])
    g_offs, g_cols = graph_oracle.knn_adjacency(w.n, w.d, w.x_offsets, w.x_cols, 10)
    assert np.array_equal(g_offs, gold["cfg1__g_offsets"])
    assert np.array_equal(g_cols, gold["cfg1__g_cols"])
    t_offs, t_cols = graph_oracle.threshold_adjacency(w.n, w.d, w.x_offsets, w.x_cols, 0.3)
    assert np.array_equal(t_offs, gold["cfg1__t030_offsets"])
    assert np.array_equal(t_cols, gold["cfg1__t030_cols"])


def _rows(supports, n_cols):
    offs = np.zeros(len(supports) + 1, dtype=np.int64)
    np.cumsum([len(s) for s in supports], out=offs[1:])
    cols = np.concatenate([np.asarray(s, dtype=np.int64) for s in supports])
    return n_cols, offs, cols


def _edges(offs, cols):
    rows = np.repeat(np.arange(offs.size - 1), np.diff(offs))
    return {(int(i), int(j)) for i, j in zip(rows, cols) if i < j}


def test_oracle_hand_cases():
    # identical pairs: sim(0,1) = sim(2,3) = 1, cross pairs share nothing
    d, offs, cols = _rows([[0, 1], [0, 1], [5, 6], [5, 6]], 8)
    assert _edges(*graph_oracle.knn_adjacency(4, d, offs, cols, 1)) == {(0, 1), (2, 3)}
    # a tie at the cutoff goes to the lower index; the union keeps one-sided picks
    d, offs, cols = _rows([[0, 1, 2, 3], [0, 1, 2, 4], [0, 1, 4, 5]], 6)
    assert _edges(*graph_oracle.knn_adjacency(3, d, offs, cols, 1)) == {(0, 1), (1, 2)}
    # no shared features: padded with the lowest non-self indices
    d, offs, cols = _rows([[0], [1], [2]], 3)
    assert _edges(*graph_oracle.knn_adjacency(3, d, offs, cols, 1)) == {(0, 1), (0, 2)}


def test_tanimoto_hand_values():
    assert G.tanimoto([0, 1], [2, 3]) == 0.0
    assert G.tanimoto([1, 2, 3], [2, 3, 4]) == 0.5
    assert G.tanimoto([5, 9], [5, 9]) == 1.0
    assert G.tanimoto([], []) == 0.0


def test_knn_validates_k_before_the_device():
    x = T.SparseMatrix.binary(2, 2, [0, 1, 2], [0, 1])
    with pytest.raises(G.GraphError):
        G.knn_graph(x, 0)
    with pytest.raises(G.GraphError):
        G.knn_graph(x, 2)      # k must leave room for self-exclusion
    with pytest.raises(ValueError):
        G.knn_graph(x, -1)


def test_laplacian_assembly():
    # path graph 0 - 1 - 2 plus an isolated vertex 3
    adj = T.SparseMatrix(4, 4, [0, 1, 3, 4, 4], [1, 0, 2, 1], np.ones(4))
    lap = G.laplacian(G.SimilarityGraph(adjacency=adj, degrees=np.array([1, 2, 1, 0])))
    dense = np.zeros((4, 4))
    rows = np.repeat(np.arange(4), np.diff(lap.matrix.row_offsets))
    dense[rows, lap.matrix.col_indices] = lap.matrix.values
    assert np.array_equal(dense, [[1, -1, 0, 0], [-1, 2, -1, 0], [0, -1, 1, 0], [0, 0, 0, 0]])
    assert lap.matrix.row_offsets[-1] == 7            # the isolated vertex stores nothing
    assert np.array_equal(lap.degrees, [1, 2, 1, 0])


def test_laplacian_of_golden_graph_is_the_reference_layout(gold):
    """Every row: ascending columns, -1 off the diagonal, the degree on it,
    row sums exactly zero (graph.py:191-195, sparse.from_scipy)."""
    offs, cols = gold["zipf__g_offsets"], gold["zipf__g_cols"].astype(np.int64)
    n = offs.size - 1
    adj = T.SparseMatrix(n, n, offs, cols, np.ones(cols.size))
    lap = G.laplacian(G.SimilarityGraph(adjacency=adj, degrees=np.diff(offs)))
    m = lap.matrix
    rows = np.repeat(np.arange(n), np.diff(m.row_offsets))
    sums = np.bincount(rows, weights=m.values, minlength=n)
    assert np.all(sums == 0.0)
    diag = rows == m.col_indices
    assert np.array_equal(m.values[diag], np.diff(offs)[rows[diag]].astype(float))
    assert np.all(m.values[~diag] == -1.0)
