"""Tanimoto k-NN and threshold graphs of the rows of X on the device
(SURVEY §8f #4).

Mirrors the reference's graph API for this construction
(/root/reference/pkg/src/sdakit/graph.py): ``knn_graph(x, k, *, block_size,
n_threads)`` (graph.py:152-166) returns a ``SimilarityGraph`` whose adjacency
is the union-symmetrized k-NN edge set with unit values, built exactly as
``_knn_rows_block`` ranks candidates (graph.py:79-111: Tanimoto of the
supports, ties toward the lower index, padding with the lowest unused
indices) and ``_adjacency_from_pairs`` stores it (graph.py:141-149); and
``threshold_graph(x, theta)`` (graph.py:169-188) keeps every pair with
similarity >= theta; ``laplacian(graph)`` (graph.py:191-195) assembles
L = D - S.

The similarity work — every pair's intersection count, the per-row ranking
and the symmetrization — runs in ``libfsda_b200.so`` (graph_gemm.cuh / graph_knn.cuh: a
hand-written int8 tcgen05 tensor-core GEMM of the 0/1 head-column matrix for
the exact counts of the frequent columns, a warp-per-row ranking scan, an exact re-ranking of the
candidates that share rarer columns, a radix-sort union).  ``block_size`` and
``n_threads`` only steer the reference's CPU blocking; the result does not
depend on them, so they are accepted and ignored.  There is no CPU fallback.
"""

from __future__ import annotations

import importlib
from dataclasses import dataclass
from typing import Optional

import numpy as np

from . import _capi
from . import types as T
from .fsda import Device, _i64, _raise_for, default_device


class GraphError(ValueError):
    """Invalid graph construction parameters (graph.py:28-29)."""


@dataclass(frozen=True)
class SimilarityGraph:
    """Undirected unweighted graph: binary symmetric adjacency, zero diagonal
    (graph.py:32-46)."""

    adjacency: T.SparseMatrix
    degrees: np.ndarray

    @property
    def n(self) -> int:
        return self.adjacency.n_rows

    @property
    def n_edges(self) -> int:
        return self.adjacency.nnz // 2


def tanimoto(support_a, support_b) -> float:
    """|a & b| / |a | b| of two index sets; 0 when both are empty (graph.py:58-66)."""
    a = np.unique(np.asarray(support_a, dtype=np.int64))
    b = np.unique(np.asarray(support_b, dtype=np.int64))
    inter = np.intersect1d(a, b, assume_unique=True).size
    union = a.size + b.size - inter
    return inter / union if union else 0.0


def _graph_types(x):
    """sdakit's SparseMatrix / SimilarityGraph / GraphError when x is sdakit's."""
    root = (type(x).__module__ or "").split(".")[0]
    if root == "sdakit":
        g = importlib.import_module("sdakit.graph")
        s = importlib.import_module("sdakit.sparse")
        return s.SparseMatrix, g.SimilarityGraph, g.GraphError, g.Laplacian
    return T.SparseMatrix, SimilarityGraph, GraphError, T.Laplacian


def head_counts(a, r0: int = 0, nb: Optional[int] = None, *, device: Optional[Device] = None) -> np.ndarray:
    """counts[b, j] = sum_k a[r0 + b, k] * a[j, k] for a 0/1 matrix a (any
    n x h): the exact int32 block the graph builds take from the hand-written
    tcgen05 head-count GEMM (csrc/graph_gemm.cuh)."""
    a = np.ascontiguousarray(a, dtype=np.int8)
    n, h = a.shape
    nb = n - r0 if nb is None else int(nb)
    out = np.empty((nb, n), dtype=np.int32)
    dev = device or default_device()
    _raise_for(_capi.lib().fsda_head_counts(dev._h, n, h, a.ctypes.data, int(r0), nb, out.ctypes.data))
    return out


def knn_graph(x, k: int, *, block_size: int = 1024, n_threads: int = 1,
              device: Optional[Device] = None):
    """Union-symmetrized k-nearest-neighbour Tanimoto graph of the rows of x
    (graph.py:152-166), built on the device."""
    SM, SG, GE, _ = _graph_types(x)
    n = int(x.n_rows)
    k = int(k)
    if not 0 < k < n:
        raise GE(f"k must satisfy 0 < k < n_samples, got k={k}, n={n}")
    if k > 64:
        raise GE(f"k={k}: the device ranking keeps at most 64 neighbours per row")
    dev = device or default_device()
    lib = _upload_pattern(dev, x)
    nnz = np.zeros(1, dtype=np.int64)
    _raise_for(lib.fsda_graph_knn(dev._h, k, _capi.i64ptr(nnz)))
    return _fetch_graph(dev, lib, n, int(nnz[0]), SM, SG)


def threshold_graph(x, theta: float, *, block_size: int = 1024, n_threads: int = 1,
                    device: Optional[Device] = None):
    """Graph with an edge wherever the Tanimoto similarity of two distinct
    rows is >= theta (graph.py:169-188), built on the device."""
    SM, SG, GE, _ = _graph_types(x)
    theta = float(theta)
    if not 0.0 < theta <= 1.0:
        raise GE(f"theta must lie in (0, 1], got {theta}")
    n = int(x.n_rows)
    dev = device or default_device()
    lib = _upload_pattern(dev, x)
    nnz = np.zeros(1, dtype=np.int64)
    _raise_for(lib.fsda_graph_threshold(dev._h, theta, _capi.i64ptr(nnz)))
    return _fetch_graph(dev, lib, n, int(nnz[0]), SM, SG)


def _upload_pattern(dev, x):
    offs, cols = _i64(x.row_offsets), _i64(x.col_indices)
    lib = _capi.lib()
    # the support pattern only (graph.py:69-73): values are not read
    _raise_for(lib.fsda_upload_x(dev._h, int(x.n_rows), int(x.n_cols), _capi.i64ptr(offs),
                                 _capi.i64ptr(cols)))
    dev.n, dev.d = int(x.n_rows), int(x.n_cols)
    dev._loaded = (None, None, None)   # the context's X changed: a resident problem re-uploads
    return lib


def _fetch_graph(dev, lib, n, nnz, SM, SG):
    g_offs = np.empty(n + 1, dtype=np.int64)
    g_cols = np.empty(nnz, dtype=np.int64)
    _raise_for(lib.fsda_graph_fetch(dev._h, _capi.i64ptr(g_offs), _capi.i64ptr(g_cols)))
    adj = SM(n, n, g_offs, g_cols, np.ones(g_cols.size))
    return SG(adjacency=adj, degrees=np.diff(g_offs).astype(np.int64))


def laplacian(graph):
    """L = D - S in CSR with ascending columns (graph.py:191-195): each row
    of a vertex with neighbours holds -1 at its neighbours and its degree on
    the diagonal; isolated vertices store nothing."""
    adj = graph.adjacency
    SM, _, _, LP = _graph_types(adj)
    n = int(adj.n_rows)
    offs = np.asarray(adj.row_offsets, dtype=np.int64)
    cols = np.asarray(adj.col_indices, dtype=np.int64)
    deg = np.asarray(graph.degrees, dtype=np.int64)
    rows = np.repeat(np.arange(n, dtype=np.int64), np.diff(offs))
    has = deg > 0
    d_rows = np.flatnonzero(has)
    all_rows = np.concatenate([rows, d_rows])
    all_cols = np.concatenate([cols, d_rows])
    all_vals = np.concatenate([-np.ones(cols.size), deg[has].astype(np.float64)])
    order = np.lexsort((all_cols, all_rows))
    counts = np.bincount(all_rows, minlength=n)
    l_offs = np.zeros(n + 1, dtype=np.int64)
    np.cumsum(counts, out=l_offs[1:])
    mat = SM(n, n, l_offs, all_cols[order], all_vals[order])
    return LP(matrix=mat, degrees=deg.copy())


def install_into_sdakit_graph(graph_module=None):
    """Route the reference's graph construction to the device: sdakit.graph's
    knn_graph / threshold_graph and the names its callers bound at import
    (cli.py:29, synthetic.py:21, __init__.py:24-27)."""
    g = graph_module or importlib.import_module("sdakit.graph")
    original = getattr(g.knn_graph, "__wrapped_reference__", g.knn_graph)

    def knn_graph_routed(x, k, *args, **kwargs):
        # the device ranking keeps at most 64 neighbours per row: larger k stays
        # on sdakit's own function, so installing never narrows what callers get
        if int(k) > 64:
            return original(x, k, *args, **kwargs)
        return knn_graph(x, k, *args, **kwargs)

    knn_graph_routed.__wrapped_reference__ = original
    knn_graph_routed.__doc__ = knn_graph.__doc__
    g.knn_graph = knn_graph_routed
    g.threshold_graph = threshold_graph
    for mod in ("sdakit", "sdakit.cli", "sdakit.synthetic"):
        try:
            m = importlib.import_module(mod)
        except Exception:
            continue
        if hasattr(m, "knn_graph"):
            m.knn_graph = knn_graph_routed
        if hasattr(m, "threshold_graph"):
            m.threshold_graph = threshold_graph
    return g
