"""Golden k-NN and threshold graphs from the UNMODIFIED reference
(sdakit.graph.knn_graph / threshold_graph).

Run in the authoring container, where /root/reference exists:

    PYTHONPATH=/root/repo python tests/golden/make_golden_graph.py

Inputs: the reference's own synthetic generators (random_sparse_binary with
and without a column-popularity power, random_sparse_rows, clustered_binary,
two_chain_fingerprints — stored as raw CSR arrays) and this package's cfg1
workload (stored as its digest; the tests regenerate it).  Outputs: each
graph's adjacency (CSR) as the reference builds it.  Nothing here is
imported at test time.
"""

from __future__ import annotations

import sys
import time
from pathlib import Path

import numpy as np

sys.path.insert(0, "/root/reference/pkg/src")

from sdakit.graph import knn_graph, threshold_graph  # noqa: E402
from sdakit.sparse import SparseMatrix  # noqa: E402
from sdakit.synthetic import (clustered_binary, random_sparse_binary,  # noqa: E402
                              random_sparse_rows, two_chain_fingerprints)

from paper_1709_04794_b200.workloads import make_workload, workload_digest  # noqa: E402

OUT = Path(__file__).resolve().parent / "graph_reference.npz"
THETAS = (0.15, 0.3, 0.5, 1.0)


def main():
    cases = []
    # (name, matrix, k)
    cases.append(("uniform", random_sparse_binary(300, 80, 2400, seed=3), 5))
    cases.append(("zipf", random_sparse_binary(500, 200, 6000, seed=4, column_power=1.1), 10))
    cases.append(("zipf_k1", random_sparse_binary(400, 150, 3000, seed=5, column_power=1.3), 1))
    cases.append(("sparse_pad", random_sparse_binary(200, 400, 150, seed=6), 4))   # many empty rows
    cases.append(("rows", random_sparse_rows(250, 60, 6, seed=7), 15))
    cases.append(("ones_column", random_sparse_binary(300, 50, 900, seed=8, ones_column=True), 7))
    x_cl, _ = clustered_binary(400, 120, seed=9)
    cases.append(("clustered", x_cl, 10))
    x_fp, _ = two_chain_fingerprints(300, seed=10)
    cases.append(("fingerprints", x_fp, 8))
    cases.append(("wide", random_sparse_binary(600, 6000, 30000, seed=11, column_power=1.05), 12))
    out = {}
    for name, x, k in cases:
        g = knn_graph(x, k)
        out[f"{name}__x_shape"] = np.array([x.n_rows, x.n_cols, k])
        out[f"{name}__x_offsets"] = np.asarray(x.row_offsets, dtype=np.int64)
        out[f"{name}__x_cols"] = np.asarray(x.col_indices, dtype=np.int32)
        out[f"{name}__g_offsets"] = np.asarray(g.adjacency.row_offsets, dtype=np.int64)
        out[f"{name}__g_cols"] = np.asarray(g.adjacency.col_indices, dtype=np.int32)
        print(name, x.n_rows, x.n_cols, x.nnz, "k", k, "edges", g.n_edges)
        for theta in THETAS:
            t = threshold_graph(x, theta)
            tag = f"{name}__t{int(round(theta * 100)):03d}"
            out[f"{tag}_offsets"] = np.asarray(t.adjacency.row_offsets, dtype=np.int64)
            out[f"{tag}_cols"] = np.asarray(t.adjacency.col_indices, dtype=np.int32)
            print("   threshold", theta, "edges", t.n_edges)
    # cfg1 (10k x 5k, Zipf 1.1, Poisson 25), k = 10 — the BASELINE plumbing size
    w = make_workload("cfg1")
    xw = SparseMatrix(w.n, w.d, w.x_offsets, w.x_cols, np.ones(w.nnz))
    t0 = time.perf_counter()
    g = knn_graph(xw, 10)
    out["cfg1__seconds"] = np.array([time.perf_counter() - t0])
    out["cfg1__digest"] = np.array([workload_digest(w)])
    out["cfg1__g_offsets"] = np.asarray(g.adjacency.row_offsets, dtype=np.int64)
    out["cfg1__g_cols"] = np.asarray(g.adjacency.col_indices, dtype=np.int32)
    print("cfg1 edges", g.n_edges, "reference seconds", out["cfg1__seconds"][0])
    t = threshold_graph(xw, 0.3)
    out["cfg1__t030_offsets"] = np.asarray(t.adjacency.row_offsets, dtype=np.int64)
    out["cfg1__t030_cols"] = np.asarray(t.adjacency.col_indices, dtype=np.int32)
    out["thetas"] = np.array(THETAS)
    print("cfg1 threshold 0.3 edges", t.n_edges)
    out["names"] = np.array([c[0] for c in cases])
    np.savez_compressed(OUT, **out)
    print("wrote", OUT)


if __name__ == "__main__":
    main()
