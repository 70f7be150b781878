"""Time the device k-NN graph build (knn_graph) on BASELINE-shaped X.

    python tools/graph_bench.py [--workload cfg2] [--k 10] [--reps 3] [--oracle]
"""
import argparse
import json
import sys
import time
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import numpy as np  # noqa: E402

import paper_1709_04794_b200 as fb  # noqa: E402
import paper_1709_04794_b200.graph as G  # noqa: E402
from paper_1709_04794_b200.workloads import make_workload  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--workload", default="cfg1")
ap.add_argument("--k", type=int, default=10)
ap.add_argument("--reps", type=int, default=3)
ap.add_argument("--oracle", action="store_true")
args = ap.parse_args()
w = make_workload(args.workload)
x = fb.SparseMatrix.binary(w.n, w.d, w.x_offsets, w.x_cols)
dev = fb.Device(0)
G.knn_graph(x, args.k, device=dev)            # warm (cuBLAS handle, allocations)
ts = []
for _ in range(args.reps):
    t0 = time.perf_counter()
    g = G.knn_graph(x, args.k, device=dev)
    ts.append(time.perf_counter() - t0)
out = {"workload": args.workload, "n": w.n, "d": w.d, "nnz": w.nnz, "k": args.k,
       "edges": g.n_edges, "gpu_s": min(ts), "gpu_s_all": ts}
if args.oracle:
    from oracle import graph_oracle
    t0 = time.perf_counter()
    go, gc = graph_oracle.knn_adjacency(w.n, w.d, w.x_offsets, w.x_cols, args.k)
    out["oracle_s"] = time.perf_counter() - t0
    out["equal_to_oracle"] = bool(np.array_equal(go, g.adjacency.row_offsets) and
                                  np.array_equal(gc, g.adjacency.col_indices))
print(json.dumps(out), flush=True)
