"""Break the drop-in call fsda_solve(p) into its host-visible phases (GPU box).

    python tools/time_e2e.py [--workload cfg2] [--reps 3]
"""
import argparse
import sys
import time
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))

import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_1709_04794_b200 as fb  # noqa: E402
from paper_1709_04794_b200.workloads import make_workload  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--workload", default="cfg2")
ap.add_argument("--reps", type=int, default=3)
args = ap.parse_args()
w = make_workload(args.workload)


def pinned(a):
    t = torch.from_numpy(np.ascontiguousarray(a)).pin_memory()
    keep.append(t)
    out = t.numpy()
    out.setflags(write=False)
    return out


keep = []
x = fb.SparseMatrix.binary(w.n, w.d, pinned(w.x_offsets), pinned(w.x_cols))
lap = fb.Laplacian(fb.SparseMatrix(w.n, w.n, pinned(w.l_offsets), pinned(w.l_cols), pinned(w.l_vals)),
                   w.degrees)
p = fb.SdaProblem(x=x, labels=fb.LabelVector(w.labels), lap=lap, alpha=w.alpha, betas=w.betas,
                  tol=w.tol, max_iter_d=w.max_iter, seed=w.seed)
dev = fb.Device(0)
for rep in range(args.reps):
    t = {}
    t0 = time.perf_counter()
    dev.upload_x(p.x)
    t["upload_x"] = time.perf_counter() - t0
    t0 = time.perf_counter()
    dev.upload_laplacian(p.lap)
    t["upload_laplacian"] = time.perf_counter() - t0
    t0 = time.perf_counter()
    dev.set_labels(p.labels)
    t["set_labels"] = time.perf_counter() - t0
    probe = w.probe()
    t0 = time.perf_counter()
    r = dev.solve_fsda(w.alpha, w.betas, w.tol, w.max_iter, probe)
    t["solve+readback"] = time.perf_counter() - t0
    t0 = time.perf_counter()
    rep_ = fb.fsda_solve(p, device=dev)
    t["fsda_solve(p) total"] = time.perf_counter() - t0
    print(rep, {k: round(v * 1e3, 2) for k, v in t.items()}, "ms", flush=True)
