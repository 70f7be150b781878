"""Run complete FSDA solves of a workload on cuda:0 (for ncu launch lists).

    python tools/ncu_solve.py [--workload cfg2] [--solves 2] [--eager]
"""
import argparse
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))

import paper_1709_04794_b200 as fb  # noqa: E402
from paper_1709_04794_b200.workloads import make_workload  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--workload", default="cfg2")
ap.add_argument("--solves", type=int, default=2)
ap.add_argument("--max-iter", type=int, default=None)
args = ap.parse_args()

w = make_workload(args.workload, max_iter=args.max_iter)
dev = fb.Device(0)
x = fb.SparseMatrix.binary(w.n, w.d, w.x_offsets, w.x_cols)
lap = fb.Laplacian(fb.SparseMatrix(w.n, w.n, w.l_offsets, w.l_cols, w.l_vals), w.degrees)
p = fb.SdaProblem(x=x, labels=fb.LabelVector(w.labels), lap=lap, alpha=w.alpha, betas=w.betas,
                  tol=w.tol, max_iter_d=w.max_iter, seed=w.seed)
dev.load_problem(p)
dev.prepare_resident(w.alpha, w.betas, w.tol, w.max_iter, w.probe())
for _ in range(args.solves):
    dev.solve_async()
r = dev.fetch(directions=False, scores=False)
print("solves", args.solves, "n_applies", r.n_applies, "launches/solve", r.launches)
