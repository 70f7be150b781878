"""Per-CTA phase timeline of k_xt_coop (the last launch of one solve).

    python tools/xt_trace.py [--workload cfg2]
"""
import argparse
import ctypes as C
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import numpy as np  # noqa: E402

import paper_1709_04794_b200 as fb  # noqa: E402
from paper_1709_04794_b200 import _capi  # noqa: E402
from paper_1709_04794_b200.workloads import make_workload  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--workload", default="cfg2")
args = ap.parse_args()
w = make_workload(args.workload)
x = fb.SparseMatrix.binary(w.n, w.d, w.x_offsets, w.x_cols)
lap = fb.Laplacian(fb.SparseMatrix(w.n, w.n, w.l_offsets, w.l_cols, w.l_vals), w.degrees)
p = fb.SdaProblem(x=x, labels=fb.LabelVector(w.labels), lap=lap, alpha=w.alpha, betas=w.betas,
                  tol=w.tol, max_iter_d=w.max_iter, seed=w.seed)
dev = fb.Device(0)
dev.load_problem(p)
dev.prepare_resident(w.alpha, w.betas, w.tol, w.max_iter, w.probe())
lib = _capi.lib()
lib.fsda_debug_xt_trace.argtypes = [C.c_int, C.c_void_p]
for _ in range(2):
    dev.solve_async()
dev.fetch(directions=False, scores=False)
lib.fsda_debug_xt_trace(1, None)
dev.solve_async()
dev.fetch(directions=False, scores=False)
buf = np.zeros((5, 1024), dtype=np.uint64)
lib.fsda_debug_xt_trace(0, buf.ctypes.data)
nb = int((buf[0] > 0).sum())
t = buf[:, :nb].astype(np.int64)
t0 = t[0].min()
rel = (t - t0) / 1000.0
print(f"CTAs {nb}; kernel span {rel[4].max():.2f} us")
names = ["start", "end 1a", "end 1b", "after sync", "end"]
for k in range(5):
    print(f"  {names[k]:>10}: min {rel[k].min():7.2f}  median {np.median(rel[k]):7.2f}  max {rel[k].max():7.2f} us")
print("  phase 1a per CTA  : median %.2f max %.2f" % (np.median(rel[1] - rel[0]), (rel[1] - rel[0]).max()))
print("  phase 1b per CTA  : median %.2f max %.2f" % (np.median(rel[2] - rel[1]), (rel[2] - rel[1]).max()))
print("  sync wait per CTA : median %.2f max %.2f" % (np.median(rel[3] - rel[2]), (rel[3] - rel[2]).max()))
print("  phase 2 per CTA   : median %.2f max %.2f" % (np.median(rel[4] - rel[3]), (rel[4] - rel[3]).max()))
