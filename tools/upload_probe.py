"""Time fsda_solve(p)'s upload (load_problem) of a workload on cuda:0, with
the current narrowing mode (FSDA_B200_DEVICE_NARROW), for pageable and
page-locked inputs; phase marks with FSDA_B200_TRACE=1.

    python tools/upload_probe.py [--workload cfg3] [--reps 2]
"""
import argparse
import json
import sys
import time
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))

import torch  # noqa: E402

import paper_1709_04794_b200 as fb  # noqa: E402
from paper_1709_04794_b200.workloads import make_workload, make_workload_chunked  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--workload", default="cfg3")
ap.add_argument("--reps", type=int, default=2)
args = ap.parse_args()
w = make_workload_chunked(args.workload) if args.workload == "cfg5" else make_workload(args.workload)


def problem(pin):
    cp = (lambda a: torch.from_numpy(a).pin_memory().numpy()) if pin else (lambda a: a)
    x = fb.SparseMatrix.binary(w.n, w.d, cp(w.x_offsets), cp(w.x_cols))
    lap = fb.Laplacian(fb.SparseMatrix(w.n, w.n, cp(w.l_offsets), cp(w.l_cols), cp(w.l_vals)), w.degrees)
    return fb.SdaProblem(x=x, labels=fb.LabelVector(w.labels), lap=lap, alpha=w.alpha, betas=w.betas,
                         tol=w.tol, max_iter_d=w.max_iter, seed=w.seed)


out = {"workload": w.name}
dev = fb.Device(0)
for pin in (False, True):
    p = problem(pin)
    ts = []
    for _ in range(args.reps):
        t0 = time.perf_counter()
        dev.load_problem(p)
        torch.cuda.synchronize()
        ts.append(time.perf_counter() - t0)
    out["pinned" if pin else "pageable"] = ts
print(json.dumps(out))
