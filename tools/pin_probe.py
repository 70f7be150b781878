"""How the host placement of the inputs moves the drop-in call (GPU box):
fsda_solve(p) with (a) pageable numpy arrays, (b) torch.pin_memory() copies
(cudaHostAlloc), (c) the same numpy arrays page-locked in place
(cudaHostRegister).

    python tools/pin_probe.py [--workload cfg3] [--reps 6]
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
ap.add_argument("--workload", default="cfg3")
ap.add_argument("--reps", type=int, default=6)
args = ap.parse_args()
w = make_workload(args.workload)
keep = []


def copy_pinned(a):
    t = torch.from_numpy(np.ascontiguousarray(a)).pin_memory()
    keep.append(t)
    out = t.numpy()
    out.setflags(write=False)
    return out


def register(a):
    a = np.ascontiguousarray(a)
    rc = torch.cuda.cudart().cudaHostRegister(a.ctypes.data, a.nbytes, 0)
    assert int(rc) == 0, rc
    keep.append(a)
    return a


def problem(f):
    x = fb.SparseMatrix.binary(w.n, w.d, f(w.x_offsets), f(w.x_cols))
    lap = fb.Laplacian(fb.SparseMatrix(w.n, w.n, f(w.l_offsets), f(w.l_cols), f(w.l_vals)), w.degrees)
    return fb.SdaProblem(x=x, labels=fb.LabelVector(w.labels), lap=lap, alpha=w.alpha, betas=w.betas,
                         tol=w.tol, max_iter_d=w.max_iter, seed=w.seed)


dev = fb.Device(0)
probs = {"pageable": problem(lambda a: a), "pin_memory copy": problem(copy_pinned)}
probs["registered in place"] = problem(register)
for name, p in probs.items():
    for _ in range(2):
        fb.fsda_solve(p, device=dev)
for rnd in range(2):
    for name, p in probs.items():
        ts = []
        for _ in range(args.reps):
            t0 = time.perf_counter()
            fb.fsda_solve(p, device=dev)
            ts.append((time.perf_counter() - t0) * 1e3)
        print(f"{name:22s} mean {np.mean(ts):7.2f} ms  median {np.median(ts):7.2f}  min {min(ts):7.2f}", flush=True)
