"""cfg5 (8M x 2M, 640M nnz, 15-NN, 30 shifts) — the largest BASELINE config —
on one B200 against the C oracle, bit for bit, at a short Krylov dimension
(the oracle needs ~1 s per iteration on the host at this size):

    python tools/cfg5_parity.py [--max-iter 3] [--storage 64,32]

Prints one JSON line: per storage mode, whether directions, scores,
residuals and iteration counts equal the oracle's exactly."""
import argparse
import json
import sys
import time
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))

import numpy as np  # noqa: E402

import paper_1709_04794_b200 as fb  # noqa: E402
from oracle import c_oracle  # noqa: E402
from paper_1709_04794_b200.workloads import make_workload_chunked  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--max-iter", type=int, default=3)
ap.add_argument("--storage", default="64,32")
args = ap.parse_args()
K = args.max_iter
t0 = time.perf_counter()
w = make_workload_chunked("cfg5", max_iter=K)
out = {"workload": "cfg5", "n": w.n, "d": w.d, "nnz": w.nnz, "laplacian_nnz": int(w.l_cols.size),
       "n_shifts": int(w.betas.size), "max_iter": K, "generate_s": time.perf_counter() - t0, "modes": {}}
p = fb.SdaProblem(x=fb.SparseMatrix.binary(w.n, w.d, w.x_offsets, w.x_cols),
                  labels=fb.LabelVector(w.labels),
                  lap=fb.Laplacian(fb.SparseMatrix(w.n, w.n, w.l_offsets, w.l_cols, w.l_vals), w.degrees),
                  alpha=w.alpha, betas=w.betas, tol=w.tol, max_iter_d=K, seed=w.seed)
dev = fb.Device(0)
for bits in [int(b) for b in args.storage.split(",")]:
    dev.set_storage(bits)
    rep = fb.fsda_solve(p, device=dev)
    mode = dev.last_shift_update_mode
    c_oracle.set_shift_mode(mode)
    c_oracle.set_storage(bits)
    t1 = time.perf_counter()
    ref = c_oracle.fsda_solve_workload(w, max_iter=K)
    t_o = time.perf_counter() - t1
    c_oracle.set_storage(64)
    c_oracle.set_shift_mode(2)
    dirs = np.stack([rep.directions[float(b)] for b in w.betas])
    scores = np.stack([rep.ratings[float(b)].scores for b in w.betas])
    out["modes"][f"fp{bits}"] = {
        "shift_update_mode": mode,
        "directions_equal": bool(np.array_equal(dirs, ref["directions"])),
        "scores_equal": bool(np.array_equal(scores, ref["scores"])),
        "residuals_equal": bool(np.array_equal(rep.regression.residuals, ref["residuals"])),
        "iterations_equal": bool(np.array_equal(rep.regression.iterations, ref["iterations"])),
        "n_applies": int(rep.regression.operator_applications),
        "oracle_s": t_o}
print(json.dumps(out))
