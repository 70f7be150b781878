"""cfg5 (8M x 2M, 640M nnz, 15-NN, 30 shifts, K=200) on ONE B200, in BASELINE's
fp32 storage with fp64 reductions (and, for comparison, fp64 storage).

    python tools/cfg5_run.py [--max-iter K] [--solves 3] [--scale 1.0] [--storage 32,64]

Generates the problem row-chunked on the host, uploads it, and times
device-resident solves with CUDA events.  Checks: two solves are bitwise
identical, every shift ran K iterations, and the labeled-row AUC of the
projected ratings.  Prints one JSON line.
"""
import argparse
import json
import sys
import time
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))

import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_1709_04794_b200 as fb  # noqa: E402
from paper_1709_04794_b200.workloads import CONFIGS, make_workload_chunked  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--max-iter", type=int, default=None)
ap.add_argument("--solves", type=int, default=3)
ap.add_argument("--scale", type=float, default=1.0, help="row/feature scale (smoke runs)")
ap.add_argument("--storage", default="32,64", help="storage modes to time, in order")
args = ap.parse_args()

cfg = CONFIGS["cfg5"]
over = {}
if args.scale != 1.0:
    over = dict(n=int(cfg["n"] * args.scale), d=int(cfg["d"] * args.scale),
                ell=int(cfg["ell"] * args.scale), n_pos=int(cfg["n_pos"] * args.scale))
t0 = time.perf_counter()
w = make_workload_chunked("cfg5", max_iter=args.max_iter, **over)
t_gen = time.perf_counter() - t0
x = fb.SparseMatrix.binary(w.n, w.d, w.x_offsets, w.x_cols)
lap = fb.Laplacian(fb.SparseMatrix(w.n, w.n, w.l_offsets, w.l_cols, w.l_vals), w.degrees)
p = fb.SdaProblem(x=x, labels=fb.LabelVector(w.labels), lap=lap, alpha=w.alpha, betas=w.betas,
                  tol=w.tol, max_iter_d=w.max_iter, seed=w.seed)
stream = torch.cuda.Stream()
torch.cuda.set_stream(stream)
dev = fb.Device(0, stream=stream.cuda_stream)
t0 = time.perf_counter()
dev.load_problem(p)
torch.cuda.synchronize()
t_up = time.perf_counter() - t0
lab = w.labels


def aucs_of(scores):
    out = []
    for s in range(scores.shape[0]):
        sc = scores[s][lab != 0]
        y = lab[lab != 0] == 1
        order = np.argsort(sc, kind="stable")
        ranks = np.empty(sc.size)
        ranks[order] = np.arange(1, sc.size + 1)
        out.append(float((ranks[y].sum() - y.sum() * (y.sum() + 1) / 2) / (y.sum() * (~y).sum())))
    return out


runs = {}
dirs = {}
for bits in [int(b) for b in args.storage.split(",")]:
    dev.set_storage(bits)
    dev.prepare_resident(w.alpha, w.betas, w.tol, w.max_iter, w.probe())
    dev.solve_async()                                   # warm (graph capture)
    torch.cuda.synchronize()
    first = dev.fetch(directions=True, scores=False)
    ms = []
    for _ in range(args.solves):
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record(stream)
        dev.solve_async()
        b.record(stream)
        torch.cuda.synchronize()
        ms.append(a.elapsed_time(b))
    res = dev.fetch(directions=True, scores=True)
    au = aucs_of(res.scores)
    dirs[bits] = res.directions
    runs[f"fp{bits}"] = {"solve_ms": ms, "solves_per_s": 1000.0 / float(np.median(ms)),
                         "n_applies": res.n_applies,
                         "bitwise_repeatable": bool(np.array_equal(first.directions, res.directions)),
                         "labeled_auc_min_max": [min(au), max(au)], "labeled_auc": au}
if 32 in dirs and 64 in dirs:
    d32, d64 = dirs[32], dirs[64]
    rel = np.linalg.norm(d32 - d64, axis=1) / np.linalg.norm(d64, axis=1)
    runs["fp32_vs_fp64_full_K"] = {
        "max_rel_dw": float(rel.max()),
        "max_abs_dauc": float(np.max(np.abs(np.array(runs["fp32"]["labeled_auc"]) -
                                            np.array(runs["fp64"]["labeled_auc"])))),
        "note": "at the full K = 200, past the Krylov stability horizon; the 1e-3 gate is stated at "
                "the stable K (tests/test_gpu_parity.py::test_fp32_storage_gate_vs_fp64)"}
for r in runs.values():
    r.pop("labeled_auc", None)
out = {
    "workload": "cfg5", "n": w.n, "d": w.d, "nnz": w.nnz, "laplacian_nnz": int(w.l_cols.size),
    "n_shifts": int(w.betas.size), "max_iter": w.max_iter, "gpus": 1, "generate_s": t_gen,
    "upload_s": t_up, "runs": runs,
    "device_mem_used_gb": (lambda fr_tot: (fr_tot[1] - fr_tot[0]) / 1e9)(torch.cuda.mem_get_info()),
}
print(json.dumps(out))
