"""Time device-resident solves of one workload under several environment
settings (each setting gets a fresh context, so knobs read at context
creation take effect) and check every setting's directions are bitwise equal.

    python tools/sweep.py --workload cfg2 --set FSDA_B200_HOT_COLS=0 --set FSDA_B200_HOT_COLS=4096
"""
import argparse
import json
import os
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))

import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_1709_04794_b200 as fb  # noqa: E402
from paper_1709_04794_b200.workloads import make_workload  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--workload", default="cfg2")
ap.add_argument("--solves", type=int, default=10)
ap.add_argument("--set", action="append", default=[], help="VAR=V[,VAR=V] per setting")
ap.add_argument("--profile", action="store_true")
args = ap.parse_args()

w = make_workload(args.workload)
x = fb.SparseMatrix.binary(w.n, w.d, w.x_offsets, w.x_cols)
lap = fb.Laplacian(fb.SparseMatrix(w.n, w.n, w.l_offsets, w.l_cols, w.l_vals), w.degrees)
p = fb.SdaProblem(x=x, labels=fb.LabelVector(w.labels), lap=lap, alpha=w.alpha, betas=w.betas,
                  tol=w.tol, max_iter_d=w.max_iter, seed=w.seed)
flush = torch.empty(256 * 1024 * 1024 // 4, dtype=torch.float32, device="cuda")
ref = None
for setting in args.set or [""]:
    env = dict(kv.split("=", 1) for kv in setting.split(",") if kv)
    old = {k: os.environ.get(k) for k in env}
    os.environ.update(env)
    stream = torch.cuda.Stream()
    torch.cuda.set_stream(stream)
    dev = fb.Device(0, stream=stream.cuda_stream)
    dev.load_problem(p)
    dev.prepare_resident(w.alpha, w.betas, w.tol, w.max_iter, w.probe())
    for _ in range(3):
        dev.solve_async()
    torch.cuda.synchronize()
    ms = []
    for k in range(args.solves):
        flush.fill_(float(k))
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record(stream)
        dev.solve_async()
        b.record(stream)
        b.synchronize()
        ms.append(a.elapsed_time(b))
    r = dev.fetch(directions=True, scores=False)
    d = np.asarray(r.directions)
    same = None
    if ref is None:
        ref = d
    else:
        same = bool(np.array_equal(ref, d))
    out = {"setting": setting, "median_ms": float(np.median(ms)), "min_ms": float(np.min(ms)),
           "solves_per_s": 1000.0 / float(np.median(ms)), "bitwise_equal_first": same}
    if args.profile:
        out["kernels"] = {k["name"]: round(k["ms"] * 1e3, 2) for k in dev.profile_kernels()}
    print(json.dumps(out), flush=True)
    del dev
    for k, v in old.items():
        if v is None:
            os.environ.pop(k, None)
        else:
            os.environ[k] = v
