"""Multi-task batch throughput (cfg4 shape) against one-at-a-time solves.

    python tools/bench_batch.py [--workload cfg4] [--tasks 64] [--max-iter K]
                                [--seq-tasks 2] [--reps 1]

X and L are resident; each batch call uploads the T label masks and probes
and returns the directions (scores stay on the device: at cfg4 they are
15 GB).  Prints one JSON line: task-solves/s batched, task-solves/s
sequential (fsda_set_label_mask + fsda_solve per task, measured on
--seq-tasks tasks), and the ratio.
"""
import argparse
import json
import sys
import time
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))

import numpy as np  # noqa: E402

import paper_1709_04794_b200 as fb  # noqa: E402
from paper_1709_04794_b200.workloads import CONFIGS, make_workload, task_masks  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--workload", default="cfg4")
ap.add_argument("--tasks", type=int, default=None)
ap.add_argument("--max-iter", type=int, default=None)
ap.add_argument("--seq-tasks", type=int, default=2)
ap.add_argument("--reps", type=int, default=1)
ap.add_argument("--storage", type=int, default=64, help="32: fp32 storage with fp64 reductions")
ap.add_argument("--cache", default=None, help="pickle the generated workload here and reuse it (variant sweeps)")
args = ap.parse_args()

cfg = CONFIGS[args.workload]
T = args.tasks or cfg.get("tasks", 32)
if args.cache and Path(args.cache).exists():
    import pickle
    with open(args.cache, "rb") as fh:
        w = pickle.load(fh)
else:
    w = make_workload(args.workload, max_iter=args.max_iter)
    if args.cache:
        import pickle
        with open(args.cache, "wb") as fh:
            pickle.dump(w, fh, protocol=4)
masks = task_masks(w.n, T, cfg.get("task_frac", 0.01), cfg.get("task_pos", 0.1), seed=77)
probes = np.stack([np.random.default_rng(s).uniform(-1, 1, w.d) for s in range(T)])
x = fb.SparseMatrix.binary(w.n, w.d, w.x_offsets, w.x_cols)
lap = fb.Laplacian(fb.SparseMatrix(w.n, w.n, w.l_offsets, w.l_cols, w.l_vals), w.degrees)
dev = fb.Device(0)
dev.set_storage(args.storage)
dev.upload_x(x)
dev.upload_laplacian(lap)

# warm: allocations at the full task count and Krylov dimension (the deferred
# shift updates keep K + 1 task-minor residuals: 39 GB at cfg4)
dev.solve_batch(masks, w.alpha, w.betas, w.tol, w.max_iter, probes, scores=False)
best = None
for _ in range(args.reps):
    t0 = time.perf_counter()
    res = dev.solve_batch(masks, w.alpha, w.betas, w.tol, w.max_iter, probes, scores=False)
    el = time.perf_counter() - t0
    best = el if best is None else min(best, el)
napp = [r.n_applies for r in res]

seq_el = 0.0
S = min(args.seq_tasks, T)
if S:
    dev.set_label_mask(masks[0])      # warm: graph capture of the single-task solve
    dev.solve_fsda(w.alpha, w.betas, w.tol, w.max_iter, probes[0], scores=False)
for t in range(S):
    dev.set_label_mask(masks[t])
    t0 = time.perf_counter()
    r = dev.solve_fsda(w.alpha, w.betas, w.tol, w.max_iter, probes[t], scores=False)
    seq_el += time.perf_counter() - t0
    np.testing.assert_array_equal(r.directions, res[t].directions)

out = {
    "workload": args.workload, "storage_bits": args.storage, "tasks": T, "n_shifts": int(w.betas.size), "max_iter": w.max_iter,
    "n_applies": [min(napp), max(napp)],
    "batch_s": best, "batch_task_solves_per_s": T / best,
    "sequential_task_s": seq_el / S if S else None,
    "sequential_task_solves_per_s": S / seq_el if S else None,
    "speedup": (T / best) / (S / seq_el) if S else None, "bitwise_equal_tasks_checked": S,
}
print(json.dumps(out))
