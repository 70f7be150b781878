"""Where the row-sharded solve's time goes at world 1 (GPU box):

    python tools/shard_probe.py [--workload cfg3] [--solves 3]

Times, with CUDA events on the rank's stream, (a) the single-GPU fsda_solve
path (resident, graph), (b) fsda_solve_sharded with the local-context
backend (eager phases, device copies), (c) fsda_solve_sharded over NCCL at
world 1 (captured iteration graph), each a whole call including the result
readback, and prints one JSON line."""
import argparse
import json
import os
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))

import numpy as np  # noqa: E402
import torch  # noqa: E402
import torch.distributed as dist  # noqa: E402

import paper_1709_04794_b200 as fb  # noqa: E402
from paper_1709_04794_b200 import sharded  # noqa: E402
from paper_1709_04794_b200.workloads import make_workload  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--workload", default="cfg3")
ap.add_argument("--solves", type=int, default=3)
args = ap.parse_args()
w = make_workload(args.workload)
n1, n2 = sharded._class_counts(w.labels)
probe = w.probe()


def timed(fn):
    fn()
    torch.cuda.synchronize()
    out = []
    for _ in range(args.solves):
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        fn()
        b.record()
        torch.cuda.synchronize()
        out.append(a.elapsed_time(b))
    return min(out)


res = {"workload": w.name}
dev = fb.Device(0)
p = fb.SdaProblem(x=fb.SparseMatrix.binary(w.n, w.d, w.x_offsets, w.x_cols),
                  labels=fb.LabelVector(w.labels),
                  lap=fb.Laplacian(fb.SparseMatrix(w.n, w.n, w.l_offsets, w.l_cols, w.l_vals), w.degrees),
                  alpha=w.alpha, betas=w.betas, tol=w.tol, max_iter_d=w.max_iter, seed=w.seed)
dev.load_problem(p)
res["single_fsda_solve_ms"] = timed(lambda: dev.solve_fsda(w.alpha, w.betas, w.tol, w.max_iter, probe,
                                                         scores=False))
del dev
b = sharded.partition_rows(w.x_offsets, 1, w.l_offsets)
loc = [sharded.ShardRank(sharded.take_shard(w.x_offsets, w.x_cols, w.d, w.l_offsets, w.l_cols, w.l_vals,
                                            w.labels, b, 0), b, 0)]
res["local_world1_ms"] = timed(lambda: sharded._solve_ranks(loc, int(w.d), w.alpha, w.betas, w.tol,
                                                            w.max_iter, probe, n1, n2, scores=False))
del loc
os.environ.setdefault("MASTER_ADDR", "127.0.0.1")
os.environ.setdefault("MASTER_PORT", "29517")
dist.init_process_group("nccl", rank=0, world_size=1, device_id=torch.device("cuda", 0))
out = sharded.solve_row_sharded(w.x_offsets, w.x_cols, w.d, w.l_offsets, w.l_cols, w.l_vals, w.labels,
                                w.alpha, w.betas, w.tol, w.max_iter, w.seed, device=0)
r = out["rank"]
res["nccl_world1_ms"] = timed(lambda: sharded._solve_ranks([r], int(w.d), w.alpha, w.betas, w.tol,
                                                           w.max_iter, probe, n1, n2, scores=False))
dist.destroy_process_group()
print(json.dumps(res))
