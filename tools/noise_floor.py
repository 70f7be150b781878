"""The reference's own noise floor per Krylov dimension.

Runs the reference-order oracle (oracle/ref_numpy.py, pinned bit for bit to
the unmodified reference) twice on a workload: once as is, once with every
operator output multiplied by (1 + 1.1e-16 * N(0, 1)) — an ulp-level
reordering of the SpMV sums.  The max over shifts of rel||dw|| at each K
tells how far any correct implementation with a different summation order
can sit from the reference; K_stable is the largest K where it stays
<= 1e-9 (so a 1e-6 gate has three orders of margin).

    python tools/noise_floor.py --workload cfg3 --kmax 60 --every 10
"""
import argparse
import json
import sys
import time
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))

import numpy as np  # noqa: E402

from oracle import ref_numpy  # noqa: E402
from paper_1709_04794_b200.workloads import make_workload  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--workload", default="cfg3")
ap.add_argument("--kmax", type=int, default=60)
ap.add_argument("--every", type=int, default=10)
ap.add_argument("--out", default=None)
args = ap.parse_args()

w = make_workload(args.workload)
prob = ref_numpy.Problem.from_workload(w)
ks = list(range(args.every, args.kmax + 1, args.every))


def run(perturb):
    snaps = {}
    rng = np.random.default_rng(12345)

    def op(alpha, mu, v):
        q = prob.operator(alpha, mu, v)
        if perturb:
            q = q * (1.0 + 1.1e-16 * rng.standard_normal(q.size))
        return q

    def on_iter(i, sols):
        if i + 1 in ks:
            snaps[i + 1] = ref_numpy.orient(prob, sols)

    ref_numpy.fsda_solve(prob, w.alpha, w.betas, w.tol, args.kmax, w.seed, on_iter=on_iter, operator=op)
    return snaps


t0 = time.time()
a = run(False)
b = run(True)
rows = []
for k in ks:
    da, db = a[k], b[k]
    rel = np.linalg.norm(da - db, axis=1) / np.linalg.norm(da, axis=1)
    rows.append({"K": k, "max_rel_dw": float(rel.max()), "median_rel_dw": float(np.median(rel))})
    print(json.dumps(rows[-1]), flush=True)
stable = max([r["K"] for r in rows if r["max_rel_dw"] <= 1e-9] or [0])
res = {"workload": args.workload, "rows": rows, "K_stable": stable,
       "perturbation": "operator output * (1 + 1.1e-16 N(0,1))", "seconds": time.time() - t0}
print(json.dumps({"K_stable": stable}))
if args.out:
    Path(args.out).write_text(json.dumps(res, indent=1) + "\n")
