"""A small run of every device path for compute-sanitizer (memcheck /
racecheck / synccheck, one tool per gpurun call):

    compute-sanitizer --tool memcheck --error-exitcode 9 python tools/sanitize_run.py

cfg1 at K=5: the FSDA sweep (graph and eager launches, fp64 and fp32
storage, both shift-update modes), a 2-task label-mask batch, the row-sharded
solve as a local group of 2 ranks, and the parity probes.  Every result is
checked bitwise against the C oracle, so a run that passes the checks and
reports no sanitizer error is clean on real data."""
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))

import numpy as np  # noqa: E402

import paper_1709_04794_b200 as fb  # noqa: E402
from oracle import c_oracle  # noqa: E402
from paper_1709_04794_b200.sharded import solve_row_sharded_local  # noqa: E402
from paper_1709_04794_b200.workloads import make_workload  # noqa: E402

K = 5
w = make_workload("cfg1", n=3000, d=1500, ell=300, n_pos=60, max_iter=K)
x = fb.SparseMatrix.binary(w.n, w.d, w.x_offsets, w.x_cols)
lap = fb.Laplacian(fb.SparseMatrix(w.n, w.n, w.l_offsets, w.l_cols, w.l_vals), w.degrees)
p = fb.SdaProblem(x=x, labels=fb.LabelVector(w.labels), lap=lap, alpha=w.alpha, betas=w.betas,
                  tol=w.tol, max_iter_d=K, seed=w.seed)


def dirs(rep):
    return np.stack([rep.directions[float(b)] for b in w.betas])


for eager in (False, True):
    for mode in (1, 2):
        dev = fb.Device(0)
        dev.set_eager(eager)
        dev.set_shift_update_mode(mode)
        got = dirs(fb.fsda_solve(p, device=dev))
        c_oracle.set_shift_mode(mode)
        assert np.array_equal(got, c_oracle.fsda_solve_workload(w)["directions"]), (eager, mode)
        c_oracle.set_shift_mode(2)
        del dev
got = dirs(fb.fsda_solve(p, storage=32))
c_oracle.set_storage(32)
assert np.array_equal(got, c_oracle.fsda_solve_workload(w)["directions"])
c_oracle.set_storage(64)

rng = np.random.default_rng(1)
masks = []
for _ in range(2):
    lab = np.zeros(w.n, dtype=np.int8)
    idx = rng.choice(w.n, size=200, replace=False)
    lab[idx] = -1
    lab[idx[:50]] = 1
    masks.append(lab)
res = fb.solve_label_sets(x, lap, masks, w.alpha, w.betas, w.tol, K, seeds=[0, 1])
for lab, r, seed in zip(masks, res, [0, 1]):
    ref = c_oracle.fsda_solve(w.x_offsets, w.x_cols, w.d, w.l_offsets, w.l_cols, w.l_vals, lab,
                              w.alpha, w.betas, w.tol, K, np.random.default_rng(seed).uniform(-1, 1, w.d))
    assert np.array_equal(r.directions, ref["directions"])

out = solve_row_sharded_local(w.x_offsets, w.x_cols, w.d, w.l_offsets, w.l_cols, w.l_vals, w.labels,
                              w.alpha, w.betas, w.tol, K, seed=w.seed, world=2)
ref = c_oracle.fsda_solve_sharded(w.x_offsets, w.x_cols, w.d, w.l_offsets, w.l_cols, w.l_vals, w.labels,
                                  w.alpha, w.betas, w.tol, K, w.probe(), out["row_bounds"])
assert np.array_equal(out["directions"], ref["directions"])

v = np.random.default_rng(3).standard_normal(w.d)
assert np.array_equal(fb.matvec(x, v), c_oracle.matvec(w.x_offsets, w.x_cols, v))
print("sanitize_run ok")
