"""Golden fixtures of the reference's own FSDA acceptance cases, for running
them through the drop-in plugin on the GPU (tests/test_gpu_acceptance.py).

Run in the authoring container, where /root/reference exists:

    PYTHONPATH=/root/repo python tests/golden/make_golden_acceptance.py

Cases (the reference's tests, reproduced by calling its own public helpers
with the same seeds; nothing of the reference is copied):
* test_sda.py::test_fsda_matches_dense_pencil_dominant_eigenvector
* test_sda.py::test_fsda_alpha_zero_is_regularized_lda
* test_sda.py::test_fsda_separable_problem_rates_perfectly
* test_sda.py::test_report_directions_consistent_with_scores (fsda)
* test_sda.py::test_fsda_is_deterministic
* test_acceptance.py criterion 1 (20 problems vs the dense centered pencil)
* test_acceptance.py criterion 4 (centering annihilation, 100 + 25 cases)
* test_acceptance.py criterion 5 (graph smoothing gain, 10 seeds x 2000 samples)

Stored per problem: the CSR arrays of X and L (int32 indices), labels, the
solve knobs, the reference's own outputs (sdakit.sda.solve(p, "fsda")
directions / scores) and each test's check data (dominant eigenvector of the
dense pencil, regularized Fisher direction, truth labels).  The check data
are computed here with numpy/scipy from the same dense assembly the
reference's tests use.
"""

from __future__ import annotations

import sys
from pathlib import Path

import numpy as np
from scipy.linalg import eigh

REF = "/root/reference/pkg/src"
sys.path.insert(0, REF)
sys.path.insert(0, "/root/reference/pkg/tests")

from sdakit.evaluation import auc_roc  # noqa: E402
from sdakit.graph import knn_graph, laplacian  # noqa: E402
from sdakit.sda import SdaProblem, solve  # noqa: E402
from sdakit.sparse import LabelVector, build_sparse  # noqa: E402
from sdakit.synthetic import (clustered_binary, knn_problem_parts,  # noqa: E402
                              labeled_first_parts, two_chain_fingerprints)
from conftest import dense_of, dense_smoother, dense_w, random_binary_matrix  # noqa: E402

OUT = Path(__file__).resolve().parent / "acceptance_reference.npz"


def put(store, key, p, extra=None, run=True):
    """Arrays of SdaProblem p under key__*, plus the reference's solve."""
    store[f"{key}__x_offsets"] = np.asarray(p.x.row_offsets, dtype=np.int32)
    store[f"{key}__x_cols"] = np.asarray(p.x.col_indices, dtype=np.int32)
    store[f"{key}__shape"] = np.array([p.x.n_rows, p.x.n_cols], dtype=np.int64)
    m = p.lap.matrix
    store[f"{key}__l_offsets"] = np.asarray(m.row_offsets, dtype=np.int32)
    store[f"{key}__l_cols"] = np.asarray(m.col_indices, dtype=np.int32)
    store[f"{key}__l_vals"] = np.asarray(m.values, dtype=np.float64)
    store[f"{key}__degrees"] = np.asarray(p.lap.degrees, dtype=np.float64)
    store[f"{key}__labels"] = np.asarray(p.labels.labels, dtype=np.int8)
    store[f"{key}__knobs"] = np.array([p.alpha, p.tol, p.max_iter_d, p.seed], dtype=np.float64)
    store[f"{key}__betas"] = np.asarray(p.betas.betas, dtype=np.float64)
    if run:
        rep = solve(p, "fsda")
        store[f"{key}__ref_directions"] = np.stack([rep.directions[float(b)] for b in p.betas.betas])
        store[f"{key}__ref_scores"] = np.stack([rep.ratings[float(b)].scores for b in p.betas.betas])
    for k, v in (extra or {}).items():
        store[f"{key}__{k}"] = np.asarray(v)


def main():
    s = {}
    # test_sda.py: dense pencil dominant eigenvector (n=60, d=8, seed 2, beta 1e-3, tol 1e-10)
    beta = 1e-3
    x, truth = clustered_binary(60, 8, seed=2)
    g, lap = knn_problem_parts(x, k=3)
    x2, lap2, labels, truth2, _ = labeled_first_parts(x, lap, truth, 6, seed=3)
    p = SdaProblem(x=x2, labels=labels, lap=lap2, alpha=0.5, betas=(beta,), tol=1e-10)
    xd = dense_of(p.x)
    mu = xd[: p.labels.n_labeled].mean(axis=0)
    xc = xd - mu
    a = xc.T @ dense_w(p.labels) @ xc
    b = xc.T @ dense_smoother(p.labels, dense_of(p.lap.matrix), 0.5) @ xc + beta * np.eye(p.d)
    put(s, "pencil", p, {"dominant": eigh(a, b)[1][:, -1]})

    # test_sda.py: alpha = 0, fully labeled -> regularized LDA (seed 3, beta 1e-2, tol 1e-12)
    beta = 1e-2
    x, truth = clustered_binary(50, 8, seed=3)
    lap = laplacian(knn_graph(x, 3))
    p = SdaProblem(x=x, labels=LabelVector(truth), lap=lap, alpha=0.0, betas=(beta,), tol=1e-12)
    xd = dense_of(x)
    xcc = xd - xd.mean(axis=0)
    fisher = np.linalg.solve(xcc.T @ xcc + beta * np.eye(8),
                             xd[truth == 1].mean(axis=0) - xd[truth == -1].mean(axis=0))
    put(s, "lda", p, {"fisher": fisher})

    # test_sda.py: class-pure features, perfectly separable held-out ranking
    from sdakit.sda import arrange_labeled_first

    tr = np.array([1, -1] * 15)
    xs = build_sparse(30, 2, list(range(30)), [0 if t == 1 else 1 for t in tr], np.ones(30))
    lab = np.zeros(30, dtype=int)
    lab[:6] = tr[:6]
    g, lap = knn_problem_parts(xs, 2)
    x2, lap2, labels2, perm = arrange_labeled_first(xs, lap, LabelVector(lab))
    p = SdaProblem(x=x2, labels=labels2, lap=lap2, alpha=0.5, betas=(1e-3,))
    put(s, "separable", p, {"truth": tr[perm]})

    # test_sda.py: directions consistent with scores; determinism (make_problem defaults)
    def make_problem(n=60, d=12, seed=0, alpha=0.5, betas=(1e-3,), n_labeled=6, k=3):
        x, truth = clustered_binary(n, d, seed=seed)
        g, lap = knn_problem_parts(x, k=k)
        x2, lap2, labels, truth2, _ = labeled_first_parts(x, lap, truth, n_labeled, seed=seed + 1)
        return SdaProblem(x=x2, labels=labels, lap=lap2, alpha=alpha, betas=betas)

    put(s, "consistent", make_problem(n=50, d=60, seed=13, betas=(1e-4, 1e-1)))
    put(s, "deterministic", make_problem(seed=5))

    # criterion 1: 20 random problems vs the dense centered pencil
    alphas, betas = (0.1, 0.5, 0.9), (1e-6, 1e-2)
    for i in range(20):
        rng = np.random.default_rng(1000 + i)
        n = int(rng.integers(40, 301))
        d = int(rng.integers(8, 51))
        alpha, beta = alphas[i % 3], betas[i % 2]
        x, truth = clustered_binary(n, d, seed=1000 + i)
        g, lap = knn_problem_parts(x, 3)
        x2, lap2, labels, _, _ = labeled_first_parts(x, lap, truth, 6, seed=2000 + i)
        p = SdaProblem(x=x2, labels=labels, lap=lap2, alpha=alpha, betas=(beta,), tol=1e-12)
        xd = dense_of(x2)
        xc = xd - xd[: labels.n_labeled].mean(axis=0)
        a = xc.T @ dense_w(labels) @ xc
        bm = xc.T @ dense_smoother(labels, dense_of(lap2.matrix), alpha) @ xc + beta * np.eye(d)
        put(s, f"crit1_{i}", p, {"w_star": eigh(a, bm)[1][:, -1]})

    # criterion 4 (a): centered transpose annihilates the labeled indicator
    for i in range(100):
        rng = np.random.default_rng(4000 + i)
        n = int(rng.integers(5, 120))
        d = int(rng.integers(2, 60))
        n_lab = int(rng.integers(1, n + 1))
        x, _ = random_binary_matrix(rng, n, d, density=0.25)
        lab = np.zeros(n, dtype=np.int64)
        lab[: max(1, n_lab // 2)] = 1
        lab[max(1, n_lab // 2): n_lab] = -1
        s[f"crit4a_{i}__x_offsets"] = np.asarray(x.row_offsets, dtype=np.int32)
        s[f"crit4a_{i}__x_cols"] = np.asarray(x.col_indices, dtype=np.int32)
        s[f"crit4a_{i}__shape"] = np.array([n, d], dtype=np.int64)
        s[f"crit4a_{i}__labels"] = lab.astype(np.int8)
    # criterion 4 (b): the operator chain kills the all-ones preimage
    for i in range(25):
        x, truth = clustered_binary(60 + i, 12, seed=5000 + i, ones_column=True)
        g, lap = knn_problem_parts(x, 4)
        x2, lap2, labels, _, _ = labeled_first_parts(x, lap, truth, 5, seed=5100 + i)
        p = SdaProblem(x=x2, labels=labels, lap=lap2, alpha=0.4, betas=(1e-3,))
        put(s, f"crit4b_{i}", p, run=False)

    # criterion 5: two-manifold data, 1% labeled, alpha 0.5 vs 0 (10 seeds)
    for seed in range(1, 11):
        x, truth = two_chain_fingerprints(2000, seed=seed, features_per_chain=600, window=12,
                                          n_noise_features=40, p_noise=0.05)
        g, lap = knn_problem_parts(x, 5)
        x2, lap2, labels, truth2, _ = labeled_first_parts(x, lap, truth, 10, seed=seed + 100)
        unl = labels.labels == 0
        aucs = []
        for alpha in (0.5, 0.0):
            p = SdaProblem(x=x2, labels=labels, lap=lap2, alpha=alpha, betas=(1e-2,), seed=seed)
            sc = solve(p, "fsda").ratings[1e-2].scores
            aucs.append(auc_roc(sc[unl], truth2[unl]))
        p = SdaProblem(x=x2, labels=labels, lap=lap2, alpha=0.5, betas=(1e-2,), seed=seed)
        put(s, f"crit5_{seed}", p, {"truth": truth2, "ref_auc": np.array(aucs)}, run=False)
    np.savez_compressed(OUT, **s)
    print(OUT, OUT.stat().st_size)


if __name__ == "__main__":
    main()
