"""The reference's own FSDA acceptance cases (pkg/tests/test_sda.py:120-239,
pkg/tests/test_acceptance.py criteria 1, 4, 5) run on the B200 through the
drop-in plugin: fb.install_into_sdakit registers the device solver in a
_SOLVERS table and every case calls solve(p, "fsda") through it.  Each case
keeps the reference test's own assertion and tolerance, and the directions
are compared with the reference's recorded outputs (same problem, same
seed) — 1e-6 per shift where the reference's solve converged."""

import numpy as np
import pytest

import paper_1709_04794_b200 as fb

from acceptance_cases import dense, keys, load, problem, sdakit_stub
from helpers import auc

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def g():
    return load()


@pytest.fixture(scope="module")
def sda():
    mod = sdakit_stub()
    fb.install_into_sdakit(mod)
    assert mod._SOLVERS["fsda"] is fb.fsda_solve
    return mod


def _cos(a, b):
    return abs(a @ b) / (np.linalg.norm(a) * np.linalg.norm(b))


def _close_to_reference(g, key, rep):
    betas = g[f"{key}__betas"]
    got = np.stack([rep.directions[float(b)] for b in betas])
    ref = g[f"{key}__ref_directions"]
    rel = np.linalg.norm(got - ref, axis=1) / np.linalg.norm(ref, axis=1)
    assert rel.max() <= 1e-6, (key, rel)


def test_dense_pencil_dominant_eigenvector(g, sda):
    p = problem(g, "pencil")
    rep = sda.solve(p, "fsda")
    beta = float(g["pencil__betas"][0])
    w_dir = np.linalg.lstsq(dense(p.x), rep.ratings[beta].scores, rcond=None)[0]
    assert _cos(g["pencil__dominant"], w_dir) >= 0.999
    _close_to_reference(g, "pencil", rep)


def test_alpha_zero_is_regularized_lda(g, sda):
    p = problem(g, "lda")
    rep = sda.solve(p, "fsda")
    beta = float(g["lda__betas"][0])
    w_dir = np.linalg.lstsq(dense(p.x), rep.ratings[beta].scores, rcond=None)[0]
    assert _cos(g["lda__fisher"], w_dir) >= 0.999
    _close_to_reference(g, "lda", rep)


def test_separable_problem_rates_perfectly(g, sda):
    p = problem(g, "separable")
    rep = sda.solve(p, "fsda")
    held = g["separable__labels"] == 0
    assert auc(rep.ratings[1e-3].scores[held], g["separable__truth"][held]) == 1.0


def test_directions_consistent_with_scores(g, sda):
    p = problem(g, "consistent")
    rep = sda.solve(p, "fsda")
    for beta, rating in rep.ratings.items():
        np.testing.assert_allclose(rating.scores, dense(p.x) @ rep.directions[beta], rtol=1e-10,
                                   atol=1e-12)
    _close_to_reference(g, "consistent", rep)


def test_fsda_is_deterministic(g, sda):
    p = problem(g, "deterministic")
    r1 = sda.solve(p, "fsda").ratings[1e-3].scores
    r2 = sda.solve(p, "fsda").ratings[1e-3].scores
    np.testing.assert_array_equal(r1, r2)


def test_criterion_1_dense_centered_pencil(g, sda):
    """20 random problems: |cos| with the dense pencil's dominant
    eigenvector >= 0.999 (the reference's gate), and within 1e-6 of the
    reference's own directions."""
    worst = 1.0
    for key in keys(g, "crit1_"):
        p = problem(g, key)
        rep = sda.solve(p, "fsda")
        beta = float(g[f"{key}__betas"][0])
        worst = min(worst, _cos(rep.directions[beta], g[f"{key}__w_star"]))
        _close_to_reference(g, key, rep)
    assert worst >= 0.999, worst


def test_criterion_4_centering_annihilation(g):
    """(a) the centred transpose annihilates the labeled indicator to
    1e-12 ||X||_F on 100 matrices; (b) the operator chain X_c^T M X kills the
    all-ones preimage to 1e-10 ||X||_F on 25 problems — on the device."""
    worst_a = 0.0
    for key in keys(g, "crit4a_"):
        n, d = (int(v) for v in g[f"{key}__shape"])
        x = fb.SparseMatrix.binary(n, d, g[f"{key}__x_offsets"].astype(np.int64),
                                   g[f"{key}__x_cols"].astype(np.int64))
        labels = fb.LabelVector(g[f"{key}__labels"].astype(np.int64))
        mu = fb.labeled_mean(x, labels)
        resid = np.linalg.norm(fb.centered_matvec_transpose(x, mu, (labels.labels != 0).astype(float)))
        worst_a = max(worst_a, resid / max(np.sqrt(x.nnz), 1e-300))
    assert worst_a <= 1e-12, worst_a
    worst_b = 0.0
    for key in keys(g, "crit4b_"):
        p = problem(g, key)
        w_nd = np.zeros(int(p.x.n_cols))
        w_nd[0] = 1.0
        out = fb.fsda_operator_apply(p, w_nd)
        worst_b = max(worst_b, np.linalg.norm(out) / np.sqrt(p.x.nnz))
    assert worst_b <= 1e-10, worst_b


def test_criterion_5_smoothing_beats_supervised(g, sda):
    """Two-manifold data, 1% labeled: alpha 0.5 beats alpha 0 by >= 0.05 mean
    unlabeled AUC over 10 seeds (the reference's gate).  These solves run up
    to max_iter_d = 1000 at tol 1e-8, far past the Krylov stability horizon,
    where the reference disagrees with itself under any reordering (SURVEY
    §8c), so each AUC is held to 1e-3 of the reference's (measured: <= 4e-6)."""
    semis, sups = [], []
    for key in keys(g, "crit5_"):
        p = problem(g, key)
        truth = g[f"{key}__truth"]
        unl = g[f"{key}__labels"] == 0
        for alpha, bucket in ((0.5, semis), (0.0, sups)):
            q = fb.SdaProblem(x=p.x, labels=p.labels, lap=p.lap, alpha=alpha, betas=(1e-2,),
                              seed=p.seed)
            bucket.append(auc(sda.solve(q, "fsda").ratings[1e-2].scores[unl], truth[unl]))
        np.testing.assert_allclose([semis[-1], sups[-1]], g[f"{key}__ref_auc"], atol=1e-3)
    assert np.mean(semis) - np.mean(sups) >= 0.05
