"""SA-SDA (sda.py:360-396): shifted CG in sample space on the
centred spectral operator.  Oracle vs the reference's outputs
(tests/golden/sa_reference.npz) on CPU; the device vs the oracle bitwise and
vs the reference on the GPU."""

from pathlib import Path

import numpy as np
import pytest

from oracle import c_oracle

from helpers import labeled_aucs, rel_rows


@pytest.fixture(scope="module")
def gold():
    return dict(np.load(Path(__file__).resolve().parent / "golden" / "sa_reference.npz"))


def _case(g, i):
    return {k[3:]: v for k, v in g.items() if k.startswith(f"s{i}_")}


def _probe(c):
    lab = c["labels"]
    m = lab != 0
    r = np.random.default_rng(int(c["seed"])).uniform(-1, 1, int(c["n"]))
    return r - r[m].sum() / int(m.sum())


@pytest.mark.parametrize("i", range(4))
def test_oracle_sa_vs_reference(gold, i):
    c = _case(gold, i)
    sols, res, its, conv, napp = c_oracle.sa_solve(
        c["l_offsets"], c["l_cols"], c["l_vals"], c["labels"], float(c["alpha"]), c["betas"],
        float(c["tol"]), int(c["max_iter"]), _probe(c))
    assert rel_rows(sols, c["scores"]) <= 1e-8
    np.testing.assert_array_equal(its, c["iterations"])
    np.testing.assert_array_equal(conv, c["converged"])
    np.testing.assert_array_equal(labeled_aucs(sols, c["labels"]), labeled_aucs(c["scores"], c["labels"]))


def test_sa_rejects_alpha_zero():
    import paper_1709_04794_b200 as fb

    n = 10
    x = fb.SparseMatrix.binary(n, 3, np.arange(n + 1), np.arange(n) % 3)
    from paper_1709_04794_b200.workloads import random_knn_laplacian

    lo, lc, lv, deg = random_knn_laplacian(n, 2, 0)
    lab = np.zeros(n, dtype=np.int8)
    lab[0], lab[1] = 1, -1
    p = fb.SdaProblem(x=x, labels=fb.LabelVector(lab),
                      lap=fb.Laplacian(fb.SparseMatrix(n, n, lo, lc, lv), deg), alpha=0.0, betas=(1e-3,))
    with pytest.raises(ValueError, match="alpha != 0"):
        fb.solve(p, "sa-sda")


@pytest.mark.gpu
@pytest.mark.parametrize("i", range(4))
def test_device_sa_bitwise_and_vs_reference(gold, i):
    import paper_1709_04794_b200 as fb

    c = _case(gold, i)
    n, d = int(c["n"]), int(c["d"])
    x = fb.SparseMatrix.binary(n, d, c["x_offsets"], c["x_cols"])
    lap = fb.Laplacian(fb.SparseMatrix(n, n, c["l_offsets"], c["l_cols"], c["l_vals"]), c["degrees"])
    p = fb.SdaProblem(x=x, labels=fb.LabelVector(c["labels"]), lap=lap, alpha=float(c["alpha"]),
                      betas=c["betas"], tol=float(c["tol"]), max_iter_n=int(c["max_iter"]),
                      seed=int(c["seed"]))
    rep = fb.solve(p, "sa-sda")
    assert rep.algorithm == "sa-sda" and rep.regression is None
    scores = np.stack([rep.ratings[float(b)].scores for b in p.betas.betas])
    sols, res, its, conv, napp = c_oracle.sa_solve(
        c["l_offsets"], c["l_cols"], c["l_vals"], c["labels"], float(c["alpha"]), c["betas"],
        float(c["tol"]), int(c["max_iter"]), _probe(c))
    np.testing.assert_array_equal(scores, sols)
    np.testing.assert_array_equal(rep.spectral.iterations, its)
    np.testing.assert_array_equal(rep.spectral.residuals, res)
    assert rep.spectral.operator_applications == napp
    assert rel_rows(scores, c["scores"]) <= 1e-8
    np.testing.assert_array_equal(rep.spectral.converged, c["converged"])
