"""Host-side logic on the CPU: the sdakit-mirroring types and their
validation (same error classes and messages as the reference), the workload
generator's distributional contract, and the drop-in plumbing."""

import sys

import numpy as np
import pytest

import paper_1709_04794_b200 as fb
from paper_1709_04794_b200 import fsda as fsda_mod
from paper_1709_04794_b200.workloads import (labels_first, make_workload, random_knn_laplacian,
                                             zipf_binary_rows)

HAND = fb.build_sparse(2, 3, [0, 0, 1], [0, 2, 1], [1.0, 2.0, 3.0])


# ------------------------------------------------------------ SparseMatrix

def test_build_sorts_and_drops_zeros():
    m = fb.build_sparse(2, 3, [1, 0, 0, 1], [1, 2, 0, 2], [3.0, 2.0, 1.0, 0.0])
    assert m.row_offsets.tolist() == [0, 2, 3]
    assert m.col_indices.tolist() == [0, 2, 1]
    assert m.values.tolist() == [1.0, 2.0, 3.0]


@pytest.mark.parametrize("rows,cols,vals,match", [
    ([0, 0], [1, 1], [1.0, 2.0], "duplicate"),
    ([0], [2], [1.0], "range"),
    ([-1], [0], [1.0], "range"),
])
def test_build_rejects(rows, cols, vals, match):
    with pytest.raises(fb.SparseFormatError, match=match):
        fb.build_sparse(2, 2, rows, cols, vals)


def test_container_invariants():
    with pytest.raises(fb.SparseFormatError):
        fb.SparseMatrix(1, 3, np.array([0, 2]), np.array([2, 0]), np.array([1.0, 1.0]))
    with pytest.raises(fb.SparseFormatError):
        fb.SparseMatrix(2, 2, np.array([0, 2, 1]), np.array([0, 1]), np.array([1.0, 1.0]))
    with pytest.raises(fb.SparseFormatError):
        fb.SparseMatrix(1, 2, np.array([0, 1]), np.array([0]), np.array([np.nan]))
    with pytest.raises(fb.SparseFormatError):
        fb.SparseMatrix(1, 2, np.array([0, 1]), np.array([0]), np.array([0.0]))
    # strictly increasing inside rows, free across row boundaries
    m = fb.SparseMatrix(2, 3, np.array([0, 2, 4]), np.array([0, 2, 0, 1]), np.ones(4))
    assert m.nnz == 4 and m.is_binary


def test_arrays_are_read_only():
    with pytest.raises(ValueError):
        HAND.values[0] = 9.0
    assert not HAND.is_binary


# ------------------------------------------------------------- labels, grid

def test_label_vector():
    lv = fb.LabelVector([1, -1, 0, 1, 0])
    assert (lv.n_class1, lv.n_class2, lv.n_labeled) == (2, 1, 3)
    assert not lv.is_labeled_first
    assert fb.LabelVector([1, -1, 0, 0]).is_labeled_first
    with pytest.raises(fb.LabelError):
        fb.LabelVector([1, 2, 0])


def test_shift_grid_validation():
    for bad in ([], [0.1, 0.1], [-1.0], [np.inf]):
        with pytest.raises(ValueError):
            fb.ShiftGrid(np.array(bad, dtype=float))
    np.testing.assert_array_equal(fb.as_shift_grid((1.0, 0.1)).betas, [0.1, 1.0])


def _lap(n, k=2, seed=0):
    lo, lc, lv, deg = random_knn_laplacian(n, k, seed)
    return fb.Laplacian(fb.SparseMatrix(n, n, lo, lc, lv), deg)


def test_problem_validation_messages():
    n, d = 20, 6
    lab = np.zeros(n, dtype=np.int8)
    lab[:2], lab[2:4] = 1, -1
    x = fb.SparseMatrix.binary(n, d, np.arange(n + 1), np.arange(n) % d)
    good = dict(x=x, labels=fb.LabelVector(lab), lap=_lap(n), alpha=0.5, betas=(1e-3,))
    fb.SdaProblem(**good)
    with pytest.raises(ValueError, match="alpha"):
        fb.SdaProblem(**{**good, "alpha": 1.5})
    with pytest.raises(ValueError, match="shift grid"):
        fb.SdaProblem(**{**good, "betas": ()})
    with pytest.raises(ValueError, match="laplacian"):
        fb.SdaProblem(**{**good, "lap": _lap(n + 1)})
    bad = lab.copy()
    bad[1], bad[10] = 0, 1
    with pytest.raises(ValueError, match="arrange_labeled_first"):
        fb.SdaProblem(**{**good, "labels": fb.LabelVector(bad)})
    one_class = np.zeros(n, dtype=np.int8)
    one_class[:3] = 1
    with pytest.raises(ValueError, match="both classes"):
        fb.SdaProblem(**{**good, "labels": fb.LabelVector(one_class)})
    with pytest.raises(ValueError, match="tolerances"):
        fb.SdaProblem(**{**good, "tol": 0.0})
    with pytest.raises(ValueError, match="budgets"):
        fb.SdaProblem(**{**good, "max_iter_d": 0})


def test_report_to_dict_roundtrip():
    ph = fb.PhaseStats(dimension=3, iterations=np.array([2, 1]), operator_applications=2,
                       residuals=np.array([0.1, 0.2]), converged=np.array([True, False]))
    rep = fb.SolveReport(algorithm="fsda", alpha=0.5, betas=np.array([0.1, 1.0]), ratings={},
                         spectral=None, regression=ph, wall_time_s=0.0)
    d = rep.to_dict()
    assert d["regression"]["iterations"] == [2, 1] and d["converged"] is False
    assert not rep.converged


def test_solve_dispatch_rejects_out_of_scope_algorithms():
    with pytest.raises(ValueError, match="unknown algorithm"):
        fb.solve(object(), "csr-sda")


def test_shifted_cg_requires_device_operator():
    op = fb.LinearOperator(3, lambda v: v)
    with pytest.raises(TypeError):
        fb.shifted_cg(op, np.ones(3), (0.1,))
    assert fb.LinearOperator.from_dense(np.eye(2))(np.ones(2)).tolist() == [1.0, 1.0]


# ------------------------------------------------------------- families

def test_family_resolution_defaults_to_own_types():
    fam = fsda_mod._family(object())
    assert fam.SolveReport is fb.SolveReport
    assert fam.SolverBreakdownError is fb.SolverBreakdownError


def test_family_resolution_for_reference_objects():
    sdakit_root = "/root/reference/pkg/src"
    import os

    if not os.path.isdir(sdakit_root):
        pytest.skip("reference not present on this host")
    sys.path.insert(0, sdakit_root)
    try:
        import sdakit.sda as rsda
        from sdakit.sparse import LabelVector

        fam = fsda_mod._family(LabelVector([1, -1]))
        assert fam.SolveReport is rsda.SolveReport
        import sdakit.krylov as rk

        assert fam.SolverBreakdownError is rk.SolverBreakdownError
        # install_into_sdakit swaps only the 'fsda' entry
        saved = dict(rsda._SOLVERS), rsda.fsda_solve, rsda.sa_sda_solve
        try:
            fb.install_into_sdakit(rsda)
            assert rsda._SOLVERS["fsda"] is fb.fsda_solve
            assert rsda._SOLVERS["sa-sda"] is fb.sa_sda_solve
            assert rsda._SOLVERS["csr-sda"] is saved[0]["csr-sda"]
        finally:
            rsda._SOLVERS.clear()
            rsda._SOLVERS.update(saved[0])
            rsda.fsda_solve = saved[1]
            rsda.sa_sda_solve = saved[2]
    finally:
        sys.path.remove(sdakit_root)


def test_graph_install_and_reference_types():
    """install_into_sdakit_graph routes sdakit's knn_graph names to the device
    build; graphs of sdakit matrices come back as sdakit types (host only)."""
    sdakit_root = "/root/reference/pkg/src"
    import os

    if not os.path.isdir(sdakit_root):
        pytest.skip("reference not present on this host")
    sys.path.insert(0, sdakit_root)
    try:
        import sdakit
        import sdakit.graph as rg
        import sdakit.synthetic as rsyn
        from sdakit.sparse import SparseMatrix as RSM

        saved = rg.knn_graph, sdakit.knn_graph, rsyn.knn_graph
        try:
            original = rg.knn_graph
            fb.install_into_sdakit_graph(rg)
            routed = rg.knn_graph
            assert routed.__wrapped_reference__ is original
            assert sdakit.knn_graph is routed and rsyn.knn_graph is routed
            # k > 64 stays on sdakit's own function (the device ranking keeps <= 64)
            x = RSM(70, 2, np.arange(71), np.zeros(70, dtype=np.int64), np.ones(70))
            got, want = routed(x, 65), original(x, 65)
            assert got.adjacency == want.adjacency and got.n == 70
            fb.install_into_sdakit_graph(rg)      # idempotent: still wraps the original
            assert rg.knn_graph.__wrapped_reference__ is original
        finally:
            rg.knn_graph, sdakit.knn_graph, rsyn.knn_graph = saved
        from paper_1709_04794_b200.graph import _graph_types

        sm, sg, ge, lp = _graph_types(RSM(2, 2, np.array([0, 1, 2]), np.array([0, 1]), np.ones(2)))
        assert sg is rg.SimilarityGraph and ge is rg.GraphError and lp is rg.Laplacian and sm is RSM
        # the host Laplacian assembly gives the reference's own layout
        adj = RSM(3, 3, np.array([0, 1, 3, 4]), np.array([1, 0, 2, 1]), np.ones(4))
        g = rg.graph_from_adjacency(adj)
        mine, ref = fb.laplacian(g), rg.laplacian(g)
        assert mine.matrix == ref.matrix and np.array_equal(mine.degrees, ref.degrees)
    finally:
        sys.path.remove(sdakit_root)


def test_label_sets_validated_before_the_device():
    """solve_label_sets rejects bad masks on the host (no GPU needed)."""
    x = fb.SparseMatrix.binary(4, 3, np.arange(5), np.array([0, 1, 2, 0]))
    lap = _lap(4)
    one_class = np.array([1, 1, 0, 0], dtype=np.int8)
    with pytest.raises(ValueError, match="both classes"):
        fb.solve_label_sets(x, lap, [one_class], 0.5, (0.1,))
    with pytest.raises(ValueError, match="one entry per sample"):
        fb.solve_label_sets(x, lap, [np.array([1, -1], dtype=np.int8)], 0.5, (0.1,))
    with pytest.raises(ValueError, match="one seed"):
        fb.solve_label_sets(x, lap, [np.array([1, -1, 0, 0], dtype=np.int8)], 0.5, (0.1,),
                            seeds=[1, 2])


def test_task_masks_shape_and_counts():
    from paper_1709_04794_b200.workloads import task_masks

    m = task_masks(1000, 5, 0.02, 0.25, seed=3)
    assert m.shape == (5, 1000) and m.dtype == np.int8
    for row in m:
        assert (row != 0).sum() == 20 and (row == 1).sum() == 5


# -------------------------------------------------------------- workloads

def test_zipf_rows_distinct_sorted_and_poisson():
    offs, cols = zipf_binary_rows(2000, 500, 20.0, 1.1, seed=3)
    assert offs[0] == 0 and offs[-1] == cols.size
    for i in range(0, 2000, 97):
        row = cols[offs[i]:offs[i + 1]]
        assert np.all(np.diff(row) > 0)
    assert abs(np.diff(offs).mean() - 20.0) < 0.5
    counts = np.bincount(cols, minlength=500)
    assert counts[0] > counts[100] > counts[499]          # low index = popular


def test_knn_laplacian_is_symmetric_with_zero_row_sums():
    lo, lc, lv, deg = random_knn_laplacian(300, 4, seed=2)
    import scipy.sparse as sp

    lap = sp.csr_matrix((lv, lc, lo), shape=(300, 300)).toarray()
    np.testing.assert_array_equal(lap, lap.T)
    np.testing.assert_array_equal(lap.sum(axis=1), np.zeros(300))
    assert deg.min() >= 4
    np.testing.assert_array_equal(np.diag(lap), deg)


def test_labels_first_counts():
    lab = labels_first(100, 30, 7, seed=1)
    assert (lab[:30] != 0).all() and (lab[30:] == 0).all()
    assert (lab == 1).sum() == 7


def test_workload_is_deterministic():
    a = make_workload("cfg1", n=500, d=200, ell=50, n_pos=10)
    b = make_workload("cfg1", n=500, d=200, ell=50, n_pos=10)
    np.testing.assert_array_equal(a.x_cols, b.x_cols)
    np.testing.assert_array_equal(a.l_cols, b.l_cols)
    np.testing.assert_array_equal(a.probe(), np.random.default_rng(0).uniform(-1, 1, 200))


def test_values_all_ones_helper_and_cache():
    """The binary-X precondition on an explicit values array (the reference's
    SparseMatrix, sparse.py:43-58): checked in C by all host threads and
    remembered per read-only array."""
    from paper_1709_04794_b200 import fsda

    ones = np.ones(300_000)
    ones.setflags(write=False)
    assert fsda._all_ones(ones) is True
    assert id(ones) in fsda._ONES_CACHE and fsda._all_ones(ones) is True
    bad = np.ones(300_000)
    bad[-1] = 2.0
    assert fsda._all_ones(bad) is False
    assert id(bad) not in fsda._ONES_CACHE          # writable arrays are not remembered
    assert fsda._all_ones(np.ones(0)) is True
    assert fsda._all_ones(np.ones(7, dtype=np.float32)) is True
    key = id(ones)
    del ones
    import gc

    gc.collect()
    assert key not in fsda._ONES_CACHE               # dropped with the array
