"""Host-side data types mirroring the reference's FSDA interface.

Same names, fields, argument meaning and error classes as sdakit
(/root/reference/pkg/src/sdakit), so code written against the reference reads
the same against this package:

  SparseMatrix, LabelVector, CenteringVector   sparse.py:41-146, 198-255
  Laplacian                                    graph.py:48-53
  ShiftGrid, as_shift_grid, ShiftedSolveResult krylov.py:69-114
  SdaProblem                                   sda.py:64-117
  RatingVector, PhaseStats, SolveReport        sda.py:182-253
  SparseFormatError, LabelError                sparse.py:28-33
  KrylovError, SolverBreakdownError,
  NumericalFailureError                        krylov.py:24-33

These are plain containers with validation; no arithmetic of the hot path
happens here (that is all on the device, see fsda.py).
"""

from __future__ import annotations

import dataclasses
from dataclasses import dataclass
from functools import cached_property
from typing import Optional, Union

import numpy as np


class SparseFormatError(ValueError):
    """Structural problem in sparse input (shape, order, duplicates, range)."""


class LabelError(ValueError):
    """Label vector unusable for two-class discriminant analysis."""


class KrylovError(RuntimeError):
    """Base class of solver failures."""


class SolverBreakdownError(KrylovError):
    """<p, B p> vanished along a search direction."""


class NumericalFailureError(KrylovError):
    """A non-finite value appeared in the iteration."""


def _frozen_array(a, dtype) -> np.ndarray:
    out = np.array(a, dtype=dtype, copy=True) if not (
        isinstance(a, np.ndarray) and a.dtype == dtype and not a.flags.writeable
    ) else a
    out.setflags(write=False)
    return out


@dataclass(frozen=True, eq=False)
class SparseMatrix:
    """Read-only CSR matrix (int64 offsets / columns, float64 values).

    Invariants checked on construction: offsets run from 0 to nnz without
    decreasing, columns are in range and strictly increasing inside a row,
    values are finite and non-zero.
    """

    n_rows: int
    n_cols: int
    row_offsets: np.ndarray
    col_indices: np.ndarray
    values: np.ndarray

    def __post_init__(self):
        if self.n_rows < 0 or self.n_cols < 0:
            raise SparseFormatError("matrix shape must be non-negative")
        offs = _frozen_array(self.row_offsets, np.int64)
        cols = _frozen_array(self.col_indices, np.int64)
        vals = _frozen_array(self.values, np.float64)
        if offs.ndim != 1 or offs.size != self.n_rows + 1:
            raise SparseFormatError("row_offsets must have length n_rows + 1")
        if cols.ndim != 1 or cols.shape != vals.shape:
            raise SparseFormatError("col_indices and values must be parallel 1-d arrays")
        steps = np.diff(offs)
        if offs[0] != 0 or offs[-1] != vals.size or (steps.size and steps.min() < 0):
            raise SparseFormatError("row_offsets must be non-decreasing from 0 to nnz")
        if vals.size:
            if cols.min() < 0 or cols.max() >= self.n_cols:
                raise SparseFormatError("column index out of range")
            rising = np.diff(cols) > 0
            new_row = np.zeros(vals.size - 1, dtype=bool)
            starts = offs[1:-1]
            starts = starts[(starts > 0) & (starts < vals.size)]
            new_row[starts - 1] = True
            if not np.all(rising | new_row):
                raise SparseFormatError(
                    "column indices must be strictly increasing within each row "
                    "(duplicate entries are rejected, not summed)")
            if not np.all(np.isfinite(vals)):
                raise SparseFormatError("values must be finite")
            if np.any(vals == 0.0):
                raise SparseFormatError("explicitly stored zero values are not allowed")
        object.__setattr__(self, "row_offsets", offs)
        object.__setattr__(self, "col_indices", cols)
        object.__setattr__(self, "values", vals)

    @property
    def nnz(self) -> int:
        return int(self.values.size)

    @property
    def shape(self) -> tuple[int, int]:
        return (self.n_rows, self.n_cols)

    @cached_property
    def is_binary(self) -> bool:
        """All stored values equal 1 (what the value-free device path needs)."""
        return bool(np.all(self.values == 1.0))

    def row_nnz(self) -> np.ndarray:
        return np.diff(self.row_offsets)

    def frobenius_norm(self) -> float:
        return float(np.linalg.norm(self.values))

    @classmethod
    def binary(cls, n_rows: int, n_cols: int, row_offsets, col_indices) -> "SparseMatrix":
        cols = np.asarray(col_indices, dtype=np.int64)
        return cls(n_rows, n_cols, row_offsets, cols, np.ones(cols.size))


def build_sparse(n_rows, n_cols, rows, cols, values) -> SparseMatrix:
    """Assemble a SparseMatrix from unordered (row, col, value) triples; zero
    values are dropped, duplicates and out-of-range indices raise."""
    r = np.asarray(rows, dtype=np.int64)
    c = np.asarray(cols, dtype=np.int64)
    v = np.asarray(values, dtype=np.float64)
    if r.ndim != 1 or r.shape != c.shape or r.shape != v.shape:
        raise SparseFormatError("rows, cols, values must be parallel 1-d arrays")
    if r.size and (r.min() < 0 or r.max() >= n_rows):
        raise SparseFormatError("row index out of range")
    if c.size and (c.min() < 0 or c.max() >= n_cols):
        raise SparseFormatError("column index out of range")
    nz = v != 0.0
    r, c, v = r[nz], c[nz], v[nz]
    key = r * max(n_cols, 1) + c
    order = np.argsort(key, kind="stable")
    key, r, c, v = key[order], r[order], c[order], v[order]
    dup = np.flatnonzero(key[1:] == key[:-1])
    if dup.size:
        k = int(dup[0])
        raise SparseFormatError(f"duplicate entry at (row={r[k]}, col={c[k]})")
    offs = np.zeros(n_rows + 1, dtype=np.int64)
    np.cumsum(np.bincount(r, minlength=n_rows), out=offs[1:])
    return SparseMatrix(n_rows, n_cols, offs, c, v)


class LabelVector:
    """Labels over N samples: +1 / -1 for the two labeled classes, 0 for
    unlabeled samples."""

    def __init__(self, labels):
        arr = np.asarray(labels)
        if arr.ndim != 1:
            raise LabelError("labels must be a 1-d array")
        if arr.size and not np.all((arr == 1) | (arr == -1) | (arr == 0)):
            raise LabelError("labels must take values in {+1, -1, 0}")
        self.labels = _frozen_array(arr, np.int8)
        self.n = int(arr.size)
        self.n_class1 = int(np.count_nonzero(self.labels == 1))
        self.n_class2 = int(np.count_nonzero(self.labels == -1))
        self.n_labeled = self.n_class1 + self.n_class2

    @cached_property
    def mask_labeled(self) -> np.ndarray:
        return _frozen_array(self.labels != 0, bool)

    @cached_property
    def mask_class1(self) -> np.ndarray:
        return _frozen_array(self.labels == 1, bool)

    @cached_property
    def mask_class2(self) -> np.ndarray:
        return _frozen_array(self.labels == -1, bool)

    @property
    def is_labeled_first(self) -> bool:
        return bool(np.all(self.labels[: self.n_labeled] != 0))

    def __len__(self) -> int:
        return self.n

    def __eq__(self, other) -> bool:
        return isinstance(other, LabelVector) and np.array_equal(self.labels, other.labels)


@dataclass(frozen=True)
class CenteringVector:
    """Labeled mean mu = X^T 1_l / l."""

    mu: np.ndarray
    n_labeled: int


@dataclass(frozen=True)
class Laplacian:
    """Graph Laplacian L = D - S (unit-weight adjacency S)."""

    matrix: SparseMatrix
    degrees: np.ndarray


@dataclass(frozen=True)
class ShiftGrid:
    """Non-empty, finite, non-negative, strictly ascending shift grid."""

    betas: np.ndarray

    def __post_init__(self):
        b = np.array(self.betas, dtype=np.float64, copy=True)
        if b.ndim != 1 or b.size == 0:
            raise ValueError("shift grid must be a non-empty 1-d array")
        if not np.all(np.isfinite(b)):
            raise ValueError("shifts must be finite")
        if b[0] < 0:
            raise ValueError("shifts must be non-negative")
        if b.size > 1 and np.min(np.diff(b)) <= 0:
            raise ValueError("shifts must be strictly ascending")
        b.setflags(write=False)
        object.__setattr__(self, "betas", b)

    @property
    def n_shifts(self) -> int:
        return int(self.betas.size)


def as_shift_grid(betas) -> ShiftGrid:
    """Wrap a grid, sorting it ascending (ShiftGrid passes through)."""
    if isinstance(betas, ShiftGrid):
        return betas
    return ShiftGrid(np.sort(np.asarray(betas, dtype=np.float64)))


@dataclass
class ShiftedSolveResult:
    """Per-shift solutions of (B + beta I) w = b (solutions is dim x n_shifts)."""

    solutions: np.ndarray
    residual_norms: np.ndarray
    iterations: np.ndarray
    converged: np.ndarray

    @property
    def all_converged(self) -> bool:
        return bool(np.all(self.converged))


@dataclass
class SdaProblem:
    """Data, labels, Laplacian and solve settings of one rating problem."""

    x: SparseMatrix
    labels: LabelVector
    lap: Laplacian
    alpha: float
    betas: Union[ShiftGrid, np.ndarray, list, tuple]
    tol: float = 1e-8
    tol_spectral: Optional[float] = None
    max_iter_n: int = 1000
    max_iter_d: int = 1000
    seed: int = 0

    def __post_init__(self):
        self.betas = as_shift_grid(self.betas)
        if self.labels.n != self.x.n_rows:
            raise ValueError(
                f"labels cover {self.labels.n} samples but x has {self.x.n_rows} rows")
        lm = self.lap.matrix
        if not (lm.n_rows == lm.n_cols == self.x.n_rows):
            raise ValueError("laplacian must be square with one row per sample")
        if not 0.0 <= self.alpha <= 1.0:
            raise ValueError(f"alpha must lie in [0, 1], got {self.alpha}")
        if self.labels.n_class1 == 0 or self.labels.n_class2 == 0:
            raise ValueError("both classes need at least one labeled sample")
        if not self.labels.is_labeled_first:
            raise ValueError("labeled samples must occupy the first rows; "
                             "use arrange_labeled_first to permute the problem")
        if self.tol <= 0 or (self.tol_spectral is not None and self.tol_spectral <= 0):
            raise ValueError("tolerances must be positive")
        if self.max_iter_n < 1 or self.max_iter_d < 1:
            raise ValueError("iteration budgets must be at least 1")

    @property
    def n(self) -> int:
        return self.x.n_rows

    @property
    def d(self) -> int:
        return self.x.n_cols


@dataclass(frozen=True)
class RatingVector:
    scores: np.ndarray
    source: str  # "projection" | "spectral"


@dataclass
class PhaseStats:
    dimension: int
    iterations: Union[np.ndarray, int]
    operator_applications: int
    residuals: Union[np.ndarray, float]
    converged: Union[np.ndarray, bool]

    @property
    def ok(self) -> bool:
        return bool(np.all(self.converged))

    def to_dict(self) -> dict:
        return {
            "dimension": self.dimension,
            "iterations": np.asarray(self.iterations).tolist(),
            "operator_applications": self.operator_applications,
            "residuals": np.asarray(self.residuals).tolist(),
            "converged": np.asarray(self.converged).tolist(),
        }


@dataclass
class SolveReport:
    algorithm: str
    alpha: float
    betas: np.ndarray
    ratings: dict
    spectral: Optional[PhaseStats]
    regression: Optional[PhaseStats]
    wall_time_s: float
    spectral_eigenvalues: Optional[np.ndarray] = None
    spectral_vectors: Optional[np.ndarray] = None
    directions: Optional[dict] = None

    @property
    def converged(self) -> bool:
        return all(ph.ok for ph in (self.spectral, self.regression) if ph is not None)

    def to_dict(self) -> dict:
        return {
            "algorithm": self.algorithm,
            "alpha": self.alpha,
            "betas": np.asarray(self.betas).tolist(),
            "converged": self.converged,
            "wall_time_s": self.wall_time_s,
            "spectral": None if self.spectral is None else self.spectral.to_dict(),
            "regression": None if self.regression is None else self.regression.to_dict(),
            "spectral_eigenvalues": None if self.spectral_eigenvalues is None
            else np.asarray(self.spectral_eigenvalues).tolist(),
        }


def replace(obj, **changes):
    return dataclasses.replace(obj, **changes)
