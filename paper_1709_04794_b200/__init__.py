"""B200-native FSDA hot path (fast semi-supervised discriminant analysis,
arXiv 1709.04794): the full regularization sweep as a device-resident
shifted-CG solve with hand-written sm_100a kernels behind a C ABI.

Public surface mirrors the reference package ``sdakit`` for this path
(/root/reference/pkg/src/sdakit/__init__.py:10-51): the data types, the
``fsda_solve`` / ``solve`` entry points, the device products used by the
operator, and a device ``shifted_cg`` for dense operators.
"""

from .types import (
    CenteringVector,
    KrylovError,
    LabelError,
    LabelVector,
    Laplacian,
    NumericalFailureError,
    PhaseStats,
    RatingVector,
    SdaProblem,
    ShiftedSolveResult,
    ShiftGrid,
    SolveReport,
    SolverBreakdownError,
    SparseFormatError,
    SparseMatrix,
    as_shift_grid,
    build_sparse,
)
from .fsda import (
    ALGORITHMS,
    Device,
    DeviceProblem,
    LinearOperator,
    apply_smoother,
    centered_matvec_transpose,
    default_device,
    fsda_operator_apply,
    fsda_solve,
    install_into_sdakit,
    labeled_mean,
    matvec,
    matvec_transpose,
    RegressionOperator,
    regression_operator,
    shifted_cg,
    sa_sda_solve,
    solve,
    solve_label_sets,
)

from .graph import (
    GraphError,
    SimilarityGraph,
    install_into_sdakit_graph,
    knn_graph,
    laplacian,
    tanimoto,
    threshold_graph,
)

__version__ = "0.1.0"

__all__ = [
    "CenteringVector", "KrylovError", "LabelError", "LabelVector", "Laplacian",
    "NumericalFailureError", "PhaseStats", "RatingVector", "SdaProblem", "ShiftedSolveResult",
    "ShiftGrid", "SolveReport", "SolverBreakdownError", "SparseFormatError", "SparseMatrix",
    "as_shift_grid", "build_sparse",
    "GraphError", "SimilarityGraph", "install_into_sdakit_graph", "knn_graph", "laplacian", "tanimoto",
    "threshold_graph",
    "ALGORITHMS", "Device", "DeviceProblem", "LinearOperator", "apply_smoother",
    "centered_matvec_transpose", "default_device", "fsda_operator_apply", "fsda_solve",
    "install_into_sdakit", "labeled_mean", "matvec", "matvec_transpose", "shifted_cg", "sa_sda_solve", "solve", "solve_label_sets", "RegressionOperator", "regression_operator",
]
