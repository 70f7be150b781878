"""ctypes binding of include/fsda_b200.h (libfsda_b200.so, built in-tree).

The product path has no fallback: if the shared library is missing or no
B200 is visible, every call raises.  Status codes are translated into the
reference's exception classes by fsda.py.
"""

from __future__ import annotations

import ctypes as C
import os
from pathlib import Path

import numpy as np

LIB_NAME = "libfsda_b200.so"
LIB_PATH = Path(__file__).resolve().parent / LIB_NAME

FSDA_OK, FSDA_EINVAL, FSDA_EBREAKDOWN, FSDA_ENONFINITE, FSDA_ECUDA, FSDA_ELABEL = range(6)

_P = C.c_void_p
_I64 = C.c_int64
_D = C.c_double
_PD = C.POINTER(C.c_double)
_PI64 = C.POINTER(C.c_int64)
_PU8 = C.POINTER(C.c_uint8)
_PI8 = C.POINTER(C.c_int8)
_PI = C.POINTER(C.c_int)

# name -> argtypes (restype is int for all but the two noted)
SIGNATURES = {
    "fsda_abi_version": [],
    "fsda_last_error": [],
    "fsda_values_all_ones": [_PD, _I64],
    "fsda_ctx_create": [C.POINTER(_P), C.c_int, _P],
    "fsda_ctx_destroy": [_P],
    "fsda_ctx_set_stream": [_P, _P],
    "fsda_upload_x": [_P, _I64, _I64, _PI64, _PI64],
    "fsda_upload_laplacian": [_P, _I64, _PI64, _PI64, _PD],
    "fsda_set_labels": [_P, _PI8],
    "fsda_upload_problem": [_P, _I64, _I64, _PI64, _PI64, _PI64, _PI64, _PD, _PI8],
    "fsda_set_label_mask": [_P, _PI8],
    "fsda_matvec": [_P, _PD, _PD],
    "fsda_matvec_transpose": [_P, _PD, _PD],
    "fsda_labeled_mean": [_P, _PD],
    "fsda_centered_matvec_transpose": [_P, _PD, _PD, _PD],
    "fsda_apply_smoother": [_P, _D, _PD, _PD],
    "fsda_operator_apply": [_P, _D, _PD, _PD],
    "fsda_solve": [_P, _D, _PD, C.c_int, _D, _I64, _PD, _PD, _PD, _PD, _PI64, _PU8, _PI64, _PI64],
    "fsda_prepare_resident": [_P, _D, _PD, C.c_int, _D, _I64, _PD],
    "fsda_solve_async": [_P],
    "fsda_set_shift_update_mode": [_P, C.c_int],
    "fsda_last_shift_update_mode": [_P],
    "fsda_set_storage": [_P, C.c_int],
    "fsda_set_eager": [_P, C.c_int],
    "fsda_nccl_unique_id": [_PU8],
    "fsda_shard_init": [_P, C.c_int, C.c_int, _PI64, _PU8],
    "fsda_solve_sharded": [C.POINTER(_P), C.c_int, _D, _PD, C.c_int, _D, _I64, _PD, _I64, _I64, _PD, _PD,
                           _PD, _PI64, _PU8, _PI64, _PI64],
    "fsda_fetch_results": [_P, _PD, _PD, _PD, _PI64, _PU8, _PI64, _PI64, _PI64],
    "fsda_profile_kernels": [_P, C.c_int, _PI, C.POINTER(C.c_char_p), _PD, _PD, _PI64],
    "fsda_shifted_cg_dense": [_P, _I64, _PD, _PD, _PD, C.c_int, _D, _I64, C.c_int, _PD, _PD,
                              _PI64, _PU8, _PI64, _PI64],
    "fsda_regression_shifted_cg": [_P, _PD, _PD, C.c_int, _D, _I64, C.c_int, _PD, _PD, _PI64,
                                   _PU8, _PI64, _PI64],
    "fsda_sa_solve": [_P, _D, _PD, C.c_int, _D, _I64, _PD, _PD, _PD, _PI64, _PU8, _PI64, _PI64],
    "fsda_solve_batch": [_P, C.c_int, _PI8, _D, _PD, C.c_int, _D, _I64, _PD, _PD, _PD, _PD, _PI64,
                         _PU8, _PI64, _PI64, _PI],
    # row-sharded building blocks (device pointers passed as c_void_p)
    "fsda_upload_laplacian_rows": [_P, _I64, _I64, _I64, _PI64, _PI64, _PD],
    "fsda_dev_xrows": [_P, _P, _P],
    "fsda_dev_smoother": [_P, _D, _P, _P],
    "fsda_dev_xt_partial": [_P, _P, _P],
    "fsda_dev_class_sums": [_P, _P, _P],
    "fsda_dev_apply_w": [_P, _D, _D, _P],
    "fsda_dev_center": [_P, _P, _P, _D],
    "fsda_dev_cg_begin": [_P, _PD, C.c_int, _D, _I64, _P],
    "fsda_dev_cg_step": [_P, _P],
    "fsda_dev_cg_direction": [_P, C.POINTER(_P)],
    "fsda_dev_cg_status": [_P, _PI, _PI64, _PI],
    "fsda_dev_project": [_P, _P, _P],
    "fsda_dev_finish": [_P, _PU8, _P, _PD, _PD, _PI64, _PU8, _PI64, _PI64],
    # Tanimoto k-NN graph (graph_knn.cuh)
    "fsda_graph_knn": [_P, C.c_int32, _PI64],
    "fsda_graph_threshold": [_P, _D, _PI64],
    "fsda_graph_fetch": [_P, _PI64, _PI64],
    "fsda_head_counts": [_P, C.c_int64, C.c_int32, _P, C.c_int64, C.c_int64, _P],
}

_lib = None


class ExtensionMissing(RuntimeError):
    """The CUDA extension was not built (run __graft_entry__.build())."""


def lib() -> C.CDLL:
    global _lib
    if _lib is not None:
        return _lib
    path = Path(os.environ.get("FSDA_B200_LIB", str(LIB_PATH)))
    if not path.exists():
        raise ExtensionMissing(
            f"{path} not found: the sm_100a extension is not built. "
            "Run `python -c 'import __graft_entry__ as g; g.build()'` first; "
            "there is no CPU fallback.")
    h = C.CDLL(str(path))
    for name, args in SIGNATURES.items():
        f = getattr(h, name)
        f.argtypes = args
        f.restype = C.c_int
    h.fsda_last_error.restype = C.c_char_p
    _lib = h
    return h


def last_error() -> str:
    msg = lib().fsda_last_error()
    return msg.decode() if msg else ""


def dptr(a: np.ndarray):
    """Pointer to a contiguous float64 array (None passes NULL)."""
    if a is None:
        return None
    assert a.dtype == np.float64 and a.flags.c_contiguous
    return a.ctypes.data_as(_PD)


def i64ptr(a: np.ndarray):
    if a is None:
        return None
    assert a.dtype == np.int64 and a.flags.c_contiguous
    return a.ctypes.data_as(_PI64)


def u8ptr(a: np.ndarray):
    assert a.dtype == np.uint8 and a.flags.c_contiguous
    return a.ctypes.data_as(_PU8)


def i8ptr(a: np.ndarray):
    assert a.dtype == np.int8 and a.flags.c_contiguous
    return a.ctypes.data_as(_PI8)
