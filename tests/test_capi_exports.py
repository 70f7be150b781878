"""The C-ABI library loads on a CPU-only host and exports every symbol the
header declares; without a GPU, context creation fails cleanly (no fallback)."""

import ctypes as C
import re
from pathlib import Path

import pytest

from paper_1709_04794_b200 import _capi

HEADER = Path(__file__).resolve().parents[1] / "include" / "fsda_b200.h"


def declared_symbols():
    text = HEADER.read_text()
    return sorted(set(re.findall(r"^\s*(?:int|const char\*)\s+(fsda_\w+)\s*\(", text, re.M)))


def test_header_declares_the_abi():
    names = declared_symbols()
    assert "fsda_solve" in names and "fsda_upload_x" in names and len(names) >= 18


def test_library_exports_every_declared_symbol():
    lib = C.CDLL(str(_capi.LIB_PATH))
    for name in declared_symbols():
        assert hasattr(lib, name), name
    assert set(declared_symbols()) == set(_capi.SIGNATURES)


def test_abi_version_and_error_channel():
    lib = _capi.lib()
    assert lib.fsda_abi_version() == 2
    assert isinstance(_capi.last_error(), str)


def test_context_creation_without_gpu_fails_loudly():
    import torch

    if torch.cuda.is_available():
        pytest.skip("a GPU is visible")
    h = C.c_void_p()
    rc = _capi.lib().fsda_ctx_create(C.byref(h), 0, None)
    assert rc == _capi.FSDA_ECUDA
    assert "device" in _capi.last_error().lower()
    import paper_1709_04794_b200 as fb

    with pytest.raises(RuntimeError):
        fb.Device(0)
