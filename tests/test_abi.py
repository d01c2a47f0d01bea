"""The C-ABI library loads and exports every symbol include/dpp_b200.h declares (CPU only)."""

from __future__ import annotations

import ctypes
import re
from pathlib import Path

from paper_1203_4938_b200 import _lib

HEADER = Path(__file__).resolve().parents[1] / "include" / "dpp_b200.h"


def declared_symbols() -> set[str]:
    text = re.sub(r"/\*.*?\*/", "", HEADER.read_text(), flags=re.S)
    return set(re.findall(r"\b(dpp_[a-z0-9_]+)\s*\(", text))


def test_header_and_binding_agree():
    assert declared_symbols() == set(_lib.SIGNATURES)


def test_library_exports_every_declared_symbol():
    lib = _lib.load()
    for name in declared_symbols():
        assert isinstance(getattr(lib, name), ctypes._CFuncPtr), name
    assert lib.dpp_abi_version() == _lib.ABI_VERSION


def test_error_path_without_a_gpu():
    lib = _lib.load()
    rc = lib.dpp_imgc_encode(None, 2, 8, 8, 16, 128, 1, None, 16, 0, 0.25, None, None, None, None, None,
                             None)
    assert rc == _lib.DPP_EINVAL
    assert "channels" in _lib.last_error()
    assert lib.dpp_fft_leaf(5, None, None, 0, None) == _lib.DPP_EINVAL


def test_library_is_sm100a():
    blob = _lib.LIB_PATH.read_bytes()
    assert b"sm_100a" in blob
