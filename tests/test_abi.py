"""The C-ABI library loads on a CPU-only host and exports every entry point
declared in include/*.h (no compute calls: there is no GPU here)."""

import ctypes
import glob
import os
import re

import pytest

from paper_1910_02371_b200 import _lib

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def declared_symbols():
    names = set()
    for h in glob.glob(os.path.join(ROOT, "include", "*.h")):
        src = open(h).read()
        src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
        names |= set(re.findall(r"\b(cpfit_\w+)\s*\(", src))
    return sorted(names)


def test_header_declares_entry_points():
    names = declared_symbols()
    assert "cpfit_tttp" in names and "cpfit_mttkrp" in names
    assert set(names) == set(_lib.SYMBOLS)


def test_library_exports_every_declared_symbol():
    if not os.path.exists(_lib.LIB_PATH):
        pytest.skip("library not built")
    L = ctypes.CDLL(_lib.LIB_PATH)
    for name in declared_symbols():
        assert hasattr(L, name), name


def test_version_and_error_without_gpu():
    if not os.path.exists(_lib.LIB_PATH):
        pytest.skip("library not built")
    L = _lib.load()
    assert b"sm_100a" in L.cpfit_version()
    # a pure argument-validation path needs no device
    out = ctypes.c_void_p()
    dims = (ctypes.c_int64 * 1)(0)
    st = L.cpfit_pattern_create(1, dims, 0, None, None, ctypes.byref(out))
    assert st == _lib.EINVAL
    assert "dimension" in _lib.last_error()
