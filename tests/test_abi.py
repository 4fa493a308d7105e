"""The C-ABI boundary: libzinf.so loads and exports every entry point include/zinf.h declares (CPU)."""

import ctypes
import os
import re

from paper_2104_07857_b200 import _lib

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def declared():
    with open(os.path.join(ROOT, "include", "zinf.h")) as f:
        src = f.read()
    return sorted(set(re.findall(r"\b(zi_[a-z0-9_]+)\s*\(", src)))


def test_header_matches_binding():
    assert declared() == sorted(_lib.exported_symbols())


def test_library_exports_every_symbol():
    lib = ctypes.CDLL(_lib.LIB_PATH)
    for name in declared():
        assert hasattr(lib, name), name
    assert _lib.load().zi_version() >= 100


def test_error_path_without_gpu():
    """Argument validation runs on the host and reports through zi_last_error."""
    L = _lib.load()
    st = L.zi_reduce_scatter_cast(None, 0, 0, 8, 8, 1.0, 1, None, None)
    assert st == _lib.ZI_EINVAL
    assert "n_contrib" in _lib.last_error()
