"""The C-ABI library loads without a GPU and exports every symbol that
include/ihdg.h declares, with struct layouts matching the ctypes mirror."""

import ctypes
import os
import re

import pytest

from paper_1711_01175_b200 import _native as N

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def declared_functions():
    src = open(os.path.join(ROOT, "include", "ihdg.h")).read()
    src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
    return sorted(set(re.findall(r"\b(ihdg_[a-z_0-9]+)\s*\(", src)))


def test_header_parses():
    names = declared_functions()
    assert "ihdg_sweep" in names and "ihdg_assemble" in names and len(names) >= 15


def test_library_exports_all_declared_symbols():
    if not os.path.exists(N.LIB_PATH):
        pytest.skip("libihdg_cuda.so not built (run __graft_entry__.build())")
    lib = ctypes.CDLL(N.LIB_PATH)
    missing = [n for n in declared_functions() if not hasattr(lib, n)]
    assert not missing, missing
    assert set(declared_functions()) == set(N.SIGNATURES)


def test_struct_layouts_and_queries():
    if not os.path.exists(N.LIB_PATH):
        pytest.skip("libihdg_cuda.so not built")
    L = N.lib()  # checks ABI version + every struct size
    assert L.ihdg_supported(2, 6, 3) == 1 and L.ihdg_supported(3, 3, 1) == 1
    assert L.ihdg_supported(2, 9, 3) == 0
    g = N.Geom()
    g.dim, g.order, g.ncomp = 2, 6, 3
    g.cells[0], g.cells[1], g.cells[2] = 2048, 2048, 1
    g.layer_begin, g.layer_end = 0, 2048
    te = L.ihdg_tile_elems(2, 6, 3)
    assert L.ihdg_tile_count(ctypes.byref(g)) == 2048 * ((2048 + te - 1) // te)
    g.layer_end = 4096
    assert L.ihdg_tile_count(ctypes.byref(g)) == -1


def test_no_cpu_fallback(monkeypatch):
    """The product refuses to run without the extension (no silent fallback)."""
    monkeypatch.setattr(N, "_lib", None)
    monkeypatch.setattr(N, "LIB_PATH", "/nonexistent/libihdg_cuda.so")
    with pytest.raises(N.NativeUnavailable):
        N.lib()
