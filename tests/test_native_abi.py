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


def _cpu_sweep_args(cfg, cells=None):
    """SweepArgs of a BASELINE config built on the host (no device pointers):
    enough for the dispatch query, which reads only the geometry and weights."""
    from paper_1711_01175_b200.assembly import build_spec
    from paper_1711_01175_b200.workloads import make_config

    wl = make_config(cfg, cells=cells)
    sp = build_spec(wl.mesh, wl.problem, wl.ops, wl.dt)
    a = N.SweepArgs()
    d = wl.mesh.dim
    a.g.dim, a.g.order, a.g.ncomp = d, wl.ops.p, sp.ncomp
    for i in range(3):
        a.g.cells[i] = wl.mesh.cells[i] if i < d else 1
        a.g.periodic[i] = int(wl.mesh.periodic[i]) if i < d else 0
    a.g.layer_begin, a.g.layer_end = 0, wl.mesh.cells[d - 1]
    for f in range(6):
        a.coupled[f] = int(sp.coupled[f])
        for c in range(4):
            a.face_w[f][c] = float(sp.face_w[f, c])
    a.norm_kind = N.NORM_VOLUME
    a.scheme = N.SCHEME_II
    return a


@pytest.mark.parametrize("cfg,cells,auto,no_v3", [
    (5, None, "k_sweep_ws", "k_sweep_ws"), (4, None, "k_sweep_v4", "k_sweep"),
    (3, None, "k_sweep_v3", "k_sweep_ws"), (2, None, "k_sweep_v5", "k_sweep_ws"), (3, 64, "k_sweep_v3", "k_sweep_ws"), (3, 192, "k_sweep_v5", "k_sweep_ws"),
    (2, 20, "k_sweep", "k_sweep"), (1, None, "k_sweep", "k_sweep")])
def test_dispatch_names(cfg, cells, auto, no_v3):
    """ihdg_sweep_kernel names the kernel each BASELINE config runs on; the
    selector switches in process (no GPU needed for the query)."""
    if not os.path.exists(N.LIB_PATH):
        pytest.skip("libihdg_cuda.so not built")
    a = _cpu_sweep_args(cfg, cells)
    try:
        assert N.sweep_kernel(a) == auto
        N.set_sweep_impl("ws")
        assert N.sweep_kernel(a) == no_v3
        N.set_sweep_impl("generic")
        assert N.sweep_kernel(a) == "k_sweep"
        N.set_sweep_impl("v3")   # v4 off: the staged-ring kernels
        assert N.sweep_kernel(a) == ("k_sweep_v3" if auto in ("k_sweep_v4", "k_sweep_v5") else auto)
    finally:
        N.set_sweep_impl("auto")
    with pytest.raises(RuntimeError):
        N.set_sweep_impl("ws9")


@pytest.mark.parametrize("order,blocks,kernel", [(2, 2, "k_sweep_gemv"), (3, 4, "k_sweep_gemv"), (1, 2, "k_sweep")])
def test_dispatch_per_element_operators(order, blocks, kernel):
    """Per-element operators with raw neighbour values (the GEMV mode) go to
    k_sweep_gemv when the element is large enough for a CTA of row threads
    (N_vol >= 108), otherwise to the generic kernel; "generic" always wins."""
    if not os.path.exists(N.LIB_PATH):
        pytest.skip("libihdg_cuda.so not built")
    a = N.SweepArgs()
    a.g.dim, a.g.order, a.g.ncomp = 3, order, 4
    for i in range(3):
        a.g.cells[i] = 16
        a.g.periodic[i] = 0
    a.g.layer_begin, a.g.layer_end = 0, 16
    a.norm_kind = N.NORM_VOLUME
    a.scheme = N.SCHEME_II if blocks == 2 else N.SCHEME_I
    a.per_element, a.raw_blocks = 1, blocks
    try:
        assert N.sweep_kernel(a) == kernel
        N.set_sweep_impl("generic")
        assert N.sweep_kernel(a) == "k_sweep"
    finally:
        N.set_sweep_impl("auto")
