"""ctypes binding of libihdg_cuda.so (include/ihdg.h).

There is no CPU fallback: if the shared library is missing or cannot be
loaded, every product entry point raises ``NativeUnavailable``.
"""

from __future__ import annotations

import ctypes as C
import os

__all__ = ["NativeUnavailable", "lib", "Geom", "IterState", "AssemblyArgs", "ClassApplyArgs",
           "FieldArgs", "QuadArgs", "SweepArgs", "FinalizeArgs", "TraceArgs", "ElemErrorArgs",
           "FaceEnergyArgs", "check",
           "LIB_PATH", "STATUS_NAMES"]

LIB_PATH = os.environ.get("IHDG_LIB") or os.path.join(os.path.dirname(os.path.abspath(__file__)),
                                                     "libihdg_cuda.so")

ABI_VERSION = 3
IHDG_OK = 0
RUNNING, CONVERGED, DIVERGED, NAN, MAXITER = 0, 1, 2, 3, 4
STATUS_NAMES = {RUNNING: "running", CONVERGED: "converged", DIVERGED: "diverged",
                NAN: "diverged", MAXITER: "max-iter"}
NORM_VOLUME, NORM_TRACE = 0, 1
SCHEME_II, SCHEME_I = 0, 1

_p = C.c_void_p
_i32 = C.c_int32
_i64 = C.c_int64
_f64 = C.c_double


class NativeUnavailable(RuntimeError):
    pass


class Geom(C.Structure):
    _fields_ = [("dim", _i32), ("order", _i32), ("ncomp", _i32), ("pad0", _i32),
                ("cells", _i64 * 3), ("periodic", _i32 * 3), ("pad1", _i32),
                ("layer_begin", _i64), ("layer_end", _i64)]


class IterState(C.Structure):
    _fields_ = [("status", _i32), ("iters", _i32), ("max_iters", _i32), ("ticket", C.c_uint32),
                ("tol", _f64), ("first_norm", _f64), ("last_norm", _f64),
                ("diverge_factor", _f64), ("last_err", _f64)]


class AssemblyArgs(C.Structure):
    _fields_ = [("dim", _i32), ("order", _i32), ("ncomp", _i32), ("n_class", _i32),
                ("n_ops", _i32), ("n_terms", _i32), ("nr", _i32), ("kin_blocks", _i32),
                ("ops1d", _p), ("op_ncols", _p), ("terms", _p), ("coefs", _p),
                ("A", _p), ("Ainv", _p), ("AinvT", _p), ("B", _p), ("R", _p),
                ("LT", _p), ("PT", _p), ("min_pivot", _p)]


class ClassApplyArgs(C.Structure):
    _fields_ = [("g", Geom), ("opT", _p), ("class_of_mask", _p), ("inp", _p), ("out", _p),
                ("in_stride", _i64), ("in_offset", _i32), ("ncols", _i32), ("in_ghost", _i32),
                ("out_ghost", _i32), ("accumulate", _i32), ("per_element", _i32)]


class FieldArgs(C.Structure):
    _fields_ = [("g", Geom), ("lo", _f64 * 3), ("h", _f64 * 3), ("ref1d", _p), ("params", _p),
                ("out", _p), ("out_stride", _i64), ("out_offset", _i32), ("out_ghost", _i32),
                ("npts1d", _i32), ("kind", _i32), ("nmodes", _i32), ("pad0", _i32)]


class QuadArgs(C.Structure):
    _fields_ = [("g", Geom), ("Bq", _p), ("fq", _p), ("out", _p), ("out_stride", _i64),
                ("out_offset", _i32), ("nq", _i32), ("jac", _f64)]


class SweepArgs(C.Structure):
    _fields_ = [("g", Geom), ("u_old", _p), ("u_new", _p), ("s", _p), ("LT", _p),
                ("class_of_mask", _p), ("chol1d", _p), ("tile_partials", _p), ("state", _p),
                ("norm_hist", _p), ("face_w", (_f64 * 4) * 6), ("comp_w", _f64 * 4),
                ("out_w", (_f64 * 4) * 6), ("jac", _f64), ("jac_face", _f64 * 3),
                ("coupled", _i32 * 6), ("out_face", _i32 * 6), ("norm_kind", _i32),
                ("finalize", _i32), ("tile_offset", _i64), ("chol", _f64 * 64),
                ("own_w", (_f64 * 4) * 6), ("scheme", _i32), ("pad1", _i32),
                ("q_store", _p), ("gram_R", _p), ("gram_kc", _i32), ("pad2", _i32),
                ("layer_sums", _p), ("grid_bar", _p),
                ("per_element", _i32), ("raw_blocks", _i32), ("raw_comp", (_i32 * 4) * 6)]


class FinalizeArgs(C.Structure):
    _fields_ = [("tile_partials", _p), ("n_tiles", _i64), ("state", _p), ("norm_hist", _p), ("row_len", _i64)]


class HaloArgs(C.Structure):
    _fields_ = [("g", Geom), ("buf", _p), ("packed", _p), ("idx", _p), ("n_idx", _i32), ("layer", _i32)]


class TraceArgs(C.Structure):
    _fields_ = [("g", Geom), ("u", _p), ("trace", _p), ("w_int_own", (_f64 * 4) * 3),
                ("w_int_nbr", (_f64 * 4) * 3), ("w_lo", (_f64 * 4) * 3), ("w_hi", (_f64 * 4) * 3)]


class ErrorArgs(C.Structure):
    _fields_ = [("g", Geom), ("u", _p), ("ue_q", _p), ("vq", _p), ("wq", _p), ("err_partials", _p),
                ("succ_partials", _p), ("n_succ", _i64), ("state", _p), ("norm_hist", _p), ("err_hist", _p),
                ("comp_w", _f64 * 4), ("jac", _f64), ("nq", _i32), ("mode", _i32)]


class ElemErrorArgs(C.Structure):
    _fields_ = [("g", Geom), ("u", _p), ("r", _p), ("chol1d", _p), ("err2", _p), ("flags", _p),
                ("total", _p), ("comp_w", _f64 * 4), ("jac", _f64), ("tol", _f64)]


class FaceEnergyArgs(C.Structure):
    _fields_ = [("g", Geom), ("t", _p), ("t_ref", _p), ("chol1d", _p), ("e2", _p), ("total", _p),
                ("jac_face", _f64 * 3)]


_STRUCTS = [Geom, IterState, AssemblyArgs, ClassApplyArgs, FieldArgs, QuadArgs, SweepArgs,
            FinalizeArgs, TraceArgs, ErrorArgs, ElemErrorArgs, FaceEnergyArgs, HaloArgs]

# exported symbol -> (restype, argtypes)
SIGNATURES = {
    "ihdg_abi_version": (_i32, []),
    "ihdg_struct_size": (_i64, [_i32]),
    "ihdg_last_error": (C.c_char_p, []),
    "ihdg_supported": (_i32, [_i32, _i32, _i32]),
    "ihdg_tile_elems": (_i32, [_i32, _i32, _i32]),
    "ihdg_tile_count": (_i64, [C.POINTER(Geom)]),
    "ihdg_assemble": (_i32, [C.POINTER(AssemblyArgs), _p]),
    "ihdg_class_apply": (_i32, [C.POINTER(ClassApplyArgs), _p]),
    "ihdg_eval_field": (_i32, [C.POINTER(FieldArgs), _p]),
    "ihdg_quad_project": (_i32, [C.POINTER(QuadArgs), _p]),
    "ihdg_sweep": (_i32, [C.POINTER(SweepArgs), _p]),
    "ihdg_stream_variant": (_i32, [C.POINTER(SweepArgs)]),
    "ihdg_sweep_kernel": (C.c_char_p, [C.POINTER(SweepArgs)]),
    "ihdg_sweep_gram_kc": (_i32, [C.POINTER(SweepArgs)]),
    "ihdg_set_sweep_impl": (_i32, [C.c_char_p]),
    "ihdg_set_graphs": (_i32, [_i32]),
    "ihdg_finalize": (_i32, [C.POINTER(FinalizeArgs), _p]),
    "ihdg_layer_sums": (_i32, [_p, _i64, _i64, _p, _p]),
    "ihdg_halo_pack": (_i32, [C.POINTER(HaloArgs), _p]),
    "ihdg_halo_unpack": (_i32, [C.POINTER(HaloArgs), _p]),
    "ihdg_extract_trace": (_i32, [C.POINTER(TraceArgs), _p]),
    "ihdg_copy_state": (_i32, [C.POINTER(Geom), _p, _p, _p]),
    "ihdg_iterate": (_i32, [C.POINTER(SweepArgs), _p, _p, _i32, _p, C.POINTER(IterState),
                            C.POINTER(_i64)]),
    "ihdg_error_norm": (_i32, [C.POINTER(ErrorArgs), _p]),
    "ihdg_error_tile_count": (_i64, [C.POINTER(Geom)]),
    "ihdg_iterate_exact": (_i32, [C.POINTER(SweepArgs), C.POINTER(ErrorArgs), _p, _p, _i32, _p,
                                  C.POINTER(IterState), C.POINTER(_i64)]),
    "ihdg_elem_error": (_i32, [C.POINTER(ElemErrorArgs), _p]),
    "ihdg_face_energy": (_i32, [C.POINTER(FaceEnergyArgs), _p]),
}

_lib = None


def lib():
    """Load libihdg_cuda.so once; raise NativeUnavailable if it is missing."""
    global _lib
    if _lib is not None:
        return _lib
    if not os.path.exists(LIB_PATH):
        raise NativeUnavailable(
            f"{LIB_PATH} is not built; run `python -c 'import __graft_entry__ as g; g.build()'` "
            "(there is no CPU fallback for the iHDG sweep)")
    try:
        L = C.CDLL(LIB_PATH)
    except OSError as exc:  # pragma: no cover - depends on the box
        raise NativeUnavailable(f"cannot load {LIB_PATH}: {exc}") from exc
    for name, (res, args) in SIGNATURES.items():
        fn = getattr(L, name)
        fn.restype = res
        fn.argtypes = args
    if L.ihdg_abi_version() != ABI_VERSION:
        raise NativeUnavailable("libihdg_cuda.so ABI version mismatch")
    for i, st in enumerate(_STRUCTS):
        if L.ihdg_struct_size(i) != C.sizeof(st):
            raise NativeUnavailable(f"ABI struct size mismatch for {st.__name__}: "
                                    f"C {L.ihdg_struct_size(i)} vs ctypes {C.sizeof(st)}")
    _lib = L
    return L


def sweep_kernel(args: "SweepArgs") -> str:
    """Name of the kernel ihdg_sweep dispatches these args to (k_sweep_ws,
    k_sweep_v4, k_sweep_v5, k_sweep_v3, k_sweep_gemv or k_sweep)."""
    s = lib().ihdg_sweep_kernel(C.byref(args))
    if s is None:
        raise RuntimeError("no sweep kernel instantiated for these args")
    return s.decode()


def set_sweep_impl(name: str) -> None:
    """Process-wide kernel selector: auto / v3 / v5 / ws / stream / generic."""
    check(lib().ihdg_set_sweep_impl(name.encode()), "ihdg_set_sweep_impl")


def set_graphs(on: bool) -> None:
    """CUDA-graph replay of sweep batches in ihdg_iterate on / off."""
    lib().ihdg_set_graphs(1 if on else 0)


def check(rc: int, what: str) -> None:
    if rc != IHDG_OK:
        msg = lib().ihdg_last_error().decode(errors="replace")
        raise RuntimeError(f"{what} failed ({rc}): {msg}")
