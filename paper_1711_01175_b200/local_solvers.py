"""Per-element API of the reference module ``ihdg.local_solvers``
(SPEC.md:230-308): ``LocalSystem``, ``TraceSnapshot``, ``assemble_transport``
/ ``assemble_shallow_water`` / ``assemble_convection_diffusion`` and
``apply_local``, as thin entry points over the device kernels.

The sweep (iteration.run) never goes through here: it applies every
element's local solve at once in the fused sweep kernel.  These entry points
exist so that code written against the reference's per-element interface
runs unchanged:

- ``assemble_*(K, problem, ops, time_cfg, mesh)`` runs K1 (ihdg_assemble) for
  the mesh's operator classes once -- factor once per (PDE, mesh, p, dt),
  SPEC.md:287, 293 -- and returns the LocalSystem of element K: its class's
  matrix (host copy), the device factorization (A^-1 and the lifted
  L = A^-1 B, P = A^-1 R), and the condition estimate.
- ``TraceSnapshot.from_state`` freezes the iterate-k face values of K's
  neighbours and the boundary data of its boundary faces.
- ``apply_local`` is the lifted local solve
      u_K^{k+1} = A^-1 b + P u^m + L q,   q_f = sum_c face_w[f][c] u^{k,+}_c (face nodes)
  evaluated by K4 (ihdg_class_apply) on a one-element strip; the face
  scalars q are the RHS builder of SPEC.md:249, 259, 269.  It is pure and
  bit-reproducible.
"""

from __future__ import annotations

import ctypes as C
from dataclasses import dataclass, field
from typing import Optional

import numpy as np

from . import _native as N
from .assembly import OperatorSpec, build_spec, face_node_indices
from .basis import ElementOperators, FieldState
from .pde import ConvectionDiffusionProblem, ShallowWaterProblem, TransportProblem

__all__ = ["LocalSystem", "TraceSnapshot", "TimeConfig", "assemble_transport", "assemble_shallow_water",
           "assemble_convection_diffusion", "apply_local"]

BOUNDARY = -1


@dataclass(frozen=True)
class TimeConfig:
    """time_cfg of the assemble_* operations: "steady", "backward-euler" /
    "locally-implicit" (dt), "crank-nicolson" (dt)."""

    mode: str = "steady"
    dt: Optional[float] = None

    def scheme(self):
        m = self.mode.lower()
        if m == "steady":
            return None, "BE"
        if self.dt is None:
            raise ValueError(f"time mode {self.mode!r} needs dt")
        if m in ("backward-euler", "be", "locally-implicit"):
            return float(self.dt), "BE"
        if m in ("crank-nicolson", "cn"):
            return float(self.dt), "CN"
        raise ValueError(f"unknown time mode {self.mode!r}")


def _time_cfg(time_cfg):
    if time_cfg is None:
        return TimeConfig()
    if isinstance(time_cfg, TimeConfig):
        return time_cfg
    if isinstance(time_cfg, (int, float)):
        return TimeConfig("backward-euler", float(time_cfg))
    if isinstance(time_cfg, str):
        return TimeConfig(time_cfg)
    if isinstance(time_cfg, tuple):
        return TimeConfig(*time_cfg)
    raise TypeError(f"unsupported time_cfg {time_cfg!r}")


@dataclass
class LocalSystem:
    """element id; the square (m (p+1)^d) matrix; a reusable
    factorization (device A^-1, L = A^-1 B, P = A^-1 R of the element's
    operator class); the RHS builder's data (face weights of the neighbour
    scalars).  ``condition`` is the 1-norm condition estimate of the matrix."""

    element: int
    matrix: np.ndarray
    class_index: int
    boundary_mask: int
    condition: float
    spec: OperatorSpec = field(repr=False)
    ops: object = field(repr=False)              # solver.AssembledOperators
    scheme: str = "iHDG-II"


def _neighbor(mesh, K: int, f: int) -> int:
    """Neighbour element of K across local face f = 2 axis + side (mesh.py:44-48)."""
    d = mesh.dim
    idx = [int(i) for i in mesh.element_multi_index(K)]
    a, s = divmod(f, 2)
    j = idx[a] + (1 if s else -1)
    if j < 0 or j >= mesh.cells[a]:
        if not mesh.periodic[a]:
            return BOUNDARY
        j %= mesh.cells[a]
    idx[a] = j
    e, mul = 0, 1
    for b in range(d):
        e += idx[b] * mul
        mul *= mesh.cells[b]
    return e


def _boundary_mask(mesh, K: int) -> int:
    return sum(1 << f for f in range(2 * mesh.dim) if _neighbor(mesh, K, f) == BOUNDARY)


_CACHE: dict = {}


def _assemble(K, problem, ops: ElementOperators, time_cfg, mesh, scheme="iHDG-II") -> LocalSystem:
    from .solver import AssembledOperators

    if mesh is None:
        raise ValueError("assemble_* needs the mesh (neighbours and boundary faces of element K)")
    dt, ts = _time_cfg(time_cfg).scheme()
    key = (id(mesh), id(problem), id(ops), dt, ts, scheme)
    hit = _CACHE.get(key)
    if hit is None or hit[0] is not mesh or hit[1] is not problem:
        spec = build_spec(mesh, problem, ops, dt, scheme=scheme, time_scheme=ts)
        _CACHE.clear()   # one factor-once set at a time (the device copies are per spec)
        hit = (mesh, problem, spec, AssembledOperators(spec))
        _CACHE[key] = hit
    _, _, spec, aops = hit
    K = int(K)
    if not 0 <= K < mesh.n_elements:
        raise IndexError(f"element {K} out of range")
    mask = _boundary_mask(mesh, K)
    c = int(spec.class_of_mask[mask])
    A = aops.A[c].cpu().numpy()
    cond = float(np.linalg.cond(A, 1))
    if not np.isfinite(cond):
        raise np.linalg.LinAlgError(f"singular local matrix at element {K} (class {c})")
    return LocalSystem(K, A, c, mask, cond, spec, aops, scheme)


def assemble_transport(K, problem: TransportProblem, ops: ElementOperators, time_cfg=None, mesh=None,
                       scheme: str = "iHDG-II") -> LocalSystem:
    """SPEC.md:246-254 (transportLocalk1 / transportLocale)."""
    if not isinstance(problem, TransportProblem):
        raise TypeError("assemble_transport needs a TransportProblem")
    return _assemble(K, problem, ops, time_cfg, mesh, scheme)


def assemble_shallow_water(K, problem: ShallowWaterProblem, ops: ElementOperators, time_cfg=None, mesh=None,
                           scheme: str = "iHDG-II") -> LocalSystem:
    """SPEC.md:256-264 (localSolverDD + phihDD)."""
    if not isinstance(problem, ShallowWaterProblem):
        raise TypeError("assemble_shallow_water needs a ShallowWaterProblem")
    if _time_cfg(time_cfg).mode == "steady":
        raise ValueError("shallow water is time dependent (backward-Euler or Crank-Nicolson dt)")
    return _assemble(K, problem, ops, time_cfg, mesh, scheme)


def assemble_convection_diffusion(K, problem: ConvectionDiffusionProblem, ops: ElementOperators, time_cfg=None,
                                  mesh=None, scheme: str = "iHDG-II") -> LocalSystem:
    """SPEC.md:266-274 (ErrorDDMCD + uhatCDR)."""
    if not isinstance(problem, ConvectionDiffusionProblem):
        raise TypeError("assemble_convection_diffusion needs a ConvectionDiffusionProblem")
    return _assemble(K, problem, ops, time_cfg, mesh, scheme)


@dataclass
class TraceSnapshot:
    """per face of element K the neighbour's iterate-k
    values of every component at the face nodes ((m, N_f), mesh.py face-node
    order), or the boundary data g at the face nodes ((N_f,)) on a boundary
    face with data, or None.  Read-only during an iteration."""

    element: int
    neighbor: dict
    boundary: dict = field(default_factory=dict)
    own: Optional[np.ndarray] = None   # iHDG-I: the element's own iterate k (m, Np)

    @classmethod
    def from_state(cls, mesh, state, K: int, boundary_data=None) -> "TraceSnapshot":
        """Freeze the neighbour face values of iterate k (``state``: FieldState
        or (Nel, m, Np)) around element K; ``boundary_data(x)`` -> (n,) gives
        g at the boundary face nodes (transport inflow / CD Dirichlet)."""
        data = state.data if isinstance(state, FieldState) else np.asarray(state)
        d = mesh.dim
        n1 = round(data.shape[-1] ** (1.0 / d))
        nbr, bnd = {}, {}
        for f in range(2 * d):
            nb = _neighbor(mesh, K, f)
            if nb != BOUNDARY:
                nbr[f] = np.array(data[nb][:, face_node_indices(d, n1, f ^ 1)], dtype=float)
            elif boundary_data is not None:
                from .basis import gll_nodes

                nodes = gll_nodes(n1 - 1)[0]
                pts = mesh.element_points(K, [nodes] * d)[face_node_indices(d, n1, f)]
                bnd[f] = np.asarray(boundary_data(pts), dtype=float).reshape(-1)
        return cls(int(K), nbr, bnd, np.array(data[K], dtype=float))


def _apply_one(aops, spec, c, opT_class_block, ncols, vec, out, accumulate):
    """K4 on a one-element strip: out (+)= opT[c]^T vec (ihdg_class_apply)."""
    torch = aops.torch
    d = spec.dim
    g = N.Geom()
    g.dim, g.order, g.ncomp = d, spec.order, spec.ncomp
    for a in range(3):
        g.cells[a] = 1
    g.layer_begin, g.layer_end = 0, 1
    com = torch.full((64,), 0, dtype=torch.int32, device=aops.device)
    a = N.ClassApplyArgs()
    a.g = g
    a.opT = int(opT_class_block.data_ptr())
    a.class_of_mask, a.inp, a.out = int(com.data_ptr()), int(vec.data_ptr()), int(out.data_ptr())
    a.in_stride, a.in_offset, a.ncols = int(vec.numel()), 0, int(ncols)
    a.in_ghost, a.out_ghost, a.accumulate = 0, 0, int(accumulate)
    N.check(aops.L.ihdg_class_apply(C.byref(a), aops._sptr), "ihdg_class_apply")


def apply_local(system: LocalSystem, snapshot: TraceSnapshot, forcing=None, prev_level=None) -> np.ndarray:
    """the element's iterate k+1, (m, Np).

    ``forcing``: the element load vector (f, v)_K, (m, Np) or (nv,), or None;
    ``prev_level``: u^m of the element, (m, Np), for time-dependent systems.
    Zero inputs give zero; repeated calls are bit-identical."""
    sp, aops, c = system.spec, system.ops, system.class_index
    torch = aops.torch
    if snapshot.element != system.element:
        raise ValueError("snapshot and local system belong to different elements")
    if sp.time_scheme == "CN":
        raise NotImplementedError("apply_local: Crank-Nicolson couples both levels' traces; use run_time_dependent")
    d, nv, npn = sp.dim, sp.nv, sp.n_nodes
    nf = sp.n1 ** (d - 1)
    dev = aops.device
    # RHS builder: neighbour face scalars q_f = sum_c face_w[f][c] u^+_c (the
    # trace formulas' neighbour parts; boundary data enter the same slot for
    # transport inflow, through L_D for convection-diffusion Dirichlet faces)
    q = np.zeros(sp.kin)
    qd = np.zeros(sp.kin)
    for f in range(2 * d):
        if f in snapshot.neighbor and sp.coupled[f]:
            vals = snapshot.neighbor[f]
            q[f * nf:(f + 1) * nf] = sum(float(sp.face_w[f, cc]) * vals[cc] for cc in range(sp.ncomp)
                                         if float(sp.face_w[f, cc]) != 0.0)
        elif f in snapshot.boundary:
            g = snapshot.boundary[f]
            if aops.LT_dir is not None:                       # CD Dirichlet: u_hat := g (L_D)
                qd[f * nf:(f + 1) * nf] = g
            elif sp.coupled[f] and float(sp.face_w[f, 0]) != 0.0:   # transport inflow u_ext = g
                q[f * nf:(f + 1) * nf] = float(sp.face_w[f, 0]) * g
    if system.scheme == "iHDG-I" and snapshot.own is not None:
        own = np.asarray(snapshot.own, dtype=float).reshape(sp.ncomp, npn)
        for f in range(2 * d):
            ids = face_node_indices(d, sp.n1, f)
            q[f * nf:(f + 1) * nf] += sum(float(sp.own_w[f, cc]) * own[cc, ids] for cc in range(sp.ncomp)
                                          if float(sp.own_w[f, cc]) != 0.0)
    out = torch.zeros(nv, dtype=torch.float64, device=dev)
    acc = 0
    if forcing is not None:
        b = torch.as_tensor(np.asarray(forcing, dtype=float).reshape(nv), device=dev)
        _apply_one(aops, sp, c, aops.AinvT[c], nv, b, out, acc)
        acc = 1
    if prev_level is not None and sp.nr > 0:
        um = np.asarray(prev_level, dtype=float).reshape(nv)[sp.time_comp0 * npn: sp.time_comp0 * npn + sp.nr]
        _apply_one(aops, sp, c, aops.PT[c], sp.nr, torch.as_tensor(np.ascontiguousarray(um), device=dev), out, acc)
        acc = 1
    # the lifted couplings face by face (a column block of L per face: K4
    # takes at most NV columns per call)
    for LTc, qq in ((aops.LT[c], q), (aops.LT_dir[c] if aops.LT_dir is not None else None, qd)):
        if LTc is None:
            continue
        for f in range(2 * d):
            seg = qq[f * nf:(f + 1) * nf]
            if np.any(seg != 0.0):     # out starts at zero: accumulating is exact
                _apply_one(aops, sp, c, LTc.view(-1)[f * nf * nv:(f + 1) * nf * nv], nf,
                           torch.as_tensor(np.ascontiguousarray(seg), device=dev), out, 1)
    aops.stream.synchronize()
    return out.cpu().numpy().reshape(sp.ncomp, npn)
