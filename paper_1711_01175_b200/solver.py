"""Device-resident iHDG-II solver for one rank's strip of the mesh.

PyTorch is used only as plumbing: it allocates device memory, provides the
CUDA stream and (for several ranks) torch.distributed.  All arithmetic of the
iteration runs in libihdg_cuda.so kernels (see include/ihdg.h).
"""

from __future__ import annotations

import ctypes as C
import time
from dataclasses import dataclass
from typing import Optional

import numpy as np

from . import _native as N
from .assembly import OperatorSpec, build_spec, face_node_indices
from .basis import ElementOperators
from .pde import FourierModes, GaussianBump, TransportProblem

__all__ = ["DeviceSolver", "IterResult"]


def _torch():
    import torch

    if not torch.cuda.is_available():
        raise N.NativeUnavailable("no CUDA device: the iHDG sweep has no CPU fallback")
    return torch


def torch_cpu_zeros_like(t):
    return t.new_zeros(t.shape, device="cpu")


def _ptr(t) -> int:
    return 0 if t is None else int(t.data_ptr())


@dataclass
class IterResult:
    iterations: int
    status: str
    norms: np.ndarray
    first_norm: float
    last_norm: float
    launched: int
    seconds: float
    errors: Optional[np.ndarray] = None   # exact-solution rule: ||u^k - u^e||_{L2} per sweep
    kernel: str = ""                      # sweep kernel ihdg_sweep dispatched to (ihdg_sweep_kernel)


class AssembledOperators:
    """K1 (ihdg_assemble) for one OperatorSpec on one device: the factor-once
    local systems of every operator class -- A, A^-1,
    the lifted L = A^-1 B, P = A^-1 R, and the Crank-Nicolson / Dirichlet-data
    lifted operators when the spec has them.  Shared by DeviceSolver (the
    sweep) and local_solvers (the per-element API)."""

    def __init__(self, spec: OperatorSpec, device=None, stream=None):
        torch = _torch()
        self.torch, self.L, self.spec = torch, N.lib(), spec
        if isinstance(device, torch.device):
            self.device = device
        else:
            self.device = torch.device("cuda", torch.cuda.current_device() if device is None else int(device))
        with torch.cuda.device(self.device):
            self.stream = stream if stream is not None else torch.cuda.current_stream(self.device)
            self._assemble()

    @property
    def _sptr(self):
        return C.c_void_p(self.stream.cuda_stream)

    def _assemble(self):
        torch, sp, dev, f64 = self.torch, self.spec, self.device, self.torch.float64
        nc, nv, kin, nr = sp.n_class, sp.nv, sp.kin, sp.nr
        self._ops1d = torch.as_tensor(sp.ops1d, dtype=f64, device=dev).contiguous()
        self._opn = torch.as_tensor(sp.op_ncols, device=dev)
        self._terms = torch.as_tensor(sp.terms, device=dev).contiguous()
        self._coefs = torch.as_tensor(sp.coefs, dtype=f64, device=dev)
        self.A = torch.zeros((nc, nv, nv), dtype=f64, device=dev)
        self.Ainv = torch.zeros_like(self.A)
        self.AinvT = torch.zeros_like(self.A)
        self.B = torch.zeros((nc, nv, kin), dtype=f64, device=dev)
        self.R = torch.zeros((nc, nv, max(nr, 1)), dtype=f64, device=dev)
        self.LT = torch.zeros((nc, kin, nv), dtype=f64, device=dev)
        self.PT = torch.zeros((nc, max(nr, 1), nv), dtype=f64, device=dev)
        self.min_pivot = torch.zeros(nc, dtype=f64, device=dev)
        a = N.AssemblyArgs()
        a.dim, a.order, a.ncomp, a.n_class = sp.dim, sp.order, sp.ncomp, nc
        a.n_ops, a.n_terms, a.nr = sp.ops1d.shape[0], sp.terms.shape[0], nr
        a.kin_blocks = sp.kin_blocks
        a.ops1d, a.op_ncols = _ptr(self._ops1d), _ptr(self._opn)
        a.terms, a.coefs = _ptr(self._terms), _ptr(self._coefs)
        a.A, a.Ainv, a.AinvT, a.B = _ptr(self.A), _ptr(self.Ainv), _ptr(self.AinvT), _ptr(self.B)
        a.R = _ptr(self.R) if nr > 0 else 0
        a.LT = _ptr(self.LT)
        a.PT = _ptr(self.PT) if nr > 0 else 0
        a.min_pivot = _ptr(self.min_pivot)
        N.check(self.L.ihdg_assemble(C.byref(a), self._sptr), "ihdg_assemble")
        self.LT_expl = None
        if sp.time_scheme == "CN":
            # L_expl = A^-1 (1 - theta) B: the explicit half of the trace couplings
            self._terms_x = torch.as_tensor(sp.terms_expl, device=dev).contiguous()
            self._coefs_x = torch.as_tensor(sp.coefs_expl, dtype=f64, device=dev)
            A2, Ai2, AiT2 = torch.zeros_like(self.A), torch.zeros_like(self.A), torch.zeros_like(self.A)
            B2 = torch.zeros_like(self.B)
            self.LT_expl = torch.zeros_like(self.LT)
            mp2 = torch.zeros_like(self.min_pivot)
            b = N.AssemblyArgs()
            b.dim, b.order, b.ncomp, b.n_class = sp.dim, sp.order, sp.ncomp, nc
            b.n_ops, b.n_terms, b.nr = sp.ops1d.shape[0], sp.terms_expl.shape[0], 0
            b.ops1d, b.op_ncols = _ptr(self._ops1d), _ptr(self._opn)
            b.terms, b.coefs = _ptr(self._terms_x), _ptr(self._coefs_x)
            b.A, b.Ainv, b.AinvT, b.B = _ptr(A2), _ptr(Ai2), _ptr(AiT2), _ptr(B2)
            b.R, b.LT, b.PT, b.min_pivot = 0, _ptr(self.LT_expl), 0, _ptr(mp2)
            N.check(self.L.ihdg_assemble(C.byref(b), self._sptr), "ihdg_assemble (CN explicit)")
            del A2, Ai2, AiT2, B2, mp2
        self.LT_dir = self.LT_dir_expl = None
        if sp.terms_dir is not None:
            # L_D = A^-1 B_D: the Dirichlet-data couplings (convection-diffusion)
            self.LT_dir = self._assemble_lifted(sp.terms_dir, sp.coefs_dir, "ihdg_assemble (Dirichlet data)")
        if sp.terms_dir_expl is not None:
            self.LT_dir_expl = self._assemble_lifted(sp.terms_dir_expl, sp.coefs_dir_expl,
                                                     "ihdg_assemble (Dirichlet data, CN old level)")
        piv = self.min_pivot.cpu().numpy()
        scale = self.A.abs().amax(dim=(1, 2)).cpu().numpy()
        bad = np.nonzero(~(piv > 1e-13 * scale))[0]
        if bad.size:
            c = int(bad[0])
            raise np.linalg.LinAlgError(
                f"singular local matrix in operator class {c} (boundary mask {sp.class_masks[c]}): "
                f"min pivot {piv[c]:.3e}, max |A| {scale[c]:.3e}")

    def _assemble_lifted(self, terms, coefs, what):
        """A^-1 B of another term list with the same A (K1), as LT [class][kin][nv]."""
        torch, sp = self.torch, self.spec
        tt = torch.as_tensor(terms, device=self.device).contiguous()
        cc = torch.as_tensor(coefs, dtype=torch.float64, device=self.device)
        A2, Ai2, AiT2 = torch.zeros_like(self.A), torch.zeros_like(self.A), torch.zeros_like(self.A)
        # the data couplings: one column per face node (g), whatever the main B's blocks
        kb = sp.kin_base
        B2 = torch.zeros((sp.n_class, sp.nv, kb), dtype=torch.float64, device=self.device)
        LT = torch.zeros((sp.n_class, kb, sp.nv), dtype=torch.float64, device=self.device)
        mp2 = torch.zeros_like(self.min_pivot)
        b = N.AssemblyArgs()
        b.dim, b.order, b.ncomp, b.n_class = sp.dim, sp.order, sp.ncomp, sp.n_class
        b.n_ops, b.n_terms, b.nr = sp.ops1d.shape[0], terms.shape[0], 0
        b.ops1d, b.op_ncols = _ptr(self._ops1d), _ptr(self._opn)
        b.terms, b.coefs = _ptr(tt), _ptr(cc)
        b.A, b.Ainv, b.AinvT, b.B = _ptr(A2), _ptr(Ai2), _ptr(AiT2), _ptr(B2)
        b.R, b.LT, b.PT, b.min_pivot = 0, _ptr(LT), 0, _ptr(mp2)
        N.check(self.L.ihdg_assemble(C.byref(b), self._sptr), what)
        self.stream.synchronize()
        return LT



class DeviceSolver:
    """Factor-once local operators + ping-pong iterate buffers on one GPU.

    ``layers`` = (begin, end) range of the slowest axis owned by this rank
    (strip partition); default the whole mesh.
    """

    def __init__(self, mesh, problem, ops: ElementOperators, dt=None, layers=None,
                 device=None, max_iters: int = 100000, spec: Optional[OperatorSpec] = None,
                 scheme: str = "iHDG-II", time_scheme: str = "BE", gram_norm: bool = False):
        torch = _torch()
        L = N.lib()
        self.torch = torch
        self.L = L
        self.mesh, self.problem, self.ops, self.dt = mesh, problem, ops, dt
        self.spec = spec if spec is not None else build_spec(mesh, problem, ops, dt, scheme=scheme,
                                                             time_scheme=time_scheme)
        sp = self.spec
        d = mesh.dim
        if not L.ihdg_supported(d, ops.p, sp.ncomp):
            raise NotImplementedError(f"no sweep kernel for dim={d}, p={ops.p}, m={sp.ncomp}")
        self.device = torch.device("cuda", torch.cuda.current_device() if device is None else device)
        nlay = mesh.cells[d - 1]
        lb, le = (0, nlay) if layers is None else (int(layers[0]), int(layers[1]))
        self.layers = (lb, le)
        g = N.Geom()
        g.dim, g.order, g.ncomp = d, ops.p, sp.ncomp
        for a in range(3):
            g.cells[a] = mesh.cells[a] if a < d else 1
            g.periodic[a] = int(mesh.periodic[a]) if a < d else 0
        g.layer_begin, g.layer_end = lb, le
        self.geom = g
        self.ls = int(np.prod(mesh.cells[: d - 1])) if d > 1 else 1
        self.nloc = (le - lb) * self.ls
        self.nv = sp.nv
        self.np_ = sp.n_nodes
        self.ntiles = int(L.ihdg_tile_count(C.byref(g)))
        if self.ntiles < 1:
            raise RuntimeError("ihdg_tile_count failed")
        self.max_iters = int(max_iters)
        dev = self.device
        f64 = torch.float64
        with torch.cuda.device(dev):
            self.stream = torch.cuda.current_stream(dev)
            self._assemble()
            npad = self.nloc + 2 * self.ls
            self.u = [torch.zeros((npad, self.nv), dtype=f64, device=dev) for _ in range(2)]
            self.cur = 0
            self.s = torch.zeros((self.nloc, self.nv), dtype=f64, device=dev)
            self.s_static = None
            self.partials = torch.zeros(self.ntiles, dtype=f64, device=dev)
            self.state_dev = torch.zeros(C.sizeof(N.IterState), dtype=torch.uint8, device=dev)
            self.norm_hist = torch.zeros(self.max_iters, dtype=f64, device=dev)
            self.chol = torch.as_tensor(ops.chol1d.copy(), dtype=f64, device=dev)
            self.class_of_mask = torch.as_tensor(sp.class_of_mask, device=dev)
            # parallel finalize of k_sweep_ws (ihdg_sweep_args.layer_sums / grid_bar)
            self.layer_sums = torch.zeros(max(le - lb, 1), dtype=f64, device=dev)
            self.grid_bar = torch.zeros(2, dtype=torch.int32, device=dev)
            self.gram_kc = 0
            if gram_norm:
                self._setup_gram()

    # -- setup -------------------------------------------------------------
    @property
    def _sptr(self):
        return C.c_void_p(self.stream.cuda_stream)

    def _assemble(self):
        """K1 through AssembledOperators; the class operators become attributes."""
        ops = AssembledOperators(self.spec, self.device, self.stream)
        self.assembled = ops
        for name in ("A", "Ainv", "AinvT", "B", "R", "LT", "PT", "min_pivot", "LT_expl", "LT_dir", "LT_dir_expl"):
            setattr(self, name, getattr(ops, name))

    def _setup_gram(self) -> None:
        """Gram-form stopping norm of the interior operator class (ihdg.h,
        ihdg_sweep_args.q_store): R upper triangular with
        R^T R = L^T (W (x) M1 (x) .. (x) M1) L over the kernel's q columns,
        so that ||u^{k+1} - u^k||^2_M = J ||R (q^k - q^{k-1})||^2 within a
        solve; plus the per-element q store.  Only for kernels that take it
        (ihdg_sweep_gram_kc > 0); otherwise the direct norm runs.

        Opt-in (``DeviceSolver(gram_norm=True)``): it replaces ~190 of the
        ~460 DMMAs per config-5 tile by 32 but adds the q store, 3 B per DOF of
        HBM traffic (+12.7%), and on B200 the sweep is bound by its memory
        throughput, so it measured 4.46 ms against 4.01 ms per sweep
        (profiles/r02_gram_ab.txt)."""
        self.gram_R = self.q_store = None
        self.gram_kc = 0
        a = self.sweep_args("volume", gram=False)
        a.u_old, a.u_new = _ptr(self.u[0]), _ptr(self.u[1])
        kc = int(self.L.ihdg_sweep_gram_kc(C.byref(a)))
        if kc <= 0:
            return
        sp, d = self.spec, self.mesh.dim
        nf = sp.n1 ** (d - 1)
        cols = [f * nf + n for f in range(2 * d) if sp.coupled[f] for n in range(nf)]
        if len(cols) != kc:
            return
        c = int(sp.class_of_mask[0])
        Lc = self.LT[c].cpu().numpy().T[:, cols]                   # (nv, kc)
        m1 = self.ops.chol1d @ self.ops.chol1d.T
        mref = m1
        for _ in range(d - 1):
            mref = np.kron(m1, mref)
        W = np.kron(np.diag(np.asarray(sp.comp_w[: sp.ncomp], dtype=float)), mref)
        G = Lc.T @ W @ Lc
        G = 0.5 * (G + G.T)
        try:
            R = np.linalg.cholesky(G).T                            # upper: G = R^T R
        except np.linalg.LinAlgError:
            return                                                 # singular: direct norm
        torch = self.torch
        self.gram_R = torch.as_tensor(np.ascontiguousarray(R), dtype=torch.float64, device=self.device)
        self.q_store = torch.zeros((self.nloc, kc), dtype=torch.float64, device=self.device)
        self.gram_kc = kc

    # -- state -------------------------------------------------------------
    def interior(self, which=None):
        t = self.u[self.cur if which is None else which]
        return t[self.ls: self.ls + self.nloc]

    def set_state(self, data) -> None:
        """Host (nloc, m, Np) array (or device tensor) -> current iterate."""
        torch = self.torch
        t = self.interior()
        src = torch.as_tensor(np.ascontiguousarray(data, dtype=np.float64)) if isinstance(data, np.ndarray) else data
        t.copy_(src.reshape(self.nloc, self.nv), non_blocking=False)
        self.u[self.cur][: self.ls].zero_()
        self.u[self.cur][self.ls + self.nloc:].zero_()

    def zero_state(self) -> None:
        self.u[self.cur].zero_()

    def get_state(self) -> np.ndarray:
        return self.interior().reshape(self.nloc, self.spec.ncomp, self.np_).cpu().numpy()

    def _field_args(self, field, ref1d_t, out, out_stride, out_offset, out_ghost):
        a = N.FieldArgs()
        a.g = self.geom
        for i in range(self.mesh.dim):
            a.lo[i] = float(self.mesh.lo[i])
            a.h[i] = float(self.mesh.h[i])
        params = self.torch.as_tensor(field.device_params(), dtype=self.torch.float64, device=self.device)
        a.ref1d, a.params, a.out = _ptr(ref1d_t), _ptr(params), _ptr(out)
        a.out_stride, a.out_offset, a.out_ghost = out_stride, out_offset, out_ghost
        a.npts1d = ref1d_t.numel()
        a.kind = 0 if isinstance(field, FourierModes) else 1
        a.nmodes = params.shape[0]
        return a, params

    def set_state_component(self, field, comp: int) -> None:
        """Nodal interpolation (project) of an analytic field into one component."""
        torch = self.torch
        if isinstance(field, (FourierModes, GaussianBump)):
            ref = torch.as_tensor(self.ops.nodes, dtype=torch.float64, device=self.device)
            a, keep = self._field_args(field, ref, self.u[self.cur], self.nv, comp * self.np_, 1)
            N.check(self.L.ihdg_eval_field(C.byref(a), self._sptr), "ihdg_eval_field")
            torch.cuda.current_stream(self.device).synchronize()
        else:
            pts = self._local_points(self.ops.nodes)
            vals = np.asarray(field(pts.reshape(-1, self.mesh.dim)), dtype=float).reshape(self.nloc, self.np_)
            self.interior().view(self.nloc, self.spec.ncomp, self.np_)[:, comp, :].copy_(
                torch.as_tensor(vals, device=self.device))

    def _local_points(self, ref):
        pts = self.mesh.all_element_points([ref] * self.mesh.dim)
        lb, le = self.layers
        return pts[lb * self.ls: le * self.ls]

    def set_forcing(self, forcing) -> None:
        """Static RHS part s_f = A^-1 (f, v)_K."""
        torch, sp, ops = self.torch, self.spec, self.ops
        nq = ops.quad_points.size
        d = self.mesh.dim
        fq = torch.zeros((self.nloc, nq ** d), dtype=torch.float64, device=self.device)
        if isinstance(forcing, (FourierModes, GaussianBump)):
            ref = torch.as_tensor(ops.quad_points, dtype=torch.float64, device=self.device)
            a, keep = self._field_args(forcing, ref, fq, nq ** d, 0, 0)
            N.check(self.L.ihdg_eval_field(C.byref(a), self._sptr), "ihdg_eval_field")
        else:
            pts = self._local_points(ops.quad_points)
            vals = np.asarray(forcing(pts.reshape(-1, d)), dtype=float).reshape(self.nloc, -1)
            fq.copy_(torch.as_tensor(vals, device=self.device))
        b = torch.zeros((self.nloc, self.nv), dtype=torch.float64, device=self.device)
        Bq = torch.as_tensor(ops.quad_to_rhs, dtype=torch.float64, device=self.device).contiguous()
        q = N.QuadArgs()
        q.g = self.geom
        q.Bq, q.fq, q.out = _ptr(Bq), _ptr(fq), _ptr(b)
        q.out_stride, q.out_offset, q.nq, q.jac = self.nv, sp.forcing_comp * self.np_, nq, sp.jac
        N.check(self.L.ihdg_quad_project(C.byref(q), self._sptr), "ihdg_quad_project")
        self.s_static = torch.zeros((self.nloc, self.nv), dtype=torch.float64, device=self.device)
        self._apply(self.AinvT, self.nv, b, self.nv, 0, 0, self.s_static, 0)
        self.stream.synchronize()

    def _apply(self, opT, ncols, inp, in_stride, in_offset, in_ghost, out, accumulate):
        a = N.ClassApplyArgs()
        a.g = self.geom
        a.opT, a.class_of_mask, a.inp, a.out = _ptr(opT), _ptr(self.class_of_mask), _ptr(inp), _ptr(out)
        a.in_stride, a.in_offset, a.ncols = in_stride, in_offset, ncols
        a.in_ghost, a.out_ghost, a.accumulate = in_ghost, 0, accumulate
        a.per_element = int(self.spec.per_element)
        N.check(self.L.ihdg_class_apply(C.byref(a), self._sptr), "ihdg_class_apply")

    def set_inflow(self, g, g_explicit=None) -> None:
        """Inflow boundary data u_ext = g,
        transport: the inflow faces' neighbour scalar on the boundary is
        q = face_w g instead of 0, so the static RHS gains s_g = L q_g (K4 with
        the lifted operator).  ``g(x)`` -> (n,) is evaluated at the boundary
        face nodes; None clears it."""
        torch, sp, d = self.torch, self.spec, self.mesh.dim
        if g is None:
            self.s_bdata, self._bdata_faces = None, None
            return
        if not isinstance(self.problem, TransportProblem) or sp.n_class != 1:
            raise NotImplementedError("inflow data is defined for transport (one operator class)")
        nf = sp.n1 ** (d - 1)
        nfc = 2 * d * nf

        def inflow_face(f):
            return bool(sp.coupled[f]) and float(sp.face_w[f, 0]) != 0.0

        def face_data(fn):
            # q = face_w g on the inflow boundary faces (the neighbour scalar)
            return self._boundary_face_data(fn, inflow_face, weight=lambda f: float(sp.face_w[f, 0]))

        self.s_bdata = torch.zeros((self.nloc, self.nv), dtype=torch.float64, device=self.device)
        # one K4 pass per inflow face with that face's column block of L
        # (transport has a single operator class, so the block is contiguous)
        parts = [(g, self.LT)]
        if sp.time_scheme == "CN":
            if g_explicit is None:
                raise ValueError("Crank-Nicolson inflow data needs the old-level data g_explicit")
            parts.append((g_explicit, self.LT_expl))
        faces = None
        for fn, LT in parts:
            q, fc = face_data(fn)
            faces = fc if faces is None else faces
            for f in fc:
                self._apply(LT.view(-1)[f * nf * self.nv:], nf, q, nfc, f * nf, 0, self.s_bdata, 1)
        self._bdata_faces = faces
        self.stream.synchronize()

    def _boundary_face_data(self, fn, face_ok, weight=None):
        """(q, faces): fn at the face nodes of every boundary face f of the
        local elements with face_ok(f) (non-periodic axes), as a
        [nloc][2d N_f] face-node array and {f: (elements, values)}."""
        torch, sp, d = self.torch, self.spec, self.mesh.dim
        nf = sp.n1 ** (d - 1)
        nfc = 2 * d * nf
        pts = self._local_points(self.ops.nodes)
        e = np.arange(self.nloc, dtype=np.int64)
        idx = [(e // int(np.prod(self.mesh.cells[:a]))) % self.mesh.cells[a] for a in range(d - 1)]
        idx.append(self.layers[0] + e // self.ls)
        qg = np.zeros((self.nloc, nfc))
        faces = {}
        for f in range(2 * d):
            a, side = divmod(f, 2)
            if self.mesh.periodic[a] or not face_ok(f):
                continue
            on = np.flatnonzero(idx[a] == (self.mesh.cells[a] - 1 if side else 0))
            if on.size == 0:
                continue
            ids = face_node_indices(d, sp.n1, f)
            vals = np.asarray(fn(pts[on][:, ids, :].reshape(-1, d)), dtype=float).reshape(on.size, nf)
            qg[on, f * nf:(f + 1) * nf] = vals if weight is None else weight(f) * vals
            faces[f] = (on, vals)
        return torch.as_tensor(qg, dtype=torch.float64, device=self.device), faces

    def set_dirichlet(self, g, g_explicit=None) -> None:
        """Dirichlet data u_hat := g_D on the boundary,
        convection-diffusion: s gains L_D q_g (K4), L_D = A^-1 B_D assembled by
        K1 from the Dirichlet-data term list; g at the boundary face nodes
        (the trace space).  The returned trace is g on the boundary.
        Crank-Nicolson: g at the new level, g_explicit at the old one, split
        like the trace couplings (theta = 1 on the sigma rows, 1/2 on u)."""
        if g is None:
            self.s_bdata, self._bdata_faces = None, None
            return
        if self.LT_dir is None:
            raise NotImplementedError("Dirichlet data needs a ConvectionDiffusionProblem built with dirichlet=")
        sp = self.spec
        q, faces = self._boundary_face_data(g, lambda f: True)
        nfc = q.shape[1]
        assert sp.kin_base == nfc, "Dirichlet data: every face slot is coupled for convection-diffusion"
        self.s_bdata = self.torch.zeros((self.nloc, self.nv), dtype=self.torch.float64, device=self.device)
        self._apply(self.LT_dir, nfc, q, nfc, 0, 0, self.s_bdata, 0)
        if self.LT_dir_expl is not None:
            if g_explicit is None:
                raise ValueError("Crank-Nicolson Dirichlet data needs the old-level data g_explicit")
            q0, _ = self._boundary_face_data(g_explicit, lambda f: True)
            self._apply(self.LT_dir_expl, nfc, q0, nfc, 0, 0, self.s_bdata, 1)
        self._bdata_faces = faces
        self.stream.synchronize()

    def prepare_steady(self) -> None:
        """s = A^-1 b (forcing) or 0, plus the inflow-data part L q_g."""
        if self.s_static is None:
            self.s.zero_()
        else:
            self.s.copy_(self.s_static)
        if getattr(self, "s_bdata", None) is not None:
            self.s.add_(self.s_bdata)

    def begin_step(self, exchange=None) -> None:
        """RHS of the next step from the current state u^m.

        Backward Euler: s = P u^m (+ A^-1 f) (K4).  Crank-Nicolson adds the
        explicit half of the trace couplings, A^-1 (1-theta) B q(u^m): one
        sweep with L_expl from u^m into the spare buffer, which becomes s
        (``exchange`` refreshes the ghost layers of u^m first, multi-rank)."""
        sp = self.spec
        if sp.nr == 0:
            raise RuntimeError("problem was assembled without a time step")
        if self.s_static is not None:
            self.s.copy_(self.s_static)
            acc = 1
        else:
            acc = 0
        if getattr(self, "s_bdata", None) is not None:
            if acc:
                self.s.add_(self.s_bdata)
            else:
                self.s.copy_(self.s_bdata)
            acc = 1
        self._apply(self.PT, sp.nr, self.u[self.cur], self.nv, sp.time_comp0 * self.np_, 1, self.s, acc)
        if sp.time_scheme == "CN":
            if exchange is not None:
                exchange()
            self.reset_state(0.0, 1)
            a = self.sweep_args("volume", finalize=0, gram=False)
            a.LT = _ptr(self.LT_expl)
            a.u_old, a.u_new = _ptr(self.u[self.cur]), _ptr(self.u[1 - self.cur])
            N.check(self.L.ihdg_sweep(C.byref(a), self._sptr), "ihdg_sweep (CN explicit half)")
            self.s.copy_(self.interior(1 - self.cur))

    # -- iteration ---------------------------------------------------------
    def sweep_args(self, norm: str, finalize: int = 1, gram: bool = True) -> N.SweepArgs:
        """Sweep arguments of the current operators; ``gram``: pass the
        Gram-form norm data when the kernel takes it (the caller keeps s and
        the operators fixed between the sweeps of one solve)."""
        sp = self.spec
        a = N.SweepArgs()
        a.g = self.geom
        a.s, a.LT = _ptr(self.s), _ptr(self.LT)
        a.class_of_mask, a.chol1d = _ptr(self.class_of_mask), _ptr(self.chol)
        ch = np.ascontiguousarray(self.ops.chol1d, dtype=np.float64).ravel()
        if ch.size <= 64:
            for i, v in enumerate(ch):
                a.chol[i] = float(v)
        a.tile_partials, a.state, a.norm_hist = _ptr(self.partials), _ptr(self.state_dev), _ptr(self.norm_hist)
        for f in range(6):
            for c in range(4):
                a.face_w[f][c] = float(sp.face_w[f, c])
                a.out_w[f][c] = float(sp.out_w[f, c])
            a.coupled[f] = int(sp.coupled[f])
            for c in range(4):
                a.own_w[f][c] = float(sp.own_w[f, c])
            a.out_face[f] = int(sp.out_face[f])
        for c in range(4):
            a.comp_w[c] = float(sp.comp_w[c])
        a.jac = sp.jac
        for i in range(3):
            a.jac_face[i] = float(sp.jac_face[i])
        a.norm_kind = N.NORM_TRACE if norm == "trace" else N.NORM_VOLUME
        a.finalize = finalize
        a.tile_offset = 0
        a.scheme = N.SCHEME_I if sp.scheme == "iHDG-I" else N.SCHEME_II
        if sp.per_element:
            # per-element operators: raw neighbour (and, iHDG-I, own) face values;
            # the own part is a column of L, not the own_w scalar trick
            a.per_element, a.raw_blocks = 1, int(sp.kin_blocks)
            for f in range(6):
                for j in range(4):
                    a.raw_comp[f][j] = int(sp.raw_comp[f, j])
            a.scheme = N.SCHEME_II
        if gram and getattr(self, "gram_kc", 0) > 0:
            a.q_store, a.gram_R, a.gram_kc = _ptr(self.q_store), _ptr(self.gram_R), self.gram_kc
        if getattr(self, "grid_bar", None) is not None and self.mesh.dim > 1:
            a.layer_sums, a.grid_bar = _ptr(self.layer_sums), _ptr(self.grid_bar)
        return a

    def reset_state(self, tol: float, max_iters: int, diverge_factor: float = 1e6) -> None:
        if int(max_iters) > self.max_iters:
            # the norm history holds one entry per sweep: grow it rather than
            # silently capping the caller's max_iters
            self.max_iters = int(max_iters)
            self.norm_hist = self.torch.zeros(self.max_iters, dtype=self.torch.float64, device=self.device)
            if getattr(self, "err_hist", None) is not None:
                self.err_hist = self.torch.zeros(self.max_iters, dtype=self.torch.float64, device=self.device)
        st = N.IterState()
        st.status, st.iters, st.max_iters, st.ticket = N.RUNNING, 0, int(max_iters), 0
        st.tol, st.first_norm, st.last_norm, st.diverge_factor = tol, 0.0, 0.0, diverge_factor
        host = self.torch.frombuffer(bytearray(bytes(st)), dtype=self.torch.uint8)
        self.state_dev.copy_(host)

    def read_state(self) -> N.IterState:
        raw = bytes(self.state_dev.cpu().numpy().tobytes())
        return N.IterState.from_buffer_copy(raw)

    def set_exact(self, exact, t: Optional[float] = None) -> None:
        """Exact solution u^e for the exact-solution stopping rule
        (PAPER.md:1303-1306), evaluated at the Gauss points of every local
        element: ``exact(x)`` or ``exact(x, t)`` -> (n,) for the problem's
        primary component or (n, m) for all components."""
        torch, sp, ops = self.torch, self.spec, self.ops
        d = self.mesh.dim
        pts = self._local_points(ops.quad_points).reshape(-1, d)
        vals = np.asarray(exact(pts) if t is None else exact(pts, t), dtype=float)
        nqd = ops.quad_points.size ** d
        ue = np.zeros((self.nloc, sp.ncomp, nqd))
        w = np.zeros(4)
        if vals.ndim == 1:
            c = sp.forcing_comp
            ue[:, c, :] = vals.reshape(self.nloc, nqd)
            w[c] = 1.0
        else:
            ue[:] = vals.reshape(self.nloc, nqd, sp.ncomp).transpose(0, 2, 1)
            w[: sp.ncomp] = 1.0
        self.ue_q = torch.as_tensor(ue, dtype=torch.float64, device=self.device).contiguous()
        self._err_w = w
        if getattr(self, "_vq", None) is None:
            self._vq = torch.as_tensor(ops.interp, dtype=torch.float64, device=self.device).contiguous()
            self._wq = torch.as_tensor(ops.quad_weights, dtype=torch.float64, device=self.device).contiguous()
            self.err_partials = torch.zeros(int(self.L.ihdg_error_tile_count(C.byref(self.geom))),
                                            dtype=torch.float64, device=self.device)
            self.err_hist = torch.zeros(self.max_iters, dtype=torch.float64, device=self.device)

    def set_reference(self, ref) -> None:
        """Reference field of the vs-direct stopping rule: a
        direct HDG solution (FieldState data (Nel, m, Np) of the local strip),
        interpolated to the Gauss points; the rule is ||u^k - u_ref||_{L2} < tol
        over all components."""
        torch, sp, ops = self.torch, self.spec, self.ops
        d = self.mesh.dim
        r = np.asarray(ref, dtype=np.float64).reshape(self.nloc, sp.ncomp, self.np_)
        vq = np.asarray(ops.interp, dtype=np.float64)          # (nq, N1)
        phi = vq
        for _ in range(d - 1):
            phi = np.kron(vq, phi)                               # (nq^d, Np), axis 0 fastest
        ue = r @ phi.T                                           # (nloc, m, nq^d)
        self.ue_q = torch.as_tensor(np.ascontiguousarray(ue), dtype=torch.float64, device=self.device)
        self._err_w = np.zeros(4)
        self._err_w[: sp.ncomp] = 1.0
        if getattr(self, "_vq", None) is None:
            self._vq = torch.as_tensor(ops.interp, dtype=torch.float64, device=self.device).contiguous()
            self._wq = torch.as_tensor(ops.quad_weights, dtype=torch.float64, device=self.device).contiguous()
            self.err_partials = torch.zeros(int(self.L.ihdg_error_tile_count(C.byref(self.geom))),
                                            dtype=torch.float64, device=self.device)
            self.err_hist = torch.zeros(self.max_iters, dtype=torch.float64, device=self.device)

    def _error_args(self, mode: int) -> N.ErrorArgs:
        e = N.ErrorArgs()
        e.g = self.geom
        e.u, e.ue_q, e.vq, e.wq = _ptr(self.u[self.cur]), _ptr(self.ue_q), _ptr(self._vq), _ptr(self._wq)
        e.err_partials, e.succ_partials, e.n_succ = _ptr(self.err_partials), _ptr(self.partials), self.ntiles
        e.state, e.norm_hist, e.err_hist = _ptr(self.state_dev), _ptr(self.norm_hist), _ptr(self.err_hist)
        for c in range(4):
            e.comp_w[c] = float(self._err_w[c])
        e.jac, e.nq, e.mode = self.spec.jac, self.ops.quad_points.size, mode
        return e

    def iterate(self, tol: float = 1e-10, max_iters: int = 10000, norm: str = "volume",
                batch: int = 16) -> IterResult:
        """Algorithm 1 from the current iterate until the
        stopping rule holds; the latest iterate becomes current.  norm
        "volume" / "trace" (successive) or "exact" (set_exact first)."""
        if norm in ("exact", "vs-direct"):
            return self._iterate_exact(tol, max_iters, batch, mode=2 if norm == "vs-direct" else 1)
        self.reset_state(tol, max_iters)
        a = self.sweep_args(norm, finalize=1)
        out = N.IterState()
        nl = C.c_int64(0)
        b0, b1 = self.u[self.cur], self.u[1 - self.cur]
        a.u_old, a.u_new = _ptr(b0), _ptr(b1)
        kernel = N.sweep_kernel(a)
        t0 = time.perf_counter()
        N.check(self.L.ihdg_iterate(C.byref(a), _ptr(b0), _ptr(b1), int(batch), self._sptr,
                                    C.byref(out), C.byref(nl)), "ihdg_iterate")
        sec = time.perf_counter() - t0
        self.cur = (self.cur + out.iters) % 2
        it = out.iters
        norms = self.norm_hist[:it].cpu().numpy().copy()
        return IterResult(it, N.STATUS_NAMES[out.status], norms, out.first_norm, out.last_norm,
                          int(nl.value), sec, kernel=kernel)

    def _iterate_exact(self, tol, max_iters, batch, mode: int = 1) -> IterResult:
        if getattr(self, "ue_q", None) is None:
            raise RuntimeError("exact-solution / vs-direct rule: call set_exact() / set_reference() first")
        if self.layers != (0, self.mesh.cells[self.mesh.dim - 1]):
            raise NotImplementedError("exact-solution rule on a partitioned mesh")
        self.reset_state(tol, max_iters)
        N.check(self.L.ihdg_error_norm(C.byref(self._error_args(0)), self._sptr), "ihdg_error_norm")
        a = self.sweep_args("volume", finalize=0)
        e = self._error_args(mode)
        out = N.IterState()
        nl = C.c_int64(0)
        b0, b1 = self.u[self.cur], self.u[1 - self.cur]
        a.u_old, a.u_new = _ptr(b0), _ptr(b1)
        kernel = N.sweep_kernel(a)
        t0 = time.perf_counter()
        N.check(self.L.ihdg_iterate_exact(C.byref(a), C.byref(e), _ptr(b0), _ptr(b1), int(batch), self._sptr,
                                          C.byref(out), C.byref(nl)), "ihdg_iterate_exact")
        sec = time.perf_counter() - t0
        self.cur = (self.cur + out.iters) % 2
        it = out.iters
        norms = self.norm_hist[:it].cpu().numpy().copy()
        errs = self.err_hist[:it].cpu().numpy().copy()
        return IterResult(it, N.STATUS_NAMES[out.status], norms, out.first_norm, out.last_norm,
                          int(nl.value), sec, errs, kernel=kernel)

    def sweep_once(self, norm: str = "volume", finalize: int = 1, a: Optional[N.SweepArgs] = None):
        """One sweep from the current iterate (used by the bench and multi-rank driver)."""
        if a is None:
            a = self.sweep_args(norm, finalize)
        a.u_old, a.u_new = _ptr(self.u[self.cur]), _ptr(self.u[1 - self.cur])
        N.check(self.L.ihdg_sweep(C.byref(a), self._sptr), "ihdg_sweep")
        self.cur = 1 - self.cur

    # -- output ------------------------------------------------------------
    def _whole_mesh(self, what: str) -> None:
        if self.layers != (0, self.mesh.cells[self.mesh.dim - 1]):
            raise NotImplementedError(f"{what} of a partitioned mesh: gather the state first")

    @property
    def primary_comp(self) -> int:
        """Component carrying the single-valued trace (phi for shallow water, u otherwise)."""
        labels = self.spec.labels
        return labels.index("phi") if "phi" in labels else labels.index("u")

    def trace_of(self, buf=None, jump: bool = False, weights=None):
        """Face array (n_faces, N_f) on the device, mesh.py face order, of the
        ghost-padded state ``buf`` (default: the current iterate).  jump=False:
        the single-valued trace; jump=True: u^- - u^+ of the primary component on
        interior faces (0 on boundary faces)."""
        self._whole_mesh("trace")
        sp = self.spec
        nf = sp.n1 ** (self.mesh.dim - 1)
        out = self.torch.zeros((self.mesh.n_faces, nf), dtype=self.torch.float64, device=self.device)
        a = N.TraceArgs()
        a.g = self.geom
        a.u, a.trace = _ptr(self.u[self.cur] if buf is None else buf), _ptr(out)
        pc = self.primary_comp
        for ax in range(3):
            for c in range(4):
                if weights is not None:      # explicit face-side weights (int_own, int_nbr, lo, hi)
                    a.w_int_own[ax][c] = float(weights["int_own"][ax, c])
                    a.w_int_nbr[ax][c] = float(weights["int_nbr"][ax, c])
                    a.w_lo[ax][c] = float(weights["lo"][ax, c])
                    a.w_hi[ax][c] = float(weights["hi"][ax, c])
                elif jump:
                    a.w_int_own[ax][c] = 1.0 if c == pc else 0.0
                    a.w_int_nbr[ax][c] = -1.0 if c == pc else 0.0
                    a.w_lo[ax][c] = a.w_hi[ax][c] = 0.0
                else:
                    a.w_int_own[ax][c] = float(sp.trace_w["int_own"][ax, c])
                    a.w_int_nbr[ax][c] = float(sp.trace_w["int_nbr"][ax, c])
                    a.w_lo[ax][c] = float(sp.trace_w["lo"][ax, c])
                    a.w_hi[ax][c] = float(sp.trace_w["hi"][ax, c])
        N.check(self.L.ihdg_extract_trace(C.byref(a), self._sptr), "ihdg_extract_trace")
        return out

    def _face_ids(self, elems, f) -> np.ndarray:
        """mesh.py face id (mesh.py:89-125) of local face f of the given elements."""
        d, cells = self.mesh.dim, self.mesh.cells
        e = np.asarray(elems, dtype=np.int64) + self.layers[0] * self.ls
        idx = [(e // int(np.prod(cells[:b]))) % cells[b] for b in range(d)]
        a, side = divmod(f, 2)
        off = 0
        for b in range(a):
            off += (cells[b] + (0 if self.mesh.periodic[b] else 1)) * int(np.prod([cells[c] for c in range(d) if c != b]))
        ntan = int(np.prod([cells[c] for c in range(d) if c != a]))
        tl, mul = np.zeros_like(e), 1
        for b in range(d):
            if b != a:
                tl += idx[b] * mul
                mul *= cells[b]
        return off + (idx[a] + side) * ntan + tl

    def trace(self) -> np.ndarray:
        """Single-valued trace (n_faces, 1, N_f) in mesh.py face order; on
        inflow boundary faces with data it is g at the face nodes."""
        if self.spec.per_element:
            raise NotImplementedError("the single-valued trace of per-element (variable-coefficient) operators "
                                      "varies along the face weights; not extracted on the device")
        t = self.trace_of()
        for f, (on, vals) in (getattr(self, "_bdata_faces", None) or {}).items():
            t[self.torch.as_tensor(self._face_ids(on, f), device=self.device)] = self.torch.as_tensor(
                vals, dtype=self.torch.float64, device=self.device)
        return t.cpu().numpy().reshape(self.mesh.n_faces, 1, t.shape[1])

    # -- diagnostics (K6) ---------------------
    def padded_copy(self, data=None):
        """Ghost-padded device copy of the current iterate, or of a host
        FieldState array (Nel, m, Np) / (Nel, nv)."""
        if data is None:
            return self.u[self.cur].clone()
        out = self.torch.zeros_like(self.u[0])
        arr = np.ascontiguousarray(np.asarray(data, dtype=np.float64).reshape(self.nloc, self.nv))
        out[self.ls: self.ls + self.nloc].copy_(self.torch.from_numpy(arr))
        return out

    def element_errors(self, ref, tol: float, buf=None):
        """Per-element ||u_K - r_K||^2_{L2(K)} (all components, the successive
        norm's weights) and the converged flags (< tol) on the device;
        returns (err2, flags, total)."""
        torch = self.torch
        if getattr(self, "_diag_err2", None) is None:
            self._diag_err2 = torch.zeros(self.nloc, dtype=torch.float64, device=self.device)
            self._diag_flags = torch.zeros(self.nloc, dtype=torch.uint8, device=self.device)
            self._diag_tot = torch.zeros(2, dtype=torch.float64, device=self.device)
        a = N.ElemErrorArgs()
        a.g = self.geom
        a.u = _ptr(self.u[self.cur] if buf is None else buf)
        a.r, a.chol1d = _ptr(ref), _ptr(self.chol)
        a.err2, a.flags, a.total = _ptr(self._diag_err2), _ptr(self._diag_flags), _ptr(self._diag_tot)
        for c in range(4):
            a.comp_w[c] = float(self.spec.comp_w[c])
        a.jac, a.tol = self.spec.jac, float(tol)
        N.check(self.L.ihdg_elem_error(C.byref(a), self._sptr), "ihdg_elem_error")
        return self._diag_err2, self._diag_flags, float(self._diag_tot[0].item())

    def energy_sides(self) -> list:
        """Face-side extraction weights of the skeleton energy of the theorems
        (PAPER.md ThmConvergenceShallowWater / ThmUpwindDDM):
        ||(phi, theta.n)||^2_{E_h} with the Phi weight on theta.n (shallow
        water), ||(sigma.n, u)||^2_{E_h} (convection-diffusion), ||u||^2_{E_h}
        (transport).  Every element's own face values over its whole boundary:
        one weight set for the owner side and one for the neighbour side of
        every face."""
        d, labels = self.mesh.dim, self.spec.labels
        fields = []   # (component per axis, weight)
        if "phi" in labels:
            fields.append(([0] * d, 1.0))
            fields.append(([1 + a for a in range(d)], float(np.sqrt(self.problem.Phi))))
        elif len(labels) > 1:   # convection-diffusion: sigma_a on axis-a faces, u
            fields.append(([labels.index("u")] * d, 1.0))
            fields.append(([a for a in range(d)], 1.0))
        else:
            fields.append(([0] * d, 1.0))
        out = []
        for comps, w in fields:
            own = {k: np.zeros((3, 4)) for k in ("int_own", "int_nbr", "lo", "hi")}
            nbr = {k: np.zeros((3, 4)) for k in ("int_own", "int_nbr", "lo", "hi")}
            for ax in range(d):
                c = comps[ax]
                own["int_own"][ax, c] = own["lo"][ax, c] = own["hi"][ax, c] = w
                nbr["int_nbr"][ax, c] = w
            out += [own, nbr]
        return out

    def skeleton_energy(self, ref_traces, buf=None) -> float:
        """sum over the energy_sides() of ||t(u) - t(r)||^2_{L2(E_h)} (K6);
        ref_traces = [trace_of(r, weights=w) for w in energy_sides()]."""
        return sum(self.face_energy(self.trace_of(buf, weights=w), tr)
                   for w, tr in zip(self.energy_sides(), ref_traces))

    def face_energy(self, t, t_ref=None) -> float:
        """sum_f ||t_f - t_ref_f||^2_{L2(f)} over the skeleton (face arrays from trace_of)."""
        torch = self.torch
        if getattr(self, "_diag_e2", None) is None:
            self._diag_e2 = torch.zeros(self.mesh.n_faces, dtype=torch.float64, device=self.device)
            self._diag_etot = torch.zeros(2, dtype=torch.float64, device=self.device)
        a = N.FaceEnergyArgs()
        a.g = self.geom
        a.t, a.t_ref = _ptr(t), (_ptr(t_ref) if t_ref is not None else None)
        a.chol1d, a.e2, a.total = _ptr(self.chol), _ptr(self._diag_e2), _ptr(self._diag_etot)
        for i in range(3):
            a.jac_face[i] = float(self.spec.jac_face[i])
        N.check(self.L.ihdg_face_energy(C.byref(a), self._sptr), "ihdg_face_energy")
        return float(self._diag_etot[0].item())


class DistributedSweeper:
    """Strip-partitioned iHDG-II over torch.distributed ranks (one GPU each).

    Per sweep:
      - halo: the face-node entries of the first / last local layer that the
        neighbouring ranks read (partition.halo_entries) are packed on the
        device, exchanged with NCCL send/recv (NVLink), and unpacked into the
        ghost layers;
      - the sweep kernel, finalize off.  With ``overlap`` the interior layers
        (which read no ghost) are launched first and the halo runs on a side
        stream meanwhile (local solves overlap the
        communication); the two boundary layers follow it as one-layer strips;
      - the layer sums of the tile partials (ihdg_layer_sums) are written into
        this rank's slice of a zeroed global array and all-reduced (one
        non-zero term per layer, so the sum is exact for any strip sizes),
        then every rank applies the fixed-order finalize (ihdg_finalize), so
        every rank derives the same device status and the norms are
        bit-identical to one rank.
    """

    # the split launch of the overlap path costs ~25 us per sweep on B200 (two
    # one-layer strips at ~11 us each; profiles/r02_strip_overhead.txt: +0.6%
    # on the 2048 layers of config 5), about what an exposed packed-halo
    # exchange costs, so it is the default only for strips tall enough to make
    # it a small fraction of the sweep
    OVERLAP_MIN_LAYERS = 512

    def __init__(self, solver: DeviceSolver, rank: int, world: int, group=None,
                 host_staging: bool = False, overlap=None):
        """``host_staging``: exchange halos and layer sums through host memory
        (gloo); used to test this path with several ranks on one GPU.
        ``overlap``: True / False, or None = by strip height (OVERLAP_MIN_LAYERS)."""
        from .partition import halo_entries

        self.sv, self.rank, self.world, self.group = solver, rank, world, group
        self.host_staging = host_staging
        torch = solver.torch
        sv = solver
        d = sv.mesh.dim
        if d < 2:
            raise NotImplementedError("strip partitions are defined for 2D / 3D meshes (layers of the slowest axis)")
        self.nlay = sv.layers[1] - sv.layers[0]
        self.nlay_global = int(sv.mesh.cells[d - 1])
        self.segs = sv.ntiles // self.nlay
        self.layer_sums = torch.zeros(self.nlay_global, dtype=torch.float64, device=sv.device)
        self.periodic_last = bool(sv.mesh.periodic[d - 1])
        if overlap is None:
            overlap = self.nlay >= self.OVERLAP_MIN_LAYERS
        self.overlap = bool(overlap) and self.nlay >= 3
        self.comm_stream = torch.cuda.Stream(sv.device) if self.overlap else None
        self.idx, self.send, self.recv = {}, {}, {}
        for direction in ("to_lower", "to_upper"):
            ent = halo_entries(sv.spec, direction)
            self.idx[direction] = torch.as_tensor(ent, dtype=torch.int32, device=sv.device) if ent else None
            n = max(len(ent), 1)
            self.send[direction] = torch.zeros((sv.ls, n), dtype=torch.float64, device=sv.device)
            self.recv[direction] = torch.zeros((sv.ls, n), dtype=torch.float64, device=sv.device)

    # -- halo ----------------------------------------------------------------
    def _halo_args(self, direction, layer, packed):
        sv = self.sv
        h = N.HaloArgs()
        h.g = sv.geom
        h.buf, h.packed = _ptr(sv.u[sv.cur]), _ptr(packed)
        h.idx, h.n_idx, h.layer = _ptr(self.idx[direction]), int(self.idx[direction].numel()), layer
        return h

    def _exchange(self, stream=None):
        """Ghost layers of the current iterate from the neighbouring ranks.
        My first layer goes to the lower rank (entries "to_lower"), my last to
        the upper rank ("to_upper"); I receive the lower rank's last layer into
        ghost_lo and the upper rank's first layer into ghost_hi."""
        import torch.distributed as dist
        from .partition import halo_plan

        sv = self.sv
        sp = C.c_void_p(stream.cuda_stream) if stream is not None else sv._sptr
        plan = halo_plan(self.rank, self.world, self.periodic_last)
        for _, sdir, _, _ in plan:
            if self.idx[sdir] is not None:
                layer = 1 if sdir == "to_lower" else 2
                N.check(sv.L.ihdg_halo_pack(C.byref(self._halo_args(sdir, layer, self.send[sdir])), sp),
                        "ihdg_halo_pack")
        if self.host_staging:
            (stream or sv.stream).synchronize()
        ops = []
        staged = {}
        for peer, sdir, rdir, _ in plan:
            if self.idx[sdir] is not None:
                t = self.send[sdir].cpu() if self.host_staging else self.send[sdir]
                ops.append(dist.P2POp(dist.isend, t, peer, self.group))
            if self.idx[rdir] is not None:
                t = torch_cpu_zeros_like(self.recv[rdir]) if self.host_staging else self.recv[rdir]
                staged[rdir] = t
                ops.append(dist.P2POp(dist.irecv, t, peer, self.group))
        if ops:
            for req in dist.batch_isend_irecv(ops):
                req.wait()
        for _, _, rdir, layer in plan:
            if self.idx[rdir] is not None:
                if self.host_staging:
                    self.recv[rdir].copy_(staged[rdir])
                N.check(sv.L.ihdg_halo_unpack(C.byref(self._halo_args(rdir, layer, self.recv[rdir])), sp),
                        "ihdg_halo_unpack")

    # -- one sweep -----------------------------------------------------------
    def _sub_args(self, a: N.SweepArgs, l0: int, l1: int) -> N.SweepArgs:
        """Sweep args of local layers [l0, l1) as a strip of its own: the
        buffers shifted by l0 layers, so its ghost rows are the neighbouring
        local layers (or the true ghosts at the strip ends)."""
        sv = self.sv
        b = N.SweepArgs.from_buffer_copy(a)
        b.g.layer_begin, b.g.layer_end = sv.layers[0] + l0, sv.layers[0] + l1
        lsz = sv.ls * sv.nv * 8
        b.u_old, b.u_new = a.u_old + l0 * lsz, a.u_new + l0 * lsz
        b.s = a.s + l0 * lsz
        b.tile_partials = a.tile_partials + l0 * self.segs * 8
        if a.q_store:
            b.q_store = a.q_store + l0 * sv.ls * sv.gram_kc * 8
        b.layer_sums = b.grid_bar = None   # sub-strips run with finalize = 0
        return b

    def sweep(self, a: N.SweepArgs) -> None:
        import torch.distributed as dist

        sv = self.sv
        torch = sv.torch
        a.u_old, a.u_new = _ptr(sv.u[sv.cur]), _ptr(sv.u[1 - sv.cur])
        if self.overlap:
            # interior layers first (no ghost reads), the halo meanwhile
            main = sv.stream
            inner = self._sub_args(a, 1, self.nlay - 1)
            self.comm_stream.wait_stream(main)          # the previous sweep wrote u_old
            N.check(sv.L.ihdg_sweep(C.byref(inner), sv._sptr), "ihdg_sweep (interior)")
            with torch.cuda.stream(self.comm_stream):
                self._exchange(self.comm_stream)
            main.wait_stream(self.comm_stream)
            for l0 in (0, self.nlay - 1):
                b = self._sub_args(a, l0, l0 + 1)
                N.check(sv.L.ihdg_sweep(C.byref(b), sv._sptr), "ihdg_sweep (boundary layer)")
        else:
            self._exchange()
            N.check(sv.L.ihdg_sweep(C.byref(a), sv._sptr), "ihdg_sweep")
        lb = sv.layers[0]
        self.layer_sums.zero_()
        N.check(sv.L.ihdg_layer_sums(_ptr(sv.partials), self.nlay, self.segs,
                                     _ptr(self.layer_sums) + lb * 8, sv._sptr), "ihdg_layer_sums")
        if self.host_staging:
            t = self.layer_sums.cpu()
            dist.all_reduce(t, group=self.group)
            self.layer_sums.copy_(t)
        else:
            dist.all_reduce(self.layer_sums, group=self.group)
        f = N.FinalizeArgs()
        f.tile_partials, f.n_tiles, f.row_len = _ptr(self.layer_sums), self.nlay_global, 1
        f.state, f.norm_hist = _ptr(sv.state_dev), _ptr(sv.norm_hist)
        N.check(sv.L.ihdg_finalize(C.byref(f), sv._sptr), "ihdg_finalize")
        sv.cur = 1 - sv.cur

    def launches_per_sweep(self) -> int:
        """Kernels of this library per sweep: the sweep (3 with overlap),
        halo packs and unpacks, layer sums, finalize (NCCL's own not counted)."""
        from .partition import halo_plan

        n = 3 if self.overlap else 1
        for _, sdir, rdir, _ in halo_plan(self.rank, self.world, self.periodic_last):
            n += (self.idx[sdir] is not None) + (self.idx[rdir] is not None)
        return n + 2

    def begin_step(self) -> None:
        self.sv.begin_step(exchange=self._exchange)

    def iterate(self, tol=1e-10, max_iters=10000, norm="volume", batch=16) -> IterResult:
        sv = self.sv
        sv.reset_state(tol, max_iters)
        a = sv.sweep_args(norm, finalize=0)
        a.u_old, a.u_new = _ptr(sv.u[sv.cur]), _ptr(sv.u[1 - sv.cur])
        kernel = N.sweep_kernel(a)
        start = sv.cur
        launched = 0
        t0 = time.perf_counter()
        while True:
            for _ in range(batch):
                self.sweep(a)
                launched += 1
            st = sv.read_state()
            if st.status != N.RUNNING:
                break
        sec = time.perf_counter() - t0
        sv.cur = (start + st.iters) % 2
        norms = sv.norm_hist[: st.iters].cpu().numpy().copy()
        return IterResult(st.iters, N.STATUS_NAMES[st.status], norms, st.first_norm, st.last_norm,
                          launched, sec, kernel=kernel)
