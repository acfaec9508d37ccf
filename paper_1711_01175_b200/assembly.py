"""Element-local iHDG-II operators as Kronecker term lists (host side of K1).

On an affine axis-aligned element every bilinear form of the substituted
iHDG-II local solvers is a sum of tensor products of 1D reference matrices:

    mass       (phi_j, phi_i)_K            = J  * (M1 x M1 x M1)
    Q_a[i, j]  (phi_j, d_a phi_i)_K        = Jf_a * (M1 .. S1^T(axis a) .. M1)
    face mass  <phi_j, phi_i>_{face (a,s)} = Jf_a * (M1 .. E_s(axis a) .. M1)
    coupling   <q_face, phi_i>_{face (a,s)}= Jf_a * (M1 .. e_s(axis a) .. M1)

with J = prod h/2, Jf_a = J / (h_a/2), S1[i,j] = int l_i l_j', E_s the endpoint
projector and e_s the endpoint column.  This module writes down, per PDE,
which coefficient multiplies which tensor product (the physics); the device
kernel K1 (``ihdg_assemble``) evaluates the entries, inverts A and forms
L = A^-1 B, P = A^-1 R.

Derivations (n = owner outward normal of face f = (a, s), sgn = +-1):

transport
    A = -sum_a beta_a Q_a + sum_{beta.n>0} (beta.n) Mf [+ (c + 1/dt) M]
    B_f = |beta.n| Bf on inflow faces; neighbour scalar q = u^k_nbr.

convection-diffusion, unknowns (sigma, u),
    u_hat = (q_own + q_nbr)/alpha,  q_X = sigma_X.n_X + (alpha + beta.n_X)/2 u_X
    alpha = sqrt((beta.n)^2 + 4), tau = (alpha - beta.n)/2, c+ = (alpha+beta.n)/2
    interior face:  (s_a,s_a) += Mf/alpha        (s_a,u) += sgn c+/alpha Mf
                    (u,s_a)  += sgn(1-tau/alpha) Mf
                    (u,u)    += (beta.n + tau - tau c+/alpha) Mf
                    B: s_a row -sgn/alpha Bf, u row tau/alpha Bf
    Dirichlet face (u_hat = g_D = 0): (u,s_a) += sgn Mf, (u,u) += (beta.n+tau) Mf
    neighbour scalar q = -sgn sigma_a,nbr + tau u_nbr.

shallow water, unknowns (phi, u, v),
    phi_hat = (q_own + q_nbr)/2, q_X = phi_X + sqrt(Phi) theta_X.n_X
    interior face:  (phi,phi) += sqrt(Phi)/2 Mf   (phi,th_a) += Phi sgn/2 Mf
                    (th_a,phi) += Phi sgn/2 Mf    (th_a,th_a) += Phi sqrt(Phi)/2 Mf
                    B: phi row sqrt(Phi)/2 Bf, th_a row -Phi sgn/2 Bf
    wall face (mirror state): phi_hat = phi + sqrt(Phi) theta.n
                    (th_a,phi) += Phi sgn Mf      (th_a,th_a) += Phi sqrt(Phi) Mf
    Coriolis f and friction gamma implicit.

iHDG-I (scheme="iHDG-I"): the trace is
the all-iterate-k u_hat^k, so the own part of every u_hat term leaves A and
enters the RHS at iterate k.  The element's own face scalar has the same
form as the neighbour's (q_own above), so face f couples through ONE scalar
per face node, q_f = q_nbr + q_own (own_w = the q_own weights), with the same
B column as iHDG-II:
    transport: outflow faces A (beta.n) -> 2 beta.n, B_f = beta.n Bf, q = u_own
    CD interior: A loses the 1/alpha terms: (s_a,s_a) 0, (s_a,u) 0,
                 (u,s_a) sgn, (u,u) beta.n + tau;  Dirichlet faces unchanged
    SW interior: (phi,phi) sqrt(Phi), (phi,th_a) Phi sgn, (th_a, .) 0
       wall:     (phi,phi) sqrt(Phi), (phi,th_a) Phi sgn,
                 B: phi row sqrt(Phi) Bf, th_a row -Phi sgn Bf  (q = q_own)
"""

from __future__ import annotations

from dataclasses import dataclass, field
from typing import Optional

import numpy as np

from .basis import ElementOperators
from .pde import ConvectionDiffusionProblem, ShallowWaterProblem, TransportProblem, stabilization

__all__ = ["OperatorSpec", "build_spec", "OPS"]

# 1D operator table indices
MASS, CONV, CONVT, E0, E1, C0, C1 = range(7)
OPS = {"mass": MASS, "conv": CONV, "convT": CONVT, "E0": E0, "E1": E1, "c0": C0, "c1": C1}
A_T, B_T, R_T = 0, 1, 2


@dataclass
class OperatorSpec:
    """Everything the device needs to assemble and sweep one problem."""

    dim: int
    order: int
    ncomp: int
    labels: tuple
    n_class: int
    class_masks: list           # boundary mask of each class
    class_of_mask: np.ndarray   # (64,) int32
    ops1d: np.ndarray           # (7, N1, N1)
    op_ncols: np.ndarray        # (7,) int32
    terms: np.ndarray           # (nt, 8) int32
    coefs: np.ndarray           # (nt,)
    nr: int                     # R columns
    time_comp0: int             # first component with a time derivative
    n_time_comp: int
    forcing_comp: int           # component row receiving (f, v)
    face_w: np.ndarray          # (6, 4)
    coupled: np.ndarray         # (6,) int32
    out_face: np.ndarray        # (6,) int32 (trace norm faces)
    out_w: np.ndarray           # (6, 4)
    own_w: np.ndarray           # (6, 4) iHDG-I own face-scalar weights (0 for iHDG-II)
    comp_w: np.ndarray          # (4,)
    trace_w: dict               # int_own, int_nbr, lo, hi : (3, 4)
    jac: float
    jac_face: np.ndarray        # (3,)
    periodic: tuple
    boundary_rhs: list = field(default_factory=list)
    scheme: str = "iHDG-II"
    time_scheme: str = "BE"
    terms_expl: Optional[np.ndarray] = None   # CN: A terms + (1 - theta) B terms (L_expl)
    coefs_expl: Optional[np.ndarray] = None
    terms_dir: Optional[np.ndarray] = None    # CD Dirichlet data: A terms + B_D terms (L_D = A^-1 B_D)
    coefs_dir: Optional[np.ndarray] = None
    terms_dir_expl: Optional[np.ndarray] = None   # CN: A terms + (1 - theta) B_D terms (old-level data)
    coefs_dir_expl: Optional[np.ndarray] = None
    # per-element operators (variable coefficients, the GEMV mode): class =
    # element, B columns = raw face-node values of raw_comp (kin_blocks per face)
    per_element: bool = False
    kin_blocks: int = 1
    raw_comp: Optional[np.ndarray] = None       # (6, 4) int32

    @property
    def kin_base(self):
        """neighbour face scalars per element (one per face node)"""
        return 2 * self.dim * self.n1 ** (self.dim - 1)

    @property
    def n1(self):
        return self.order + 1

    @property
    def n_nodes(self):
        return self.n1 ** self.dim

    @property
    def nv(self):
        return self.ncomp * self.n_nodes

    @property
    def kin(self):
        return 2 * self.dim * self.n1 ** (self.dim - 1) * max(1, self.kin_blocks)


class _Terms:
    def __init__(self, dim):
        self.dim = dim
        self.rows = []
        self.coefs = []
        self.time = []    # True: a 1/dt mass term (not part of the spatial operator)

    def add(self, cls, target, rc, cb, axis_ops, coef, time=False):
        if coef == 0.0:
            return
        ops = list(axis_ops) + [MASS] * (3 - len(axis_ops))
        self.rows.append([cls, target, rc, cb, ops[0], ops[1], ops[2], 0])
        self.coefs.append(float(coef))
        self.time.append(bool(time or target == R_T))

    def vol(self, cls, target, rc, cb, coef, axis=None, op=None, time=False):
        ops = [MASS] * self.dim
        if axis is not None:
            ops[axis] = op
        self.add(cls, target, rc, cb, ops, coef, time)

    def crank_nicolson(self, theta, time_comp0):
        """Trapezoidal split of the spatial operator S:
        rows of component c get theta_c S on the LHS (and theta_c B for the
        iterate-k couplings) and -(1 - theta_c) S in the explicit operator R,
        whose columns become absolute components.  Returns the term list of
        the explicit couplings (1 - theta_c) B (with the same A) for L_expl."""
        rows, coefs = [], []
        ex_rows, ex_coefs = [], []
        for r, c, t in zip(self.rows, self.coefs, self.time):
            cls, target, rc, cb = r[:4]
            th = theta[rc]
            if target == R_T:
                rows.append([cls, R_T, rc, cb + time_comp0] + r[4:])
                coefs.append(c)
            elif target == A_T and t:
                rows.append(r)
                coefs.append(c)
                ex_rows.append(r)
                ex_coefs.append(c)
            elif target == A_T:
                rows.append(r)
                coefs.append(th * c)
                ex_rows.append(r)
                ex_coefs.append(th * c)
                if th != 1.0:
                    rows.append([cls, R_T, rc, cb] + r[4:])
                    coefs.append(-(1.0 - th) * c)
            else:  # B_T
                rows.append(r)
                coefs.append(th * c)
                if th != 1.0:
                    ex_rows.append(r)
                    ex_coefs.append((1.0 - th) * c)
        self.rows, self.coefs = rows, coefs
        return (np.asarray(ex_rows, dtype=np.int32).reshape(-1, 8), np.asarray(ex_coefs, dtype=float))


def _ops_table(ops: ElementOperators) -> tuple[np.ndarray, np.ndarray]:
    n1 = ops.n1
    T = np.zeros((7, n1, n1))
    T[MASS] = ops.mass1d
    T[CONV] = ops.conv1d
    T[CONVT] = ops.conv1d.T
    T[E0][0, 0] = 1.0
    T[E1][n1 - 1, n1 - 1] = 1.0
    T[C0][0, 0] = 1.0
    T[C1][n1 - 1, 0] = 1.0
    ncols = np.array([n1, n1, n1, n1, n1, 1, 1], dtype=np.int32)
    return T, ncols


def _class_masks(mesh) -> list[int]:
    """Boundary masks (bit 2a+s = face (a,s) on the physical boundary) that occur."""
    per_axis = []
    for a in range(mesh.dim):
        lo, hi = 1 << (2 * a), 1 << (2 * a + 1)
        n = mesh.cells[a]
        if mesh.periodic[a]:
            pats = [0]
        elif n == 1:
            pats = [lo | hi]
        elif n == 2:
            pats = [lo, hi]
        else:
            pats = [0, lo, hi]
        per_axis.append(pats)
    masks = [0]
    for pats in per_axis:
        masks = [m | p for m in masks for p in pats]
    return sorted(set(masks))


SCHEMES = ("iHDG-II", "iHDG-I")


TIME_SCHEMES = ("BE", "CN")


def build_spec(mesh, problem, ops: ElementOperators, dt=None, norm="auto", scheme: str = "iHDG-II",
               time_scheme: str = "BE") -> OperatorSpec:
    if scheme not in SCHEMES:
        raise ValueError(f"unknown scheme {scheme!r}")
    if time_scheme not in TIME_SCHEMES:
        raise ValueError(f"unknown time scheme {time_scheme!r} (BE or CN)")
    if time_scheme == "CN" and dt is None:
        raise ValueError("Crank-Nicolson needs a time step")
    one = scheme == "iHDG-I"
    d = mesh.dim
    if ops.dim != d:
        raise ValueError("ops.dim != mesh.dim")
    if not np.allclose(ops.h, mesh.h, rtol=1e-14, atol=0.0):
        raise ValueError("ops.h does not match mesh.h")
    h = mesh.h
    J = float(np.prod(h / 2.0))
    Jf = np.array([float(np.prod([h[b] / 2.0 for b in range(d) if b != a])) for a in range(d)])
    jac_face = np.zeros(3)
    jac_face[:d] = Jf
    T, ncols = _ops_table(ops)
    terms = _Terms(d)
    face_w = np.zeros((6, 4))
    coupled = np.zeros(6, dtype=np.int32)
    out_face = np.zeros(6, dtype=np.int32)
    out_w = np.zeros((6, 4))
    own_w = np.zeros((6, 4))
    comp_w = np.zeros(4)
    tw = {k: np.zeros((3, 4)) for k in ("int_own", "int_nbr", "lo", "hi")}
    inv_dt = 0.0 if dt is None else 1.0 / float(dt)

    def E(s):
        return E1 if s else E0

    def Cc(s):
        return C1 if s else C0

    if isinstance(problem, TransportProblem):
        beta = problem.beta_const(d)
        if beta is None:
            raise NotImplementedError("device path needs a constant beta (shared operator)")
        m = 1
        masks = [0]
        class_of_mask = np.zeros(64, dtype=np.int32)
        cls = 0
        for a in range(d):
            terms.vol(cls, A_T, 0, 0, -beta[a] * Jf[a], axis=a, op=CONVT)
        terms.vol(cls, A_T, 0, 0, problem.reaction * J)
        terms.vol(cls, A_T, 0, 0, inv_dt * J, time=True)
        for f in range(2 * d):
            a, s = divmod(f, 2)
            sgn = 1.0 if s else -1.0
            bn = beta[a] * sgn
            if bn > 0:
                terms.vol(cls, A_T, 0, 0, (2.0 if one else 1.0) * bn * Jf[a], axis=a, op=E(s))
                out_face[f] = 1
                out_w[f, 0] = 1.0
                if one:
                    terms.vol(cls, B_T, 0, f, bn * Jf[a], axis=a, op=Cc(s))
                    coupled[f] = 1
                    own_w[f, 0] = 1.0
            elif bn < 0:
                terms.vol(cls, B_T, 0, f, -bn * Jf[a], axis=a, op=Cc(s))
                coupled[f] = 1
                face_w[f, 0] = 1.0
        for a in range(d):
            if beta[a] > 0:
                tw["int_own"][a, 0] = 1.0
            elif beta[a] < 0:
                tw["int_nbr"][a, 0] = 1.0
            else:
                tw["int_own"][a, 0] = tw["int_nbr"][a, 0] = 0.5
            tw["lo"][a, 0] = 1.0 if -beta[a] >= 0 else 0.0  # outflow: u_hat = u^-, inflow: g = 0
            tw["hi"][a, 0] = 1.0 if beta[a] >= 0 else 0.0
        if dt is not None:
            terms.vol(cls, R_T, 0, 0, J * inv_dt)
        nr = ops.n_nodes if dt is not None else 0
        tc0, ntc, fcomp = 0, 1, 0
        comp_w[0] = 1.0
        labels = ("u",)   # inflow data g enters s as L q_g (DeviceSolver.set_inflow)
    elif isinstance(problem, ConvectionDiffusionProblem):
        beta = problem.beta_const(d)
        if beta is None:
            return build_spec_variable(mesh, problem, ops, dt, scheme=scheme, time_scheme=time_scheme)
        dterms = _Terms(d) if problem.dirichlet is not None else None
        m = d + 1
        U = d
        masks = _class_masks(mesh)
        class_of_mask = np.zeros(64, dtype=np.int32)
        for ci, mk in enumerate(masks):
            class_of_mask[mk] = ci
        kinv = 1.0 / problem.kappa
        for ci, mk in enumerate(masks):
            for a in range(d):
                terms.vol(ci, A_T, a, a, kinv * J)
                terms.vol(ci, A_T, a, U, -Jf[a], axis=a, op=CONVT)
                terms.vol(ci, A_T, U, a, -Jf[a], axis=a, op=CONVT)
                terms.vol(ci, A_T, U, U, -beta[a] * Jf[a], axis=a, op=CONVT)
            terms.vol(ci, A_T, U, U, problem.nu * J)
            terms.vol(ci, A_T, U, U, inv_dt * J, time=True)
            for f in range(2 * d):
                a, s = divmod(f, 2)
                sgn = 1.0 if s else -1.0
                bn = beta[a] * sgn
                st = stabilization(problem, bn)   # alpha, tau at this face
                alpha, tau = float(st.alpha), float(st.tau)
                cp = 0.5 * (alpha + bn)
                if mk & (1 << f):
                    terms.vol(ci, A_T, U, a, sgn * Jf[a], axis=a, op=E(s))
                    terms.vol(ci, A_T, U, U, (bn + tau) * Jf[a], axis=a, op=E(s))
                    if dterms is not None:
                        # u_hat := g_D: -<g, tau.n> (sigma rows)
                        # and +tau <g, v> (u row) move to the RHS; g lives at
                        # the face nodes, coupled like a neighbour scalar
                        dterms.vol(ci, B_T, a, f, -sgn * Jf[a], axis=a, op=Cc(s))
                        dterms.vol(ci, B_T, U, f, tau * Jf[a], axis=a, op=Cc(s))
                elif one:
                    terms.vol(ci, A_T, U, a, sgn * Jf[a], axis=a, op=E(s))
                    terms.vol(ci, A_T, U, U, (bn + tau) * Jf[a], axis=a, op=E(s))
                    terms.vol(ci, B_T, a, f, -sgn / alpha * Jf[a], axis=a, op=Cc(s))
                    terms.vol(ci, B_T, U, f, tau / alpha * Jf[a], axis=a, op=Cc(s))
                else:
                    terms.vol(ci, A_T, a, a, Jf[a] / alpha, axis=a, op=E(s))
                    terms.vol(ci, A_T, a, U, sgn * cp / alpha * Jf[a], axis=a, op=E(s))
                    terms.vol(ci, A_T, U, a, sgn * (1.0 - tau / alpha) * Jf[a], axis=a, op=E(s))
                    terms.vol(ci, A_T, U, U, (bn + tau - tau * cp / alpha) * Jf[a], axis=a, op=E(s))
                    terms.vol(ci, B_T, a, f, -sgn / alpha * Jf[a], axis=a, op=Cc(s))
                    terms.vol(ci, B_T, U, f, tau / alpha * Jf[a], axis=a, op=Cc(s))
            if dt is not None:
                terms.vol(ci, R_T, U, 0, J * inv_dt)
        for f in range(2 * d):
            a, s = divmod(f, 2)
            sgn = 1.0 if s else -1.0
            bn = beta[a] * sgn
            alpha = np.sqrt(bn * bn + 4.0)
            face_w[f, a] = -sgn
            face_w[f, U] = 0.5 * (alpha - bn)
            coupled[f] = 1
            if one:
                own_w[f, a] = sgn
                own_w[f, U] = 0.5 * (alpha + bn)
        for a in range(d):
            alpha = np.sqrt(beta[a] ** 2 + 4.0)
            tw["int_own"][a, a] = 1.0 / alpha
            tw["int_own"][a, U] = 0.5 * (alpha + beta[a]) / alpha
            tw["int_nbr"][a, a] = -1.0 / alpha
            tw["int_nbr"][a, U] = 0.5 * (alpha - beta[a]) / alpha
        nr = ops.n_nodes if dt is not None else 0
        tc0, ntc, fcomp = U, 1, U
        comp_w[:m] = 1.0
        labels = problem.labels(d)
    elif isinstance(problem, ShallowWaterProblem):
        if d != 2:
            raise ValueError("shallow water is 2D")
        if dt is None:
            raise ValueError("shallow water needs a time step (backward Euler)")
        if problem.beta_cor != 0.0:
            raise NotImplementedError("variable Coriolis parameter (beta_cor != 0) not on the device path")
        if any(t != 0.0 for t in problem.tau):
            raise NotImplementedError("wind stress forcing not on the device path")
        m = 3
        P = float(problem.Phi)
        sP = np.sqrt(P)
        fc = float(problem.f0)
        masks = _class_masks(mesh)
        class_of_mask = np.zeros(64, dtype=np.int32)
        for ci, mk in enumerate(masks):
            class_of_mask[mk] = ci
        for ci, mk in enumerate(masks):
            terms.vol(ci, A_T, 0, 0, J * inv_dt, time=True)
            for a in range(2):
                th = 1 + a
                terms.vol(ci, A_T, 0, th, -P * Jf[a], axis=a, op=CONVT)
                terms.vol(ci, A_T, th, 0, -P * Jf[a], axis=a, op=CONVT)
                terms.vol(ci, A_T, th, th, P * inv_dt * J, time=True)
                terms.vol(ci, A_T, th, th, problem.gamma * P * J)
            terms.vol(ci, A_T, 1, 2, -fc * P * J)
            terms.vol(ci, A_T, 2, 1, fc * P * J)
            for f in range(4):
                a, s = divmod(f, 2)
                sgn = 1.0 if s else -1.0
                th = 1 + a
                if one:
                    terms.vol(ci, A_T, 0, 0, sP * Jf[a], axis=a, op=E(s))
                    terms.vol(ci, A_T, 0, th, P * sgn * Jf[a], axis=a, op=E(s))
                    w = 1.0 if mk & (1 << f) else 0.5   # wall: phi_hat^k = q_own
                    terms.vol(ci, B_T, 0, f, w * sP * Jf[a], axis=a, op=Cc(s))
                    terms.vol(ci, B_T, th, f, -w * P * sgn * Jf[a], axis=a, op=Cc(s))
                elif mk & (1 << f):  # reflective wall
                    terms.vol(ci, A_T, th, 0, P * sgn * Jf[a], axis=a, op=E(s))
                    terms.vol(ci, A_T, th, th, P * sP * Jf[a], axis=a, op=E(s))
                else:
                    terms.vol(ci, A_T, 0, 0, 0.5 * sP * Jf[a], axis=a, op=E(s))
                    terms.vol(ci, A_T, 0, th, 0.5 * P * sgn * Jf[a], axis=a, op=E(s))
                    terms.vol(ci, A_T, th, 0, 0.5 * P * sgn * Jf[a], axis=a, op=E(s))
                    terms.vol(ci, A_T, th, th, 0.5 * P * sP * Jf[a], axis=a, op=E(s))
                    terms.vol(ci, B_T, 0, f, 0.5 * sP * Jf[a], axis=a, op=Cc(s))
                    terms.vol(ci, B_T, th, f, -0.5 * P * sgn * Jf[a], axis=a, op=Cc(s))
            terms.vol(ci, R_T, 0, 0, J * inv_dt)
            terms.vol(ci, R_T, 1, 1, P * J * inv_dt)
            terms.vol(ci, R_T, 2, 2, P * J * inv_dt)
        for f in range(4):
            a, s = divmod(f, 2)
            sgn = 1.0 if s else -1.0
            face_w[f, 0] = 1.0
            face_w[f, 1 + a] = -sP * sgn
            coupled[f] = 1
            if one:
                own_w[f, 0] = 1.0
                own_w[f, 1 + a] = sP * sgn
        for a in range(2):
            tw["int_own"][a, 0] = 0.5
            tw["int_own"][a, 1 + a] = 0.5 * sP
            tw["int_nbr"][a, 0] = 0.5
            tw["int_nbr"][a, 1 + a] = -0.5 * sP
            tw["lo"][a, 0] = 1.0
            tw["lo"][a, 1 + a] = -sP
            tw["hi"][a, 0] = 1.0
            tw["hi"][a, 1 + a] = sP
        nr = 3 * ops.n_nodes
        tc0, ntc, fcomp = 0, 3, 0
        comp_w[:3] = 1.0
        labels = problem.labels(d)
    else:
        raise TypeError(f"unsupported problem type {type(problem).__name__}")

    terms_expl = coefs_expl = None
    theta_rows = None
    if time_scheme == "CN":
        theta_rows = np.ones(m)
        theta_rows[tc0:tc0 + ntc] = 0.5
        # theta = 1/2 on rows with a time derivative, 1 on algebraic rows (sigma)
        theta = np.ones(m)
        theta[tc0:tc0 + ntc] = 0.5
        terms_expl, coefs_expl = terms.crank_nicolson(theta, tc0)
        nr, tc0, ntc = m * ops.n_nodes, 0, m
    terms_dir = coefs_dir = terms_dir_expl = coefs_dir_expl = None
    if isinstance(problem, ConvectionDiffusionProblem) and dterms is not None:
        # the A terms after the (possible) Crank-Nicolson split; the data
        # couplings split like the trace couplings: theta_c B_D on the new
        # level, (1 - theta_c) B_D on the old one
        keep = [i for i, r in enumerate(terms.rows) if r[1] == A_T]
        a_rows = [terms.rows[i] for i in keep]
        a_coefs = [terms.coefs[i] for i in keep]
        th = [1.0 if theta_rows is None else float(theta_rows[r[2]]) for r in dterms.rows]
        terms_dir = np.asarray(a_rows + dterms.rows, dtype=np.int32).reshape(-1, 8)
        coefs_dir = np.asarray(a_coefs + [t * c for t, c in zip(th, dterms.coefs)], dtype=float)
        if theta_rows is not None:
            ex = [(r, (1.0 - t) * c) for r, t, c in zip(dterms.rows, th, dterms.coefs) if t != 1.0]
            terms_dir_expl = np.asarray(a_rows + [r for r, _ in ex], dtype=np.int32).reshape(-1, 8)
            coefs_dir_expl = np.asarray(a_coefs + [c for _, c in ex], dtype=float)
    terms_arr = np.asarray(terms.rows, dtype=np.int32).reshape(-1, 8)
    return OperatorSpec(
        dim=d, order=ops.p, ncomp=m, labels=tuple(labels), n_class=len(masks),
        class_masks=list(masks), class_of_mask=class_of_mask, ops1d=T, op_ncols=ncols,
        terms=terms_arr, coefs=np.asarray(terms.coefs, dtype=float), nr=nr,
        time_comp0=tc0, n_time_comp=ntc, forcing_comp=fcomp, face_w=face_w, coupled=coupled,
        out_face=out_face, out_w=out_w, own_w=own_w, comp_w=comp_w, trace_w=tw, jac=J, jac_face=jac_face,
        periodic=tuple(mesh.periodic), scheme=scheme, time_scheme=time_scheme, terms_expl=terms_expl,
        coefs_expl=coefs_expl, terms_dir=terms_dir, coefs_dir=coefs_dir, terms_dir_expl=terms_dir_expl,
        coefs_dir_expl=coefs_dir_expl)


def evaluate_terms(spec: OperatorSpec, expl: bool = False, which: str = "main"):
    """Host evaluation of the term list -> (A, B, R) per class (expl /
    which="expl": the Crank-Nicolson explicit-coupling list, B = (1 - theta) B;
    which="dir": the Dirichlet-data list, B = B_D).

    Mirror of the first stage of K1 (k_assemble_build), used by the CPU tests
    to check the physics against the oracle without a GPU.  Not on the
    product path.
    """
    d, n1 = spec.dim, spec.n1
    npn, nv, nf, kin = spec.n_nodes, spec.nv, n1 ** (d - 1), spec.kin
    A = np.zeros((spec.n_class, nv, nv))
    B = np.zeros((spec.n_class, nv, kin))
    R = np.zeros((spec.n_class, nv, max(spec.nr, 1)))
    if expl:
        which = "expl"
    rows, coefs = {"main": (spec.terms, spec.coefs), "expl": (spec.terms_expl, spec.coefs_expl),
                   "dir": (spec.terms_dir, spec.coefs_dir),
                   "dir_expl": (spec.terms_dir_expl, spec.coefs_dir_expl)}[which]
    for row, coef in zip(rows, coefs):
        cls, target, rc, cb = (int(x) for x in row[:4])
        mats = []
        for a in range(d):
            op = spec.ops1d[row[4 + a]]
            mats.append(op[:, : spec.op_ncols[row[4 + a]]])
        K = np.ones((1, 1))
        for mtx in mats:
            K = np.kron(mtx, K)
        K = coef * K
        if target == A_T:
            A[cls, rc * npn:(rc + 1) * npn, cb * npn:(cb + 1) * npn] += K
        elif target == B_T:
            B[cls, rc * npn:(rc + 1) * npn, cb * nf:(cb + 1) * nf] += K
        else:
            R[cls, rc * npn:(rc + 1) * npn, cb * npn:(cb + 1) * npn] += K
    return A, B, R


def face_node_indices(dim: int, n1: int, f: int) -> np.ndarray:
    """Volume node index of each node of local face f (tangential axes
    increasing, the smallest fastest: mesh.py:166-187).  Mirrors
    ihdg::face_node_vidx in csrc/ihdg_common.cuh."""
    a, s = divmod(f, 2)
    out = []
    for n in range(n1 ** (dim - 1)):
        v, mul, rem = 0, 1, n
        for b in range(dim):
            if b == a:
                ib = n1 - 1 if s else 0
            else:
                ib = rem % n1
                rem //= n1
            v += ib * mul
            mul *= n1
        out.append(v)
    return np.array(out, dtype=np.int64)


def own_coupling(spec: OperatorSpec, B: np.ndarray, mask: int) -> np.ndarray:
    """(NV x NV) map own iterate-k volume state -> RHS (iHDG-I): sum over faces
    of B[:, face block f] @ (q_own extraction with own_w from the own face f).
    Host mirror of the own-face part of the gather in k_sweep (tests only)."""
    npn, nv, nf = spec.n_nodes, spec.nv, spec.n1 ** (spec.dim - 1)
    out = np.zeros((nv, nv))
    for f in range(2 * spec.dim):
        W = np.zeros((nf, nv))
        idx = face_node_indices(spec.dim, spec.n1, f)
        for c in range(spec.ncomp):
            W[np.arange(nf), c * npn + idx] = spec.own_w[f, c]
        out += B[:, f * nf:(f + 1) * nf] @ W
    return out


def neighbor_coupling(spec: OperatorSpec, B: np.ndarray, f: int) -> np.ndarray:
    """(NV x NV) map neighbour iterate-k volume state -> RHS of face f:
    B[:, face block f] @ (q extraction with face_w from the neighbour's
    opposite face).  Host mirror of the gather in k_sweep (tests only)."""
    npn, nv, nf = spec.n_nodes, spec.nv, spec.n1 ** (spec.dim - 1)
    W = np.zeros((nf, nv))
    idx = face_node_indices(spec.dim, spec.n1, f ^ 1)
    for c in range(spec.ncomp):
        W[np.arange(nf), c * npn + idx] = spec.face_w[f, c]
    return B[:, f * nf:(f + 1) * nf] @ W


def beta_dependence(beta, dim, lo, hi, rng_seed=0) -> list:
    """For a callable velocity beta(x) -> (n, dim): the coordinate each
    component depends on (None = constant), checked on random points.  The
    per-element term lists need every component to vary along at most one
    axis, different from its own (so div beta = 0 and the face coefficients
    of an a-face vary along one tangential axis) -- e.g. the cdr_manufactured
    velocity (1 + z, 1 + x, 1 + y) of PAPER.md:1664-1666."""
    rng = np.random.default_rng(rng_seed)
    lo, hi = np.asarray(lo, float), np.asarray(hi, float)
    x = lo + (hi - lo) * rng.uniform(size=(64, dim))
    b0 = np.asarray(beta(x), float).reshape(64, dim)
    dep = []
    for a in range(dim):
        axes = []
        for c in range(dim):
            y = x.copy()
            y[:, c] = lo[c] + (hi[c] - lo[c]) * rng.uniform(size=64)
            if not np.allclose(np.asarray(beta(y), float).reshape(64, dim)[:, a], b0[:, a], rtol=1e-13, atol=1e-13):
                axes.append(c)
        if len(axes) > 1 or (axes and axes[0] == a):
            raise NotImplementedError(f"beta component {a} depends on axes {axes}: the per-element term lists "
                                      "need each component to vary along one axis other than its own")
        dep.append(axes[0] if axes else None)
    return dep


def build_spec_variable(mesh, problem, ops: ElementOperators, dt=None, scheme: str = "iHDG-II",
                        time_scheme: str = "BE") -> OperatorSpec:
    """Per-element operators of convection-diffusion with a variable velocity
    beta(x) (the GEMV mode; Table 7):
    the same substituted local equations as the constant case
    (ErrorDDMCD + uhatCDR) with beta.n, alpha, tau
    evaluated at the (p+2) Gauss points -- as weighted 1D mass matrices along
    the axis the coefficient varies on.  Every element is its own operator
    class; the neighbour enters through raw face-node values (sigma_a^+ and
    u^+, 2 blocks per face; iHDG-I adds the element's own 2), because the
    trace weights vary along the face."""
    if time_scheme != "BE":
        raise NotImplementedError("per-element operators: steady or backward Euler")
    one = scheme == "iHDG-I"
    d = mesh.dim
    m, U = d + 1, d
    h = mesh.h
    J = float(np.prod(h / 2.0))
    Jf = np.array([float(np.prod([h[b] / 2.0 for b in range(d) if b != a])) for a in range(d)])
    jac_face = np.zeros(3)
    jac_face[:d] = Jf
    T0, nc0 = _ops_table(ops)
    dep = beta_dependence(problem.beta, d, mesh.lo, mesh.hi)
    center = 0.5 * (np.asarray(mesh.lo, float) + np.asarray(mesh.hi, float))
    qx, qw, V = ops.quad_points, ops.quad_weights, ops.interp     # V[q, i] = l_i(x_q)
    extra, cache = [], {}

    def beta_1d(a, b, xs):
        pts = np.tile(center, (len(xs), 1))
        if b is not None:
            pts[:, b] = xs
        return np.asarray(problem.beta(pts), float).reshape(len(xs), d)[:, a]

    def wop(key, wq):
        """1D mass weighted by wq() at the Gauss points: sum_q w_q wq l_i l_j.
        The weights depend on the element only through its index along the
        axis the coefficient varies on (part of the key), so they are
        evaluated on a cache miss only (cells x faces x tags operators, not
        elements x faces x tags evaluations of beta)."""
        if key not in cache:
            cache[key] = len(T0) + len(extra)
            extra.append((V * (qw * wq())[:, None]).T @ V)
        return cache[key]

    BOUND = -1
    nel = mesh.n_elements
    strides = [int(np.prod(mesh.cells[:a])) for a in range(d)]
    terms = _Terms(d)
    dterms = _Terms(d) if problem.dirichlet is not None else None
    blocks = 4 if one else 2
    kinv = 1.0 / problem.kappa
    inv_dt = 0.0 if dt is None else 1.0 / float(dt)

    def E(s):
        return E1 if s else E0

    def Cc(s):
        return C1 if s else C0

    for e in range(nel):
        idx = [(e // strides[a]) % mesh.cells[a] for a in range(d)]

        def xq(b):
            return mesh.lo[b] + (idx[b] + 0.5 * (qx + 1.0)) * h[b]

        for a in range(d):
            terms.vol(e, A_T, a, a, kinv * J)
            terms.vol(e, A_T, a, U, -Jf[a], axis=a, op=CONVT)
            terms.vol(e, A_T, U, a, -Jf[a], axis=a, op=CONVT)
            b = dep[a]
            if b is None:
                terms.vol(e, A_T, U, U, -float(beta_1d(a, None, np.array([0.0]))[0]) * Jf[a], axis=a, op=CONVT)
            else:
                ops_ = [MASS] * d
                ops_[a] = CONVT
                ops_[b] = wop(("beta", a, b, idx[b]), lambda: beta_1d(a, b, xq(b)))
                terms.add(e, A_T, U, U, ops_, -Jf[a])
        terms.vol(e, A_T, U, U, problem.nu * J)
        terms.vol(e, A_T, U, U, inv_dt * J, time=True)
        for f in range(2 * d):
            a, s = divmod(f, 2)
            sgn = 1.0 if s else -1.0
            b = dep[a]
            boundary = (idx[a] == 0 and not s or idx[a] == mesh.cells[a] - 1 and s) and not mesh.periodic[a]

            def coeffs(xs):
                bn = sgn * beta_1d(a, b, xs)
                al = np.sqrt(bn * bn + 4.0)
                tau = 0.5 * (al - bn)
                cp = 0.5 * (al + bn)
                return bn, al, tau, cp

            def face(target, rc, cb, op_a, fn, tag):
                ops_ = [MASS] * d
                ops_[a] = op_a
                if b is None:
                    val = float(fn(*coeffs(np.array([0.0])))[0])
                    (dterms if target == "D" else terms).add(e, B_T if target in ("B", "D") else A_T, rc, cb,
                                                             ops_, val * Jf[a])
                else:
                    ops_[b] = wop((tag, f, b, idx[b]), lambda: fn(*coeffs(xq(b))))
                    (dterms if target == "D" else terms).add(e, B_T if target in ("B", "D") else A_T, rc, cb,
                                                             ops_, Jf[a])

            if boundary:
                terms.add(e, A_T, U, a, [E(s) if c == a else MASS for c in range(d)], sgn * Jf[a])
                face("A", U, U, E(s), lambda bn, al, tau, cp: bn + tau, "A_uu_bnd")
                if dterms is not None:
                    dterms.add(e, B_T, a, f, [Cc(s) if c == a else MASS for c in range(d)], -sgn * Jf[a])
                    face("D", U, f, Cc(s), lambda bn, al, tau, cp: tau, "D_u")
                continue
            cb0 = f * blocks
            if one:
                terms.add(e, A_T, U, a, [E(s) if c == a else MASS for c in range(d)], sgn * Jf[a])
                face("A", U, U, E(s), lambda bn, al, tau, cp: bn + tau, "A1_uu")
            else:
                face("A", a, a, E(s), lambda bn, al, tau, cp: 1.0 / al, "A_ss")
                face("A", a, U, E(s), lambda bn, al, tau, cp: sgn * cp / al, "A_su")
                face("A", U, a, E(s), lambda bn, al, tau, cp: sgn * (1.0 - tau / al), "A_us")
                face("A", U, U, E(s), lambda bn, al, tau, cp: bn + tau - tau * cp / al, "A_uu")
            # neighbour raw values sigma_a^+ (block 0) and u^+ (block 1):
            # q_nbr = -sgn sigma_a^+ + tau u^+, sigma rows -sgn/alpha q, u row tau/alpha q
            face("B", a, cb0 + 0, Cc(s), lambda bn, al, tau, cp: 1.0 / al, "B_s0")
            face("B", a, cb0 + 1, Cc(s), lambda bn, al, tau, cp: -sgn * tau / al, "B_s1")
            face("B", U, cb0 + 0, Cc(s), lambda bn, al, tau, cp: -sgn * tau / al, "B_u0")
            face("B", U, cb0 + 1, Cc(s), lambda bn, al, tau, cp: tau * tau / al, "B_u1")
            if one:
                # iHDG-I: the element's own iterate-k trace part, q_own = sgn sigma_a + cp u
                face("B", a, cb0 + 2, Cc(s), lambda bn, al, tau, cp: -1.0 / al, "B_s2")
                face("B", a, cb0 + 3, Cc(s), lambda bn, al, tau, cp: -sgn * cp / al, "B_s3")
                face("B", U, cb0 + 2, Cc(s), lambda bn, al, tau, cp: sgn * tau / al, "B_u2")
                face("B", U, cb0 + 3, Cc(s), lambda bn, al, tau, cp: tau * cp / al, "B_u3")
        if dt is not None:
            terms.vol(e, R_T, U, 0, J * inv_dt)
    T = np.concatenate([T0, np.asarray(extra).reshape(-1, ops.n1, ops.n1)]) if extra else T0
    ncols = np.concatenate([nc0, np.full(len(extra), ops.n1, dtype=np.int32)]).astype(np.int32)
    raw_comp = np.zeros((6, 4), dtype=np.int32)
    coupled = np.zeros(6, dtype=np.int32)
    for f in range(2 * d):
        raw_comp[f] = [f // 2, U, f // 2, U]
        coupled[f] = 1
    comp_w = np.zeros(4)
    comp_w[:m] = 1.0
    terms_dir = coefs_dir = None
    if dterms is not None:
        keep = [i for i, r in enumerate(terms.rows) if r[1] == A_T]
        terms_dir = np.asarray([terms.rows[i] for i in keep] + dterms.rows, dtype=np.int32).reshape(-1, 8)
        coefs_dir = np.asarray([terms.coefs[i] for i in keep] + dterms.coefs, dtype=float)
    tw = {k: np.zeros((3, 4)) for k in ("int_own", "int_nbr", "lo", "hi")}
    return OperatorSpec(
        dim=d, order=ops.p, ncomp=m, labels=problem.labels(d), n_class=nel,
        class_masks=[], class_of_mask=np.zeros(64, dtype=np.int32), ops1d=T, op_ncols=ncols,
        terms=np.asarray(terms.rows, dtype=np.int32).reshape(-1, 8), coefs=np.asarray(terms.coefs, dtype=float),
        nr=ops.n_nodes if dt is not None else 0, time_comp0=U, n_time_comp=1, forcing_comp=U,
        face_w=np.zeros((6, 4)), coupled=coupled, out_face=np.zeros(6, dtype=np.int32), out_w=np.zeros((6, 4)),
        own_w=np.zeros((6, 4)), comp_w=comp_w, trace_w=tw, jac=J, jac_face=jac_face,
        periodic=tuple(mesh.periodic), scheme=scheme, time_scheme=time_scheme,
        terms_dir=terms_dir, coefs_dir=coefs_dir, per_element=True, kin_blocks=blocks, raw_comp=raw_comp)
