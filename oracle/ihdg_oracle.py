"""CPU ORACLE for the iHDG-II sweep -- TEST INFRASTRUCTURE ONLY.

Only ``tests/``, ``__graft_entry__.smoke()`` and ``bench.py``'s reference /
cpu_baseline legs may import this module, and only as the checker or the
timed reference arm.  The product path (``paper_1711_01175_b200``) never
imports it.

What it restates
----------------
The reference package's hot path (``ihdg.local_solvers`` + ``ihdg.iteration``
+ the Cython map ``ihdg._kernels._sweep_cy``, pkg/setup.py:13-19) has no
source in /root/reference, so this is a restatement of its documented
algorithm, written independently of the product code:

- basis: GLL nodes from the roots of P_p' (Newton-polished),
  Lagrange polynomials by their product formula, (p+2)-point Gauss
  quadrature, element matrices by explicit quadrature on the tensor grid
  (the product uses Kronecker term lists instead);
- local solvers: the local equation with the iHDG-II trace
  substituted, assembled at face quadrature points from the trace formulas
  themselves -- transport PAPER.md:409-420 (transportLocalk1/transportLocale),
  shallow water PAPER.md:714-727 (localSolverDD + phihDD),
  convection-diffusion PAPER.md:1067-1077 (ErrorDDMCD + uhatCDR);
  own iterate-(k+1) terms -> LHS, neighbour iterate-k terms -> RHS
  (SPEC.md:259, 269, 292); Dirichlet u_hat := g_D and inflow u_ext = g
  (SPEC.md:214); mirror walls for SW;
- factor once: scipy LU per operator class, then every
  sweep is one LU solve per element (the `_sweep_cy` role);
- iteration: ping-pong buffers, stopping
  rule ||u^k - u^{k-1}||_{L2} < tol evaluated by quadrature
   or the skeleton trace-update norm,
  divergence at 1e6 x the first norm, count = sweeps executed
  (SPEC.md:391).

Parity pins: golden fixtures generated from the
reference's own mesh.py (tests/golden/make_golden.py), the SPEC.md
known-answer examples, and the paper's Table-2 iteration counts.
"""

from __future__ import annotations

import ctypes
import os
from dataclasses import dataclass, field

import numpy as np
import scipy.linalg as sla
from numpy.polynomial import legendre as npleg

__all__ = ["Basis1D", "OracleProblem", "OracleSolver", "structured_neighbors",
           "load_c_sweep", "gll_nodes_oracle"]

BOUNDARY = -1


# --------------------------------------------------------------------------
# basis
# --------------------------------------------------------------------------

def gll_nodes_oracle(p: int) -> np.ndarray:
    """GLL nodes: +-1 and the roots of P_p' (companion roots, Newton-polished)."""
    if p == 1:
        return np.array([-1.0, 1.0])
    c = np.zeros(p + 1)
    c[p] = 1.0
    dc = npleg.legder(c)
    r = np.sort(np.real(npleg.legroots(dc)))
    d2c = npleg.legder(dc)
    for _ in range(5):
        r = r - npleg.legval(r, dc) / npleg.legval(r, d2c)
    x = np.concatenate([[-1.0], r, [1.0]])
    return 0.5 * (x - x[::-1])


def lagrange_values(nodes: np.ndarray, x: np.ndarray) -> np.ndarray:
    """[q, j] = l_j(x_q) = prod_{m != j} (x_q - x_m) / (x_j - x_m)."""
    n = nodes.size
    out = np.ones((x.size, n))
    for j in range(n):
        for m in range(n):
            if m != j:
                out[:, j] *= (x - nodes[m]) / (nodes[j] - nodes[m])
    return out


def lagrange_derivs(nodes: np.ndarray, x: np.ndarray) -> np.ndarray:
    """[q, j] = l_j'(x_q) by the product rule."""
    n = nodes.size
    out = np.zeros((x.size, n))
    for j in range(n):
        for k in range(n):
            if k == j:
                continue
            term = np.full(x.size, 1.0 / (nodes[j] - nodes[k]))
            for m in range(n):
                if m != j and m != k:
                    term *= (x - nodes[m]) / (nodes[j] - nodes[m])
            out[:, j] += term
    return out


@dataclass
class Basis1D:
    p: int
    nodes: np.ndarray = field(init=False)
    qx: np.ndarray = field(init=False)
    qw: np.ndarray = field(init=False)
    V: np.ndarray = field(init=False)    # l_j at Gauss points
    dV: np.ndarray = field(init=False)   # l_j' at Gauss points

    def __post_init__(self):
        self.nodes = gll_nodes_oracle(self.p)
        self.qx, self.qw = npleg.leggauss(self.p + 2)
        self.V = lagrange_values(self.nodes, self.qx)
        self.dV = lagrange_derivs(self.nodes, self.qx)


def _kron_axes(mats):
    """Tensor product with axis 0 fastest: mats[a] is (rows_a, cols_a)."""
    out = np.ones((1, 1))
    for m in mats:
        out = np.kron(m, out)
    return out


# --------------------------------------------------------------------------
# structured connectivity (mesh.py:43-48, 81-140), index arithmetic
# --------------------------------------------------------------------------

def structured_neighbors(cells, periodic=None):
    """(Nel, 2d) neighbour element per local face slot 2*axis+side, BOUNDARY = -1."""
    cells = list(cells)
    d = len(cells)
    periodic = [False] * d if periodic is None else list(periodic)
    nel = int(np.prod(cells))
    e = np.arange(nel, dtype=np.int64)
    strides = [int(np.prod(cells[:a])) for a in range(d)]
    idx = [(e // strides[a]) % cells[a] for a in range(d)]
    nbr = np.full((nel, 2 * d), BOUNDARY, dtype=np.int64)
    for a in range(d):
        for s, step in ((0, -1), (1, 1)):
            j = idx[a] + step
            if periodic[a]:
                j = j % cells[a]
                ok = np.ones(nel, dtype=bool)
            else:
                ok = (j >= 0) & (j < cells[a])
            nb = e + (j - idx[a]) * strides[a]
            nbr[ok, 2 * a + s] = nb[ok]
    return nbr


# --------------------------------------------------------------------------
# problems
# --------------------------------------------------------------------------

@dataclass
class OracleProblem:
    """kind in {"transport", "cd", "sw"}; constant coefficients."""

    kind: str
    dim: int
    beta: np.ndarray = None
    kappa: float = 1.0
    nu: float = 0.0
    reaction: float = 0.0
    Phi: float = 1.0
    f_cor: float = 0.0
    gamma: float = 0.0
    forcing: object = None     # callable x -> (n,)

    @property
    def m(self):
        return {"transport": 1, "cd": self.dim + 1, "sw": 3}[self.kind]

    @property
    def time_comps(self):
        return {"transport": [0], "cd": [self.dim], "sw": [0, 1, 2]}[self.kind]

    @property
    def forcing_comp(self):
        return {"transport": 0, "cd": self.dim, "sw": 0}[self.kind]


# --------------------------------------------------------------------------
# local operators by quadrature with the trace substituted
# --------------------------------------------------------------------------

class _Element:
    """Reference-element evaluation data for order p in d dims, element size h."""

    def __init__(self, b: Basis1D, d: int, h):
        self.b, self.d = b, d
        self.h = np.asarray(h, dtype=float)
        n1 = b.p + 1
        self.n1, self.np = n1, n1 ** d
        self.J = float(np.prod(self.h / 2))
        # volume quadrature
        self.Phi = _kron_axes([b.V] * d)                       # (nq^d, Np)
        self.W = _kron_axes([b.qw[:, None]] * d)[:, 0] * self.J
        self.dPhi = []
        for a in range(d):
            mats = [b.V] * d
            mats = list(mats)
            mats[a] = b.dV * (2.0 / self.h[a])
            self.dPhi.append(_kron_axes(mats))
        # face quadrature: own basis at the face points of local face f
        self.Pf, self.Wf = [], []
        one = np.ones((1, 1))
        for f in range(2 * d):
            a, s = divmod(f, 2)
            end = lagrange_values(b.nodes, np.array([1.0 if s else -1.0]))  # (1, n1)
            mats = [end if c == a else b.V for c in range(d)]
            self.Pf.append(_kron_axes(mats))
            wmats = [one if c == a else b.qw[:, None] for c in range(d)]
            Jf = float(np.prod([self.h[c] / 2 for c in range(d) if c != a]))
            self.Wf.append(_kron_axes(wmats)[:, 0] * Jf)
        # face-node evaluation (for the returned trace)
        self.Pn = []
        for f in range(2 * d):
            a, s = divmod(f, 2)
            end = lagrange_values(b.nodes, np.array([1.0 if s else -1.0]))
            mats = [end if c == a else lagrange_values(b.nodes, b.nodes) for c in range(d)]
            self.Pn.append(_kron_axes(mats))

    def mass(self):
        return self.Phi.T @ (self.W[:, None] * self.Phi)

    # physical points of an element with lower corner x0 (variable coefficients)
    def _grid(self, x0, per_axis):
        d = self.d
        n = [len(v) for v in per_axis]
        pts = np.zeros((int(np.prod(n)), d))
        idx = np.indices(n[::-1]).reshape(d, -1)[::-1]     # axis 0 fastest
        for a in range(d):
            pts[:, a] = np.asarray(per_axis[a])[idx[a]]
        return pts

    def vol_points(self, x0):
        return self._grid(x0, [x0[a] + 0.5 * self.h[a] * (self.b.qx + 1.0) for a in range(self.d)])

    def face_points(self, x0, f, nodes=False):
        a, s = divmod(f, 2)
        ref = self.b.nodes if nodes else self.b.qx
        axes = [np.array([x0[c] + (self.h[c] if s else 0.0)]) if c == a
                else x0[c] + 0.5 * self.h[c] * (ref + 1.0) for c in range(self.d)]
        return self._grid(x0, axes)

    def Qw(self, a, w):
        """Q with a pointwise weight at the volume quadrature points: (w phi_j, d_a phi_i)_K."""
        return self.dPhi[a].T @ ((self.W * w)[:, None] * self.Phi)

    def Q(self, a):
        """Q[i, j] = (phi_j, d_a phi_i)_K."""
        return self.dPhi[a].T @ (self.W[:, None] * self.Phi)

    def fmass(self, f, L, R):
        """<R_j, L_i>_face for face-point maps L (nq, nl), R (nq, nr)."""
        return L.T @ (self.Wf[f][:, None] * R)


def _blocks(m, npn):
    return [slice(c * npn, (c + 1) * npn) for c in range(m)]


def _beta_at(prob, pts):
    """beta at physical points: constant vector or callable beta(x) -> (n, d)."""
    b = prob.beta
    if callable(b):
        return np.asarray(b(pts), dtype=float).reshape(len(pts), -1)
    return np.broadcast_to(np.asarray(b, dtype=float), (len(pts), len(b)))


def local_operators(prob: OracleProblem, el: _Element, mask: int, dt=None, scheme: str = "II", x0=None):
    """A (own, LHS), N[f] (neighbour iterate-k -> RHS), R (time level -> RHS),
    H_own[f], H_nbr[f] (trace at face NODES as maps of own / neighbour state),
    Own (own iterate-k -> RHS; zero for iHDG-II).

    scheme "II": the trace u_hat^{k,k+1} takes the element's own iterate k+1
    (iHDGtrace).  scheme "I" (iHDG-I, PAPER.md:272-279,
    SPEC.md:249, 295): the all-iterate-k trace u_hat^k, i.e. the own part T
    of every u_hat term moves from the LHS to the RHS at iterate k:
    A_I = A_II - T, Own = -T."""
    d, npn, m = el.d, el.np, prob.m
    nv = m * npn
    sl = _blocks(m, npn)
    M = el.mass()
    A = np.zeros((nv, nv))
    Nf = [np.zeros((nv, nv)) for _ in range(2 * d)]
    Hown = [np.zeros((el.n1 ** (d - 1), nv)) for _ in range(2 * d)]
    Hnbr = [np.zeros((el.n1 ** (d - 1), nv)) for _ in range(2 * d)]
    inv_dt = 0.0 if dt is None else 1.0 / dt
    R = np.zeros((nv, nv))
    T = np.zeros((nv, nv))   # own-iterate part of the u_hat terms in A

    def fl(f):  # opposite face of the neighbour
        return f ^ 1

    if prob.kind == "transport":
        beta = prob.beta
        for a in range(d):
            A -= beta[a] * el.Q(a)
        A += (prob.reaction + inv_dt) * M
        R[:, :] = inv_dt * M
        for f in range(2 * d):
            a, s = divmod(f, 2)
            sgn = 1.0 if s else -1.0
            bn = beta[a] * sgn
            ab = abs(bn)
            P, Pn = el.Pf[f], el.Pf[fl(f)]
            boundary = bool(mask & (1 << f))
            # face term <beta.n u + |beta.n| (u - u_hat), v>, with
            # 2|bn| u_hat = (bn+|bn|) u^- + (|bn|-bn) u^+ (transportLocale)
            if not boundary:
                A += el.fmass(f, P, (bn + ab - 0.5 * (bn + ab)) * P)
                T -= 0.5 * (bn + ab) * el.fmass(f, P, P)
                Nf[f] += 0.5 * (ab - bn) * el.fmass(f, P, Pn)
                if ab > 0:
                    Hown[f] = (bn + ab) / (2 * ab) * el.Pn[f]
                    Hnbr[f] = (ab - bn) / (2 * ab) * el.Pn[fl(f)]
                else:
                    Hown[f] = 0.5 * el.Pn[f]
                    Hnbr[f] = 0.5 * el.Pn[fl(f)]
            elif bn < 0:   # inflow boundary: u_hat = g (= 0): LHS (bn+|bn|) u = 0
                pass
            else:          # outflow boundary: u_hat = u^-
                A += el.fmass(f, P, bn * P)
                T -= bn * el.fmass(f, P, P)
                Hown[f] = el.Pn[f]
    elif prob.kind == "cd":
        # beta constant, or beta(x) (per-element operators, x0 = the element's
        # lower corner): coefficients at the quadrature points
        var = callable(prob.beta)
        U = d
        bq = _beta_at(prob, el.vol_points(x0)) if var else None
        for a in range(d):
            A[sl[a], sl[a]] += M / prob.kappa
            A[sl[a], sl[U]] -= el.Q(a)
            A[sl[U], sl[a]] -= el.Q(a)
            A[sl[U], sl[U]] -= el.Qw(a, bq[:, a]) if var else prob.beta[a] * el.Q(a)
        A[sl[U], sl[U]] += (prob.nu + inv_dt) * M
        R[sl[U], sl[U]] = inv_dt * M
        for f in range(2 * d):
            a, s = divmod(f, 2)
            sgn = 1.0 if s else -1.0
            # beta.n at the face quadrature points (a column of row weights)
            bn = (_beta_at(prob, el.face_points(x0, f))[:, a] * sgn)[:, None] if var else prob.beta[a] * sgn
            alpha = np.sqrt(bn * bn + 4.0)
            tm = 0.5 * (alpha - bn)          # tau^-
            tp = 0.5 * (alpha + bn)          # tau^+ (beta.n^+ = -bn)
            P, Pn = el.Pf[f], el.Pf[fl(f)]
            boundary = bool(mask & (1 << f))
            # u_hat = [s^-.n + s^+.n^+ + bn u^- - bn u^+ + tau^- u^- + tau^+ u^+] / alpha
            Ho = np.zeros((P.shape[0], nv))
            Hn = np.zeros((P.shape[0], nv))
            if not boundary:
                Ho[:, sl[a]] = sgn / alpha * P
                Ho[:, sl[U]] = (bn + tm) / alpha * P
                Hn[:, sl[a]] = -sgn / alpha * Pn
                Hn[:, sl[U]] = (-bn + tp) / alpha * Pn
                # the same formula at the face NODES (returned trace)
                if var:
                    bnn = (_beta_at(prob, el.face_points(x0, f, nodes=True))[:, a] * sgn)[:, None]
                else:
                    bnn = bn
                an = np.sqrt(bnn * bnn + 4.0)
                tmn, tpn = 0.5 * (an - bnn), 0.5 * (an + bnn)
                Hown[f][:, sl[a]] = sgn / an * el.Pn[f]
                Hown[f][:, sl[U]] = (bnn + tmn) / an * el.Pn[f]
                Hnbr[f][:, sl[a]] = -sgn / an * el.Pn[fl(f)]
                Hnbr[f][:, sl[U]] = (-bnn + tpn) / an * el.Pn[fl(f)]
            # sigma_a rows: + <u_hat n_a, w>
            A[sl[a], :] += sgn * el.fmass(f, P, Ho)
            T[sl[a], :] += sgn * el.fmass(f, P, Ho)
            Nf[f][sl[a], :] -= sgn * el.fmass(f, P, Hn)
            # u rows: <bn u + s.n + tau (u - u_hat), v>
            own = np.zeros((P.shape[0], nv))
            own[:, sl[U]] = (bn + tm) * P
            own[:, sl[a]] += sgn * P
            own -= tm * Ho
            A[sl[U], :] += el.fmass(f, P, own)
            T[sl[U], :] -= el.fmass(f, P, tm * Ho)
            Nf[f][sl[U], :] += el.fmass(f, P, tm * Hn)
    elif prob.kind == "sw":
        if d != 2:
            raise ValueError("sw is 2D")
        Phi, sP = prob.Phi, np.sqrt(prob.Phi)
        A[sl[0], sl[0]] += inv_dt * M
        R[sl[0], sl[0]] = inv_dt * M
        for a in range(2):
            th = 1 + a
            A[sl[0], sl[th]] -= Phi * el.Q(a)
            A[sl[th], sl[0]] -= Phi * el.Q(a)
            A[sl[th], sl[th]] += (Phi * inv_dt + prob.gamma * Phi) * M
            R[sl[th], sl[th]] = Phi * inv_dt * M
        A[sl[1], sl[2]] -= prob.f_cor * Phi * M
        A[sl[2], sl[1]] += prob.f_cor * Phi * M
        for f in range(4):
            a, s = divmod(f, 2)
            sgn = 1.0 if s else -1.0
            th = 1 + a
            P, Pn = el.Pf[f], el.Pf[fl(f)]
            boundary = bool(mask & (1 << f))
            Ho = np.zeros((P.shape[0], nv))
            Hn = np.zeros((P.shape[0], nv))
            if not boundary:   # phi_hat = (phi^- + phi^+)/2 + sqrt(Phi)/2 (th^-.n^- + th^+.n^+)
                Ho[:, sl[0]] = 0.5 * P
                Ho[:, sl[th]] = 0.5 * sP * sgn * P
                Hn[:, sl[0]] = 0.5 * Pn
                Hn[:, sl[th]] = -0.5 * sP * sgn * Pn
                Hown[f][:, sl[0]] = 0.5 * el.Pn[f]
                Hown[f][:, sl[th]] = 0.5 * sP * sgn * el.Pn[f]
                Hnbr[f][:, sl[0]] = 0.5 * el.Pn[fl(f)]
                Hnbr[f][:, sl[th]] = -0.5 * sP * sgn * el.Pn[fl(f)]
            else:              # mirror wall: phi^+ = phi^-, th^+.n^+ = th^-.n^-
                Ho[:, sl[0]] = P
                Ho[:, sl[th]] = sP * sgn * P
                Hown[f][:, sl[0]] = el.Pn[f]
                Hown[f][:, sl[th]] = sP * sgn * el.Pn[f]
            # phi rows: <Phi th.n + sqrt(Phi) (phi - phi_hat), phi1>
            own = np.zeros((P.shape[0], nv))
            own[:, sl[th]] = Phi * sgn * P
            own[:, sl[0]] += sP * P
            own -= sP * Ho
            A[sl[0], :] += el.fmass(f, P, own)
            T[sl[0], :] -= sP * el.fmass(f, P, Ho)
            Nf[f][sl[0], :] += sP * el.fmass(f, P, Hn)
            # theta_a rows: <Phi phi_hat n_a, phi2>
            A[sl[th], :] += Phi * sgn * el.fmass(f, P, Ho)
            T[sl[th], :] += Phi * sgn * el.fmass(f, P, Ho)
            Nf[f][sl[th], :] -= Phi * sgn * el.fmass(f, P, Hn)
    else:
        raise ValueError(prob.kind)
    if scheme == "I":
        return A - T, Nf, R, Hown, Hnbr, -T
    if scheme != "II":
        raise ValueError(scheme)
    return A, Nf, R, Hown, Hnbr, np.zeros((nv, nv))


# --------------------------------------------------------------------------
# the C/OpenMP sweep (the `_sweep_cy` role) -- oracle/sweep.c
# --------------------------------------------------------------------------

_C = None


def load_c_sweep():
    """Load oracle/liboracle_sweep.so (built by oracle/Makefile)."""
    global _C
    if _C is not None:
        return _C
    path = os.path.join(os.path.dirname(os.path.abspath(__file__)), "liboracle_sweep.so")
    if not os.path.exists(path):
        raise FileNotFoundError(f"{path} missing: run `make -C oracle`")
    lib = ctypes.CDLL(path)
    P = ctypes.c_void_p
    lib.oracle_sweep.restype = ctypes.c_double
    lib.oracle_sweep.argtypes = [ctypes.c_int64, ctypes.c_int32, ctypes.c_int32, P, P, P, P,
                                 ctypes.c_int32, P, P, P, P, P, P, ctypes.c_int32, P, ctypes.c_int32,
                                 ctypes.c_int32]
    lib.oracle_max_threads.restype = ctypes.c_int32
    _C = lib
    return lib


def _p(a):
    return a.ctypes.data_as(ctypes.c_void_p)


# --------------------------------------------------------------------------
# solver
# --------------------------------------------------------------------------

class OracleSolver:
    """Factor-once local systems + the iHDG-II iteration on the CPU."""

    def __init__(self, prob: OracleProblem, cells, p: int, box=None, periodic=None, dt=None,
                 scheme: str = "II", time_scheme: str = "BE"):
        """time_scheme "BE" (backward Euler) or "CN" (Crank-Nicolson):
        with the spatial operator S = A - R of the local system, theta = 1/2 on
        rows with a time derivative and 1 on algebraic rows (sigma, CD):
            LHS = R + Theta S,   iterate-k couplings Theta N_f (Theta Own),
            RHS = f + (R - (1-Theta) S) u^m + (1-Theta) (sum_f N_f u^m_nbr + Own u^m)."""
        d = prob.dim
        self.prob, self.p, self.dt, self.scheme = prob, p, dt, scheme
        if time_scheme not in ("BE", "CN"):
            raise ValueError(time_scheme)
        if time_scheme == "CN" and dt is None:
            raise ValueError("Crank-Nicolson needs a time step")
        self.time_scheme = time_scheme
        self.cells = [int(c) for c in cells]
        self.periodic = [False] * d if periodic is None else [bool(x) for x in periodic]
        lo = np.zeros(d) if box is None else np.asarray(box[0], float)
        hi = np.ones(d) if box is None else np.asarray(box[1], float)
        self.lo, self.h = lo, (hi - lo) / np.asarray(self.cells, float)
        self.b = Basis1D(p)
        self.el = _Element(self.b, d, self.h)
        self.nel = int(np.prod(self.cells))
        self.nbr = structured_neighbors(self.cells, self.periodic)
        self.mask = np.zeros(self.nel, dtype=np.int64)
        for f in range(2 * d):
            self.mask |= (self.nbr[:, f] == BOUNDARY).astype(np.int64) << f
        m = prob.m
        self.m, self.npn, self.nv = m, self.el.np, m * self.el.np
        self.classes = {}
        self.cls = np.zeros(self.nel, dtype=np.int32)
        masks = sorted(set(self.mask.tolist())) if prob.kind != "transport" else [0]
        # variable coefficients (beta(x), convection-diffusion): one operator
        # per element (the GEMV mode of the device); keys are element ids
        self.per_element = callable(prob.beta)
        if self.per_element and prob.kind != "cd":
            raise NotImplementedError("variable beta: convection-diffusion")
        if self.per_element:
            e = np.arange(self.nel)
            strides = [int(np.prod(self.cells[:a])) for a in range(d)]
            self.x0 = np.stack([self.lo[a] + ((e // strides[a]) % self.cells[a]) * self.h[a] for a in range(d)], 1)
            masks = list(range(self.nel))
        for ci, mk in enumerate(masks):
            if self.per_element:
                A, Nf, R, Ho, Hn, Own = local_operators(prob, self.el, int(self.mask[mk]), dt, scheme, x0=self.x0[mk])
            else:
                A, Nf, R, Ho, Hn, Own = local_operators(prob, self.el, mk if prob.kind != "transport" else 0, dt,
                                                        scheme)
            Nx, Ownx = None, None
            if time_scheme == "CN":
                th = np.ones(prob.m)
                th[prob.time_comps] = 0.5
                th = np.repeat(th, self.el.np)[:, None]
                S = A - R
                A = R + th * S
                R = R - (1.0 - th) * S
                Nx = [(1.0 - th) * x for x in Nf]
                Ownx = (1.0 - th) * Own
                Nf = [th * x for x in Nf]
                Own = th * Own
            lu, piv = sla.lu_factor(A)
            self.classes[mk] = dict(idx=ci, A=A, N=Nf, R=R, lu=lu, piv=piv, Hown=Ho, Hnbr=Hn, Own=Own,
                                    Nx=Nx, Ownx=Ownx)
        if prob.kind == "transport":
            self.cls[:] = 0
            self.class_list = [self.classes[0]]
            # boundary handling for transport uses the per-face masks (inflow u_ext = g = 0)
            _, _, _, Hob, _, _ = local_operators(prob, self.el, (1 << (2 * d)) - 1, dt)
            self._transport_bnd_H = Hob
        elif self.per_element:
            self.class_list = [self.classes[e] for e in masks]
            self.cls = np.arange(self.nel, dtype=np.int32)
        else:
            self.class_list = [self.classes[mk] for mk in masks]
            lut = {mk: i for i, mk in enumerate(masks)}
            self.cls = np.array([lut[x] for x in self.mask.tolist()], dtype=np.int32)
        self.b_static = np.zeros((self.nel, self.nv))
        self.s = np.zeros((self.nel, self.nv))

    # -- inputs ------------------------------------------------------------
    def element_points(self, ref):
        d = self.prob.dim
        e = np.arange(self.nel)
        strides = [int(np.prod(self.cells[:a])) for a in range(d)]
        cols = []
        for a in range(d):
            ia = (e // strides[a]) % self.cells[a]
            orig = self.lo[a] + ia * self.h[a]
            cols.append(orig[:, None] + 0.5 * self.h[a] * (ref[None, :] + 1.0))
        n1 = ref.size
        pts = np.empty((self.nel, n1 ** d, d))
        for a in range(d):
            rep = n1 ** a
            tile = n1 ** (d - 1 - a)
            pts[:, :, a] = np.tile(np.repeat(cols[a], rep, axis=1), (1, tile))
        return pts

    def interpolate(self, f):
        pts = self.element_points(self.b.nodes)
        return np.asarray(f(pts.reshape(-1, self.prob.dim)), float).reshape(self.nel, self.npn)

    def set_forcing(self, f):
        """(f, v)_K by (p+2)^d Gauss quadrature."""
        pts = self.element_points(self.b.qx)
        fq = np.asarray(f(pts.reshape(-1, self.prob.dim)), float).reshape(self.nel, -1)
        bvals = (fq * self.el.W[None, :]) @ self.el.Phi
        c = self.prob.forcing_comp
        self.b_static[:, c * self.npn:(c + 1) * self.npn] = bvals

    def _face_node_ids(self, f):
        """Volume node indices of local face f (tangential axes increasing,
        smallest fastest; mesh.py:166-187)."""
        d, n1 = self.prob.dim, self.p + 1
        a, s = divmod(f, 2)
        grid = np.indices([n1] * d).reshape(d, -1)[::-1]   # grid[b] = index along axis b, axis 0 fastest
        keep = grid[a] == (n1 - 1 if s else 0)
        return np.flatnonzero(keep)

    def set_inflow(self, g, g_old=None):
        """Transport inflow data u_ext = g, taken in the
        trace space: g at the face GLL nodes, interpolated over the face.
        RHS += <(|b.n| - b.n)/2 g_h, v> on every inflow boundary face.
        Crank-Nicolson (theta = 1/2 on the transport row): half of the term at
        the new level g, half at the old level g_old."""
        d = self.prob.dim
        self.b_inflow = np.zeros((self.nel, self.nv))
        self.inflow_nodes = {}
        if g is None:
            return
        if self.time_scheme == "CN":
            if g_old is None:
                raise ValueError("Crank-Nicolson inflow data needs g_old")
            self.time_scheme = "BE"
            try:
                self.set_inflow(g)
                b_new, nodes = self.b_inflow, self.inflow_nodes
                self.set_inflow(g_old)
            finally:
                self.time_scheme = "CN"
            self.b_inflow = 0.5 * (b_new + self.b_inflow)
            self.inflow_nodes = nodes
            return
        pts = self.element_points(self.b.nodes)
        Vf = _kron_axes([self.b.V] * (d - 1)) if d > 1 else np.ones((1, 1))
        for f in range(2 * d):
            a, s = divmod(f, 2)
            bn = self.prob.beta[a] * (1.0 if s else -1.0)
            if bn >= 0 or self.periodic[a]:
                continue
            on = np.flatnonzero(self.nbr[:, f] == BOUNDARY)
            ids = self._face_node_ids(f)
            gv = np.asarray(g(pts[on][:, ids, :].reshape(-1, d)), float).reshape(on.size, -1)
            M = self.el.fmass(f, self.el.Pf[f], Vf)          # (Np, N_f)
            self.b_inflow[on, :self.npn] += 0.5 * (abs(bn) - bn) * gv @ M.T
            self.inflow_nodes[f] = (on, gv)

    def set_dirichlet(self, g, g_old=None):
        """Convection-diffusion Dirichlet data u_hat := g_D on the boundary
        (SPEC.md:214, 269), in the trace space (g at the face GLL nodes):
        the sigma_a rows gain -<g_h, tau.n> = -sgn <g_h, phi>_f and the u row
        +tau <g_h, v>_f, tau = (alpha - beta.n)/2."""
        d = self.prob.dim
        self.b_inflow = np.zeros((self.nel, self.nv))
        self.inflow_nodes = {}
        if g is None:
            return
        if self.prob.kind != "cd":
            raise NotImplementedError("Dirichlet data: convection-diffusion")
        if self.time_scheme == "CN" and g_old is None:
            raise ValueError("Crank-Nicolson Dirichlet data needs g_old")
        pts = self.element_points(self.b.nodes)
        Vf = _kron_axes([self.b.V] * (d - 1)) if d > 1 else np.ones((1, 1))
        U = d
        for f in range(2 * d):
            a, s = divmod(f, 2)
            if self.periodic[a]:
                continue
            sgn = 1.0 if s else -1.0
            on = np.flatnonzero(self.nbr[:, f] == BOUNDARY)
            ids = self._face_node_ids(f)
            gv = np.asarray(g(pts[on][:, ids, :].reshape(-1, d)), float).reshape(on.size, -1)
            M = self.el.fmass(f, self.el.Pf[f], Vf)          # (Np, N_f)
            val = gv @ M.T
            # Crank-Nicolson: the algebraic sigma rows take the new level only,
            # the u row (time derivative) the average of the two levels
            val_u = val
            if self.time_scheme == "CN":
                g0 = np.asarray(g_old(pts[on][:, ids, :].reshape(-1, d)), float).reshape(on.size, -1)
                val_u = 0.5 * (val + g0 @ M.T)
            self.b_inflow[on, a * self.npn:(a + 1) * self.npn] += -sgn * val
            if self.per_element:
                # tau(x) at the face quadrature points of each boundary element
                for i, e in enumerate(on):
                    bq = _beta_at(self.prob, self.el.face_points(self.x0[e], f))[:, a] * sgn
                    tq = 0.5 * (np.sqrt(bq * bq + 4.0) - bq)
                    Mt = self.el.fmass(f, self.el.Pf[f], tq[:, None] * Vf)
                    self.b_inflow[e, U * self.npn:(U + 1) * self.npn] += Mt @ (
                        gv[i] if self.time_scheme != "CN" else 0.5 * (gv[i] + g0[i]))
            else:
                bn = self.prob.beta[a] * sgn
                tau = 0.5 * (np.sqrt(bn * bn + 4.0) - bn)
                self.b_inflow[on, U * self.npn:(U + 1) * self.npn] += tau * val_u
            self.inflow_nodes[f] = (on, gv)

    # -- sweep -------------------------------------------------------------
    def rhs_static(self, u_prev=None):
        rhs = self.b_static.copy()
        if getattr(self, "b_inflow", None) is not None:
            rhs += self.b_inflow
        if u_prev is not None and self.dt is not None:
            d = self.prob.dim
            for ci, C in enumerate(self.class_list):
                sel = np.nonzero(self.cls == ci)[0]
                rhs[sel] += u_prev[sel] @ C["R"].T
                if self.time_scheme == "CN":   # explicit half of the neighbour / own trace terms
                    rhs[sel] += u_prev[sel] @ C["Ownx"].T
                    for f in range(2 * d):
                        nb = self.nbr[sel, f]
                        ok = nb != BOUNDARY
                        if np.any(ok):
                            rhs[sel[ok]] += u_prev[nb[ok]] @ C["Nx"][f].T
        return rhs

    def sweep(self, u_old, rhs):
        """One sweep: u^{k+1}_K = A_K^-1 (rhs_K + sum_f N_f u^k_nbr(f) [+ Own u^k_K, iHDG-I])."""
        d = self.prob.dim
        u_new = np.empty_like(u_old)
        for ci, C in enumerate(self.class_list):
            sel = np.nonzero(self.cls == ci)[0]
            r = rhs[sel].copy()
            if self.scheme == "I":
                r += u_old[sel] @ C["Own"].T
            for f in range(2 * d):
                nb = self.nbr[sel, f]
                ok = nb != BOUNDARY
                if np.any(ok):
                    r[ok] += u_old[nb[ok]] @ C["N"][f].T
            u_new[sel] = sla.lu_solve((C["lu"], C["piv"]), r.T).T
        return u_new

    def set_exact(self, exact, t=None):
        """u^e at the Gauss points for the exact-solution rule:
        exact(x[, t]) -> (n,) (the primary component) or (n, m) (all)."""
        pts = self.element_points(self.b.qx).reshape(-1, self.prob.dim)
        vals = np.asarray(exact(pts) if t is None else exact(pts, t), float)
        nq = self.el.W.size
        self.ue_q = np.zeros((self.nel, self.m, nq))
        self.err_w = np.zeros(self.m)
        if vals.ndim == 1:
            c = self.prob.forcing_comp
            self.ue_q[:, c, :] = vals.reshape(self.nel, nq)
            self.err_w[c] = 1.0
        else:
            self.ue_q[:] = vals.reshape(self.nel, nq, self.m).transpose(0, 2, 1)
            self.err_w[:] = 1.0

    def err_norm(self, u):
        """||u - u^e||_{L2} by quadrature, element sums in order."""
        vals = u.reshape(self.nel, self.m, self.npn) @ self.el.Phi.T - self.ue_q
        per = np.einsum("emq,q,m->e", vals * vals, self.el.W, self.err_w)
        return float(np.sqrt(np.add.accumulate(per)[-1]))

    def vol_norm(self, delta):
        """||delta||_{L2} by quadrature, element sums in lexicographic order."""
        vals = delta.reshape(self.nel, self.m, self.npn) @ self.el.Phi.T  # (nel, m, nq)
        per = np.einsum("emq,q->e", vals * vals, self.el.W)
        return float(np.sqrt(np.add.accumulate(per)[-1]))

    def trace_norm(self, delta):
        """Skeleton L2 norm of the upwind-trace update (transport)."""
        d = self.prob.dim
        beta = self.prob.beta
        tot = np.zeros(self.nel)
        for f in range(2 * d):
            a, s = divmod(f, 2)
            bn = beta[a] * (1.0 if s else -1.0)
            if bn > 0:
                v = delta @ self.el.Pf[f].T
                tot += (v * v) @ self.el.Wf[f]
        return float(np.sqrt(np.add.accumulate(tot)[-1]))

    def run(self, u0=None, tol=1e-10, max_iters=10000, norm="volume", u_prev=None,
            diverge_factor=1e6, keep_history=False, engine="numpy", threads=0, reference=None):
        """Algorithm 1; returns (u, iterations, status, norms).  engine
        "numpy": scipy LU solves + quadrature norms; "c": the C/OpenMP map
        (oracle/sweep.c: the same LU solve per element, norm sum_K delta^T M
        delta) for full-size parity runs (volume rule, iHDG-II, BE/steady).
        norm "vs-direct": stop when ||u^k - reference||_{L2} < tol (
        reference = the direct HDG solution, oracle/reference_hdg.py)."""
        u = np.zeros((self.nel, self.nv)) if u0 is None else np.array(u0, float).reshape(self.nel, self.nv)
        rhs = self.rhs_static(u_prev)
        norms = []
        errs = []
        status = "max-iter"
        first = None
        e_prev = self.err_norm(u) if norm == "exact" else None
        if norm == "vs-direct":
            if reference is None:
                raise ValueError("vs-direct needs the reference (direct HDG) solution")
            reference = np.asarray(reference, float).reshape(self.nel, self.nv)
        hist = [u.copy()] if keep_history else None
        if engine == "c":
            if norm != "volume" or self.scheme != "II" or self.time_scheme != "BE":
                raise NotImplementedError("engine='c': volume rule, iHDG-II, steady / backward Euler")
            if getattr(self, "_cdata", None) is None:
                self._cdata = self.c_sweep_data()
            u = np.ascontiguousarray(u)
            rhs = np.ascontiguousarray(rhs)
            spare = np.empty_like(u)
        for k in range(1, max_iters + 1):
            if engine == "c":
                total = self.c_sweep(self._cdata, u, rhs, spare, threads)
                un, spare = spare, u
                nrm = float(np.sqrt(total))
            else:
                un = self.sweep(u, rhs)
                delta = un - u
                nrm = self.trace_norm(delta) if norm == "trace" else self.vol_norm(delta)
            norms.append(nrm)
            if norm == "exact":
                e = self.err_norm(un)
                errs.append(e)
            elif norm == "vs-direct":
                e = self.vol_norm(un - reference)
                errs.append(e)
            u = un
            if keep_history:
                hist.append(u.copy())
            if first is None:
                first = nrm
            if not np.isfinite(nrm):
                status = "diverged"
                break
            if norm == "exact":
                done = abs(e - e_prev) < tol
                e_prev = e
                if done:
                    status = "converged"
                    break
            elif norm == "vs-direct":
                if e < tol:
                    status = "converged"
                    break
            elif nrm < tol:
                status = "converged"
                break
            if k > 1 and nrm > diverge_factor * first:
                status = "diverged"
                break
        out = dict(u=u, iterations=len(norms), status=status, norms=np.array(norms), errors=np.array(errs))
        if keep_history:
            out["history"] = hist
        return out

    def run_time_dependent(self, u0, nsteps, tol=1e-10, max_iters=10000, norm="volume", exact=None,
                           forcing=None, inflow=None, dirichlet=None, engine="numpy", threads=0):
        """forcing(x, t) / inflow(x, t): time-dependent data, taken at the new
        level (BE) or averaged / split between the levels (CN)."""
        u = np.array(u0, float).reshape(self.nel, self.nv)
        reports = []
        for step in range(nsteps):
            t0, t1 = step * self.dt, (step + 1) * self.dt
            if forcing is not None:
                if self.time_scheme == "CN":
                    self.set_forcing(lambda x: 0.5 * (forcing(x, t0) + forcing(x, t1)))
                else:
                    self.set_forcing(lambda x: forcing(x, t1))
            if inflow is not None:
                self.set_inflow(lambda x: inflow(x, t1), lambda x: inflow(x, t0))
            if dirichlet is not None:
                self.set_dirichlet(lambda x: dirichlet(x, t1), lambda x: dirichlet(x, t0))
            if norm == "exact":
                self.set_exact(exact, (step + 1) * self.dt)
            r = self.run(u0=u, tol=tol, max_iters=max_iters, norm=norm, u_prev=u, engine=engine, threads=threads)
            reports.append(r)
            u = r["u"]
            if r["status"] != "converged":
                break
        return u, reports

    # -- trace -------------------------------------------------------------
    def trace(self, u):
        """Single-valued trace at face nodes, face order of mesh.py:89-125."""
        d = self.prob.dim
        cells = self.cells
        strides = [int(np.prod(cells[:a])) for a in range(d)]
        out = []
        for a in range(d):
            tang = [b for b in range(d) if b != a]
            ntan = int(np.prod([cells[b] for b in tang])) if tang else 1
            planes = cells[a] + (0 if self.periodic[a] else 1)
            tl = np.arange(ntan)
            base = np.zeros(ntan, dtype=np.int64)
            rem = tl.copy()
            for b in tang:
                base += (rem % cells[b]) * strides[b]
                rem //= cells[b]
            for pl in range(planes):
                if self.periodic[a] or 0 < pl < cells[a]:
                    lower = pl - 1 if pl > 0 else cells[a] - 1
                    eo = base + lower * strides[a]
                    en = base + (pl % cells[a]) * strides[a]
                    C = self.class_list[self.cls[eo[0]]]
                    f = 2 * a + 1
                    tr = u[eo] @ C["Hown"][f].T + u[en] @ C["Hnbr"][f].T
                else:
                    if pl == 0:
                        eo, f = base, 2 * a
                    else:
                        eo, f = base + (cells[a] - 1) * strides[a], 2 * a + 1
                    if self.prob.kind == "transport":
                        H = self._transport_bnd_H[f]
                    else:
                        H = self.class_list[self.cls[eo[0]]]["Hown"][f]
                    tr = u[eo] @ H.T
                    data = getattr(self, "inflow_nodes", {}).get(f)
                    if data is not None:   # inflow boundary: u_hat = g
                        pos = {int(e): i for i, e in enumerate(data[0])}
                        tr = tr + np.stack([data[1][pos[int(e)]] for e in eo])
                out.append(tr)
        return np.concatenate(out, axis=0)[:, None, :]

    # -- diagnostics ------------------------
    def elem_errors(self, u, ref):
        """Per-element ||u_K - r_K||^2_{L2(K)} by quadrature, all components."""
        vals = (np.asarray(u) - np.asarray(ref)).reshape(self.nel, self.m, self.npn) @ self.el.Phi.T
        return np.einsum("emq,q->e", vals * vals, self.el.W)

    def face_energy(self, t, t_ref=None):
        """sum_f ||t_f - t_ref_f||^2_{L2(f)} for face-node arrays in mesh.py face
        order (as returned by trace()), by face Gauss quadrature."""
        d = self.prob.dim
        t = np.asarray(t, float).reshape(t.shape[0], -1)
        if t_ref is not None:
            t = t - np.asarray(t_ref, float).reshape(t.shape)
        b = self.b
        Vf = _kron_axes([b.V] * (d - 1)) if d > 1 else np.ones((1, 1))
        wf = _kron_axes([b.qw[:, None]] * (d - 1))[:, 0] if d > 1 else np.ones(1)
        tot, off = 0.0, 0
        for a in range(d):
            ntan = int(np.prod([self.cells[c] for c in range(d) if c != a])) if d > 1 else 1
            nfa = (self.cells[a] + (0 if self.periodic[a] else 1)) * ntan
            Jf = float(np.prod([self.h[c] / 2 for c in range(d) if c != a]))
            v = t[off: off + nfa] @ Vf.T
            tot += Jf * float(np.sum((v * v) @ wf))
            off += nfa
        return tot

    def jump_faces(self, u, comp):
        """u^- - u^+ of component ``comp`` at the face nodes of every face
        (0 on boundary faces), mesh.py face order."""
        d = self.prob.dim
        cells = self.cells
        u = np.asarray(u, float).reshape(self.nel, self.m, self.npn)[:, comp, :]
        strides = [int(np.prod(cells[:a])) for a in range(d)]
        out = []
        for a in range(d):
            tang = [b for b in range(d) if b != a]
            ntan = int(np.prod([cells[b] for b in tang])) if tang else 1
            planes = cells[a] + (0 if self.periodic[a] else 1)
            base = np.zeros(ntan, dtype=np.int64)
            rem = np.arange(ntan)
            for b in tang:
                base += (rem % cells[b]) * strides[b]
                rem //= cells[b]
            Phi_hi, Phi_lo = self.el.Pn[2 * a + 1], self.el.Pn[2 * a]
            for pl in range(planes):
                if self.periodic[a] or 0 < pl < cells[a]:
                    lower = pl - 1 if pl > 0 else cells[a] - 1
                    eo = base + lower * strides[a]
                    en = base + (pl % cells[a]) * strides[a]
                    out.append(u[eo] @ Phi_hi.T - u[en] @ Phi_lo.T)
                else:
                    out.append(np.zeros((ntan, Phi_hi.shape[0])))
        return np.concatenate(out, axis=0)

    def side_faces(self, u, comps, w=1.0):
        """Owner-side and neighbour-side face-node values, mesh.py face order,
        of component comps[a] on the axis-a faces (scaled by w); the
        neighbour side is 0 on boundary faces."""
        d = self.prob.dim
        cells = self.cells
        u = np.asarray(u, float).reshape(self.nel, self.m, self.npn)
        strides = [int(np.prod(cells[:a])) for a in range(d)]
        own, nbr = [], []
        for a in range(d):
            c = comps[a]
            tang = [b for b in range(d) if b != a]
            ntan = int(np.prod([cells[b] for b in tang])) if tang else 1
            planes = cells[a] + (0 if self.periodic[a] else 1)
            base = np.zeros(ntan, dtype=np.int64)
            rem = np.arange(ntan)
            for b in tang:
                base += (rem % cells[b]) * strides[b]
                rem //= cells[b]
            P_hi, P_lo = self.el.Pn[2 * a + 1], self.el.Pn[2 * a]
            for pl in range(planes):
                if self.periodic[a] or 0 < pl < cells[a]:
                    lower = pl - 1 if pl > 0 else cells[a] - 1
                    own.append(w * u[base + lower * strides[a], c] @ P_hi.T)
                    nbr.append(w * u[base + (pl % cells[a]) * strides[a], c] @ P_lo.T)
                elif pl == 0:
                    own.append(w * u[base, c] @ P_lo.T)
                    nbr.append(np.zeros((ntan, P_lo.shape[0])))
                else:
                    own.append(w * u[base + (cells[a] - 1) * strides[a], c] @ P_hi.T)
                    nbr.append(np.zeros((ntan, P_hi.shape[0])))
        return np.concatenate(own, axis=0), np.concatenate(nbr, axis=0)

    def skeleton_energy(self, u):
        """The theorems' skeleton norm squared:
        ||(phi, theta.n)||^2_{E_h} with the Phi weight (SW), ||(sigma.n, u)||^2
        (CD), ||u||^2 (transport), each element's own values over its boundary."""
        d, kind = self.prob.dim, self.prob.kind
        if kind == "sw":
            fields = [([0] * d, 1.0), ([1 + a for a in range(d)], float(np.sqrt(self.prob.Phi)))]
        elif kind == "cd":
            fields = [([d] * d, 1.0), (list(range(d)), 1.0)]
        else:
            fields = [([0] * d, 1.0)]
        tot = 0.0
        for comps, w in fields:
            o, n = self.side_faces(u, comps, w)
            tot += self.face_energy(o) + self.face_energy(n)
        return tot

    def diagnostics(self, hist, ref, tol=1e-10):
        """Per-iteration trace energy, jump norm and converged-element map of
        a run(keep_history=True) history against the reference state."""
        comp = 0 if self.prob.kind != "cd" else self.prob.dim
        energy, jump, maps = [], [], []
        for u in hist[1:]:
            energy.append(self.skeleton_energy(np.asarray(u) - np.asarray(ref)))
            jump.append(np.sqrt(self.face_energy(self.jump_faces(u, comp))))
            maps.append(self.elem_errors(u, ref) < tol * tol)
        return dict(trace_energy=np.array(energy), jump_norm=np.array(jump), maps=maps)

    # -- C sweep (CPU baseline / `_sweep_cy` role) --------------------------
    def c_sweep_data(self):
        """Compressed neighbour blocks + LU factors for oracle/sweep.c."""
        d = self.prob.dim
        nv, npn, n1 = self.nv, self.npn, self.b.p + 1
        nfn = n1 ** (d - 1)
        rows, cols = [], []
        for f in range(2 * d):
            a, s = divmod(f, 2)
            own = [i for i in range(npn) if (i // n1 ** a) % n1 == (n1 - 1 if s else 0)]
            opp = [i for i in range(npn) if (i // n1 ** a) % n1 == (0 if s else n1 - 1)]
            rows.append([c * npn + i for c in range(self.m) for i in own])
            cols.append([c * npn + i for c in range(self.m) for i in opp])
        nr = len(rows[0])
        assert nr == self.m * nfn
        ncls = len(self.class_list)
        blk = np.zeros((ncls, 2 * d, nr, nr))
        for ci, C in enumerate(self.class_list):
            for f in range(2 * d):
                Nf = C["N"][f]
                sub = Nf[np.ix_(rows[f], cols[f])]
                rest = Nf.copy()
                rest[np.ix_(rows[f], cols[f])] = 0.0
                assert np.max(np.abs(rest)) <= 1e-12 * max(1.0, np.max(np.abs(Nf))), "coupling not face-local"
                blk[ci, f] = sub
        LU = np.ascontiguousarray(np.stack([C["lu"] for C in self.class_list]))
        PIV = np.ascontiguousarray(np.stack([C["piv"] for C in self.class_list]).astype(np.int32))
        # mass matrix for the norm (volume rule)
        Mq = np.ascontiguousarray(self.el.mass())
        return dict(rows=np.ascontiguousarray(np.array(rows, dtype=np.int32)),
                    cols=np.ascontiguousarray(np.array(cols, dtype=np.int32)),
                    blk=np.ascontiguousarray(blk), LU=LU, PIV=PIV, nr=nr, mass=Mq)

    def c_sweep(self, data, u_old, rhs, u_new, nthreads=0):
        """One sweep + sum_K delta^T M delta through the C/OpenMP kernel."""
        lib = load_c_sweep()
        d = self.prob.dim
        nbr = np.ascontiguousarray(self.nbr)
        cls = np.ascontiguousarray(self.cls.astype(np.int32))
        return lib.oracle_sweep(self.nel, self.nv, 2 * d, _p(nbr), _p(cls), _p(data["LU"]),
                                _p(data["PIV"]), data["nr"], _p(data["rows"]), _p(data["cols"]),
                                _p(data["blk"]), _p(rhs), _p(u_old), _p(u_new), self.npn,
                                _p(data["mass"]), self.m, nthreads)
