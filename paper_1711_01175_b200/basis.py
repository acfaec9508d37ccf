"""Nodal tensor-product basis.

Host-side setup only: the 1D reference matrices built here are tiny and are
shipped to the device, where K1 (``ihdg_assemble``) evaluates the tensorised
element operators.  Conventions:

- nodes: Gauss-Lobatto-Legendre, p+1 per axis, lexicographic with axis 0
  fastest (mesh.py:155-164);
- quadrature: (p+2)-point Gauss-Legendre for volume and face integrals;
- full (consistent) mass matrices, no lumping.
"""

from __future__ import annotations

from dataclasses import dataclass, field
from functools import cached_property

import numpy as np
from numpy.polynomial.legendre import leggauss

__all__ = [
    "gll_nodes",
    "gauss_rule",
    "lagrange_eval",
    "lagrange_diff",
    "ElementOperators",
    "FieldState",
    "build_operators",
    "project",
    "l2_norm",
    "l2_error",
]

P_MIN, P_MAX = 1, 10


def gll_nodes(p: int) -> tuple[np.ndarray, np.ndarray]:
    """Gauss-Lobatto-Legendre nodes/weights on [-1, 1] (p+1 points).

    Interior nodes are the roots of P_p'; Newton iteration on
    (1 - x^2) P_p'(x) from the Chebyshev-Gauss-Lobatto points.
    """
    n = p + 1
    x = -np.cos(np.pi * np.arange(n) / p)
    for _ in range(100):
        # Legendre recurrence for P_p and P_{p-1}
        P0 = np.ones_like(x)
        P1 = x.copy()
        for k in range(2, p + 1):
            P0, P1 = P1, ((2 * k - 1) * x * P1 - (k - 1) * P0) / k
        if p == 1:
            P0, P1 = np.ones_like(x), x.copy()
        # interior update: x <- x - (x P_p - P_{p-1}) / (n P_p)
        dx = (x * P1 - P0) / (n * P1)
        dx[0] = dx[-1] = 0.0
        x = x - dx
        if np.max(np.abs(dx)) < 1e-16:
            break
    x[0], x[-1] = -1.0, 1.0
    x = 0.5 * (x - x[::-1])  # exact symmetry
    # weights 2 / (p (p+1) P_p(x)^2)
    P0 = np.ones_like(x)
    P1 = x.copy()
    for k in range(2, p + 1):
        P0, P1 = P1, ((2 * k - 1) * x * P1 - (k - 1) * P0) / k
    w = 2.0 / (p * (p + 1) * P1 ** 2)
    return x, w


def gauss_rule(n: int) -> tuple[np.ndarray, np.ndarray]:
    """n-point Gauss-Legendre rule on [-1, 1] (exact to degree 2n-1)."""
    return leggauss(n)


def _bary_weights(nodes: np.ndarray) -> np.ndarray:
    d = nodes[:, None] - nodes[None, :]
    np.fill_diagonal(d, 1.0)
    return 1.0 / np.prod(d, axis=1)


def lagrange_eval(nodes: np.ndarray, x: np.ndarray) -> np.ndarray:
    """V[q, i] = l_i(x_q) for the Lagrange basis on ``nodes`` (barycentric)."""
    nodes = np.asarray(nodes, dtype=float)
    x = np.atleast_1d(np.asarray(x, dtype=float))
    w = _bary_weights(nodes)
    diff = x[:, None] - nodes[None, :]
    exact = diff == 0.0
    with np.errstate(divide="ignore", invalid="ignore"):
        t = w[None, :] / diff
        V = t / np.sum(t, axis=1, keepdims=True)
    rows = np.any(exact, axis=1)
    V[rows] = exact[rows].astype(float)
    return V


def lagrange_diff(nodes: np.ndarray) -> np.ndarray:
    """D[i, j] = l_j'(x_i) (nodal differentiation matrix)."""
    nodes = np.asarray(nodes, dtype=float)
    n = nodes.size
    w = _bary_weights(nodes)
    D = np.zeros((n, n))
    for i in range(n):
        for j in range(n):
            if i != j:
                D[i, j] = (w[j] / w[i]) / (nodes[i] - nodes[j])
        D[i, i] = -np.sum(D[i, :])  # rows annihilate constants
    return D


@dataclass(frozen=True)
class ElementOperators:
    """Per-order basis data.

    ``mass1d``, ``conv1d`` and ``diff1d`` are reference-element ([-1, 1])
    matrices; physical scaling uses ``h`` (affine axis-aligned elements,
    SPEC.md:71).
    """

    p: int
    dim: int
    h: np.ndarray
    nodes: np.ndarray            # GLL nodes (p+1)
    node_weights: np.ndarray     # GLL weights (not used for integration)
    quad_points: np.ndarray      # (p+2) Gauss points
    quad_weights: np.ndarray
    interp: np.ndarray           # V[q, i] = l_i(x_q), (p+2, p+1)
    diff1d: np.ndarray           # D[i, j] = l_j'(x_i)
    mass1d: np.ndarray           # M1[i, j] = int l_i l_j
    conv1d: np.ndarray           # S1[i, j] = int l_i l_j'
    chol1d: np.ndarray = field(repr=False)  # lower C, M1 = C C^T

    @property
    def n1(self) -> int:
        return self.p + 1

    @property
    def n_nodes(self) -> int:
        return self.n1 ** self.dim

    @property
    def n_face_nodes(self) -> int:
        return self.n1 ** (self.dim - 1)

    @property
    def jacobian(self) -> float:
        return float(np.prod(self.h / 2.0))

    def face_jacobian(self, axis: int) -> float:
        return float(np.prod([self.h[b] / 2.0 for b in range(self.dim) if b != axis]))

    @cached_property
    def mass(self) -> np.ndarray:
        """Physical element mass matrix (N_p x N_p), axis 0 fastest."""
        M = np.ones((1, 1))
        for a in range(self.dim):
            M = np.kron(self.mass1d * (self.h[a] / 2.0), M)
        return M

    @cached_property
    def quad_to_rhs(self) -> np.ndarray:
        """Bq[i, q] = w_q l_i(x_q): (f, l_i) = J sum_q Bq[i,q] f_q (per axis)."""
        return (self.interp * self.quad_weights[:, None]).T.copy()

    @cached_property
    def face_maps(self) -> list[np.ndarray]:
        """Volume nodes -> face quadrature points, one (nq^(d-1), N_p) map per face."""
        n1, nq = self.n1, self.quad_points.size
        maps = []
        for f in range(2 * self.dim):
            a, s = divmod(f, 2)
            mats = []
            for b in range(self.dim):
                if b == a:
                    e = np.zeros((1, n1))
                    e[0, n1 - 1 if s else 0] = 1.0
                    mats.append(e)
                else:
                    mats.append(self.interp)
            F = np.ones((1, 1))
            for m in mats:
                F = np.kron(m, F)
            maps.append(F.reshape(-1, n1 ** self.dim))
        return maps


def build_operators(p: int, dim: int, h) -> ElementOperators:
    """Build the order-p operators for ``dim`` dimensions and element size h."""
    if not (P_MIN <= int(p) <= P_MAX):
        raise ValueError(f"order p must be in [{P_MIN}, {P_MAX}], got {p}")
    if dim not in (1, 2, 3):
        raise ValueError(f"dim must be 1, 2 or 3, got {dim}")
    p = int(p)
    h = np.broadcast_to(np.asarray(h, dtype=float), (dim,)).copy()
    nodes, nw = gll_nodes(p)
    qx, qw = gauss_rule(p + 2)
    V = lagrange_eval(nodes, qx)
    D = lagrange_diff(nodes)
    M1 = V.T @ (qw[:, None] * V)
    M1 = 0.5 * (M1 + M1.T)
    S1 = V.T @ (qw[:, None] * (V @ D))
    C = np.linalg.cholesky(M1)
    return ElementOperators(p=p, dim=dim, h=h, nodes=nodes, node_weights=nw,
                            quad_points=qx, quad_weights=qw, interp=V, diff1d=D,
                            mass1d=M1, conv1d=S1, chol1d=C)


@dataclass
class FieldState:
    """Per-element coefficients: data[Nel, m, (p+1)^d]."""

    data: np.ndarray
    labels: tuple = ("u",)
    k: int = 0
    m: int = 0

    @property
    def n_elements(self) -> int:
        return self.data.shape[0]

    @property
    def n_components(self) -> int:
        return self.data.shape[1]

    def component(self, name: str) -> np.ndarray:
        return self.data[:, self.labels.index(name), :]

    def copy(self) -> "FieldState":
        return FieldState(self.data.copy(), tuple(self.labels), self.k, self.m)


def _eval_points(f, pts: np.ndarray, ncomp: int) -> np.ndarray:
    v = np.asarray(f(pts), dtype=float)
    if ncomp == 1:
        return v.reshape(pts.shape[0], 1)
    return v.reshape(pts.shape[0], ncomp)


def project(f, mesh, ops: ElementOperators, ncomp: int = 1, labels=None) -> FieldState:
    """Nodal interpolation at GLL nodes.

    ``f`` maps an (npts, dim) array to (npts,) or (npts, ncomp).
    """
    pts = mesh.all_element_points([ops.nodes] * mesh.dim)  # (Nel, Np, dim)
    nel, npn, dim = pts.shape
    vals = _eval_points(f, pts.reshape(-1, dim), ncomp).reshape(nel, npn, ncomp)
    data = np.ascontiguousarray(np.transpose(vals, (0, 2, 1)))
    if labels is None:
        labels = ("u",) if ncomp == 1 else tuple(f"c{i}" for i in range(ncomp))
    return FieldState(data, tuple(labels))


def _elementwise_sq(data: np.ndarray, ops: ElementOperators) -> np.ndarray:
    """Per-element sum over components of u_c^T M_K u_c."""
    nel, m, npn = data.shape
    n1, d = ops.n1, ops.dim
    x = data.reshape((nel * m,) + (n1,) * d)  # axis order: (..., i_{d-1}, ..., i_0)
    y = x
    for a in range(d):
        ax = d - a  # array axis of reference axis a (axis 0 fastest == last)
        y = np.moveaxis(np.tensordot(y, ops.mass1d, axes=([ax], [1])), -1, ax)
    s = np.sum((x * y).reshape(nel, m, -1), axis=(1, 2))
    return ops.jacobian * s


def l2_norm(state, mesh, ops: ElementOperators) -> float:
    """sqrt(sum_K sum_c u_c^T M_K u_c), summed element by element in
    lexicographic order."""
    data = state.data if isinstance(state, FieldState) else np.asarray(state)
    per = _elementwise_sq(data, ops)
    return float(np.sqrt(np.add.accumulate(per)[-1])) if per.size else 0.0


def l2_error(state, exact, mesh, ops: ElementOperators, component: int = 0) -> float:
    """||u_h - exact||_{L2} by (p+2)^d Gauss quadrature."""
    data = state.data if isinstance(state, FieldState) else np.asarray(state)
    d = ops.dim
    qpts = mesh.all_element_points([ops.quad_points] * d)  # (Nel, nq^d, dim)
    nel, nq, _ = qpts.shape
    V = np.ones((1, 1))
    W = np.ones(1)
    for _ in range(d):
        V = np.kron(ops.interp, V)
        W = np.kron(ops.quad_weights, W)
    uh = data[:, component, :] @ V.T
    ue = np.asarray(exact(qpts.reshape(-1, d)), dtype=float).reshape(nel, nq)
    err = np.sum(W[None, :] * (uh - ue) ** 2, axis=1) * ops.jacobian
    return float(np.sqrt(np.add.accumulate(err)[-1]))
