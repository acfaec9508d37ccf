"""The paper's contraction / iteration-count predictors (SPEC.md:325-329,
361-377): ``predict_sw`` and ``predict_cdr``
(PAPER.md:1090-1133), plus the inverse-trace constant c of the nodal basis
(PAPER.md FEMTraceIn).  Closed forms on the host; they are compared with the
measured skeleton-energy contraction of a diagnostic run
(``IterationConfig(diagnostics=True)``)."""

from __future__ import annotations

from dataclasses import dataclass, field
from typing import Optional

import numpy as np

__all__ = ["ContractionEstimate", "predict_sw", "predict_cdr", "trace_inequality_constant"]


@dataclass
class ContractionEstimate:
    """SPEC.md:325-329."""

    kind: str
    inputs: dict
    admissible: bool
    epsilon: float
    contraction: float             # C (shallow water) or D (convection-diffusion)
    k_predicted: float
    constants: dict = field(default_factory=dict)


def predict_sw(h: float, p: int, dt: float, Phi: float, c: float = 1.0, gamma: float = 0.0) -> ContractionEstimate:
    """Shallow water (PAPER.md ContractionConstant, coarse_constraint,
    epsilon, khp_estimate).  Admissible iff the coarse constraint holds and
    B = min(B1, B2) > 0; C = A / B with the epsilon of Eq. (epsilon)."""
    if min(h, dt, Phi, c) <= 0 or p < 0:
        raise ValueError("positive inputs required")
    q = (p + 1) * (p + 2)
    sq = np.sqrt(Phi)
    top = max(1.0, Phi) + sq
    chq = c * h / (dt * q)
    constraint = chq / top
    eps = (2.0 * chq + sq) / top
    A = top / (4.0 * eps)
    G = eps * top / 4.0
    B1 = chq + (2.0 * sq - (Phi + sq) * eps) / 4.0
    B2 = (gamma + 1.0 / dt) * c * h / q + (2.0 * sq - (1.0 + sq) * eps) / 4.0
    B = min(B1, B2)
    C = A / B if B > 0 else float("inf")
    closed = (top / sq / (1.0 + 2.0 * c * h / (sq * dt * q))) ** 2
    return ContractionEstimate("sw", dict(h=h, p=p, dt=dt, Phi=Phi, c=c, gamma=gamma),
                               bool(constraint > 0.5 and B > 0), eps, C, dt * q * sq / (4.0 * c * h),
                               dict(constraint=constraint, A=A, G=G, B1=B1, B2=B2, B=B, C_closed_form=closed))


def _cdr_constants(eps, h, p, d, kappa, lam, bn_inf, tau_bar, a_bar, a_star, c):
    q = (p + 1) * (p + 2)
    C1 = (bn_inf + tau_bar) * (tau_bar + 1.0) / (2.0 * eps * a_star)
    C2 = (tau_bar + 1.0) / (2.0 * eps * a_star)
    C3 = eps * tau_bar * (1.0 + tau_bar + bn_inf) / (2.0 * a_star)
    C4 = eps * (1.0 + tau_bar + bn_inf) / (2.0 * a_star)
    A = max(C1, C2)
    B1 = 2.0 * c * h / (kappa * d * q) + 1.0 / (2.0 * a_bar) - C4
    B2 = 2.0 * c * h * lam / (d * q) + 1.0 / a_bar - C3
    B = min(B1, B2)
    m = min(1.0 / kappa, lam)
    return dict(C1=C1, C2=C2, C3=C3, C4=C4, A=A, B1=B1, B2=B2, B=B,
                D=A / B if B > 0 else float("inf"), E=max(C3, C4) / m, F=A / m)


def predict_cdr(h: float, p: int, d: int, kappa: float, lam: float, beta, c: float = 1.0,
                dt: Optional[float] = None) -> ContractionEstimate:
    """Convection-diffusion (PAPER.md DefineC1-DefineB, khp_estimate_CDR).
    beta: the constant velocity, or a dict of the bounds (bn_inf, tau_bar,
    a_bar, a_star) for a variable one; the face bounds |beta.n|_inf, tau_bar,
    alpha_bar, alpha_* follow from beta.n = +-beta_a with alpha =
    sqrt((beta.n)^2 + 4) and tau = (alpha - beta.n)/2.  With
    dt, lambda becomes lambda + 1/dt.  epsilon minimises D over B > 0
    (log-grid search refined by golden section)."""
    if min(h, kappa, c) <= 0 or p < 0 or lam < 0 or (lam == 0 and not dt):
        raise ValueError("positive inputs required (lambda may be 0 with a time step)")
    lam_eff = lam + (1.0 / dt if dt else 0.0)
    if isinstance(beta, dict):      # beta_bounds of SPEC.md:372 (variable beta)
        bounds = {k: float(beta[k]) for k in ("bn_inf", "tau_bar", "a_bar", "a_star")}
        b = np.zeros(0)
    else:
        b = np.abs(np.asarray(beta, dtype=float).reshape(-1))
        bn = np.concatenate([b, -b]) if b.size else np.zeros(1)
        alpha = np.sqrt(bn ** 2 + 4.0)
        tau = (alpha - bn) / 2.0
        bounds = dict(bn_inf=float(np.max(np.abs(bn))), tau_bar=float(np.max(tau)), a_bar=float(np.max(alpha)),
                      a_star=float(np.min(alpha)))
    args = (h, p, d, kappa, lam_eff, bounds["bn_inf"], bounds["tau_bar"], bounds["a_bar"], bounds["a_star"], c)
    grid = np.logspace(-6, 3, 2000)
    Ds = np.array([_cdr_constants(e, *args)["D"] for e in grid])
    i = int(np.argmin(Ds))
    lo, hi = grid[max(i - 1, 0)], grid[min(i + 1, grid.size - 1)]
    g = (np.sqrt(5.0) - 1.0) / 2.0
    for _ in range(80):
        x1, x2 = hi - g * (hi - lo), lo + g * (hi - lo)
        if _cdr_constants(x1, *args)["D"] < _cdr_constants(x2, *args)["D"]:
            hi = x2
        else:
            lo = x1
    eps = 0.5 * (lo + hi)
    k = _cdr_constants(eps, *args)
    k_pred = d * (p + 1) * (p + 2) / (8.0 * bounds["a_bar"] * c * h * min(1.0 / kappa, lam_eff))
    k.update(bounds)
    return ContractionEstimate("cdr", dict(h=h, p=p, d=d, kappa=kappa, lam=lam, beta=list(map(float, b)), c=c, dt=dt),
                               bool(k["B"] > 0 and k["D"] < 1.0), eps, k["D"], k_pred, k)


def trace_inequality_constant(p: int, d: int) -> float:
    """Largest c with (u,u)_K >= 2ch/(d(p+1)(p+2)) <u,u>_dK for every u in
    Q_p (PAPER.md FEMTraceIn), on the reference element [-1,1]^d (h = 2):
    1/mu_max of <u,u>_dK = mu (u,u)_K, times d(p+1)(p+2)/(2h).  This is the
    "c calibrated per basis" of SPEC.md:510 (the basis spans Q_p, so c does
    not depend on the nodes)."""
    import scipy.linalg as sla

    x, _ = np.polynomial.legendre.leggauss(p + 1)          # any p+1 nodes span P_p
    qx, qw = np.polynomial.legendre.leggauss(p + 2)
    n1 = p + 1

    def lag(t):
        return np.array([np.prod([(t - x[m]) / (x[j] - x[m]) for m in range(n1) if m != j]) for j in range(n1)])

    V = np.array([lag(t) for t in qx])
    M1 = V.T @ (qw[:, None] * V)
    ends = np.array([lag(-1.0), lag(1.0)])
    E1 = ends.T @ ends                                       # <u,u> at the two end points
    Mv = np.ones((1, 1))
    for _ in range(d):
        Mv = np.kron(M1, Mv)
    Mb = np.zeros_like(Mv)
    for a in range(d):
        term = np.ones((1, 1))
        for b in range(d):
            term = np.kron(E1 if b == a else M1, term)
        Mb += term
    mu_max = float(np.max(sla.eigh(Mb, Mv, eigvals_only=True)))
    h = 2.0
    return d * (p + 1) * (p + 2) / (2.0 * h * mu_max)
