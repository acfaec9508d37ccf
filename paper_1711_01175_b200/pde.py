"""PDE problem definitions and stabilisation.

Transport, linearised shallow water and
convection-diffusion in first-order form.  Coefficients
used by the device path must be constant on the mesh (shared element operator,
BASELINE.json north_star); variable fields are accepted by the host API and
rejected by the device path with a clear error.
"""

from __future__ import annotations

from dataclasses import dataclass, field
from typing import Callable, Optional

import numpy as np

__all__ = ["TransportProblem", "ShallowWaterProblem", "ConvectionDiffusionProblem",
           "StabilizationData", "upwind_flux_matrix", "stabilization", "FourierModes",
           "GaussianBump", "preset_problems"]


@dataclass(frozen=True)
class FourierModes:
    """f(x) = sum_j a_j sin(2 pi k_j . x + phi_j) (seeded synthetic field)."""

    amplitudes: np.ndarray   # (n,)
    wavevectors: np.ndarray  # (n, dim)
    phases: np.ndarray       # (n,)
    scale: float = 1.0

    def __call__(self, x):
        x = np.atleast_2d(np.asarray(x, dtype=float))
        arg = 2.0 * np.pi * (x @ self.wavevectors.T) + self.phases[None, :]
        return self.scale * (np.sin(arg) @ self.amplitudes)

    def device_params(self) -> np.ndarray:
        n, d = self.wavevectors.shape
        P = np.empty((n, 2 + d))
        P[:, 0] = self.scale * self.amplitudes
        P[:, 1:1 + d] = self.wavevectors
        P[:, 1 + d] = self.phases
        return P


@dataclass(frozen=True)
class GaussianBump:
    """f(x) = a exp(-|x - c|^2 / (2 w^2))."""

    center: np.ndarray
    width: float
    amplitude: float = 1.0

    def __call__(self, x):
        x = np.atleast_2d(np.asarray(x, dtype=float))
        r2 = np.sum((x - self.center[None, :]) ** 2, axis=1)
        return self.amplitude * np.exp(-r2 / (2.0 * self.width ** 2))

    def device_params(self) -> np.ndarray:
        d = self.center.size
        P = np.empty((1, 2 + d))
        P[0, 0] = self.amplitude
        P[0, 1:1 + d] = self.center
        P[0, 1 + d] = self.width
        return P


def _const_vector(v, dim) -> Optional[np.ndarray]:
    if callable(v):
        return None
    a = np.asarray(v, dtype=float).reshape(-1)
    if a.size != dim:
        raise ValueError(f"expected a {dim}-vector, got {a}")
    return a


@dataclass
class TransportProblem:
    """beta . grad u + c u = f in Omega, u = g on the inflow boundary."""

    beta: object                      # constant (dim,) vector or callable x -> (n, dim)
    forcing: Optional[Callable] = None
    inflow: Optional[Callable] = None  # g; None = 0
    reaction: float = 0.0
    exact: Optional[Callable] = None
    alpha_div: Optional[float] = None
    kind: str = field(default="transport", init=False)

    def beta_const(self, dim):
        return _const_vector(self.beta, dim)

    def n_components(self, dim):
        return 1

    def labels(self, dim):
        return ("u",)


@dataclass
class ConvectionDiffusionProblem:
    """kappa^-1 sigma + grad u = 0, div sigma + beta.grad u + nu u = f."""

    kappa: float
    beta: object
    nu: float = 0.0
    forcing: Optional[Callable] = None
    dirichlet: Optional[Callable] = None  # g_D; None = 0
    lam: Optional[float] = None
    exact: Optional[Callable] = None
    kind: str = field(default="cd", init=False)

    def __post_init__(self):
        if not self.kappa > 0:
            raise ValueError("kappa must be > 0")

    def beta_const(self, dim):
        return _const_vector(self.beta, dim)

    def n_components(self, dim):
        return dim + 1

    def labels(self, dim):
        return tuple(f"sigma{a}" for a in range(dim)) + ("u",)


@dataclass
class ShallowWaterProblem:
    """Linearised oceanic shallow water (phi, u, v)."""

    Phi: float = 1.0
    gamma: float = 0.0
    f0: float = 0.0
    beta_cor: float = 0.0
    y_m: float = 0.0
    tau: tuple = (0.0, 0.0)
    rho: float = 1.0
    exact: Optional[Callable] = None
    kind: str = field(default="sw", init=False)

    def __post_init__(self):
        if not self.Phi > 0:
            raise ValueError("Phi must be > 0")
        if self.gamma < 0:
            raise ValueError("gamma must be >= 0")

    def n_components(self, dim):
        if dim != 2:
            raise ValueError("the shallow water system is two-dimensional")
        return 3

    def labels(self, dim):
        return ("phi", "u", "v")


@dataclass(frozen=True)
class StabilizationData:
    """Face-point stabilisation: beta.n, |beta.n|, alpha, tau, sqrt(Phi)."""

    bn: np.ndarray
    abs_bn: np.ndarray
    alpha: np.ndarray
    tau: np.ndarray
    sqrt_phi: Optional[float] = None

    @property
    def tau_bar(self):
        return float(np.max(self.tau))

    @property
    def alpha_bar(self):
        return float(np.max(self.alpha))

    @property
    def alpha_star(self):
        return float(np.min(self.alpha))


def stabilization(problem, bn) -> StabilizationData:
    """alpha = sqrt(|beta.n|^2 + 4), tau = (alpha - beta.n)/2."""
    bn = np.asarray(bn, dtype=float)
    alpha = np.sqrt(bn ** 2 + 4.0)
    tau = 0.5 * (alpha - bn)
    sp = np.sqrt(problem.Phi) if isinstance(problem, ShallowWaterProblem) else None
    return StabilizationData(bn, np.abs(bn), alpha, tau, sp)


def upwind_flux_matrix(problem, n, beta=None):
    """(A, |A|) with A = sum_k A_k n_k, |A| = R|S|R^-1."""
    n = np.asarray(n, dtype=float)
    if abs(np.linalg.norm(n) - 1.0) > 1e-12:
        raise ValueError("normal must have unit length")
    if isinstance(problem, ShallowWaterProblem):
        P = problem.Phi
        A = np.array([[0.0, P * n[0], P * n[1]],
                      [n[0], 0.0, 0.0],
                      [n[1], 0.0, 0.0]])
        # flux of (phi, Phi u, Phi v) in terms of (phi, u, v): symmetrise with
        # diag(1, Phi, Phi) -> eigen-decomposition of the symmetric form
        S = np.diag([1.0, np.sqrt(P), np.sqrt(P)])
        Sinv = np.diag(1.0 / np.diag(S))
        As = S @ A @ Sinv
        As = 0.5 * (As + As.T)
        lam, R = np.linalg.eigh(As)
        absA = Sinv @ (R @ np.diag(np.abs(lam)) @ R.T) @ S
        return Sinv @ As @ S, absA
    b = beta if beta is not None else problem.beta
    b = np.asarray(b(n[None, :]) if callable(b) else b, dtype=float).reshape(-1)
    bn = float(b @ n)
    return np.array([[bn]]), np.array([[abs(bn)]])


def _gauss_timedep(x, t):
    x = np.asarray(x, dtype=float)
    return np.exp(-5.0 * np.sum((x - 0.35 * t) ** 2, axis=1))


def cdr_manufactured(kappa: float = 1e-2) -> "ConvectionDiffusionProblem":
    """SPEC.md:198 / PAPER.md:1661-1666: u^e = sin(pi x) cos(pi y) sin(pi z) / pi,
    beta = (1 + z, 1 + x, 1 + y) (div beta = 0), nu = 1, forcing
    f = -kappa Lap u^e + beta . grad u^e + nu u^e, Dirichlet data u^e on [0,1]^3."""
    pi = np.pi

    def ue(x):
        x = np.asarray(x, dtype=float)
        return np.sin(pi * x[:, 0]) * np.cos(pi * x[:, 1]) * np.sin(pi * x[:, 2]) / pi

    def beta(x):
        x = np.asarray(x, dtype=float)
        return np.stack([1.0 + x[:, 2], 1.0 + x[:, 0], 1.0 + x[:, 1]], axis=1)

    def forcing(x):
        x = np.asarray(x, dtype=float)
        X, Y, Z = x[:, 0], x[:, 1], x[:, 2]
        ux = np.cos(pi * X) * np.cos(pi * Y) * np.sin(pi * Z)
        uy = -np.sin(pi * X) * np.sin(pi * Y) * np.sin(pi * Z)
        uz = np.sin(pi * X) * np.cos(pi * Y) * np.cos(pi * Z)
        b = beta(x)
        u = ue(x)
        return kappa * 3.0 * pi * pi * u + b[:, 0] * ux + b[:, 1] * uy + b[:, 2] * uz + 1.0 * u

    return ConvectionDiffusionProblem(kappa=kappa, beta=beta, nu=1.0, forcing=forcing, dirichlet=ue, lam=1.0,
                                      exact=ue)


def elliptic_manufactured(kappa: float = 1.0) -> "ConvectionDiffusionProblem":
    """The elliptic regime of PAPER.md section 6.3 ("elliptic with
    kappa = 1 and beta = 0") on the manufactured solution of cdr_manufactured:
    -kappa Lap u + nu u = f with u^e = sin(pi x) cos(pi y) sin(pi z) / pi,
    nu = 1, f = (3 pi^2 kappa + nu) u^e, Dirichlet data u^e on [0,1]^3.  The
    velocity is constant (zero), so the operators are shared per class."""
    pi = np.pi

    def ue(x):
        x = np.asarray(x, dtype=float)
        return np.sin(pi * x[:, 0]) * np.cos(pi * x[:, 1]) * np.sin(pi * x[:, 2]) / pi

    def forcing(x):
        return (3.0 * pi * pi * kappa + 1.0) * ue(x)

    return ConvectionDiffusionProblem(kappa=kappa, beta=np.zeros(3), nu=1.0, forcing=forcing, dirichlet=ue, lam=1.0,
                                      exact=ue)


def preset_problems():
    """Named presets usable through the same API."""
    s2 = np.sqrt(2.0)
    cat = {
        "transport2d_diag": TransportProblem(beta=np.array([1.0, 1.0])),
        "transport3d_diag": TransportProblem(beta=np.array([1.0, 1.0, 1.0])),
        # u^e = exp(-5 |x - 0.35 t|^2); f = u_t + beta . grad u
        # = 1.5 u sum_i (x_i - 0.35 t) manufactured, inflow data g = u^e
        "transport3d_timedep": TransportProblem(
            beta=np.array([0.2, 0.2, 0.2]),
            exact=lambda x, t=0.0: _gauss_timedep(x, t),
            forcing=lambda x, t=0.0: 1.5 * np.sum(np.asarray(x) - 0.35 * t, axis=1) * _gauss_timedep(x, t),
            inflow=lambda x, t=0.0: _gauss_timedep(x, t)),
        "sw_standing_wave": ShallowWaterProblem(
            Phi=1.0,
            exact=lambda x, t=0.0: np.stack([
                np.cos(np.pi * x[:, 0]) * np.cos(np.pi * x[:, 1]) * np.cos(s2 * np.pi * t),
                np.sin(np.pi * x[:, 0]) * np.cos(np.pi * x[:, 1]) * np.sin(s2 * np.pi * t) / s2,
                np.cos(np.pi * x[:, 0]) * np.sin(np.pi * x[:, 1]) * np.sin(s2 * np.pi * t) / s2],
                axis=1)),
        "elliptic": ConvectionDiffusionProblem(kappa=1.0, beta=np.zeros(3), nu=1.0, lam=1.0),
        "elliptic_manufactured": elliptic_manufactured(1.0),
        "cdr_manufactured": cdr_manufactured(1e-2),
    }
    return cat
