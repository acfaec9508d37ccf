"""Seeded synthetic inputs for the BASELINE.json configurations.

BASELINE.json names no dataset; every input is synthetic and seeded from
``np.random.default_rng(seed)``.  The formulas are pinned here once and used by
the product path, the tests (against the CPU oracle) and bench.py
(SURVEY.md 8d, Appendix B.4-B.7):

- Fourier field: f(x) = s * sum_{j<8} a_j sin(2 pi k_j . x + phi_j),
  a_j ~ N(0,1), k_j uniform in {1..4}^d, phi_j ~ U[0, 2 pi);
- Gaussian bump: exp(-|x - c|^2 / (2 * 0.05^2)), c ~ U[0.3, 0.7]^2.

Configs (BASELINE.json "configs", 1-based as in SURVEY.md):
 1  2D steady transport, beta=(1,0.5), 16^2, p=2, Fourier forcing, zero inflow,
    stop on the trace update < 1e-10
 2  2D convection-diffusion, kappa=1e-2, beta=(1,1), 128^2, p=4, BE dt=1e-2 x 10,
    Gaussian-bump u0, homogeneous Dirichlet (f = 0, nu = 0: App. B.5)
 3  2D linearised shallow water, Phi=1, f=1, gamma=0, 256^2, p=4, BE dt=5e-3 x 20,
    phi0 = 1e-2 * Fourier, zero velocity, periodic
 4  3D steady transport, beta=(1,0.7,0.4), 64^3, p=3, Fourier forcing, zero inflow
 5  2D convection-diffusion, kappa in {1e-1, 1e-3}, beta=(1,1), 2048^2, p=6,
    BE dt = h/p x 5, Fourier u0, homogeneous Dirichlet
Initial sigma = 0 for convection-diffusion.
"""

from __future__ import annotations

from dataclasses import dataclass, field
from typing import Optional

import numpy as np

from .basis import build_operators
from .mesh import build_mesh
from .pde import ConvectionDiffusionProblem, FourierModes, GaussianBump, ShallowWaterProblem, TransportProblem

__all__ = ["Workload", "fourier_modes", "gaussian_bump", "make_config", "CONFIG_CELLS"]

CONFIG_CELLS = {1: 16, 2: 128, 3: 256, 4: 64, 5: 2048}


def fourier_modes(rng: np.random.Generator, dim: int, n: int = 8, kmax: int = 4,
                  scale: float = 1.0) -> FourierModes:
    a = rng.normal(size=n)
    k = rng.integers(1, kmax + 1, size=(n, dim)).astype(float)
    ph = rng.uniform(0.0, 2.0 * np.pi, size=n)
    return FourierModes(a, k, ph, scale)


def gaussian_bump(rng: np.random.Generator, width: float = 0.05) -> GaussianBump:
    c = rng.uniform(0.3, 0.7, size=2)
    return GaussianBump(c, width, 1.0)


@dataclass
class Workload:
    config: int
    name: str
    mesh: object
    problem: object
    ops: object
    dt: Optional[float]
    n_steps: int
    initial: dict = field(default_factory=dict)   # label -> field (None = zero)
    stop: str = "successive"
    params: dict = field(default_factory=dict)

    @property
    def dofs(self) -> int:
        return self.mesh.n_elements * self.problem.n_components(self.mesh.dim) * self.ops.n_nodes


def make_config(config: int, seed: int = 0, cells: Optional[int] = None, kappa: Optional[float] = None,
                order: Optional[int] = None, n_steps: Optional[int] = None) -> Workload:
    """Build BASELINE config ``config`` (1..5); ``cells``/``order``/``n_steps``
    shrink it for parity tests (same formulas, smaller mesh)."""
    rng = np.random.default_rng(seed)
    n = CONFIG_CELLS[config] if cells is None else int(cells)
    if config == 1:
        p = 2 if order is None else order
        mesh = build_mesh(2, [n, n])
        prob = TransportProblem(beta=np.array([1.0, 0.5]), forcing=fourier_modes(rng, 2))
        return Workload(1, f"transport2d_{n}x{n}_p{p}", mesh, prob, build_operators(p, 2, mesh.h),
                        None, 0, {}, "trace", {"beta": [1.0, 0.5], "seed": seed})
    if config == 2:
        p = 4 if order is None else order
        mesh = build_mesh(2, [n, n])
        prob = ConvectionDiffusionProblem(kappa=1e-2, beta=np.array([1.0, 1.0]), nu=0.0)
        init = {"u": gaussian_bump(rng)}
        return Workload(2, f"cd2d_{n}x{n}_p{p}", mesh, prob, build_operators(p, 2, mesh.h),
                        1e-2, 10 if n_steps is None else n_steps, init, "successive",
                        {"kappa": 1e-2, "beta": [1.0, 1.0], "seed": seed})
    if config == 3:
        p = 4 if order is None else order
        mesh = build_mesh(2, [n, n], periodic=True)
        prob = ShallowWaterProblem(Phi=1.0, gamma=0.0, f0=1.0)
        init = {"phi": fourier_modes(rng, 2, scale=1e-2)}
        return Workload(3, f"sw2d_{n}x{n}_p{p}", mesh, prob, build_operators(p, 2, mesh.h),
                        5e-3, 20 if n_steps is None else n_steps, init, "successive",
                        {"Phi": 1.0, "f": 1.0, "seed": seed})
    if config == 4:
        p = 3 if order is None else order
        mesh = build_mesh(3, [n, n, n])
        prob = TransportProblem(beta=np.array([1.0, 0.7, 0.4]), forcing=fourier_modes(rng, 3))
        return Workload(4, f"transport3d_{n}^3_p{p}", mesh, prob, build_operators(p, 3, mesh.h),
                        None, 0, {}, "successive", {"beta": [1.0, 0.7, 0.4], "seed": seed})
    if config == 5:
        p = 6 if order is None else order
        k = 1e-3 if kappa is None else float(kappa)
        mesh = build_mesh(2, [n, n])
        prob = ConvectionDiffusionProblem(kappa=k, beta=np.array([1.0, 1.0]), nu=0.0)
        dt = float(mesh.h[0]) / p
        init = {"u": fourier_modes(rng, 2)}
        return Workload(5, f"cd2d_{n}x{n}_p{p}_k{k:g}", mesh, prob, build_operators(p, 2, mesh.h),
                        dt, 5 if n_steps is None else n_steps, init, "successive",
                        {"kappa": k, "beta": [1.0, 1.0], "dt": dt, "seed": seed})
    raise ValueError(f"unknown config {config}")
