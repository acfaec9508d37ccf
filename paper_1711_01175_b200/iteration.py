"""Algorithm 1 drivers: ``run`` and ``run_time_dependent``.

Same call shapes as the reference module ``ihdg.iteration``; the parallel
element map behind them is the sm_100a sweep of libihdg_cuda.so (the
reference's ``_kernels._sweep_cy`` seam, pkg/setup.py:13-19).  Inputs and
outputs are host numpy arrays (``FieldState``); everything in between stays in
HBM: one upload, sweeps batched with a device-side convergence flag (exact
iteration count, no per-sweep host sync), one download.
"""

from __future__ import annotations

import time
from dataclasses import dataclass, field
from typing import Optional

import numpy as np

from .basis import ElementOperators, FieldState
from .pde import ConvectionDiffusionProblem, FourierModes, GaussianBump, ShallowWaterProblem, TransportProblem
from .solver import DeviceSolver

__all__ = ["IterationConfig", "IterationReport", "run", "run_time_dependent", "default_max_iters"]


@dataclass
class IterationConfig:
    """SPEC.md:315-318.  ``stop``: "successive" (||u^k - u^{k-1}||_{L2} < tol,
    PAPER.md:1308-1311), "exact" (| ||u^k - u^e|| - ||u^{k-1} - u^e|| | < tol,
    PAPER.md:1303-1306, needs problem.exact) or "trace" (skeleton L2 norm of
    the trace update; transport only)."""

    scheme: str = "iHDG-II"
    stop: str = "successive"
    tol: float = 1e-10
    max_iters: Optional[int] = None
    initial_guess: object = None
    workers: Optional[int] = None      # API parity; the device owns parallelism
    check_every: int = 16              # sweeps per host poll of the device flag
    diverge_factor: float = 1e6

    def __post_init__(self):
        if not self.tol > 0:
            raise ValueError("tolerance must be > 0")
        if self.max_iters is not None and self.max_iters < 1:
            raise ValueError("max_iters must be >= 1")
        if self.scheme not in ("iHDG-II", "iHDG-I"):
            raise ValueError(f"unknown scheme {self.scheme!r} (iHDG-I or iHDG-II)")
        if self.stop == "exact-solution":
            self.stop = "exact"
        if self.stop not in ("successive", "trace", "exact"):
            raise NotImplementedError(f"stopping rule {self.stop!r} not on the device path")


@dataclass
class IterationReport:
    """SPEC.md:320-323 (device subset)."""

    iterations: int
    status: str
    successive_norms: np.ndarray
    wall_time: float
    state: Optional[FieldState] = None
    trace: Optional[np.ndarray] = None
    first_norm: float = 0.0
    final_norm: float = 0.0
    sweeps_launched: int = 0
    extra: dict = field(default_factory=dict)


def default_max_iters(mesh) -> int:
    """SPEC.md:389 sets 10 * (predicted k + Nel^(1/d) * d); the closed-form
    predictor underestimates diffusion-dominated cells by ~50x (measured
    spectral radii), so the default is floored at 100000."""
    n = mesh.n_elements ** (1.0 / mesh.dim)
    return max(int(10 * (n * mesh.dim) + 100), 100000)


def _exact_at(exact, t):
    """exact(x) (steady) or exact(x, t) at the new time level -> a function of x."""
    if t is None:
        return lambda x: exact(x)
    return lambda x: exact(x, t)


def _norm_name(cfg: IterationConfig, problem) -> str:
    if cfg.stop == "trace" and not isinstance(problem, TransportProblem):
        raise NotImplementedError("the trace stopping rule is defined for transport")
    if cfg.stop == "exact":
        if getattr(problem, "exact", None) is None:
            raise ValueError("the exact-solution stopping rule needs problem.exact")
        return "exact"
    return "trace" if cfg.stop == "trace" else "volume"


def _set_initial(solver: DeviceSolver, init):
    if init is None:
        solver.zero_state()
    elif isinstance(init, FieldState):
        solver.set_state(init.data)
    elif isinstance(init, np.ndarray):
        solver.set_state(init)
    elif isinstance(init, dict):  # component label -> field
        solver.zero_state()
        labels = solver.spec.labels
        for name, fld in init.items():
            solver.set_state_component(fld, labels.index(name))
    else:
        raise TypeError(f"unsupported initial guess {type(init).__name__}")


def run(mesh, problem, ops: ElementOperators, cfg: Optional[IterationConfig] = None,
        solver: Optional[DeviceSolver] = None, return_state: bool = True,
        return_trace: bool = True) -> IterationReport:
    """Steady solve (Algorithm 1); cfg.scheme selects
    iHDG-II (default) or iHDG-I (all-iterate-k trace)."""
    cfg = cfg or IterationConfig()
    t0 = time.perf_counter()
    if solver is None:
        solver = DeviceSolver(mesh, problem, ops, dt=None,
                              max_iters=cfg.max_iters or default_max_iters(mesh), scheme=cfg.scheme)
    forcing = getattr(problem, "forcing", None)
    if forcing is not None and solver.s_static is None:
        solver.set_forcing(forcing)
    solver.prepare_steady()
    _set_initial(solver, cfg.initial_guess)
    if cfg.stop == "exact":
        solver.set_exact(_exact_at(problem.exact, None))
    res = solver.iterate(tol=cfg.tol, max_iters=cfg.max_iters or default_max_iters(mesh),
                         norm=_norm_name(cfg, problem), batch=cfg.check_every)
    state = FieldState(solver.get_state(), solver.spec.labels, k=res.iterations) if return_state else None
    tr = solver.trace() if (return_trace and solver.layers[0] == 0
                            and solver.layers[1] == mesh.cells[-1]) else None
    return IterationReport(res.iterations, res.status, res.norms, time.perf_counter() - t0,
                           state, tr, res.first_norm, res.last_norm, res.launched,
                           extra={"device_seconds": res.seconds, "l2_errors": res.errors})


def run_time_dependent(mesh, problem, ops: ElementOperators, cfg: Optional[IterationConfig],
                       dt: float, T: Optional[float] = None, n_steps: Optional[int] = None,
                       initial=None, solver: Optional[DeviceSolver] = None,
                       keep_states: bool = False, time_scheme: str = "backward-euler") -> list:
    """Time steps; each step iterates from u^m.
    ``time_scheme``: "backward-euler" or "crank-nicolson" (trapezoidal split of
    the spatial operator).  Divergence at any step aborts
    the run (the last report says which step)."""
    cfg = cfg or IterationConfig()
    ts = {"backward-euler": "BE", "be": "BE", "crank-nicolson": "CN", "cn": "CN"}.get(time_scheme.lower())
    if ts is None:
        raise ValueError(f"unknown time scheme {time_scheme!r}")
    if n_steps is None:
        if T is None:
            raise ValueError("give T or n_steps")
        n_steps = int(round(T / dt))
    if solver is None:
        solver = DeviceSolver(mesh, problem, ops, dt=dt,
                              max_iters=cfg.max_iters or default_max_iters(mesh), scheme=cfg.scheme,
                              time_scheme=ts)
    forcing = getattr(problem, "forcing", None)
    if forcing is not None and solver.s_static is None:
        solver.set_forcing(forcing)
    _set_initial(solver, initial if initial is not None else cfg.initial_guess)
    reports = []
    for m in range(n_steps):
        t0 = time.perf_counter()
        solver.begin_step()
        if cfg.stop == "exact":
            solver.set_exact(_exact_at(problem.exact, (m + 1) * dt))
        res = solver.iterate(tol=cfg.tol, max_iters=cfg.max_iters or default_max_iters(mesh),
                             norm=_norm_name(cfg, problem), batch=cfg.check_every)
        last = m == n_steps - 1 or res.status != "converged"
        st = (FieldState(solver.get_state(), solver.spec.labels, k=res.iterations, m=m + 1)
              if (keep_states or last) else None)
        reports.append(IterationReport(res.iterations, res.status, res.norms,
                                       time.perf_counter() - t0, st, None, res.first_norm,
                                       res.last_norm, res.launched,
                                       extra={"step": m + 1, "device_seconds": res.seconds,
                                              "l2_errors": res.errors}))
        if res.status != "converged":
            break
    return reports
