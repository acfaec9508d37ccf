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

__all__ = ["IterationConfig", "IterationReport", "run", "run_time_dependent", "default_max_iters",
           "layer_convergence_map", "write_history_csv", "HISTORY_COLUMNS", "cfl_number",
           "contraction_factor"]

HISTORY_COLUMNS = ("iteration", "l2_error", "successive_norm", "trace_energy", "converged_elements",
                   "elapsed_ms")


@dataclass
class IterationConfig:
    """SPEC.md:315-318.  ``stop``: "successive" (||u^k - u^{k-1}||_{L2} < tol,
    PAPER.md:1308-1311), "exact" (| ||u^k - u^e|| - ||u^{k-1} - u^e|| | < tol,
    PAPER.md:1303-1306, needs problem.exact), "vs-direct" (||u^k - u_direct||
    < tol, SPEC.md:316 / PAPER.md section 6.3, ``reference`` = the direct HDG
    solution) or "trace" (skeleton L2 norm of the trace update, SURVEY.md
    App. B.2; transport only)."""

    scheme: str = "iHDG-II"
    stop: str = "successive"
    tol: float = 1e-10
    max_iters: Optional[int] = None
    initial_guess: object = None
    workers: Optional[int] = None      # API parity; the device owns parallelism
    check_every: int = 16              # sweeps per host poll of the device flag
    diverge_factor: float = 1e6
    # per-iteration diagnostics: sweep-by-sweep,
    # against ``reference`` (the converged HDG solution; computed by a first
    # solve from the same initial guess when None)
    diagnostics: bool = False
    reference: object = None

    def __post_init__(self):
        if not self.tol > 0:
            raise ValueError("tolerance must be > 0")
        if self.max_iters is not None and self.max_iters < 1:
            raise ValueError("max_iters must be >= 1")
        if self.scheme not in ("iHDG-II", "iHDG-I"):
            raise ValueError(f"unknown scheme {self.scheme!r} (iHDG-I or iHDG-II)")
        if self.stop == "exact-solution":
            self.stop = "exact"
        if self.stop not in ("successive", "trace", "exact", "vs-direct"):
            raise NotImplementedError(f"stopping rule {self.stop!r} not on the device path")
        if self.stop == "vs-direct" and self.reference is None:
            raise ValueError("the vs-direct stopping rule needs IterationConfig(reference=<direct HDG solution>)")


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


def _takes_time(fn) -> bool:
    """True for a data callable of (x, t) (time-dependent forcing / boundary data)."""
    if fn is None or isinstance(fn, (FourierModes, GaussianBump)):
        return False
    import inspect
    try:
        return len(inspect.signature(fn).parameters) >= 2
    except (TypeError, ValueError):
        return False


def _norm_name(cfg: IterationConfig, problem) -> str:
    if cfg.stop == "trace" and not isinstance(problem, TransportProblem):
        raise NotImplementedError("the trace stopping rule is defined for transport")
    if cfg.stop == "exact":
        if getattr(problem, "exact", None) is None:
            raise ValueError("the exact-solution stopping rule needs problem.exact")
        return "exact"
    if cfg.stop == "vs-direct":
        return "vs-direct"
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


def _diagnostic_iterate(solver: DeviceSolver, cfg: IterationConfig, norm: str, max_iters: int) -> dict:
    """Algorithm 1 one sweep at a time with the per-iteration diagnostics of
    SPEC.md:321 on the device (K6): successive norm, L2 error vs exact (when
    known), trace energy ||(phi, theta.n)(u^k - r)||^2_{E_h} (shallow water;
    (sigma.n, u) for convection-diffusion, u for transport) -- the skeleton
    norm the contraction theorems bound --,
    skeleton jump norm ||u^- - u^+||_{L2(E_h)} of the trace variable, and the
    element convergence map {K : ||u^k - r||_{L2(K)} < tol}.  r is cfg.reference or the
    converged solution of a first (batched) solve from the same iterate."""
    import ctypes as C
    from . import _native as N
    torch = solver.torch
    start = solver.padded_copy()
    cur0 = solver.cur
    if cfg.reference is not None:
        ref_data = cfg.reference.data if isinstance(cfg.reference, FieldState) else cfg.reference
        ref = solver.padded_copy(ref_data)
    else:
        pre = solver.iterate(tol=cfg.tol, max_iters=max_iters, norm=norm, batch=cfg.check_every)
        if pre.status != "converged":
            raise RuntimeError(f"diagnostics: the reference solve did not converge ({pre.status})")
        ref = solver.padded_copy()
        solver.cur = cur0
        solver.u[cur0].copy_(start)
    side_refs = [solver.trace_of(ref, weights=w) for w in solver.energy_sides()]
    has_exact = getattr(solver, "ue_q", None) is not None
    solver.reset_state(cfg.tol, max_iters, cfg.diverge_factor)
    err_rule = {"exact": 1, "vs-direct": 2}.get(norm, 0)   # K5 mode of the stop rule
    if err_rule:
        N.check(solver.L.ihdg_error_norm(C.byref(solver._error_args(0)), solver._sptr), "ihdg_error_norm")
        a = solver.sweep_args("volume", finalize=0)
    else:
        a = solver.sweep_args(norm, finalize=1)
    cols = {k: [] for k in HISTORY_COLUMNS}
    maps = []
    t0 = time.perf_counter()
    status = "running"
    for k in range(1, max_iters + 1):
        solver.sweep_once(a=a)
        if err_rule:
            e = solver._error_args(err_rule)
            N.check(solver.L.ihdg_error_norm(C.byref(e), solver._sptr), "ihdg_error_norm")
        st = solver.read_state()
        err = float("nan")
        if err_rule:
            err = st.last_err
        elif has_exact:
            e = solver._error_args(0)
            N.check(solver.L.ihdg_error_norm(C.byref(e), solver._sptr), "ihdg_error_norm")
            err = solver.read_state().last_err
        energy = solver.skeleton_energy(side_refs)
        _, flags, _ = solver.element_errors(ref, cfg.tol)
        fl = flags.cpu().numpy().astype(bool)
        maps.append(fl)
        cols["iteration"].append(k)
        cols["l2_error"].append(err)
        cols["successive_norm"].append(st.last_norm)
        cols["trace_energy"].append(energy)
        cols["converged_elements"].append(int(fl.sum()))
        cols["elapsed_ms"].append((time.perf_counter() - t0) * 1e3)
        cols.setdefault("jump_norm", []).append(np.sqrt(solver.face_energy(solver.trace_of(jump=True))))
        status = N.STATUS_NAMES[st.status]
        if st.status != N.RUNNING:
            break
    hist = {k: np.asarray(v) for k, v in cols.items()}
    return dict(iterations=len(maps), status=status, history=hist, maps=maps, first_norm=st.first_norm,
                last_norm=st.last_norm, contraction=contraction_factor(hist["trace_energy"], cfg.tol),
                seconds=time.perf_counter() - t0)


def contraction_factor(energy, tol: float = 1e-10) -> float:
    """Measured contraction factor: geometric mean of the
    successive trace-energy ratios E_{k+1}/E_k after the first iteration
    (E is the squared skeleton norm, so this is comparable with the C / D of
    the theorems), over the energies above (1e3 tol)^2 (below that the
    reference solution's own stopping error dominates)."""
    e = np.asarray(energy, dtype=float)
    r = [e[k + 1] / e[k] for k in range(1, len(e) - 1) if e[k] > 0 and e[k + 1] > (1e3 * tol) ** 2]
    return float(np.exp(np.mean(np.log(r)))) if r else float("nan")


def layer_convergence_map(report: "IterationReport") -> list:
    """per-iteration converged-element sets (element ids in
    mesh order) of a run with cfg.diagnostics=True."""
    maps = report.extra.get("convergence_map")
    if maps is None:
        raise ValueError("layer_convergence_map needs a run with IterationConfig(diagnostics=True)")
    return [set(np.flatnonzero(m).tolist()) for m in maps]


def write_history_csv(report: "IterationReport", path) -> None:
    """Per-iteration CSV rows: iteration, l2_error,
    successive_norm, trace_energy, converged_elements, elapsed_ms."""
    import csv
    hist = report.extra.get("history")
    if hist is None:
        raise ValueError("write_history_csv needs a run with IterationConfig(diagnostics=True)")
    with open(path, "w", newline="") as fh:
        w = csv.writer(fh)
        w.writerow(HISTORY_COLUMNS)
        for i in range(len(hist["iteration"])):
            w.writerow([int(hist["iteration"][i])] + [repr(float(hist[c][i])) for c in HISTORY_COLUMNS[1:4]]
                       + [int(hist["converged_elements"][i]), f"{hist['elapsed_ms'][i]:.3f}"])


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
    if getattr(problem, "inflow", None) is not None:
        solver.set_inflow(problem.inflow)
    if getattr(problem, "dirichlet", None) is not None:
        solver.set_dirichlet(problem.dirichlet)
    solver.prepare_steady()
    _set_initial(solver, cfg.initial_guess)
    if cfg.stop == "exact" or (cfg.diagnostics and getattr(problem, "exact", None) is not None):
        solver.set_exact(_exact_at(problem.exact, None))
    if cfg.stop == "vs-direct":
        solver.set_reference(cfg.reference.data if isinstance(cfg.reference, FieldState) else cfg.reference)
    if cfg.diagnostics:
        return _diagnostic_report(solver, cfg, _norm_name(cfg, problem), cfg.max_iters or default_max_iters(mesh),
                                  t0, return_state, return_trace)
    res = solver.iterate(tol=cfg.tol, max_iters=cfg.max_iters or default_max_iters(mesh),
                         norm=_norm_name(cfg, problem), batch=cfg.check_every)
    state = FieldState(solver.get_state(), solver.spec.labels, k=res.iterations) if return_state else None
    tr = solver.trace() if (return_trace and not solver.spec.per_element and solver.layers[0] == 0
                            and solver.layers[1] == mesh.cells[-1]) else None
    return IterationReport(res.iterations, res.status, res.norms, time.perf_counter() - t0,
                           state, tr, res.first_norm, res.last_norm, res.launched,
                           extra={"device_seconds": res.seconds, "l2_errors": res.errors,
                                  "kernel": res.kernel})


def cfl_number(problem, mesh, p: int, dt: float) -> float:
    """CFL = |beta|_max dt (p+1)^2 / h (the DG estimate of
    PAPER.md section 4.4); |beta| is the Euclidean speed, h the smallest
    element size.  Shallow water uses the gravity-wave speed sqrt(Phi)."""
    if hasattr(problem, "beta") and callable(problem.beta):
        # variable velocity: the largest speed at the element centres
        c = np.asarray(mesh.all_element_points([np.zeros(1)] * mesh.dim), float).reshape(-1, mesh.dim)
        speed = float(np.max(np.linalg.norm(np.asarray(problem.beta(c), float).reshape(len(c), -1), axis=1)))
    elif hasattr(problem, "beta"):
        speed = float(np.linalg.norm(np.asarray(problem.beta, float)))
    elif hasattr(problem, "Phi"):
        speed = float(np.sqrt(problem.Phi))
    else:
        speed = 0.0
    return speed * dt * (p + 1) ** 2 / float(np.min(mesh.h))


def _diagnostic_report(solver, cfg, norm, max_iters, t0, return_state, return_trace, extra=None):
    d = _diagnostic_iterate(solver, cfg, norm, max_iters)
    h = d["history"]
    state = FieldState(solver.get_state(), solver.spec.labels, k=d["iterations"]) if return_state else None
    tr = solver.trace() if return_trace else None
    ex = {"device_seconds": d["seconds"], "l2_errors": h["l2_error"], "history": h,
          "convergence_map": d["maps"], "contraction_factor": d["contraction"],
          "trace_energy": h["trace_energy"], "jump_norm": h["jump_norm"]}
    ex.update(extra or {})
    return IterationReport(d["iterations"], d["status"], h["successive_norm"], time.perf_counter() - t0,
                           state, tr, d["first_norm"], d["last_norm"], d["iterations"], extra=ex)


def run_time_dependent(mesh, problem, ops: ElementOperators, cfg: Optional[IterationConfig],
                       dt: float, T: Optional[float] = None, n_steps: Optional[int] = None,
                       initial=None, solver: Optional[DeviceSolver] = None,
                       keep_states: bool = False, time_scheme: str = "backward-euler",
                       return_trace: bool = True) -> list:
    """Time steps; each step iterates from u^m.
    ``time_scheme``: "backward-euler" (= "locally-implicit": the implicit
    Euler HDG step solved by iHDG from the initial guess u^m, PAPER.md:593-653,
    SPEC.md:248) or "crank-nicolson" (trapezoidal split of the spatial
    operator).  Each report records the step's CFL number
    (SPEC.md:355, 400).  Divergence at any step aborts the run (the last report
    says which step)."""
    cfg = cfg or IterationConfig()
    ts = {"backward-euler": "BE", "be": "BE", "locally-implicit": "BE", "crank-nicolson": "CN",
          "cn": "CN"}.get(time_scheme.lower())
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
    f_t = _takes_time(forcing)
    if forcing is not None and solver.s_static is None and not f_t:
        solver.set_forcing(forcing)
    inflow = getattr(problem, "inflow", None)
    _set_initial(solver, initial if initial is not None else cfg.initial_guess)
    reports = []
    cfl = cfl_number(problem, mesh, ops.p, dt)
    for m in range(n_steps):
        t0 = time.perf_counter()
        t_old, t_new = m * dt, (m + 1) * dt
        # time-dependent forcing / inflow data: the new level (implicit Euler);
        # Crank-Nicolson averages the forcing and splits the boundary coupling
        # between the levels like the trace couplings
        if f_t:
            if ts == "CN":
                solver.set_forcing(lambda x, a=t_old, b=t_new: 0.5 * (np.asarray(forcing(x, a))
                                                                      + np.asarray(forcing(x, b))))
            else:
                solver.set_forcing(_exact_at(forcing, t_new))
        dirichlet = getattr(problem, "dirichlet", None)
        if dirichlet is not None:
            d_t = _takes_time(dirichlet)
            solver.set_dirichlet(_exact_at(dirichlet, t_new) if d_t else dirichlet,
                                 (_exact_at(dirichlet, t_old) if d_t else dirichlet) if ts == "CN" else None)
        if inflow is not None:
            g_t = _takes_time(inflow)
            solver.set_inflow(_exact_at(inflow, t_new) if g_t else inflow,
                              (_exact_at(inflow, t_old) if g_t else inflow) if ts == "CN" else None)
        solver.begin_step()
        if cfg.stop == "exact" or (cfg.diagnostics and getattr(problem, "exact", None) is not None):
            solver.set_exact(_exact_at(problem.exact, (m + 1) * dt))
        if cfg.stop == "vs-direct":   # one direct solution per step (a list), or one for all
            r = cfg.reference[m] if isinstance(cfg.reference, (list, tuple)) else cfg.reference
            solver.set_reference(r.data if isinstance(r, FieldState) else r)
        if cfg.diagnostics:
            keep = keep_states or m == n_steps - 1
            rep = _diagnostic_report(solver, cfg, _norm_name(cfg, problem),
                                     cfg.max_iters or default_max_iters(mesh), t0,
                                     keep, keep and return_trace, extra={"step": m + 1, "cfl": cfl})
            if rep.state is not None:
                rep.state.m = m + 1
            reports.append(rep)
            if rep.status != "converged":
                break
            continue
        res = solver.iterate(tol=cfg.tol, max_iters=cfg.max_iters or default_max_iters(mesh),
                             norm=_norm_name(cfg, problem), batch=cfg.check_every)
        last = m == n_steps - 1 or res.status != "converged"
        keep = keep_states or last
        st = (FieldState(solver.get_state(), solver.spec.labels, k=res.iterations, m=m + 1)
              if keep else None)
        # the step's single-valued trace with every state returned
        tr = solver.trace() if (keep and return_trace and not solver.spec.per_element and solver.layers[0] == 0
                                and solver.layers[1] == mesh.cells[-1]) else None
        reports.append(IterationReport(res.iterations, res.status, res.norms,
                                       time.perf_counter() - t0, st, tr, res.first_norm,
                                       res.last_norm, res.launched,
                                       extra={"step": m + 1, "device_seconds": res.seconds,
                                              "l2_errors": res.errors, "cfl": cfl, "kernel": res.kernel}))
        if res.status != "converged":
            break
    return reports
