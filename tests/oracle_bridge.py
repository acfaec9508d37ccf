"""Map product workloads onto the CPU oracle (test infrastructure)."""

from __future__ import annotations

import numpy as np

from oracle.ihdg_oracle import OracleProblem, OracleSolver
from paper_1711_01175_b200.pde import ConvectionDiffusionProblem, ShallowWaterProblem, TransportProblem


def oracle_problem(problem, dim) -> OracleProblem:
    if isinstance(problem, TransportProblem):
        return OracleProblem("transport", dim, beta=np.asarray(problem.beta, float),
                             reaction=problem.reaction)
    if isinstance(problem, ConvectionDiffusionProblem):
        return OracleProblem("cd", dim, beta=np.asarray(problem.beta, float), kappa=problem.kappa,
                             nu=problem.nu)
    if isinstance(problem, ShallowWaterProblem):
        return OracleProblem("sw", dim, Phi=problem.Phi, f_cor=problem.f0, gamma=problem.gamma)
    raise TypeError(type(problem))


def oracle_solver(wl) -> OracleSolver:
    mesh = wl.mesh
    prob = oracle_problem(wl.problem, mesh.dim)
    S = OracleSolver(prob, mesh.cells, wl.ops.p, box=(mesh.lo, mesh.hi), periodic=mesh.periodic,
                     dt=wl.dt)
    forcing = getattr(wl.problem, "forcing", None)
    if forcing is not None:
        S.set_forcing(forcing)
    return S


def oracle_initial(wl, S: OracleSolver) -> np.ndarray:
    labels = wl.problem.labels(wl.mesh.dim)
    u0 = np.zeros((S.nel, S.m, S.npn))
    for name, fld in wl.initial.items():
        u0[:, labels.index(name), :] = S.interpolate(fld)
    return u0.reshape(S.nel, S.nv)


def rel_l2(a, b) -> float:
    a = np.asarray(a, float).ravel()
    b = np.asarray(b, float).ravel()
    den = np.linalg.norm(b)
    return float(np.linalg.norm(a - b) / (den if den > 0 else 1.0))
