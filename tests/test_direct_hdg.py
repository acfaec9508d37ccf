"""The direct HDG oracle (oracle/reference_hdg.py): its
known-answer examples and its agreement with the
iteration oracle's fixed point -- two independent formulations (trace as an
unknown vs trace formula substituted) of the same HDG solution."""

import numpy as np
import pytest

from oracle.ihdg_oracle import OracleProblem
from oracle.reference_hdg import DirectHDG, solve_direct
from tests.oracle_bridge import oracle_initial, oracle_problem, oracle_solver, rel_l2


def _exact_at_nodes(D, fn):
    return fn(D.element_points(D.b.nodes).reshape(-1, D.d)).reshape(D.nel, D.npn)


@pytest.mark.parametrize("dim,p", [(2, 2), (2, 3), (3, 2)])
def test_transport_polynomial_exactness(dim, p):
    """a manufactured polynomial of degree <= p is recovered to 1e-11."""
    beta = np.array([1.0, 0.5, 0.25])[:dim]
    if dim == 2:
        u = lambda x: 3.0 + x[:, 0] ** 2 + x[:, 0] * x[:, 1]
        f = lambda x: beta[0] * (2 * x[:, 0] + x[:, 1]) + beta[1] * x[:, 0]
    else:
        u = lambda x: 1.0 + x[:, 0] * x[:, 2] + x[:, 1] ** 2
        f = lambda x: beta[0] * x[:, 2] + beta[1] * 2 * x[:, 1] + beta[2] * x[:, 0]
    D = DirectHDG(OracleProblem("transport", dim, beta=beta), [3] * dim, p)
    uu, t = D.solve(forcing=f, inflow=u)
    assert np.max(np.abs(uu - _exact_at_nodes(D, u))) < 1e-11


def test_cd_polynomial_exactness():
    """Convection-diffusion: u in Q_p, Dirichlet data = u, sigma = -kappa grad u."""
    kappa, beta = 0.1, np.array([1.0, 0.5])
    u = lambda x: 1.0 + x[:, 0] + x[:, 1] ** 2
    f = lambda x: -kappa * 2.0 + beta[0] * 1.0 + beta[1] * 2 * x[:, 1]
    D = DirectHDG(OracleProblem("cd", 2, beta=beta, kappa=kappa), [3, 3], 2)
    uu, _ = D.solve(forcing=f, dirichlet=u)
    ue = _exact_at_nodes(D, u)
    assert np.max(np.abs(uu[:, 2 * D.npn:] - ue)) < 1e-11
    sx = -kappa * np.ones_like(ue)
    assert np.max(np.abs(uu[:, :D.npn] - sx)) < 1e-11


@pytest.mark.parametrize("p", [1, 2, 3])
def test_cd_refinement_rate(p):
    """L2 error(h) / error(h/2) >= 2^p under refinement
    (2D manufactured u = sin(pi x) sin(pi y), constant beta)."""
    kappa, beta = 1.0, np.array([1.0, 1.0])
    pi = np.pi
    u = lambda x: np.sin(pi * x[:, 0]) * np.sin(pi * x[:, 1])
    f = lambda x: (2 * kappa * pi ** 2 * u(x) + pi * (beta[0] * np.cos(pi * x[:, 0]) * np.sin(pi * x[:, 1])
                                                     + beta[1] * np.sin(pi * x[:, 0]) * np.cos(pi * x[:, 1])))
    errs = []
    for n in (4, 8):
        D = DirectHDG(OracleProblem("cd", 2, beta=beta, kappa=kappa), [n, n], p)
        uu, _ = D.solve(forcing=f)
        pts = D.element_points(D.b.qx).reshape(-1, 2)
        uq = uu[:, 2 * D.npn:] @ D.el.Phi.T
        e2 = ((uq - u(pts).reshape(D.nel, -1)) ** 2 * D.el.W[None, :]).sum()
        errs.append(np.sqrt(e2))
    assert errs[0] / errs[1] >= 2 ** p, errs


@pytest.mark.parametrize("cfg,kw", [(1, {}), (2, {"cells": 8, "n_steps": 1}), (3, {"cells": 8, "n_steps": 1}),
                                    (4, {"cells": 4}), (5, {"cells": 8, "n_steps": 1, "kappa": 1e-1})])
def test_iteration_fixed_point_is_the_hdg_solution(cfg, kw):
    """The iteration oracle converged to 1e-14 equals the direct HDG solve
    (volume and trace) on every BASELINE configuration, reduced."""
    from paper_1711_01175_b200.workloads import make_config

    wl = make_config(cfg, **kw)
    S = oracle_solver(wl)
    m = wl.mesh
    D = DirectHDG(oracle_problem(wl.problem, m.dim), m.cells, wl.ops.p, box=(m.lo, m.hi),
                  periodic=m.periodic, dt=wl.dt)
    f = getattr(wl.problem, "forcing", None)
    if wl.dt is None:
        r = S.run(tol=1e-14, max_iters=100000)
        u, t = D.solve(forcing=f)
    else:
        u0 = oracle_initial(wl, S)
        r = S.run(u0=u0, u_prev=u0, tol=1e-14, max_iters=100000)
        u, t = D.solve(forcing=f, u_prev=u0)
    assert r["status"] == "converged"
    assert rel_l2(u, r["u"]) < 1e-10
    assert rel_l2(t[:, None, :], S.trace(r["u"])) < 1e-10


def test_shallow_water_walls_fixed_point():
    """Mirror walls: the direct solve's wall condition against the iteration."""
    prob = OracleProblem("sw", 2, Phi=1.0, f_cor=1.0, gamma=0.0)
    from oracle.ihdg_oracle import OracleSolver

    S = OracleSolver(prob, [6, 6], 2, dt=1e-2)
    rng = np.random.default_rng(1)
    u0 = rng.normal(size=(S.nel, S.nv))
    r = S.run(u0=u0, u_prev=u0, tol=1e-14, max_iters=100000)
    u, t = DirectHDG(prob, [6, 6], 2, dt=1e-2).solve(u_prev=u0)
    assert rel_l2(u, r["u"]) < 1e-10
    assert rel_l2(t[:, None, :], S.trace(r["u"])) < 1e-10


def test_solve_direct_shapes_and_size_limit():
    prob = OracleProblem("transport", 2, beta=np.array([1.0, 1.0]))
    u, t = solve_direct(prob, [4, 4], 2)
    assert u.shape == (16, 1, 9) and t.shape == (40, 1, 3)
    assert np.all(u == 0.0)          # f = 0, g = 0 -> zero
    with pytest.raises(ValueError):
        DirectHDG(OracleProblem("cd", 2, beta=np.ones(2)), [64, 64], 6)
