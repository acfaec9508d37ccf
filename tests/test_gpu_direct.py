"""Device iHDG against the direct HDG oracle (oracle/reference_hdg.py):
acceptance 2 (||u_iHDG - u_direct||_{L2} < 1e-8 at termination
for the Table-2 configurations) on the BASELINE configurations reduced, and
the vs-direct stopping rule against the oracle's count."""

import numpy as np
import pytest

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module", autouse=True)
def _gpu():
    import torch

    if not torch.cuda.is_available():
        pytest.skip("needs a CUDA device")
    torch.cuda.set_device(0)


def _direct(wl, u_prev=None):
    from oracle.reference_hdg import DirectHDG
    from tests.oracle_bridge import oracle_problem

    m = wl.mesh
    D = DirectHDG(oracle_problem(wl.problem, m.dim), m.cells, wl.ops.p, box=(m.lo, m.hi),
                  periodic=m.periodic, dt=wl.dt)
    u, t = D.solve(forcing=getattr(wl.problem, "forcing", None), u_prev=u_prev)
    return D, u, t


TABLE2 = [(2, n, p) for n in (4, 8, 16, 32) for p in (1, 2)] + [(3, n, p) for n in (2, 4, 8) for p in (1, 2)] \
    + [(3, 16, 1)]


@pytest.mark.parametrize("dim,n,p", TABLE2, ids=[f"{d}d_{n}_p{p}" for d, n, p in TABLE2])
def test_acceptance2_table2_vs_direct(dim, n, p):
    """Table-2 transport (beta = 1, seeded forcing), trace rule at 1e-10 on
    the device: the terminated iterate is the HDG solution to 1e-8 (L2)."""
    from oracle.reference_hdg import DirectHDG
    from oracle.ihdg_oracle import OracleProblem
    from paper_1711_01175_b200.basis import build_operators
    from paper_1711_01175_b200.iteration import IterationConfig, run
    from paper_1711_01175_b200.mesh import build_mesh
    from paper_1711_01175_b200.pde import TransportProblem
    from paper_1711_01175_b200.workloads import fourier_modes

    mesh = build_mesh(dim, [n] * dim)
    f = fourier_modes(np.random.default_rng(3), dim)
    rep = run(mesh, TransportProblem(beta=np.ones(dim), forcing=f), build_operators(p, dim, mesh.h),
              IterationConfig(stop="trace", tol=1e-10))
    assert rep.status == "converged"
    D = DirectHDG(OracleProblem("transport", dim, beta=np.ones(dim)), [n] * dim, p)
    u, t = D.solve(forcing=f)
    diff = rep.state.data.reshape(D.nel, -1) - u
    assert D.l2_norm(diff) < 1e-8
    assert np.max(np.abs(rep.trace[:, 0, :] - t)) < 1e-8


@pytest.mark.parametrize("cfg,kw", [(1, {}), (2, {"cells": 16}), (3, {"cells": 16}), (4, {"cells": 8}),
                                    (5, {"cells": 16, "kappa": 1e-1}), (5, {"cells": 16, "kappa": 1e-3})])
def test_baseline_configs_vs_direct(cfg, kw):
    """Every BASELINE configuration (reduced, first step): the converged
    device iterate against the direct HDG solve, volume and trace."""
    from paper_1711_01175_b200.iteration import IterationConfig, run, run_time_dependent
    from paper_1711_01175_b200.workloads import make_config
    from tests.oracle_bridge import oracle_initial, oracle_solver

    wl = make_config(cfg, n_steps=1, **kw)
    if wl.dt is None:
        rep = run(wl.mesh, wl.problem, wl.ops, IterationConfig(stop="successive", tol=1e-10))
        D, u, t = _direct(wl)
    else:
        rep = run_time_dependent(wl.mesh, wl.problem, wl.ops, IterationConfig(tol=1e-10), wl.dt, n_steps=1,
                                 initial=wl.initial)[0]
        S = oracle_solver(wl)
        D, u, t = _direct(wl, u_prev=oracle_initial(wl, S))
    assert rep.status == "converged"
    assert D.l2_norm(rep.state.data.reshape(D.nel, -1) - u) < 1e-8
    assert np.max(np.abs(rep.trace[:, 0, :] - t)) < 1e-7 * max(1.0, np.max(np.abs(t)))


@pytest.mark.parametrize("cfg,kw", [(1, {}), (4, {"cells": 8}), (5, {"cells": 16, "kappa": 1e-1})])
def test_vs_direct_stopping_rule(cfg, kw):
    """stop = "vs-direct": ||u^k - u_direct||_{L2} < tol, evaluated on the
    device (K5 mode 2) every sweep; same count as the oracle with the same
    rule, final distance below tol."""
    from paper_1711_01175_b200.basis import FieldState
    from paper_1711_01175_b200.iteration import IterationConfig, run, run_time_dependent
    from paper_1711_01175_b200.workloads import make_config
    from tests.oracle_bridge import oracle_initial, oracle_solver, rel_l2

    tol = 1e-9
    wl = make_config(cfg, n_steps=1, **kw)
    S = oracle_solver(wl)
    if wl.dt is None:
        D, u, _ = _direct(wl)
        ref = S.run(tol=tol, norm="vs-direct", reference=u)
        cfgi = IterationConfig(stop="vs-direct", tol=tol, reference=FieldState(u.reshape(D.nel, D.m, D.npn),
                                                                              wl.problem.labels(wl.mesh.dim)))
        rep = run(wl.mesh, wl.problem, wl.ops, cfgi)
    else:
        u0 = oracle_initial(wl, S)
        D, u, _ = _direct(wl, u_prev=u0)
        ref = S.run(u0=u0, u_prev=u0, tol=tol, norm="vs-direct", reference=u)
        rep = run_time_dependent(wl.mesh, wl.problem, wl.ops,
                                 IterationConfig(stop="vs-direct", tol=tol, reference=u), wl.dt, n_steps=1,
                                 initial=wl.initial)[0]
    assert rep.status == ref["status"] == "converged"
    assert rep.iterations == ref["iterations"]
    errs = rep.extra["l2_errors"]
    assert errs[-1] < tol <= errs[-2]
    assert np.allclose(errs, ref["errors"], rtol=1e-6, atol=1e-14)
    assert rel_l2(rep.state.data.reshape(S.nel, -1), ref["u"]) < 1e-10
