"""Device parity with the CPU oracle beyond the BASELINE configs: other
orders, dimensions and boundary treatments, each through the same C-ABI
(generic and streaming kernels).  Bar: same iteration count, fields within
1e-10 relative L2."""

import numpy as np
import pytest

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module", autouse=True)
def _gpu():
    import torch

    if not torch.cuda.is_available():
        pytest.skip("needs a CUDA device")
    torch.cuda.set_device(0)


def _fields(dim, seed):
    from paper_1711_01175_b200.workloads import fourier_modes

    return fourier_modes(np.random.default_rng(seed), dim)


CASES = [
    # name, dim, cells, p, kind, params, dt, periodic, init comp
    ("transport2d_negbeta_p3", 2, [8, 6], 3, "transport", dict(beta=[-0.7, 0.4]), None, False, None),
    ("transport3d_p2_generic", 3, [4, 3, 5], 2, "transport", dict(beta=[0.5, 1.0, 0.3]), None, False, None),
    ("transport1d_p4", 1, [12], 4, "transport", dict(beta=[1.0]), None, False, None),
    ("cd2d_steady_p2", 2, [6, 5], 2, "cd", dict(kappa=0.3, beta=[0.5, -1.0], nu=1.0), None, False, None),
    ("cd2d_be_p3", 2, [8, 8], 3, "cd", dict(kappa=1e-2, beta=[1.0, 1.0]), 0.02, False, "u"),
    ("cd3d_be_p1", 3, [3, 4, 3], 1, "cd", dict(kappa=0.1, beta=[1.0, 0.5, 0.2]), 0.05, False, "u"),
    ("cd1d_steady_p3", 1, [7], 3, "cd", dict(kappa=1.0, beta=[0.0], nu=1.0), None, False, None),
    ("sw_walls_p3", 2, [6, 6], 3, "sw", dict(Phi=1.0, f0=0.5, gamma=0.1), 1e-2, False, "phi"),
    ("sw_periodic_p2", 2, [8, 4], 2, "sw", dict(Phi=2.0, f0=1.0), 5e-3, True, "phi"),
]


@pytest.mark.parametrize("name,dim,cells,p,kind,params,dt,periodic,init", CASES, ids=[c[0] for c in CASES])
def test_variant_parity(name, dim, cells, p, kind, params, dt, periodic, init):
    from oracle.ihdg_oracle import OracleProblem, OracleSolver
    from paper_1711_01175_b200.basis import build_operators
    from paper_1711_01175_b200.iteration import IterationConfig, run, run_time_dependent
    from paper_1711_01175_b200.mesh import build_mesh
    from paper_1711_01175_b200.pde import ConvectionDiffusionProblem, ShallowWaterProblem, TransportProblem
    from tests.oracle_bridge import rel_l2

    mesh = build_mesh(dim, cells, periodic=periodic)
    ops = build_operators(p, dim, mesh.h)
    f = _fields(dim, 11)
    if kind == "transport":
        prob = TransportProblem(beta=np.array(params["beta"]), forcing=f)
        oprob = OracleProblem("transport", dim, beta=np.array(params["beta"]))
    elif kind == "cd":
        prob = ConvectionDiffusionProblem(kappa=params["kappa"], beta=np.array(params["beta"]),
                                          nu=params.get("nu", 0.0), forcing=None if dt else f)
        oprob = OracleProblem("cd", dim, beta=np.array(params["beta"]), kappa=params["kappa"],
                              nu=params.get("nu", 0.0))
    else:
        prob = ShallowWaterProblem(Phi=params["Phi"], f0=params["f0"], gamma=params.get("gamma", 0.0))
        oprob = OracleProblem("sw", dim, Phi=params["Phi"], f_cor=params["f0"], gamma=params.get("gamma", 0.0))
    S = OracleSolver(oprob, cells, p, periodic=[periodic] * dim, dt=dt)
    if getattr(prob, "forcing", None) is not None:
        S.set_forcing(prob.forcing)
    cfg = IterationConfig(tol=1e-10)
    if dt is None:
        rep = run(mesh, prob, ops, cfg)
        ref = S.run(tol=1e-10)
        assert rep.iterations == ref["iterations"]
        assert rep.status == ref["status"] == "converged"
        assert rel_l2(rep.state.data.reshape(S.nel, -1), ref["u"]) < 1e-10
        assert rel_l2(rep.trace, S.trace(ref["u"])) < 1e-10
    else:
        labels = prob.labels(dim)
        reps = run_time_dependent(mesh, prob, ops, cfg, dt, n_steps=2, initial={init: f}, keep_states=True)
        u0 = np.zeros((S.nel, S.m, S.npn))
        u0[:, labels.index(init), :] = S.interpolate(f)
        _, refs = S.run_time_dependent(u0.reshape(S.nel, -1), 2, tol=1e-10)
        assert [r.iterations for r in reps] == [r["iterations"] for r in refs]
        for r, o in zip(reps, refs):
            assert rel_l2(r.state.data.reshape(S.nel, -1), o["u"]) < 1e-10


def test_unsupported_order_raises():
    from paper_1711_01175_b200.basis import build_operators
    from paper_1711_01175_b200.iteration import run
    from paper_1711_01175_b200.mesh import build_mesh
    from paper_1711_01175_b200.pde import TransportProblem

    mesh = build_mesh(2, [4, 4])
    with pytest.raises(NotImplementedError):
        run(mesh, TransportProblem(beta=np.array([1.0, 1.0])), build_operators(8, 2, mesh.h))
