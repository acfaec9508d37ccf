"""Locally-implicit time stepping:
each implicit-Euler HDG step is solved by iHDG from the initial guess u^m.
Acceptance 10 and the SPEC.md:357 example on the device, and
parity of the mode with the CPU oracle."""

import numpy as np
import pytest

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module", autouse=True)
def _gpu():
    import torch

    if not torch.cuda.is_available():
        pytest.skip("needs a CUDA device")
    torch.cuda.set_device(0)


def _setup(cells, p):
    from paper_1711_01175_b200.basis import build_operators
    from paper_1711_01175_b200.mesh import build_mesh
    from paper_1711_01175_b200.pde import preset_problems

    mesh = build_mesh(3, cells)
    ops = build_operators(p, 3, mesh.h)
    # transport3d_timedep: manufactured forcing, inflow g = u^e
    prob = preset_problems()["transport3d_timedep"]
    init = lambda x: prob.exact(x, 0.0)   # noqa: E731
    return mesh, ops, prob, init


def _iters_per_step(mesh, ops, prob, init, dt, steps=3):
    from paper_1711_01175_b200.iteration import IterationConfig, run_time_dependent

    reps = run_time_dependent(mesh, prob, ops, IterationConfig(tol=1e-10), dt, n_steps=steps,
                              initial={"u": init}, time_scheme="locally-implicit")
    assert all(r.status == "converged" for r in reps)
    return float(np.mean([r.iterations for r in reps])), reps[0].extra["cfl"]


def test_acceptance10_cfl_iterations_grow_mildly():
    """iterations/step at CFL ~5 <= 3x iterations/step at CFL ~1."""
    mesh, ops, prob, init = _setup([8, 8, 8], 4)
    speed = np.linalg.norm(prob.beta)
    dt1 = 1.0 * mesh.h[0] / (speed * 25)
    k1, c1 = _iters_per_step(mesh, ops, prob, init, dt1)
    k5, c5 = _iters_per_step(mesh, ops, prob, init, 5 * dt1)
    assert np.isclose(c1, 1.0) and np.isclose(c5, 5.0)
    assert k5 <= 3 * k1, (k1, k5)


def test_spec357_cfl_045_vs_18():
    """8^3, p = 4: iterations/step at CFL ~1.8 vs ~0.45 grows < 2x."""
    mesh, ops, prob, init = _setup([8, 8, 8], 4)
    unit = mesh.h[0] / (np.linalg.norm(prob.beta) * 25)   # dt of CFL 1
    k_hi, c_hi = _iters_per_step(mesh, ops, prob, init, 1.8 * unit)
    k_lo, c_lo = _iters_per_step(mesh, ops, prob, init, 0.45 * unit)
    assert np.isclose(c_hi, 1.8) and np.isclose(c_lo, 0.45)
    assert k_hi < 2 * k_lo, (k_lo, k_hi)


@pytest.mark.parametrize("stop", ["successive", "exact"])
def test_locally_implicit_parity_with_oracle(stop):
    """Two locally-implicit steps of transport3d_timedep (time-dependent
    forcing and inflow data) at CFL 5 on 4^3, p = 3: same iterations per step
    as the oracle under both stopping rules, fields within 1e-10 relative L2;
    the solution tracks u^e (implicit-Euler error at CFL 5 < 5e-2; ||u^e|| ~ 0.4)."""
    from oracle.ihdg_oracle import OracleProblem, OracleSolver
    from paper_1711_01175_b200.iteration import IterationConfig, run_time_dependent
    from tests.oracle_bridge import rel_l2

    mesh, ops, prob, init = _setup([4, 4, 4], 3)
    dt = 5 * mesh.h[0] / (np.linalg.norm(prob.beta) * 16)
    reps = run_time_dependent(mesh, prob, ops, IterationConfig(tol=1e-10, stop=stop), dt, n_steps=2,
                              initial={"u": init}, keep_states=True, time_scheme="locally-implicit")
    S = OracleSolver(OracleProblem("transport", 3, beta=prob.beta), [4, 4, 4], 3, dt=dt)
    u = S.interpolate(init).reshape(S.nel, -1)
    for m, r in enumerate(reps):
        t = (m + 1) * dt
        S.set_forcing(lambda x: prob.forcing(x, t))
        S.set_inflow(lambda x: prob.inflow(x, t))
        if stop == "exact":
            S.set_exact(prob.exact, t)
        o = S.run(u0=u, u_prev=u, tol=1e-10, norm="volume" if stop == "successive" else "exact")
        assert r.iterations == o["iterations"] and r.status == o["status"] == "converged"
        assert rel_l2(r.state.data.reshape(S.nel, -1), o["u"]) < 1e-10
        u = o["u"]
        S.set_exact(prob.exact, t)
        assert S.err_norm(u) < 5e-2


def test_inflow_data_steady_parity():
    """Steady 2D transport with non-zero inflow data g and Fourier forcing:
    same count as the oracle, volume and trace (g on inflow faces) within
    1e-10 relative L2."""
    from oracle.ihdg_oracle import OracleProblem, OracleSolver
    from paper_1711_01175_b200.basis import build_operators
    from paper_1711_01175_b200.iteration import IterationConfig, run
    from paper_1711_01175_b200.mesh import build_mesh
    from paper_1711_01175_b200.pde import TransportProblem
    from paper_1711_01175_b200.workloads import fourier_modes
    from tests.oracle_bridge import rel_l2

    beta = np.array([0.7, -0.4])
    g = lambda x: 1.0 + np.sin(3 * x[:, 0]) * x[:, 1] + x[:, 0] ** 2   # noqa: E731
    f = fourier_modes(np.random.default_rng(2), 2)
    mesh = build_mesh(2, [6, 5])
    ops = build_operators(3, 2, mesh.h)
    rep = run(mesh, TransportProblem(beta=beta, forcing=f, inflow=g), ops, IterationConfig(tol=1e-10))
    S = OracleSolver(OracleProblem("transport", 2, beta=beta), [6, 5], 3)
    S.set_forcing(f)
    S.set_inflow(g)
    o = S.run(tol=1e-10)
    assert rep.iterations == o["iterations"] and rep.status == "converged"
    assert rel_l2(rep.state.data.reshape(S.nel, -1), o["u"]) < 1e-10
    assert rel_l2(rep.trace, S.trace(o["u"])) < 1e-10


def test_inflow_constant_transported_1d():
    """SPEC.md:253 on the device: 1D, beta = 1, p = 1, f = 0, g = 1 -> u = 1."""
    from paper_1711_01175_b200.basis import build_operators
    from paper_1711_01175_b200.iteration import IterationConfig, run
    from paper_1711_01175_b200.mesh import build_mesh
    from paper_1711_01175_b200.pde import TransportProblem

    mesh = build_mesh(1, [6])
    rep = run(mesh, TransportProblem(beta=np.array([1.0]), inflow=lambda x: np.ones(len(x))),
              build_operators(1, 1, mesh.h), IterationConfig(tol=1e-12))
    assert rep.status == "converged"
    assert np.max(np.abs(rep.state.data - 1.0)) < 1e-13
    assert np.allclose(rep.trace, 1.0, atol=1e-13)


def _cd_manufactured():
    """u^e = exp(x) sin(y) + 0.5 (harmonic part), kappa = 0.1, beta = (1, 0.5),
    nu = 1: f = beta . grad u + nu u, g_D = u^e."""
    from paper_1711_01175_b200.pde import ConvectionDiffusionProblem

    ue = lambda x: np.exp(x[:, 0]) * np.sin(x[:, 1]) + 0.5   # noqa: E731
    f = lambda x: (np.exp(x[:, 0]) * (1.0 * np.sin(x[:, 1]) + 0.5 * np.cos(x[:, 1]))  # noqa: E731
                   + ue(x))
    return ConvectionDiffusionProblem(kappa=0.1, beta=np.array([1.0, 0.5]), nu=1.0, forcing=f, dirichlet=ue,
                                      exact=ue), ue


def test_dirichlet_data_steady_parity_and_accuracy():
    """Steady convection-diffusion with Dirichlet data g_D = u^e and the
    manufactured forcing: same count as the oracle, volume and trace (g on
    the boundary) within 1e-10 relative L2, and the solution is u^e to the
    discretisation error."""
    from oracle.ihdg_oracle import OracleProblem, OracleSolver
    from paper_1711_01175_b200.basis import build_operators
    from paper_1711_01175_b200.iteration import IterationConfig, run
    from paper_1711_01175_b200.mesh import build_mesh
    from tests.oracle_bridge import rel_l2

    prob, ue = _cd_manufactured()
    mesh = build_mesh(2, [6, 5])
    ops = build_operators(3, 2, mesh.h)
    rep = run(mesh, prob, ops, IterationConfig(tol=1e-10))
    S = OracleSolver(OracleProblem("cd", 2, beta=prob.beta, kappa=0.1, nu=1.0), [6, 5], 3)
    S.set_forcing(prob.forcing)
    S.set_dirichlet(ue)
    o = S.run(tol=1e-10)
    assert rep.iterations == o["iterations"] and rep.status == o["status"] == "converged"
    assert rel_l2(rep.state.data.reshape(S.nel, -1), o["u"]) < 1e-10
    assert rel_l2(rep.trace, S.trace(o["u"])) < 1e-10
    S.set_exact(ue)
    u_only = np.zeros_like(o["u"]).reshape(S.nel, S.m, S.npn)
    u_only[:, 2, :] = o["u"].reshape(S.nel, S.m, S.npn)[:, 2, :]
    assert S.err_norm(u_only.reshape(S.nel, -1)) < 1e-4


@pytest.mark.parametrize("ts", ["BE", "CN"])
def test_dirichlet_data_time_dependent_parity(ts):
    """Two backward-Euler / Crank-Nicolson steps with time-dependent Dirichlet
    data g(x, t): iterations per step and fields as the oracle."""
    from oracle.ihdg_oracle import OracleProblem, OracleSolver
    from paper_1711_01175_b200.basis import build_operators
    from paper_1711_01175_b200.iteration import IterationConfig, run_time_dependent
    from paper_1711_01175_b200.mesh import build_mesh
    from paper_1711_01175_b200.pde import ConvectionDiffusionProblem
    from paper_1711_01175_b200.workloads import fourier_modes
    from tests.oracle_bridge import rel_l2

    g = lambda x, t=0.0: np.cos(x[:, 0] + 2 * t) * (1 + x[:, 1])   # noqa: E731
    prob = ConvectionDiffusionProblem(kappa=0.02, beta=np.array([1.0, 1.0]), dirichlet=g)
    mesh = build_mesh(2, [8, 8])
    ops = build_operators(2, 2, mesh.h)
    f0 = fourier_modes(np.random.default_rng(6), 2)
    dt = 0.02
    reps = run_time_dependent(mesh, prob, ops, IterationConfig(tol=1e-10), dt, n_steps=2, initial={"u": f0},
                              keep_states=True, time_scheme="crank-nicolson" if ts == "CN" else "backward-euler")
    S = OracleSolver(OracleProblem("cd", 2, beta=prob.beta, kappa=0.02), [8, 8], 2, dt=dt, time_scheme=ts)
    u = np.zeros((S.nel, S.m, S.npn))
    u[:, 2, :] = S.interpolate(f0)
    u = u.reshape(S.nel, -1)
    for m, r in enumerate(reps):
        t = (m + 1) * dt
        S.set_dirichlet(lambda x: g(x, t), lambda x: g(x, t - dt))
        o = S.run(u0=u, u_prev=u, tol=1e-10)
        assert r.iterations == o["iterations"] and r.status == o["status"] == "converged"
        assert rel_l2(r.state.data.reshape(S.nel, -1), o["u"]) < 1e-10
        u = o["u"]
