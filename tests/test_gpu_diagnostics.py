"""Per-iteration diagnostics of iteration.run on the device (K6) against the
CPU oracle: element convergence map / layer_convergence_map,
trace energy and skeleton jump norm, measured contraction
factor and the per-iteration CSV."""

import csv

import numpy as np
import pytest

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module", autouse=True)
def _gpu():
    import torch

    if not torch.cuda.is_available():
        pytest.skip("needs a CUDA device")
    torch.cuda.set_device(0)


def _transport(dim, cells, p, beta, seed=5):
    from oracle.ihdg_oracle import OracleProblem, OracleSolver
    from paper_1711_01175_b200.basis import build_operators
    from paper_1711_01175_b200.mesh import build_mesh
    from paper_1711_01175_b200.pde import TransportProblem
    from paper_1711_01175_b200.workloads import fourier_modes

    mesh = build_mesh(dim, cells)
    ops = build_operators(p, dim, mesh.h)
    f = fourier_modes(np.random.default_rng(seed), dim)
    prob = TransportProblem(beta=np.array(beta, float), forcing=f)
    S = OracleSolver(OracleProblem("transport", dim, beta=np.array(beta, float)), cells, p)
    S.set_forcing(f)
    return mesh, ops, prob, S


def _diag_run(mesh, prob, ops, **kw):
    from paper_1711_01175_b200.iteration import IterationConfig, run

    return run(mesh, prob, ops, IterationConfig(tol=1e-10, diagnostics=True, **kw))


def test_layer_map_2d_4x4_diagonal_flow():
    """4x4, beta=(1,1): full coverage after 2*4-1 = 7 sweeps,
    after sweep 1 exactly the inflow corner; set j = first j anti-diagonals."""
    from paper_1711_01175_b200.iteration import layer_convergence_map

    mesh, ops, prob, S = _transport(2, [4, 4], 2, [1.0, 1.0])
    rep = _diag_run(mesh, prob, ops)
    sets = layer_convergence_map(rep)
    assert sets[0] == {0}
    full = next(j for j, s in enumerate(sets, 1) if len(s) == 16)
    assert full == 7
    for j, s in enumerate(sets, 1):
        expect = {i + 4 * k for i in range(4) for k in range(4) if i + k <= j - 1}
        assert s == expect, j
    # the oracle's own map (its history against its converged solution)
    o = S.run(tol=1e-10, keep_history=True)
    od = S.diagnostics(o["history"], o["u"])
    assert len(od["maps"]) == rep.iterations
    for dm, om in zip(rep.extra["convergence_map"], od["maps"]):
        assert np.array_equal(dm, om)


def test_layer_map_1d_element_j_at_iteration_j():
    """1D, 5 elements, beta=1: element j converged at iteration j."""
    from paper_1711_01175_b200.iteration import layer_convergence_map

    mesh, ops, prob, _ = _transport(1, [5], 3, [1.0])
    sets = layer_convergence_map(_diag_run(mesh, prob, ops))
    for j in range(1, 6):
        assert sets[j - 1] == set(range(j))


def test_layer_map_3d_monotone_and_layer_count():
    """Monotone layer sweep: nested sets, at least one full
    anti-diagonal layer per iteration, sum(N_i - 1) + 1 layers to coverage."""
    from paper_1711_01175_b200.iteration import layer_convergence_map

    cells = [4, 3, 5]
    mesh, ops, prob, _ = _transport(3, cells, 2, [0.5, 1.0, 0.3])
    sets = layer_convergence_map(_diag_run(mesh, prob, ops))
    n = int(np.prod(cells))
    for a, b in zip(sets, sets[1:]):
        assert a <= b
    full = next(j for j, s in enumerate(sets, 1) if len(s) == n)
    assert full == sum(c - 1 for c in cells) + 1


@pytest.mark.parametrize("kind", ["cd", "sw"])
def test_trace_energy_jump_and_contraction_vs_oracle(kind, tmp_path):
    """Skeleton energy ||(phi, theta.n)(u^k - u_HDG)||^2_{E_h} (or (sigma.n, u))
    and the skeleton jump norm per iteration agree with the oracle; the converged-element counts
    agree exactly; the contraction factor is < 1; the CSV has one row per
    iteration with the SPEC.md:398 columns."""
    from oracle.ihdg_oracle import OracleProblem, OracleSolver
    from paper_1711_01175_b200.basis import build_operators
    from paper_1711_01175_b200.iteration import (HISTORY_COLUMNS, IterationConfig, run_time_dependent,
                                                 write_history_csv)
    from paper_1711_01175_b200.mesh import build_mesh
    from paper_1711_01175_b200.pde import ConvectionDiffusionProblem, ShallowWaterProblem
    from paper_1711_01175_b200.workloads import fourier_modes

    dim, cells, p, dt = 2, [6, 5], 3, 0.02
    mesh = build_mesh(dim, cells)
    ops = build_operators(p, dim, mesh.h)
    f = fourier_modes(np.random.default_rng(3), dim)
    if kind == "cd":
        prob = ConvectionDiffusionProblem(kappa=0.05, beta=np.array([1.0, 0.5]))
        S = OracleSolver(OracleProblem("cd", dim, beta=np.array([1.0, 0.5]), kappa=0.05), cells, p, dt=dt)
        init = "u"
    else:
        prob = ShallowWaterProblem(Phi=1.0, f0=1.0)
        S = OracleSolver(OracleProblem("sw", dim, Phi=1.0, f_cor=1.0), cells, p, dt=dt)
        init = "phi"
    labels = prob.labels(dim)
    reps = run_time_dependent(mesh, prob, ops, IterationConfig(tol=1e-10, diagnostics=True), dt, n_steps=1,
                              initial={init: f})
    rep = reps[0]
    u0 = np.zeros((S.nel, S.m, S.npn))
    u0[:, labels.index(init), :] = S.interpolate(f)
    u0 = u0.reshape(S.nel, -1)
    o = S.run(u0=u0, u_prev=u0, tol=1e-10, keep_history=True)
    assert rep.iterations == o["iterations"] and rep.status == o["status"] == "converged"
    od = S.diagnostics(o["history"], o["u"])
    e_dev, e_or = rep.extra["trace_energy"], od["trace_energy"]
    big = e_or > 1e-14
    assert big.sum() >= 3
    assert np.allclose(e_dev[big], e_or[big], rtol=1e-7, atol=0)
    j_dev, j_or = rep.extra["jump_norm"], od["jump_norm"]
    assert np.allclose(j_dev, j_or, rtol=1e-8, atol=1e-13)
    counts_or = [int(m.sum()) for m in od["maps"]]
    assert list(rep.extra["history"]["converged_elements"]) == counts_or
    assert counts_or[-1] == S.nel
    rho = rep.extra["contraction_factor"]
    assert 0.0 < rho < 1.0
    path = tmp_path / "hist.csv"
    write_history_csv(rep, path)
    rows = list(csv.reader(open(path)))
    assert tuple(rows[0]) == HISTORY_COLUMNS
    assert len(rows) == rep.iterations + 1
    assert float(rows[-1][2]) == rep.successive_norms[-1]


def test_diagnostics_same_count_as_batched_run():
    """Diagnostic mode runs sweep by sweep but stops at the same sweep, with
    bit-identical successive norms, as the batched graph-replay path."""
    from paper_1711_01175_b200.iteration import IterationConfig, run

    mesh, ops, prob, _ = _transport(2, [8, 8], 2, [1.0, 0.5])
    a = run(mesh, prob, ops, IterationConfig(tol=1e-10))
    b = _diag_run(mesh, prob, ops)
    assert a.iterations == b.iterations
    assert np.array_equal(a.successive_norms, b.successive_norms)
    assert np.array_equal(a.state.data, b.state.data)


@pytest.mark.parametrize("kind", ["sw", "cd"])
def test_contraction_bound_acceptance8(kind):
    """SPEC.md:384 / acceptance 8: on admissible configs the
    measured skeleton-energy ratio E_{k+1}/E_k (the theorems' norm,
    ||(phi, theta.n)||^2 or ||(sigma.n, u)||^2 of the error iterate) is <= the
    predicted C (shallow water) or D (convection-diffusion,
    PAPER.md:1090-1111) for every iteration after the first, with c = 1/2
    calibrated for the basis (theory.trace_inequality_constant)."""
    from paper_1711_01175_b200.basis import build_operators
    from paper_1711_01175_b200.iteration import IterationConfig, run_time_dependent
    from paper_1711_01175_b200.mesh import build_mesh
    from paper_1711_01175_b200.pde import ConvectionDiffusionProblem, ShallowWaterProblem
    from paper_1711_01175_b200.theory import predict_cdr, predict_sw, trace_inequality_constant
    from paper_1711_01175_b200.workloads import fourier_modes

    n = 8
    h = 1.0 / n
    if kind == "sw":
        p, dt = 1, 0.005
        prob = ShallowWaterProblem(Phi=1.0)
        est = predict_sw(h, p, dt, 1.0, c=trace_inequality_constant(p, 2))
        init = "phi"
    else:
        p, dt = 2, 1e-3
        prob = ConvectionDiffusionProblem(kappa=1e-3, beta=np.array([1.0, 0.5]))
        est = predict_cdr(h, p, 2, 1e-3, 0.0, [1.0, 0.5], c=trace_inequality_constant(p, 2), dt=dt)
        init = "u"
    assert est.admissible and est.contraction < 1
    mesh = build_mesh(2, [n, n])
    ops = build_operators(p, 2, mesh.h)
    f = fourier_modes(np.random.default_rng(4), 2)
    rep = run_time_dependent(mesh, prob, ops, IterationConfig(tol=1e-10, diagnostics=True), dt, n_steps=1,
                             initial={init: f})[0]
    assert rep.status == "converged"
    e = rep.extra["trace_energy"]
    ratios = [e[k + 1] / e[k] for k in range(1, len(e) - 1) if e[k + 1] > 1e-14]
    assert len(ratios) >= 1
    assert max(ratios) <= est.contraction, (max(ratios), est.contraction)
    assert rep.extra["contraction_factor"] <= est.contraction
