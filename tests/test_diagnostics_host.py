"""Host side of the per-iteration diagnostics (no GPU): the oracle's layer
map against SPEC.md:346-348, its trace-energy / jump restatement against
direct quadrature, and the report helpers (contraction factor, CSV, map)."""

import csv

import numpy as np
import pytest


def _oracle_transport(dim, cells, p, beta, seed=5):
    from oracle.ihdg_oracle import OracleProblem, OracleSolver
    from paper_1711_01175_b200.workloads import fourier_modes

    S = OracleSolver(OracleProblem("transport", dim, beta=np.array(beta, float)), cells, p)
    S.set_forcing(fourier_modes(np.random.default_rng(seed), dim))
    return S


def test_oracle_layer_map_4x4():
    """SPEC.md:346-347 on the oracle: 7 layers to coverage, corner first."""
    S = _oracle_transport(2, [4, 4], 2, [1.0, 1.0])
    o = S.run(tol=1e-10, keep_history=True)
    maps = S.diagnostics(o["history"], o["u"])["maps"]
    assert np.flatnonzero(maps[0]).tolist() == [0]
    assert next(j for j, m in enumerate(maps, 1) if m.all()) == 7


def test_oracle_layer_map_1d():
    """element j converged at iteration j."""
    S = _oracle_transport(1, [5], 2, [1.0])
    o = S.run(tol=1e-10, keep_history=True)
    maps = S.diagnostics(o["history"], o["u"])["maps"]
    for j in range(1, 6):
        assert np.flatnonzero(maps[j - 1]).tolist() == list(range(j))


def test_oracle_face_energy_of_constant_trace():
    """||1||^2 over the skeleton = total face measure (2D: 2 N (N+1) h)."""
    S = _oracle_transport(2, [3, 3], 3, [1.0, 1.0])
    t = S.trace(np.zeros((S.nel, S.nv)))
    ones = np.ones_like(t)
    n, h = 3, 1.0 / 3
    assert np.isclose(S.face_energy(ones), 2 * n * (n + 1) * h, rtol=1e-13)
    assert S.face_energy(ones, ones) == 0.0


def test_oracle_jump_of_continuous_field_is_zero():
    """A globally continuous polynomial (degree <= p) has no skeleton jump."""
    S = _oracle_transport(2, [3, 2], 2, [1.0, 1.0])
    u = S.interpolate(lambda x: 1.0 + x[:, 0] * x[:, 1] - x[:, 1] ** 2)
    assert np.max(np.abs(S.jump_faces(u.reshape(S.nel, -1), 0))) < 1e-13


def test_contraction_factor_geometric_mean():
    from paper_1711_01175_b200.iteration import contraction_factor

    e = 3.0 * 0.5 ** np.arange(12)
    assert np.isclose(contraction_factor(e), 0.5, rtol=1e-12)
    assert np.isnan(contraction_factor([1.0]))


def test_history_csv_and_map_helpers(tmp_path):
    from paper_1711_01175_b200.iteration import (HISTORY_COLUMNS, IterationReport, layer_convergence_map,
                                                 write_history_csv)

    hist = {"iteration": np.array([1, 2]), "l2_error": np.array([np.nan, np.nan]),
            "successive_norm": np.array([1.0, 1e-11]), "trace_energy": np.array([0.5, 0.0]),
            "converged_elements": np.array([1, 2]), "elapsed_ms": np.array([0.1, 0.2])}
    maps = [np.array([True, False]), np.array([True, True])]
    rep = IterationReport(2, "converged", hist["successive_norm"], 0.0,
                          extra={"history": hist, "convergence_map": maps})
    assert layer_convergence_map(rep) == [{0}, {0, 1}]
    p = tmp_path / "h.csv"
    write_history_csv(rep, p)
    rows = list(csv.reader(open(p)))
    assert tuple(rows[0]) == HISTORY_COLUMNS and len(rows) == 3
    assert float(rows[2][2]) == 1e-11 and rows[2][4] == "2"
    with pytest.raises(ValueError):
        layer_convergence_map(IterationReport(1, "converged", np.zeros(1), 0.0))


def test_cfl_number_definition():
    """CFL = |beta|_max dt (p+1)^2 / h."""
    from paper_1711_01175_b200.iteration import cfl_number
    from paper_1711_01175_b200.mesh import build_mesh
    from paper_1711_01175_b200.pde import ShallowWaterProblem, TransportProblem

    mesh = build_mesh(3, [8, 8, 8])
    prob = TransportProblem(beta=np.array([0.2, 0.2, 0.2]))
    assert np.isclose(cfl_number(prob, mesh, 4, 0.01), np.sqrt(3) * 0.2 * 0.01 * 25 * 8)
    mesh2 = build_mesh(2, [4, 8])
    assert np.isclose(cfl_number(ShallowWaterProblem(Phi=4.0), mesh2, 1, 0.1), 2.0 * 0.1 * 4 * 8)


def test_oracle_inflow_constant_is_transported():
    """1D, beta = 1, p = 1, f = 0, inflow value 1 -> solution 1."""
    from oracle.ihdg_oracle import OracleProblem, OracleSolver

    S = OracleSolver(OracleProblem("transport", 1, beta=np.array([1.0])), [4], 1)
    S.set_inflow(lambda x: np.ones(len(x)))
    o = S.run(tol=1e-12)
    assert o["status"] == "converged"
    assert np.max(np.abs(o["u"] - 1.0)) < 1e-13
    assert np.allclose(S.trace(o["u"]), 1.0, atol=1e-13)


def test_oracle_manufactured_transport3d_timedep_forcing():
    """The preset's manufactured forcing is the strong residual of u^e."""
    from paper_1711_01175_b200.pde import preset_problems

    pr = preset_problems()["transport3d_timedep"]
    rng = np.random.default_rng(0)
    x, t, eps = rng.random((20, 3)), 0.3, 1e-6
    ut = (pr.exact(x, t + eps) - pr.exact(x, t - eps)) / (2 * eps)
    grad = np.stack([(pr.exact(x + eps * np.eye(3)[a], t) - pr.exact(x - eps * np.eye(3)[a], t)) / (2 * eps)
                     for a in range(3)], axis=1)
    res = ut + grad @ pr.beta - pr.forcing(x, t)
    assert np.max(np.abs(res)) < 1e-8


def test_oracle_cn_inflow_is_the_level_average():
    """Crank-Nicolson inflow term = half new-level + half old-level data."""
    from oracle.ihdg_oracle import OracleProblem, OracleSolver

    pr = OracleProblem("transport", 2, beta=np.array([1.0, 0.5]))
    S = OracleSolver(pr, [3, 3], 2, dt=0.1, time_scheme="CN")
    B = OracleSolver(pr, [3, 3], 2, dt=0.1)
    g1, g0 = (lambda x: 1.0 + x[:, 0]), (lambda x: x[:, 1] ** 2)
    S.set_inflow(g1, g0)
    B.set_inflow(g1)
    b1 = B.b_inflow.copy()
    B.set_inflow(g0)
    assert np.allclose(S.b_inflow, 0.5 * (b1 + B.b_inflow), rtol=0, atol=1e-15)


@pytest.mark.parametrize("dim,cells,p", [(2, [3, 4], 2), (3, [2, 2, 3], 1), (1, [5], 3)])
def test_dirichlet_data_terms_match_oracle(dim, cells, p):
    """The product's Dirichlet-data couplings B_D (term lists, K1's input)
    applied to g at the boundary face nodes = the oracle's quadrature of
    -<g, tau.n> and +tau <g, v>, for every element."""
    from oracle.ihdg_oracle import OracleProblem, OracleSolver
    from paper_1711_01175_b200.assembly import build_spec, evaluate_terms, face_node_indices
    from paper_1711_01175_b200.basis import build_operators
    from paper_1711_01175_b200.mesh import build_mesh
    from paper_1711_01175_b200.pde import ConvectionDiffusionProblem

    beta = np.array([1.0, -0.5, 0.3])[:dim]
    g = lambda x: 1.0 + np.sin(2 * x[:, 0]) + (x[:, -1] ** 2 if x.shape[1] > 1 else 0.0)  # noqa: E731
    mesh = build_mesh(dim, cells)
    ops = build_operators(p, dim, mesh.h)
    prob = ConvectionDiffusionProblem(kappa=0.1, beta=beta, dirichlet=g)
    sp = build_spec(mesh, prob, ops, 0.05)
    _, BD, _ = evaluate_terms(sp, which="dir")
    S = OracleSolver(OracleProblem("cd", dim, beta=beta, kappa=0.1), cells, p, dt=0.05)
    S.set_dirichlet(g)
    pts = S.element_points(S.b.nodes)
    nf = (p + 1) ** (dim - 1)
    for e in range(S.nel):
        q = np.zeros(2 * dim * nf)
        for f in range(2 * dim):
            if S.nbr[e, f] == -1:
                q[f * nf:(f + 1) * nf] = g(pts[e][face_node_indices(dim, p + 1, f)])
        c = sp.class_of_mask[S.mask[e]]
        assert np.allclose(BD[c] @ q, S.b_inflow[e], rtol=1e-12, atol=1e-13)


def test_dirichlet_data_terms_crank_nicolson_match_oracle():
    """Crank-Nicolson split of the Dirichlet-data couplings (theta = 1 on the
    sigma rows, 1/2 on the u row): theta B_D q(g_new) + (1 - theta) B_D q(g_old)
    equals the oracle's CN data term for every element."""
    from oracle.ihdg_oracle import OracleProblem, OracleSolver
    from paper_1711_01175_b200.assembly import build_spec, evaluate_terms, face_node_indices
    from paper_1711_01175_b200.basis import build_operators
    from paper_1711_01175_b200.mesh import build_mesh
    from paper_1711_01175_b200.pde import ConvectionDiffusionProblem

    dim, cells, p = 2, [3, 3], 2
    beta = np.array([1.0, -0.5])
    g1 = lambda x: 1.0 + x[:, 0] * x[:, 1]   # noqa: E731
    g0 = lambda x: np.cos(x[:, 1])           # noqa: E731
    mesh = build_mesh(dim, cells)
    ops = build_operators(p, dim, mesh.h)
    sp = build_spec(mesh, ConvectionDiffusionProblem(kappa=0.1, beta=beta, dirichlet=g1), ops, 0.05,
                    time_scheme="CN")
    _, B1, _ = evaluate_terms(sp, which="dir")
    _, B0, _ = evaluate_terms(sp, which="dir_expl")
    S = OracleSolver(OracleProblem("cd", dim, beta=beta, kappa=0.1), cells, p, dt=0.05, time_scheme="CN")
    S.set_dirichlet(g1, g0)
    pts = S.element_points(S.b.nodes)
    nf = p + 1
    for e in range(S.nel):
        q1, q0 = np.zeros(4 * nf), np.zeros(4 * nf)
        for f in range(4):
            if S.nbr[e, f] == -1:
                ids = face_node_indices(dim, p + 1, f)
                q1[f * nf:(f + 1) * nf] = g1(pts[e][ids])
                q0[f * nf:(f + 1) * nf] = g0(pts[e][ids])
        c = sp.class_of_mask[S.mask[e]]
        assert np.allclose(B1[c] @ q1 + B0[c] @ q0, S.b_inflow[e], rtol=1e-12, atol=1e-13)
