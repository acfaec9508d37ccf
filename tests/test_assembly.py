"""The product's Kronecker term lists (input of K1) against the oracle's
quadrature assembly of the same iHDG-II local solvers."""

import numpy as np
import pytest

from oracle.ihdg_oracle import OracleSolver
from paper_1711_01175_b200.assembly import build_spec, evaluate_terms, neighbor_coupling, own_coupling
from paper_1711_01175_b200.basis import build_operators
from paper_1711_01175_b200.mesh import build_mesh
from paper_1711_01175_b200.pde import ConvectionDiffusionProblem, ShallowWaterProblem, TransportProblem
from tests.oracle_bridge import oracle_problem

CASES = [
    ("transport2d", 2, [5, 4], 2, TransportProblem(beta=np.array([1.0, 0.5])), None, False),
    ("transport2d_neg", 2, [3, 3], 3, TransportProblem(beta=np.array([-0.3, 0.8])), None, False),
    ("transport3d", 3, [3, 3, 3], 2, TransportProblem(beta=np.array([1.0, 0.7, 0.4])), None, False),
    ("transport1d", 1, [5], 3, TransportProblem(beta=np.array([1.0])), 0.1, False),
    ("cd2d", 2, [4, 4], 3, ConvectionDiffusionProblem(kappa=1e-2, beta=np.array([1.0, 1.0])), 1e-2, False),
    ("cd2d_steady", 2, [3, 3], 2, ConvectionDiffusionProblem(kappa=0.5, beta=np.array([0.3, -1.0]), nu=1.0), None, False),
    ("cd3d", 3, [3, 3, 3], 1, ConvectionDiffusionProblem(kappa=1e-1, beta=np.array([1.0, 0.5, -0.2])), 0.05, False),
    ("cd1d", 1, [4], 2, ConvectionDiffusionProblem(kappa=1.0, beta=np.array([0.0]), nu=1.0), None, False),
    ("sw_periodic", 2, [4, 4], 3, ShallowWaterProblem(Phi=1.0, f0=1.0), 5e-3, True),
    ("sw_walls", 2, [3, 3], 2, ShallowWaterProblem(Phi=2.0, f0=0.3, gamma=0.1), 1e-2, False),
]


@pytest.mark.parametrize("name,dim,cells,p,prob,dt,periodic", CASES, ids=[c[0] for c in CASES])
def test_local_operators_match_oracle(name, dim, cells, p, prob, dt, periodic):
    mesh = build_mesh(dim, cells, periodic=periodic)
    ops = build_operators(p, dim, mesh.h)
    spec = build_spec(mesh, prob, ops, dt)
    A, B, R = evaluate_terms(spec)
    S = OracleSolver(oracle_problem(prob, dim), cells, p, periodic=[periodic] * dim, dt=dt)
    masks = spec.class_masks
    for ci, mk in enumerate(masks):
        C = S.classes[mk if prob.kind != "transport" else 0]
        scale = np.max(np.abs(C["A"]))
        assert np.max(np.abs(A[ci] - C["A"])) <= 1e-12 * scale, f"A mismatch class {mk}"
        for f in range(2 * dim):
            if mk & (1 << f):
                continue
            Np_ = neighbor_coupling(spec, B[ci], f)
            No = C["N"][f]
            assert np.max(np.abs(Np_ - No)) <= 1e-12 * max(scale, 1.0), f"coupling face {f} class {mk}"
        if dt is not None:
            npn = spec.n_nodes
            cols = slice(spec.time_comp0 * npn, (spec.time_comp0 + spec.n_time_comp) * npn)
            assert np.max(np.abs(R[ci][:, : spec.nr] - C["R"][:, cols])) <= 1e-12 * scale
    # lifted form L = A^-1 B is well defined (factor once)
    for ci in range(spec.n_class):
        assert np.isfinite(np.linalg.cond(A[ci]))


@pytest.mark.parametrize("name,dim,cells,p,prob,dt,periodic", CASES, ids=[c[0] for c in CASES])
def test_ihdg1_operators_match_oracle(name, dim, cells, p, prob, dt, periodic):
    """iHDG-I (all-iterate-k trace): A_I, neighbour and own
    couplings from the term lists vs the oracle's A - T and Own = -T."""
    mesh = build_mesh(dim, cells, periodic=periodic)
    ops = build_operators(p, dim, mesh.h)
    spec = build_spec(mesh, prob, ops, dt, scheme="iHDG-I")
    A, B, R = evaluate_terms(spec)
    S = OracleSolver(oracle_problem(prob, dim), cells, p, periodic=[periodic] * dim, dt=dt, scheme="I")
    for ci, mk in enumerate(spec.class_masks):
        C = S.classes[mk if prob.kind != "transport" else 0]
        scale = max(np.max(np.abs(C["A"])), 1.0)
        assert np.max(np.abs(A[ci] - C["A"])) <= 1e-12 * scale, f"A_I mismatch class {mk}"
        for f in range(2 * dim):
            if mk & (1 << f):
                continue
            assert np.max(np.abs(neighbor_coupling(spec, B[ci], f) - C["N"][f])) <= 1e-12 * scale
        assert np.max(np.abs(own_coupling(spec, B[ci], mk) - C["Own"])) <= 1e-12 * scale, f"own class {mk}"
        assert np.isfinite(np.linalg.cond(A[ci]))


CN_CASES = [c for c in CASES if c[5] is not None]


@pytest.mark.parametrize("scheme", ["iHDG-II", "iHDG-I"])
@pytest.mark.parametrize("name,dim,cells,p,prob,dt,periodic", CN_CASES, ids=[c[0] for c in CN_CASES])
def test_crank_nicolson_operators_match_oracle(name, dim, cells, p, prob, dt, periodic, scheme):
    """Crank-Nicolson split: LHS R + Theta S, iterate-k
    couplings Theta B, explicit R - (1-Theta) S and (1-Theta) B, against the
    oracle's trapezoidal operators."""
    mesh = build_mesh(dim, cells, periodic=periodic)
    ops = build_operators(p, dim, mesh.h)
    spec = build_spec(mesh, prob, ops, dt, scheme=scheme, time_scheme="CN")
    A, B, R = evaluate_terms(spec)
    Ax, Bx, _ = evaluate_terms(spec, expl=True)
    S = OracleSolver(oracle_problem(prob, dim), cells, p, periodic=[periodic] * dim, dt=dt,
                     scheme="I" if scheme == "iHDG-I" else "II", time_scheme="CN")
    assert spec.nr == spec.nv and spec.time_comp0 == 0
    for ci, mk in enumerate(spec.class_masks):
        C = S.classes[mk if prob.kind != "transport" else 0]
        scale = max(np.max(np.abs(C["A"])), 1.0)
        assert np.max(np.abs(A[ci] - C["A"])) <= 1e-12 * scale
        assert np.max(np.abs(Ax[ci] - C["A"])) <= 1e-12 * scale
        assert np.max(np.abs(R[ci][:, : spec.nr] - C["R"])) <= 1e-12 * scale
        for f in range(2 * dim):
            if mk & (1 << f):
                continue
            assert np.max(np.abs(neighbor_coupling(spec, B[ci], f) - C["N"][f])) <= 1e-12 * scale
            assert np.max(np.abs(neighbor_coupling(spec, Bx[ci], f) - C["Nx"][f])) <= 1e-12 * scale
        assert np.max(np.abs(own_coupling(spec, B[ci], mk) - C["Own"])) <= 1e-12 * scale
        assert np.max(np.abs(own_coupling(spec, Bx[ci], mk) - C["Ownx"])) <= 1e-12 * scale


def test_class_enumeration():
    mesh = build_mesh(2, [5, 5])
    ops = build_operators(1, 2, mesh.h)
    spec = build_spec(mesh, ConvectionDiffusionProblem(kappa=1.0, beta=np.zeros(2), nu=1.0), ops)
    assert spec.n_class == 9
    mesh = build_mesh(2, [5, 5], periodic=True)
    spec = build_spec(mesh, ShallowWaterProblem(), build_operators(1, 2, mesh.h), dt=0.1)
    assert spec.n_class == 1
    mesh = build_mesh(3, [2, 1, 4])
    spec = build_spec(mesh, ConvectionDiffusionProblem(kappa=1.0, beta=np.zeros(3), nu=1.0),
                      build_operators(1, 3, mesh.h))
    assert spec.n_class == 2 * 1 * 3


def test_homogeneous_local_solve_is_zero():
    """zero neighbour data, zero forcing -> zero."""
    for prob, dt, dim in [(TransportProblem(beta=np.array([1.0, 0.5])), None, 2),
                          (ConvectionDiffusionProblem(kappa=1e-2, beta=np.array([1.0, 1.0])), 1e-2, 2),
                          (ShallowWaterProblem(), 1e-2, 2)]:
        mesh = build_mesh(dim, [3, 3])
        spec = build_spec(mesh, prob, build_operators(2, dim, mesh.h), dt)
        A, B, R = evaluate_terms(spec)
        for ci in range(spec.n_class):
            x = np.linalg.solve(A[ci], np.zeros(spec.nv))
            assert np.all(x == 0)


def test_1d_constant_transport():
    """1D [0,h], beta=1, p=1, f=0, inflow u_ext=1 -> u == 1."""
    mesh = build_mesh(1, [1], (np.zeros(1), np.array([0.3])))
    spec = build_spec(mesh, TransportProblem(beta=np.array([1.0])), build_operators(1, 1, mesh.h))
    A, B, R = evaluate_terms(spec)
    q = np.zeros(spec.kin)
    q[0] = 1.0  # inflow face (low side) neighbour value
    u = np.linalg.solve(A[0], B[0] @ q)
    assert np.allclose(u, 1.0, atol=1e-14)
