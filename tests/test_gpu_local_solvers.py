"""The per-element local_solvers API on the device against
one sweep of the fused kernel (the same local solves, all elements at once)
and its SPEC examples."""

import numpy as np
import pytest

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module", autouse=True)
def _gpu():
    import torch

    if not torch.cuda.is_available():
        pytest.skip("needs a CUDA device")
    torch.cuda.set_device(0)


def _one_sweep(wl, u0, forcing=None):
    from paper_1711_01175_b200.solver import DeviceSolver

    sv = DeviceSolver(wl.mesh, wl.problem, wl.ops, dt=wl.dt, max_iters=10)
    if forcing is not None:
        sv.set_forcing(forcing)
    sv.set_state(u0)
    if wl.dt is not None:
        sv.begin_step()
    else:
        sv.prepare_steady()
    sv.reset_state(1e-300, 1)
    sv.sweep_once(a=sv.sweep_args("volume", 1))
    return sv.get_state()


def _load_vector(wl, K, f):
    """(f, v)_K on the forcing component by the basis' quadrature (host)."""
    ops, d = wl.ops, wl.mesh.dim
    qp = wl.mesh.element_points(K, [ops.quad_points] * d)
    Bq = ops.quad_to_rhs
    Bd = Bq
    for _ in range(d - 1):
        Bd = np.kron(Bq, Bd)
    return ops.jacobian * (Bd @ np.asarray(f(qp), float))


@pytest.mark.parametrize("cfg,kw", [(5, {"cells": 16, "kappa": 1e-1}), (2, {"cells": 8}), (3, {"cells": 8})])
def test_apply_local_matches_the_sweep(cfg, kw):
    from paper_1711_01175_b200.local_solvers import (TraceSnapshot, apply_local, assemble_convection_diffusion,
                                                     assemble_shallow_water)
    from paper_1711_01175_b200.pde import ShallowWaterProblem
    from paper_1711_01175_b200.workloads import make_config

    wl = make_config(cfg, n_steps=1, **kw)
    m, npn = wl.problem.n_components(wl.mesh.dim), wl.ops.n_nodes
    u0 = np.random.default_rng(4).normal(size=(wl.mesh.n_elements, m, npn))
    ref = _one_sweep(wl, u0)
    asm = assemble_shallow_water if isinstance(wl.problem, ShallowWaterProblem) else assemble_convection_diffusion
    n = wl.mesh.cells[0]
    for K in (0, n - 1, n + 1, wl.mesh.n_elements - 1, wl.mesh.n_elements // 2 + 3):
        sysK = asm(K, wl.problem, wl.ops, ("backward-euler", wl.dt), mesh=wl.mesh)
        snap = TraceSnapshot.from_state(wl.mesh, u0, K)
        uK = apply_local(sysK, snap, forcing=None, prev_level=u0[K])
        assert np.max(np.abs(uK - ref[K])) <= 1e-12 * max(1.0, np.max(np.abs(ref[K])))
        assert np.array_equal(uK, apply_local(sysK, snap, prev_level=u0[K]))   # bit-identical repeat
        assert sysK.condition > 1 and np.isfinite(sysK.condition)


def test_apply_local_transport_with_forcing():
    from paper_1711_01175_b200.local_solvers import TraceSnapshot, apply_local, assemble_transport
    from paper_1711_01175_b200.workloads import make_config

    wl = make_config(4, cells=4)
    u0 = np.random.default_rng(5).normal(size=(wl.mesh.n_elements, 1, wl.ops.n_nodes))
    f = wl.problem.forcing
    ref = _one_sweep(wl, u0, forcing=f)
    for K in (0, 21, 63):
        sysK = assemble_transport(K, wl.problem, wl.ops, "steady", mesh=wl.mesh)
        uK = apply_local(sysK, TraceSnapshot.from_state(wl.mesh, u0, K), forcing=_load_vector(wl, K, f))
        assert np.max(np.abs(uK - ref[K])) <= 1e-12 * max(1.0, np.max(np.abs(ref[K])))


def test_local_solver_examples():
    """zero inputs -> zero; 1D element, beta = 1, p = 1,
    f = 0, inflow u_ext = 1 -> the local solution is identically 1."""
    from paper_1711_01175_b200.basis import build_operators
    from paper_1711_01175_b200.local_solvers import TraceSnapshot, apply_local, assemble_transport
    from paper_1711_01175_b200.mesh import build_mesh
    from paper_1711_01175_b200.pde import TransportProblem

    mesh = build_mesh(1, [1], (np.zeros(1), np.array([0.5])))
    ops = build_operators(1, 1, mesh.h)
    prob = TransportProblem(beta=np.array([1.0]))
    sysK = assemble_transport(0, prob, ops, "steady", mesh=mesh)
    zero = apply_local(sysK, TraceSnapshot(0, {}))
    assert np.all(zero == 0.0)
    one = apply_local(sysK, TraceSnapshot(0, {}, {0: np.array([1.0])}))
    assert np.max(np.abs(one - 1.0)) < 1e-13
