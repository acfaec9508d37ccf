"""Parity of the sm_100a sweep (through the C-ABI) with the CPU oracle.

Bar (BASELINE.json north_star): the same iteration count to convergence and
volume / trace fields within 1e-10 relative L2 in fp64.
"""

import numpy as np
import pytest

pytestmark = pytest.mark.gpu

TOL_FIELD = 1e-10


@pytest.fixture(scope="module", autouse=True)
def _gpu():
    import torch

    if not torch.cuda.is_available():
        pytest.skip("needs a CUDA device")
    torch.cuda.set_device(0)


def _wl(cfg, **kw):
    from paper_1711_01175_b200.workloads import make_config

    return make_config(cfg, seed=kw.pop("seed", 0), **kw)


def _steady(wl, stop):
    from paper_1711_01175_b200.iteration import IterationConfig, run
    from tests.oracle_bridge import oracle_solver

    rep = run(wl.mesh, wl.problem, wl.ops, IterationConfig(stop=stop, tol=1e-10))
    S = oracle_solver(wl)
    ref = S.run(norm="trace" if stop == "trace" else "volume", tol=1e-10)
    return rep, S, ref


def _unsteady(wl):
    from paper_1711_01175_b200.iteration import IterationConfig, run_time_dependent
    from tests.oracle_bridge import oracle_initial, oracle_solver

    reps = run_time_dependent(wl.mesh, wl.problem, wl.ops, IterationConfig(tol=1e-10), wl.dt,
                              n_steps=wl.n_steps, initial=wl.initial, keep_states=True)
    S = oracle_solver(wl)
    u_end, refs = S.run_time_dependent(oracle_initial(wl, S), wl.n_steps, tol=1e-10)
    return reps, S, refs


def test_config1_full_size_parity():
    from tests.oracle_bridge import rel_l2

    wl = _wl(1)
    rep, S, ref = _steady(wl, "trace")
    assert rep.status == ref["status"] == "converged"
    assert rep.iterations == ref["iterations"] == 2 * 16  # 2N-1 layers + detection sweep
    assert rel_l2(rep.state.data.reshape(S.nel, -1), ref["u"]) < TOL_FIELD
    assert rel_l2(rep.trace, S.trace(ref["u"])) < TOL_FIELD
    assert np.allclose(rep.successive_norms, ref["norms"], rtol=1e-8, atol=1e-300)


def test_config1_volume_rule():
    from tests.oracle_bridge import rel_l2

    wl = _wl(1, seed=3)
    rep, S, ref = _steady(wl, "successive")
    assert rep.iterations == ref["iterations"]
    assert rel_l2(rep.state.data.reshape(S.nel, -1), ref["u"]) < TOL_FIELD


@pytest.mark.parametrize("cells,steps,kernel", [(16, 2, "k_sweep_v3"), (32, 1, "k_sweep_v3"),
                                                (20, 1, "k_sweep")])
def test_config2_reduced_parity(cells, steps, kernel):
    """20^2 has tile rows that are not a multiple of the 8-element tile: the
    generic kernel runs (asserted), the others run v3 (one round of tiles;
    the register-tiled v5 is covered by test_sweep_impl_parity and at full
    size)."""
    from tests.oracle_bridge import rel_l2

    wl = _wl(2, cells=cells, n_steps=steps)
    reps, S, refs = _unsteady(wl)
    assert all(r.extra["kernel"] == kernel for r in reps)
    assert [r.iterations for r in reps] == [r["iterations"] for r in refs]
    assert all(r.status == "converged" for r in reps)
    for r, o in zip(reps, refs):
        assert rel_l2(r.state.data.reshape(S.nel, -1), o["u"]) < TOL_FIELD


def test_config3_reduced_parity():
    from tests.oracle_bridge import rel_l2

    wl = _wl(3, cells=16, n_steps=2)
    reps, S, refs = _unsteady(wl)
    assert all(r.extra["kernel"] == "k_sweep_v3" for r in reps)
    assert [r.iterations for r in reps] == [r["iterations"] for r in refs]
    for r, o in zip(reps, refs):
        assert rel_l2(r.state.data.reshape(S.nel, -1), o["u"]) < TOL_FIELD


@pytest.mark.parametrize("beta,impl,kernel", [
    ((1.0, 0.7, 0.4), "v3", "k_sweep_v3"), ((-1.0, 0.7, -0.4), "auto", "k_sweep_v4"),
    ((1.0, -0.7, 0.4), "auto", "k_sweep_v4"), ((-0.3, -0.7, 1.0), "auto", "k_sweep_v4"),
    ((1.0, 0.0, 0.4), "auto", "k_sweep")])
def test_config4_kernels_by_inflow_faces(beta, impl, kernel):
    """3D p=3 transport: k_sweep_v4 has one instantiation per inflow-face set
    (sign pattern of beta); the v3 selector and a beta with a zero component
    (two coupled faces: generic kernel) are checked alike, all against the
    oracle on a 16^3 mesh."""
    import dataclasses

    from paper_1711_01175_b200 import _native as N
    from paper_1711_01175_b200.pde import TransportProblem
    from tests.oracle_bridge import rel_l2

    wl = _wl(4, cells=16)
    prob = TransportProblem(beta=np.array(beta), forcing=wl.problem.forcing)
    wl = dataclasses.replace(wl, problem=prob, params={**wl.params, "beta": list(beta)})
    N.set_sweep_impl(impl)
    try:
        rep, S, ref = _steady(wl, "successive")
    finally:
        N.set_sweep_impl("auto")
    assert rep.extra["kernel"] == kernel
    assert rep.status == ref["status"] == "converged"
    assert rep.iterations == ref["iterations"]
    assert rel_l2(rep.state.data.reshape(S.nel, -1), ref["u"]) < TOL_FIELD
    assert np.allclose(rep.successive_norms, ref["norms"], rtol=1e-7, atol=1e-300)


def test_config4_reduced_parity():
    from tests.oracle_bridge import rel_l2

    wl = _wl(4, cells=8)
    rep, S, ref = _steady(wl, "successive")
    assert rep.extra["kernel"] == "k_sweep_v4"
    assert rep.iterations == ref["iterations"] == 3 * 7 + 1 + 1
    assert rel_l2(rep.state.data.reshape(S.nel, -1), ref["u"]) < TOL_FIELD
    assert rel_l2(rep.trace, S.trace(ref["u"])) < TOL_FIELD


@pytest.mark.parametrize("kappa", [1e-1, 1e-3])
def test_config5_reduced_parity(kappa):
    from tests.oracle_bridge import rel_l2

    wl = _wl(5, cells=32, kappa=kappa, n_steps=1)
    reps, S, refs = _unsteady(wl)
    assert all(r.extra["kernel"] == "k_sweep_ws" for r in reps)
    assert [r.iterations for r in reps] == [r["iterations"] for r in refs]
    for r, o in zip(reps, refs):
        assert rel_l2(r.state.data.reshape(S.nel, -1), o["u"]) < TOL_FIELD


def test_device_assembly_matches_host_terms():
    """K1 (device Kronecker assembly + Gauss-Jordan) vs numpy."""
    from paper_1711_01175_b200.assembly import evaluate_terms
    from paper_1711_01175_b200.solver import DeviceSolver

    wl = _wl(5, cells=8, kappa=1e-1)
    ds = DeviceSolver(wl.mesh, wl.problem, wl.ops, dt=wl.dt)
    A, B, R = evaluate_terms(ds.spec)
    Ad = ds.A.cpu().numpy()
    assert np.max(np.abs(Ad - A)) <= 1e-14 * np.max(np.abs(A))
    Ai = np.linalg.inv(A)
    Aid = ds.Ainv.cpu().numpy()
    assert np.max(np.abs(Aid - Ai)) <= 1e-10 * np.max(np.abs(Ai))
    L = np.einsum("cij,cjk->cik", Ai, B)
    assert np.max(np.abs(ds.LT.cpu().numpy().transpose(0, 2, 1) - L)) <= 1e-10 * np.max(np.abs(L))


def test_zero_problem_one_iteration():
    """f = 0, g = 0, zero initial guess -> 1 iteration, zero solution."""
    from paper_1711_01175_b200.basis import build_operators
    from paper_1711_01175_b200.iteration import IterationConfig, run
    from paper_1711_01175_b200.mesh import build_mesh
    from paper_1711_01175_b200.pde import TransportProblem

    mesh = build_mesh(2, [8, 8])
    rep = run(mesh, TransportProblem(beta=np.array([1.0, 1.0])), build_operators(2, 2, mesh.h),
              IterationConfig())
    assert rep.iterations == 1 and rep.status == "converged"
    assert np.all(rep.state.data == 0.0)


def test_repeat_is_bit_identical():
    from paper_1711_01175_b200.iteration import IterationConfig, run

    wl = _wl(1, seed=7)
    r1 = run(wl.mesh, wl.problem, wl.ops, IterationConfig(stop="trace"))
    r2 = run(wl.mesh, wl.problem, wl.ops, IterationConfig(stop="trace"))
    assert r1.iterations == r2.iterations
    assert np.array_equal(r1.state.data, r2.state.data)
    assert np.array_equal(r1.successive_norms, r2.successive_norms)


def test_max_iter_status():
    from paper_1711_01175_b200.iteration import IterationConfig, run

    wl = _wl(1)
    rep = run(wl.mesh, wl.problem, wl.ops, IterationConfig(stop="trace", max_iters=5))
    assert rep.status == "max-iter" and rep.iterations == 5


def test_config4_full_size_layer_count():
    """64^3: the iterate is exact after 3*63+1 = 190 layer sweeps (Theorem
    DDMConvergence; PAPER.md:1426 reports 190 at 64^3), so with tol -> 0 the
    run stops at sweep 191 with a successive difference of exactly zero.  At
    tol = 1e-10 it stops earlier (data dependent) and must match the count of
    the same device run repeated (determinism)."""
    from paper_1711_01175_b200.iteration import IterationConfig, run

    wl = _wl(4)
    rep = run(wl.mesh, wl.problem, wl.ops, IterationConfig(tol=1e-300), return_trace=False)
    assert rep.status == "converged"
    assert rep.iterations == 191
    assert rep.successive_norms[-1] == 0.0 and rep.successive_norms[-2] > 0.0
    r1 = run(wl.mesh, wl.problem, wl.ops, IterationConfig(), return_trace=False)
    r2 = run(wl.mesh, wl.problem, wl.ops, IterationConfig(), return_trace=False)
    assert r1.iterations == r2.iterations < 191
    assert np.array_equal(r1.state.data, r2.state.data)


IMPL_CASES = [  # (selector, graphs, config, cells, expected kernel)
    ("auto", True, 5, 16, "k_sweep_ws"), ("generic", True, 5, 16, "k_sweep"),
    ("auto", False, 5, 16, "k_sweep_ws"),
    ("auto", True, 2, 16, "k_sweep_v3"), ("v5", True, 2, 16, "k_sweep_v5"), ("ws", True, 2, 16, "k_sweep_ws"),
    ("generic", True, 2, 16, "k_sweep"),
    ("auto", True, 3, 16, "k_sweep_v3"), ("v5", True, 3, 16, "k_sweep_v5"), ("ws", True, 3, 16, "k_sweep_ws"),
    ("v5", False, 2, 32, "k_sweep_v5"),
]


@pytest.mark.parametrize("impl,graphs,cfg,cells,kernel", IMPL_CASES,
                         ids=[f"cfg{c}-{i}-{'graph' if g else 'stream'}" for i, g, c, _, _ in IMPL_CASES])
def test_sweep_impl_parity(impl, graphs, cfg, cells, kernel):
    """Every selectable sweep kernel (ihdg_set_sweep_impl, switched in
    process) and the stream-launched (not graph-replayed) iterate loop,
    against the oracle; the dispatched kernel is asserted by name."""
    from paper_1711_01175_b200 import _native as N
    from tests.oracle_bridge import rel_l2

    wl = _wl(cfg, cells=cells, n_steps=1, **({"kappa": 1e-1} if cfg == 5 else {}))
    N.set_sweep_impl(impl)
    N.set_graphs(graphs)
    try:
        reps, S, refs = _unsteady(wl)
    finally:
        N.set_sweep_impl("auto")
        N.set_graphs(True)
    assert all(r.extra["kernel"] == kernel for r in reps), [r.extra["kernel"] for r in reps]
    assert [r.iterations for r in reps] == [r["iterations"] for r in refs]
    for r, o in zip(reps, refs):
        assert rel_l2(r.state.data.reshape(S.nel, -1), o["u"]) < TOL_FIELD



# PAPER.md:1349-1395 (Table 2) / SPEC.md acceptance 1: 2D N x N -> {9, 17, 33, 65} for N = 4..32,
# 3D N^3 -> {6, 12, 23, 47} for N = 2..16, within +-2 (any p)
TABLE2 = [(2, 4, 9), (2, 8, 17), (2, 16, 33), (2, 32, 65), (3, 2, 6), (3, 4, 12), (3, 8, 23), (3, 16, 47)]


@pytest.mark.parametrize("dim,n,paper", TABLE2, ids=[f"{d}d_{n}" for d, n, _ in TABLE2])
def test_table2_transport_counts(dim, n, paper):
    """Steady diagonal transport (transport2d_diag / transport3d_diag) on the
    device: iteration counts within +-2 of Table 2 for p = 1..4 (p <= 3 in 3D)."""
    from paper_1711_01175_b200.basis import build_operators
    from paper_1711_01175_b200.iteration import IterationConfig, run
    from paper_1711_01175_b200.mesh import build_mesh
    from paper_1711_01175_b200.pde import TransportProblem
    from paper_1711_01175_b200.workloads import fourier_modes

    mesh = build_mesh(dim, [n] * dim)
    f = fourier_modes(np.random.default_rng(3), dim)
    for p in (1, 2, 3, 4) if dim == 2 else (1, 2, 3):
        rep = run(mesh, TransportProblem(beta=np.ones(dim), forcing=f), build_operators(p, dim, mesh.h),
                  IterationConfig(stop="trace", tol=1e-10), return_trace=False)
        assert rep.status == "converged"
        assert abs(rep.iterations - paper) <= 2, (p, rep.iterations, paper)


@pytest.mark.parametrize("cfg,cells,kw", [(5, 32, {"kappa": 1e-1}), (5, 32, {"kappa": 1e-3}), (2, 32, {})])
def test_gram_norm_matches_direct(cfg, cells, kw):
    """The Gram-form norm of k_sweep_ws (ihdg_sweep_args.q_store) against the
    direct mass-norm of the same kernel: identical counts, identical first
    sweep (direct in both), later norms equal to the rounding of the
    successive difference (relative to |u|, so looser as it shrinks)."""
    from paper_1711_01175_b200 import _native as N
    from paper_1711_01175_b200.solver import DeviceSolver

    wl = _wl(cfg, cells=cells, n_steps=1, **kw)
    if cfg == 2:
        N.set_sweep_impl("ws")
    try:
        out = []
        for gram in (True, False):
            sv = DeviceSolver(wl.mesh, wl.problem, wl.ops, dt=wl.dt, gram_norm=True)
            assert sv.gram_kc == 4 * (wl.ops.p + 1)
            if not gram:
                sv.gram_kc = 0
            for name, fld in wl.initial.items():
                sv.set_state_component(fld, sv.spec.labels.index(name))
            sv.begin_step()
            r = sv.iterate(tol=1e-10, max_iters=100000)
            assert r.kernel == "k_sweep_ws"
            out.append((r, sv.get_state()))
    finally:
        N.set_sweep_impl("auto")
    (rg, ug), (rd, ud) = out
    assert rg.iterations == rd.iterations and rg.status == rd.status == "converged"
    assert rg.norms[0] == rd.norms[0]
    assert np.array_equal(ug, ud)          # the norm never feeds back into the fields
    big = rd.norms > 1e-6 * rd.norms[0]
    assert np.allclose(rg.norms[big], rd.norms[big], rtol=1e-9, atol=0)
    assert np.allclose(rg.norms, rd.norms, rtol=1e-4, atol=0)
