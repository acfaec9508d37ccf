"""pde module known answers and invariants
(SPEC.md:205-207): upwind_flux_matrix, stabilization data, presets."""

import numpy as np
import pytest

from paper_1711_01175_b200.pde import (ConvectionDiffusionProblem, ShallowWaterProblem, TransportProblem,
                                       preset_problems, stabilization, upwind_flux_matrix)


def test_transport_flux_kat():
    """beta.n = -0.5 -> A = -0.5, |A| = 0.5."""
    A, absA = upwind_flux_matrix(TransportProblem(beta=np.array([0.5, 0.0])), np.array([-1.0, 0.0]))
    assert A.shape == (1, 1) and A[0, 0] == -0.5 and absA[0, 0] == 0.5


def test_shallow_water_flux_kat():
    """Phi = 1, n = (1, 0): eig(A) = {-1, 0, 1}; |A| symmetric PSD with
    eigenvalues {1, 0, 1}."""
    A, absA = upwind_flux_matrix(ShallowWaterProblem(Phi=1.0), np.array([1.0, 0.0]))
    assert np.allclose(np.sort(np.linalg.eigvals(A).real), [-1.0, 0.0, 1.0], atol=1e-12)
    assert np.allclose(absA, absA.T, atol=1e-12)
    ev = np.sort(np.linalg.eigvalsh(absA))
    assert np.allclose(ev, [0.0, 1.0, 1.0], atol=1e-12) and ev.min() >= -1e-12


@pytest.mark.parametrize("Phi", [0.25, 1.0, 4.0])
def test_shallow_water_flux_reconstruction(Phi):
    """|A| = R |S| R^-1 from the eigendecomposition of A = R S R^-1, which
    reconstructs A to 1e-12; |A| A = A |A| and eigenvalues {+-sqrt(Phi), 0}
    for every unit normal."""
    rng = np.random.default_rng(0)
    for _ in range(20):
        n = rng.normal(size=2)
        n /= np.linalg.norm(n)
        A, absA = upwind_flux_matrix(ShallowWaterProblem(Phi=Phi), n)
        lam, R = np.linalg.eig(A)
        assert np.allclose(R @ np.diag(lam) @ np.linalg.inv(R), A, atol=1e-12)
        assert np.allclose(R @ np.diag(np.abs(lam)) @ np.linalg.inv(R), absA, atol=1e-12)
        assert np.allclose(np.sort(lam.real), [-np.sqrt(Phi), 0.0, np.sqrt(Phi)], atol=1e-12)


def test_cdr_stabilization_kat():
    """beta.n = 0 -> alpha = 2, tau = 1; alpha >= 2, tau > 0 always."""
    st = stabilization(ConvectionDiffusionProblem(kappa=1.0, beta=np.zeros(2)), 0.0)
    assert float(st.alpha) == 2.0 and float(st.tau) == 1.0
    bn = np.random.default_rng(1).normal(scale=10.0, size=1000)
    st = stabilization(ConvectionDiffusionProblem(kappa=1.0, beta=np.ones(2)), bn)
    assert np.all(st.alpha >= 2.0) and np.all(st.tau > 0.0)
    assert np.allclose(st.tau + stabilization(None, -bn).tau, st.alpha)   # tau^- + tau^+ = alpha


def test_non_unit_normal_rejected():
    with pytest.raises(ValueError):
        upwind_flux_matrix(TransportProblem(beta=np.ones(2)), np.array([1.0, 1.0]))


def test_sw_standing_wave_preset():
    """t = 0: u = v = 0, phi(0, 0) = 1, phi(0.5, 0.5) ~ 0."""
    sw = preset_problems()["sw_standing_wave"]
    x = np.array([[0.0, 0.0], [0.5, 0.5], [0.3, 0.7]])
    e = sw.exact(x, 0.0)
    assert abs(e[0, 0] - 1.0) < 1e-15 and abs(e[1, 0]) < 1e-15
    assert np.all(e[:, 1:] == 0.0)


def test_timedep_transport_forcing_is_manufactured():
    """transport3d_timedep: f = u_t + beta . grad u of the exact solution at
    random points, by central differences (residual < 1e-6 with h = 1e-5)."""
    tr = preset_problems()["transport3d_timedep"]
    rng = np.random.default_rng(2)
    x = rng.uniform(size=(50, 3))
    t, h = 0.3, 1e-5
    ut = (tr.exact(x, t + h) - tr.exact(x, t - h)) / (2 * h)
    grad = np.stack([(tr.exact(x + h * np.eye(3)[i], t) - tr.exact(x - h * np.eye(3)[i], t)) / (2 * h)
                     for i in range(3)], axis=1)
    res = ut + grad @ np.asarray(tr.beta) - tr.forcing(x, t)
    assert np.max(np.abs(res)) < 1e-6


def test_cdr_manufactured_preset():
    """div beta = 0 (so lambda = nu = 1); the forcing is
    kappa (-Lap u^e) + beta . grad u^e + nu u^e at sample points (central differences)."""
    cdr = preset_problems()["cdr_manufactured"]
    rng = np.random.default_rng(3)
    x = rng.uniform(size=(40, 3))
    h = 1e-4
    div = sum((cdr.beta(x + h * np.eye(3)[i])[:, i] - cdr.beta(x - h * np.eye(3)[i])[:, i]) / (2 * h) for i in range(3))
    assert np.max(np.abs(div)) < 1e-9 and cdr.nu == 1.0
    lap = sum((cdr.exact(x + h * np.eye(3)[i]) - 2 * cdr.exact(x) + cdr.exact(x - h * np.eye(3)[i])) / h ** 2
              for i in range(3))
    grad = np.stack([(cdr.exact(x + h * np.eye(3)[i]) - cdr.exact(x - h * np.eye(3)[i])) / (2 * h)
                     for i in range(3)], 1)
    res = -cdr.kappa * lap + np.sum(cdr.beta(x) * grad, 1) + cdr.nu * cdr.exact(x) - cdr.forcing(x)
    assert np.max(np.abs(res)) < 1e-5
