"""Discrete energy identities of the local solvers (
acceptance 9), checked on the product's assembled operators
(the Kronecker term lists K1 evaluates, assembly.evaluate_terms) against the
closed forms of the paper evaluated by independent quadrature (the oracle's
element helpers), for random own iterates u^{k+1} and neighbour face scalars q:

  u^T A u = the positive terms of the identity (its left-hand side),
  u^T B q = its right-hand side coupling.

  transport  (wellposednesstransport; div beta = 0):
      LHS = ||u||^2_{|b.n|/2, dK} (+ ||u||^2/dt)    RHS = <(b.n^+ + |b.n|)/2 u^+, u>_dK
  shallow water (localsolver1), per element before the sum:
      LHS = ||phi||^2/dt + (gamma + 1/dt) ||theta||^2_Phi + sqrt(Phi)/2 ||phi||^2_dK
            + sqrt(Phi)/2 ||theta.n||^2_{Phi, dK}
      RHS = <q, sqrt(Phi)/2 phi - Phi/2 theta.n>_dK,   q = phi^+ + sqrt(Phi) theta^+.n^+
  convection-diffusion (ErrorDDMCD5):
      LHS = ||sigma||^2/kappa + ((nu + 1/dt) u, u) + <(|b.n|^2+2)/(2 alpha) u, u>_dK
            + <sigma.n, sigma.n>_dK / alpha + <b.n u, sigma.n>_dK / alpha
      RHS = <(tau^- u - sigma.n)/alpha, q>_dK,   q = sigma^+.n^+ + tau^- u^+
Both to 1e-9 relative on 100 random iterates per PDE (acceptance 9)."""

import numpy as np
import pytest

from oracle.ihdg_oracle import Basis1D, _Element, _kron_axes
from paper_1711_01175_b200.assembly import build_spec, evaluate_terms
from paper_1711_01175_b200.basis import build_operators
from paper_1711_01175_b200.mesh import build_mesh
from paper_1711_01175_b200.pde import ConvectionDiffusionProblem, ShallowWaterProblem, TransportProblem


def _setup(problem, dim, p, dt, cells=4):
    mesh = build_mesh(dim, [cells] * dim)
    ops = build_operators(p, dim, mesh.h)
    spec = build_spec(mesh, problem, ops, dt)
    A, B, _ = evaluate_terms(spec)
    c = int(spec.class_of_mask[0])          # interior class: every face coupled
    el = _Element(Basis1D(p), dim, mesh.h)
    Mu = _kron_axes([el.b.V] * (dim - 1)) if dim > 1 else np.ones((1, 1))
    return spec, A[c], B[c], el, Mu


@pytest.mark.parametrize("dim,p,dt", [(2, 2, None), (2, 4, 0.1), (3, 2, None)])
def test_transport_energy_identity(dim, p, dt):
    beta = np.array([1.0, 0.7, 0.4])[:dim]
    spec, A, B, el, Mu = _setup(TransportProblem(beta=beta), dim, p, dt)
    rng = np.random.default_rng(0)
    nf = (p + 1) ** (dim - 1)
    for _ in range(100):
        u = rng.normal(size=spec.nv)
        q = rng.normal(size=spec.kin)
        lhs = 0.0 if dt is None else (u @ el.mass() @ u) / dt
        rhs = 0.0
        for f in range(2 * dim):
            a, s = divmod(f, 2)
            bn = beta[a] * (1.0 if s else -1.0)
            uf = el.Pf[f] @ u
            lhs += 0.5 * abs(bn) * np.sum(el.Wf[f] * uf * uf)
            if spec.coupled[f]:
                # the product's neighbour scalar is q = face_w u^+; the identity's
                # coupling is (b.n^+ + |b.n|)/2 u^+ = (|b.n| - b.n)/2 u^+
                up = (Mu @ q[f * nf:(f + 1) * nf]) / float(spec.face_w[f, 0])
                rhs += 0.5 * (abs(bn) - bn) * np.sum(el.Wf[f] * up * uf)
        assert abs(u @ A @ u - lhs) <= 1e-9 * abs(lhs)
        assert abs(u @ B @ q - rhs) <= 1e-9 * max(abs(rhs), 1e-300) + 1e-12


@pytest.mark.parametrize("p,dt,gamma,Phi", [(2, 0.1, 0.0, 1.0), (4, 0.01, 0.5, 2.0)])
def test_shallow_water_energy_identity(p, dt, gamma, Phi):
    spec, A, B, el, Mu = _setup(ShallowWaterProblem(Phi=Phi, gamma=gamma, f0=0.0), 2, p, dt)
    rng = np.random.default_rng(1)
    npn, nf = el.np, p + 1
    M = el.mass()
    sP = np.sqrt(Phi)
    for _ in range(100):
        u = rng.normal(size=spec.nv)
        q = rng.normal(size=spec.kin)
        phi, th = u[:npn], [u[npn:2 * npn], u[2 * npn:]]
        lhs = (phi @ M @ phi) / dt + (gamma + 1.0 / dt) * Phi * sum(t @ M @ t for t in th)
        rhs = 0.0
        for f in range(4):
            a, s = divmod(f, 2)
            sgn = 1.0 if s else -1.0
            pf = el.Pf[f] @ phi
            tn = sgn * (el.Pf[f] @ th[a])
            lhs += 0.5 * sP * np.sum(el.Wf[f] * pf * pf) + 0.5 * sP * Phi * np.sum(el.Wf[f] * tn * tn)
            qf = Mu @ q[f * nf:(f + 1) * nf]
            rhs += np.sum(el.Wf[f] * qf * (0.5 * sP * pf - 0.5 * Phi * tn))
        assert abs(u @ A @ u - lhs) <= 1e-9 * abs(lhs)
        assert abs(u @ B @ q - rhs) <= 1e-9 * abs(rhs) + 1e-12


@pytest.mark.parametrize("dim,p,dt,kappa,nu", [(2, 2, None, 1e-2, 1.0), (2, 6, 1e-3, 1e-3, 0.0),
                                               (3, 2, 0.1, 0.1, 0.5)])
def test_cd_energy_identity(dim, p, dt, kappa, nu):
    beta = np.array([1.0, -0.6, 0.3])[:dim]
    spec, A, B, el, Mu = _setup(ConvectionDiffusionProblem(kappa=kappa, beta=beta, nu=nu), dim, p, dt)
    rng = np.random.default_rng(2)
    npn, nf = el.np, (p + 1) ** (dim - 1)
    M = el.mass()
    for _ in range(100):
        u = rng.normal(size=spec.nv)
        q = rng.normal(size=spec.kin)
        sig, uu = [u[a * npn:(a + 1) * npn] for a in range(dim)], u[dim * npn:]
        lhs = sum(s @ M @ s for s in sig) / kappa + (nu + (0.0 if dt is None else 1.0 / dt)) * (uu @ M @ uu)
        rhs = 0.0
        for f in range(2 * dim):
            a, s = divmod(f, 2)
            sgn = 1.0 if s else -1.0
            bn = beta[a] * sgn
            alpha = np.sqrt(bn * bn + 4.0)
            tau = 0.5 * (alpha - bn)
            uf = el.Pf[f] @ uu
            sn = sgn * (el.Pf[f] @ sig[a])
            w = el.Wf[f]
            lhs += np.sum(w * ((bn * bn + 2.0) / (2 * alpha) * uf * uf + sn * sn / alpha + bn / alpha * uf * sn))
            qf = Mu @ q[f * nf:(f + 1) * nf]
            rhs += np.sum(w * (tau * uf - sn) / alpha * qf)
        assert abs(u @ A @ u - lhs) <= 1e-9 * abs(lhs)
        assert abs(u @ B @ q - rhs) <= 1e-9 * abs(rhs) + 1e-12
