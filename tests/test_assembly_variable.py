"""Per-element operators (variable beta, the GEMV mode):
the product's term lists (weighted 1D masses, raw neighbour columns) against
the oracle's quadrature assembly, element by element (CPU)."""

import numpy as np
import pytest

from oracle.ihdg_oracle import OracleProblem, OracleSolver
from paper_1711_01175_b200.assembly import beta_dependence, build_spec, evaluate_terms, face_node_indices
from paper_1711_01175_b200.basis import build_operators
from paper_1711_01175_b200.mesh import build_mesh
from paper_1711_01175_b200.pde import ConvectionDiffusionProblem



def beta3(x):
    return np.stack([1 + x[:, 2], 1 + x[:, 0], 1 + x[:, 1]], 1)


def beta2(x):
    return np.stack([1 + 0.5 * np.sin(3 * x[:, 1]), -0.3 + x[:, 0] ** 2], 1)


def test_beta_dependence():
    assert beta_dependence(beta3, 3, np.zeros(3), np.ones(3)) == [2, 0, 1]
    assert beta_dependence(beta2, 2, np.zeros(2), np.ones(2)) == [1, 0]
    with pytest.raises(NotImplementedError):
        beta_dependence(lambda x: np.stack([x[:, 0], x[:, 1]], 1), 2, np.zeros(2), np.ones(2))


@pytest.mark.parametrize("dim,beta,p,scheme,dt", [(3, beta3, 1, "iHDG-II", None), (3, beta3, 2, "iHDG-II", None),
                                                  (2, beta2, 3, "iHDG-II", 0.05), (3, beta3, 1, "iHDG-I", None),
                                                  (2, beta2, 2, "iHDG-I", None)])
def test_per_element_operators_match_oracle(dim, beta, p, scheme, dt):
    cells = [3] * dim
    mesh = build_mesh(dim, cells)
    ops = build_operators(p, dim, mesh.h)
    prob = ConvectionDiffusionProblem(kappa=0.05, beta=beta, nu=1.0)
    sp = build_spec(mesh, prob, ops, dt, scheme=scheme)
    assert sp.per_element and sp.n_class == mesh.n_elements
    A, B, R = evaluate_terms(sp)
    S = OracleSolver(OracleProblem("cd", dim, beta=beta, kappa=0.05, nu=1.0), cells, p, dt=dt,
                     scheme="I" if scheme == "iHDG-I" else "II")
    n1, npn = p + 1, (p + 1) ** dim
    nf = n1 ** (dim - 1)
    blocks = sp.kin_blocks
    for e in range(mesh.n_elements):
        C = S.class_list[e]
        scale = np.max(np.abs(C["A"]))
        assert np.max(np.abs(A[e] - C["A"])) <= 1e-12 * scale
        own = np.zeros_like(C["A"])
        for f in range(2 * dim):
            Nf = np.zeros_like(C["A"])
            for j in range(blocks):
                comp = int(sp.raw_comp[f, j])
                for n in range(nf):
                    col = (f * blocks + j) * nf + n
                    if j < 2:
                        Nf[:, comp * npn + face_node_indices(dim, n1, f ^ 1)[n]] += B[e][:, col]
                    else:
                        own[:, comp * npn + face_node_indices(dim, n1, f)[n]] += B[e][:, col]
            if S.nbr[e, f] >= 0:
                assert np.max(np.abs(Nf - C["N"][f])) <= 1e-12 * scale, (e, f)
        assert np.max(np.abs(own - C["Own"])) <= 1e-12 * scale
        if dt is not None:
            assert np.max(np.abs(R[e][:, :npn] - C["R"][:, dim * npn:])) <= 1e-12 * scale
