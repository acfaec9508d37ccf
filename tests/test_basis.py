"""Basis known-answer tests."""

import numpy as np
import pytest

from oracle.ihdg_oracle import gll_nodes_oracle
from paper_1711_01175_b200.basis import build_operators, gll_nodes, l2_error, l2_norm, project
from paper_1711_01175_b200.mesh import build_mesh


def test_mass_p1_1d():
    h = 0.37
    ops = build_operators(1, 1, h)
    assert np.allclose(ops.mass, (h / 6.0) * np.array([[2.0, 1.0], [1.0, 2.0]]), atol=1e-15, rtol=1e-14)


def test_diff_reproduces_derivative():
    ops = build_operators(2, 1, 1.0)
    x = ops.nodes
    assert np.max(np.abs(ops.diff1d @ x ** 2 - 2 * x)) < 1e-13


@pytest.mark.parametrize("p", range(1, 11))
def test_diff_rows_and_quadrature(p):
    ops = build_operators(p, 1, 1.0)
    assert np.max(np.abs(ops.diff1d.sum(axis=1))) < 1e-12
    # (p+2)-point Gauss is exact to degree 2p+3
    for k in range(2 * p + 4):
        exact = 0.0 if k % 2 else 2.0 / (k + 1)
        assert abs(np.sum(ops.quad_weights * ops.quad_points ** k) - exact) < 1e-13
    # independent GLL construction in the oracle agrees
    assert np.max(np.abs(gll_nodes(p)[0] - gll_nodes_oracle(p))) < 1e-14
    M1 = ops.mass1d
    assert np.allclose(M1, M1.T) and np.all(np.linalg.eigvalsh(M1) > 0)
    assert np.allclose(ops.chol1d @ ops.chol1d.T, M1, atol=1e-15)


def test_quadrature_of_one_p3_2d():
    ops = build_operators(3, 2, np.array([1.0, 1.0]))
    W = np.kron(ops.quad_weights, ops.quad_weights)
    assert abs(W.sum() * ops.jacobian - 1.0) < 1e-14


def test_project_and_norms():
    m = build_mesh(2, [3, 3])
    ops = build_operators(2, 2, m.h)
    z = project(lambda x: np.zeros(x.shape[0]), m, ops)
    assert np.all(z.data == 0) and l2_norm(z, m, ops) == 0.0
    one = project(lambda x: np.ones(x.shape[0]), m, ops)
    assert abs(l2_norm(one, m, ops) - 1.0) < 1e-14
    poly = lambda x: 1 + x[:, 0] ** 2 - 3 * x[:, 0] * x[:, 1]
    s = project(poly, m, ops)
    assert l2_error(s, poly, m, ops) < 1e-12
    m1 = build_mesh(1, [8])
    o1 = build_operators(4, 1, m1.h)
    s1 = project(lambda x: np.sin(np.pi * x[:, 0]), m1, o1)
    assert abs(l2_norm(s1, m1, o1) - 1 / np.sqrt(2)) < 1e-8


def test_project_3d_error():
    m = build_mesh(3, [8, 8, 8])
    ops = build_operators(4, 3, m.h)
    f = lambda x: np.sin(np.pi * x[:, 0]) * np.cos(np.pi * x[:, 1]) * np.sin(np.pi * x[:, 2]) / np.pi
    assert l2_error(project(f, m, ops), f, m, ops) < 1e-6


def test_reject_order():
    with pytest.raises(ValueError):
        build_operators(0, 2, 1.0)
    with pytest.raises(ValueError):
        build_operators(11, 2, 1.0)
