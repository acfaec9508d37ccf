"""Predictors of SPEC.md:361-377 (no GPU): the SPEC examples and the
inverse-trace constant of the basis."""

import numpy as np
import pytest

from paper_1711_01175_b200.theory import predict_cdr, predict_sw, trace_inequality_constant


def test_predict_sw_spec_examples():
    e = predict_sw(0.25, 1, 0.01, 1.0, c=1.0)
    assert e.admissible
    assert np.isclose(e.constants["constraint"], (0.25 / 0.06) / 2)
    assert np.isclose(e.epsilon, (2 * 0.25 / 0.06 + 1) / 2)
    assert np.isclose(e.contraction, (2 / (1 + 2 * 0.25 / 0.06)) ** 2)
    assert np.isclose(e.contraction, e.constants["C_closed_form"])
    bad = predict_sw(0.0625, 4, 1.0, 1.0, c=1.0)
    assert not bad.admissible and np.isclose(bad.constants["constraint"], (0.0625 / 30) / 2)
    assert np.isclose(predict_sw(0.25, 1, 0.1, 1.0, c=1.0).k_predicted, 0.6)


def test_predict_cdr_spec_examples():
    # cdr_manufactured: d=3, p=1, h=0.5, c=1, lambda=1, alpha_bar=sqrt(8)
    bounds = dict(bn_inf=2.0, tau_bar=(np.sqrt(8) + 2) / 2, a_bar=np.sqrt(8), a_star=np.sqrt(5))
    e = predict_cdr(0.5, 1, 3, 1.0, 1.0, bounds, c=1.0)
    assert np.isclose(e.k_predicted, 18 / (8 * np.sqrt(8) * 0.5))
    # elliptic (beta = 0): alpha = 2 everywhere, k = d(p+1)(p+2)/(16 c h min(1/kappa, lambda))
    el = predict_cdr(0.25, 2, 2, 1.0, 1.0, [0.0, 0.0], c=1.0)
    assert el.constants["a_bar"] == el.constants["a_star"] == 2.0 and el.constants["tau_bar"] == 1.0
    assert np.isclose(el.k_predicted, 2 * 3 * 4 / (16 * 0.25))
    # p-ratio (PAPER.md Asymptotics column): k(p)/k(1) = (p+1)(p+2)/6
    r = [predict_cdr(0.25, p, 2, 1.0, 1.0, [0.0, 0.0]).k_predicted / predict_cdr(0.25, 1, 2, 1.0, 1.0, [0.0, 0.0]).k_predicted
         for p in (2, 3, 4)]
    assert np.allclose(r, [2.0, 10 / 3, 5.0])
    # time-dependent: lambda -> lambda + 1/dt
    a = predict_cdr(0.125, 1, 2, 1e-4, 0.0, [1.0, 0.5], c=0.5, dt=1e-4)
    assert a.admissible and 0 < a.contraction < 1 and a.constants["B"] > 0
    with pytest.raises(ValueError):
        predict_cdr(0.125, 1, 2, 1e-4, 0.0, [1.0, 0.5])


def test_trace_inequality_constant_is_sharp_half():
    """(u,u)_K >= h/(d(p+1)(p+2)) <u,u>_dK is sharp on Q_p: c = 1/2."""
    for p in (1, 2, 4, 6):
        for d in (1, 2, 3):
            assert np.isclose(trace_inequality_constant(p, d), 0.5, rtol=1e-9)
