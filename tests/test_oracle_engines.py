"""The oracle's two sweep engines (scipy LU + quadrature norm, and the
C/OpenMP map of oracle/sweep.c) agree: same iteration counts, fields to
1e-12, norms to 1e-6 (the successive difference cancels, so its rounding
is relative to |u|, not to the norm; CPU only; the C engine carries the full-size GPU parity
tests)."""

import numpy as np
import pytest

from tests.oracle_bridge import oracle_initial, oracle_solver, rel_l2


@pytest.mark.parametrize("cfg,cells", [(2, 12), (3, 8), (5, 8)])
def test_engines_agree_time_dependent(cfg, cells):
    from paper_1711_01175_b200.workloads import make_config

    wl = make_config(cfg, cells=cells, n_steps=2)
    S = oracle_solver(wl)
    u0 = oracle_initial(wl, S)
    _, ra = S.run_time_dependent(u0, 2, tol=1e-10)
    _, rb = S.run_time_dependent(u0, 2, tol=1e-10, engine="c", threads=2)
    assert [r["iterations"] for r in ra] == [r["iterations"] for r in rb]
    for a, b in zip(ra, rb):
        assert rel_l2(b["u"], a["u"]) < 1e-12
        assert np.allclose(b["norms"], a["norms"], rtol=1e-6, atol=1e-300)


def test_engines_agree_steady_transport():
    from paper_1711_01175_b200.workloads import make_config

    wl = make_config(4, cells=4)
    S = oracle_solver(wl)
    ra = S.run(tol=1e-10)
    rb = S.run(tol=1e-10, engine="c", threads=2)
    assert ra["iterations"] == rb["iterations"]
    assert rel_l2(rb["u"], ra["u"]) < 1e-12
