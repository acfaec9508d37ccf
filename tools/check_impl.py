#!/usr/bin/env python
"""Compare two sweep-kernel selectors on one BASELINE config (steady configs
run to convergence, unsteady ones for one step): iteration counts, successive
norms and fields.   python tools/check_impl.py <config> <cells> <implA> <implB>"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402

from paper_1711_01175_b200 import _native as N  # noqa: E402
from paper_1711_01175_b200.iteration import IterationConfig, run, run_time_dependent  # noqa: E402
from paper_1711_01175_b200.workloads import make_config  # noqa: E402


def solve(wl, impl):
    N.set_sweep_impl(impl)
    try:
        if wl.dt is None:
            return run(wl.mesh, wl.problem, wl.ops, IterationConfig(tol=1e-10), return_trace=False)
        return run_time_dependent(wl.mesh, wl.problem, wl.ops, IterationConfig(tol=1e-10), wl.dt, n_steps=1,
                                  initial=wl.initial)[-1]
    finally:
        N.set_sweep_impl("auto")


def main():
    cfg, cells, ia, ib = int(sys.argv[1]), int(sys.argv[2]), sys.argv[3], sys.argv[4]
    wl = make_config(cfg, cells=cells)
    ra, rb = solve(wl, ia), solve(wl, ib)
    da, db = ra.state.data, rb.state.data
    rel = float(np.linalg.norm(da - db) / max(np.linalg.norm(da), 1e-300))
    na, nb = np.asarray(ra.successive_norms), np.asarray(rb.successive_norms)
    n = min(len(na), len(nb))
    nrel = float(np.max(np.abs(na[:n] - nb[:n]) / np.maximum(np.abs(na[:n]), 1e-300))) if n else 0.0
    print(f"config {cfg} cells {cells}: {ia}={ra.extra['kernel']} {ra.iterations} its {ra.status}; "
          f"{ib}={rb.extra['kernel']} {rb.iterations} its {rb.status}; field rel {rel:.3e}; norms rel {nrel:.3e}; "
          f"bit-identical fields {bool(np.array_equal(da, db))}")
    ok = ra.iterations == rb.iterations and rel < 1e-12 and nrel < 1e-9
    sys.exit(0 if ok else 1)


if __name__ == "__main__":
    main()
