#!/usr/bin/env python
"""Time sweeps of the per-element-operator (GEMV) mode on cdr_manufactured and
compare the dispatched kernel with the generic one (fields and norms bitwise).

    python tools/sweep_gemv.py [cells=16] [order=2] [n_sweeps=20]"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

from paper_1711_01175_b200 import _native as N  # noqa: E402
from paper_1711_01175_b200.basis import build_operators  # noqa: E402
from paper_1711_01175_b200.mesh import build_mesh  # noqa: E402
from paper_1711_01175_b200.pde import cdr_manufactured  # noqa: E402
from paper_1711_01175_b200.solver import DeviceSolver  # noqa: E402


def run(cells, order, n, impl):
    N.set_sweep_impl(impl)
    try:
        m = build_mesh(3, [cells] * 3)
        pr = cdr_manufactured(1e-3)
        sv = DeviceSolver(m, pr, build_operators(order, 3, m.h), max_iters=1000)
        sv.set_forcing(pr.forcing)
        sv.set_dirichlet(pr.dirichlet)
        sv.prepare_steady()
        sv.reset_state(tol=0.0, max_iters=1000)
        a = sv.sweep_args("volume", 1)
        name = N.sweep_kernel(a)
        for _ in range(3):
            sv.sweep_once(a=a)
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        torch.cuda.synchronize()
        e0.record(sv.stream)
        for _ in range(n):
            sv.sweep_once(a=a)
        e1.record(sv.stream)
        torch.cuda.synchronize()
        ms = e0.elapsed_time(e1) / n
        dofs = sv.nloc * sv.nv
        bpd = 8 * (sv.spec.kin + 3)
        print(f"{impl}: {name} {ms:.4f} ms/sweep, {bpd * dofs / ms / 1e6:.1f} GB/s of 8(K_raw+3) = {bpd} B/DOF, {dofs} DOFs")
        return sv.get_state().copy(), sv.norm_hist[: 3 + n].cpu().numpy().copy()
    finally:
        N.set_sweep_impl("auto")


def main():
    cells = int(sys.argv[1]) if len(sys.argv) > 1 else 16
    order = int(sys.argv[2]) if len(sys.argv) > 2 else 2
    n = int(sys.argv[3]) if len(sys.argv) > 3 else 20
    ua, na = run(cells, order, n, "auto")
    ug, ng = run(cells, order, n, "generic")
    print("fields bitwise", bool(np.array_equal(ua, ug)), "norms bitwise", bool(np.array_equal(na, ng)),
          "max rel field diff", float(np.max(np.abs(ua - ug)) / max(np.max(np.abs(ug)), 1e-300)))


if __name__ == "__main__":
    main()
