#!/usr/bin/env python
"""h- and p-ratio asymptotics of the iHDG-II iteration counts on the device
(SPEC.md acceptance 4, 5, 6; PAPER.md Figs. tab:p_var, h_var_CDR,
tab:h_p_var_elliptic), exact-solution stopping rule:

  sw        sw_standing_wave, one Crank-Nicolson step, Nel = 16..1024, dt 0.1 / 0.01
  cdr       cdr_manufactured, h = 0.5 .. 0.0625, kappa = 1e-2, 1e-3, 1e-6
  elliptic  elliptic_manufactured (kappa = 1, beta = 0), h = 0.5 .. 0.125, p = 1..4, under the
            paper's vs-direct rule for this regime

    python tools/ratios.py [sw] [cdr] [elliptic] [--pmax P] [--nmax N]
"""
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

from paper_1711_01175_b200.basis import build_operators  # noqa: E402
from paper_1711_01175_b200.iteration import IterationConfig, run, run_time_dependent  # noqa: E402
from paper_1711_01175_b200.mesh import build_mesh  # noqa: E402
from paper_1711_01175_b200.pde import cdr_manufactured, elliptic_manufactured, preset_problems  # noqa: E402


def sw_count(nel, p, dt):
    n = int(round(np.sqrt(nel)))
    mesh = build_mesh(2, [n, n])
    reps = run_time_dependent(mesh, preset_problems()["sw_standing_wave"], build_operators(p, 2, mesh.h),
                              IterationConfig(scheme="iHDG-II", tol=1e-10, max_iters=5000, stop="exact"), dt,
                              n_steps=1, initial={"phi": lambda x: np.cos(np.pi * x[:, 0]) * np.cos(np.pi * x[:, 1])},
                              time_scheme="crank-nicolson")
    return reps[-1].iterations


def steady_count(problem, n, p, max_iters=200000):
    mesh = build_mesh(3, [n] * 3)
    rep = run(mesh, problem, build_operators(p, 3, mesh.h),
              IterationConfig(scheme="iHDG-II", stop="exact", tol=1e-10, max_iters=max_iters))
    return rep.iterations if rep.status == "converged" else None


def vs_direct_count(problem, n, p, max_iters=400000):
    """||u^k - u_direct|| < 1e-10.  The direct HDG solution is
    the iteration's fixed point, taken here from a first solve to 1e-14 with
    the successive rule (no CPU solver on the product path)."""
    mesh = build_mesh(3, [n] * 3)
    ops = build_operators(p, 3, mesh.h)
    fix = run(mesh, problem, ops, IterationConfig(scheme="iHDG-II", stop="successive", tol=1e-14, max_iters=max_iters))
    if fix.status != "converged":
        return None
    rep = run(mesh, problem, ops, IterationConfig(scheme="iHDG-II", stop="vs-direct", tol=1e-10, max_iters=max_iters,
                                                  reference=fix.state))
    return rep.iterations if rep.status == "converged" else None


def ratios(c):
    return [round(b / a, 2) if a and b else None for a, b in zip(c[:-1], c[1:])]


def main():
    args = [a for a in sys.argv[1:] if not a.startswith("--")] or ["sw", "cdr", "elliptic"]
    pmax = int(sys.argv[sys.argv.index("--pmax") + 1]) if "--pmax" in sys.argv else 3
    nmax = int(sys.argv[sys.argv.index("--nmax") + 1]) if "--nmax" in sys.argv else 16
    if "sw" in args:
        print("# shallow water (Table 6 / Fig. tab:p_var): counts at Nel = 16, 64, 256, 1024; h ratios; dt = 0.1 / dt = 0.01 factor")
        for p in range(1, 5):
            c1 = [sw_count(nel, p, 0.1) for nel in (16, 64, 256, 1024)]
            c2 = [sw_count(nel, p, 0.01) for nel in (16, 64, 256, 1024)]
            print(f"p={p}: dt=0.1 {c1} ratios {ratios(c1)}; dt=0.01 {c2}; dt factor {[round(a / b, 2) for a, b in zip(c1, c2)]}")
    ns = [n for n in (2, 4, 8, 16) if n <= nmax]
    if "cdr" in args:
        print("# convection-diffusion (Table 7 / Fig. h_var_CDR): counts at h = 1/2 .. 1/%d; h ratios" % ns[-1])
        for kappa in (1e-2, 1e-3, 1e-6):
            for p in range(1, min(pmax, 2) + 1):
                c = [steady_count(cdr_manufactured(kappa), n, p) for n in ns]
                print(f"kappa={kappa:g} p={p}: {c} ratios {ratios(c)}")
    if "elliptic" in args:
        print("# elliptic (kappa = 1, beta = 0; Fig. tab:h_p_var_elliptic): counts at h = 1/2 .. ; h ratios; p ratios k(p)/k(1)")
        ne = [n for n in (2, 4, 8, 16) if n <= nmax]
        table = {}
        for p in range(1, pmax + 1):
            table[p] = [vs_direct_count(elliptic_manufactured(1.0), n, p) for n in ne]
            print(f"p={p}: {table[p]} ratios {ratios(table[p])}")
        for p in range(2, pmax + 1):
            pr = [round(a / b, 2) if a and b else None for a, b in zip(table[p], table[1])]
            print(f"k({p})/k(1) at h = 1/2 ..: {pr}; asymptotics {(p + 1) * (p + 2) / 6:.2f}")


if __name__ == "__main__":
    main()
