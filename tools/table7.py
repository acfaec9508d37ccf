#!/usr/bin/env python
"""Table 7 of the paper on the device (SPEC.md acceptance 7):
cdr_manufactured (beta = (1+z, 1+x, 1+y), nu = 1, exact-solution rule, 3D),
iHDG-I and iHDG-II iteration counts per (h, p, kappa), per-element operators
(the GEMV mode).  Prints one row per entry with the paper's value.

    python tools/table7.py [max_cells] [max_p]
"""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

from paper_1711_01175_b200.basis import build_operators  # noqa: E402
from paper_1711_01175_b200.iteration import IterationConfig, run  # noqa: E402
from paper_1711_01175_b200.mesh import build_mesh  # noqa: E402
from paper_1711_01175_b200.pde import cdr_manufactured  # noqa: E402

# (h, p): (iHDG-I k=1e-2, 1e-3, 1e-6, iHDG-II k=1e-2, 1e-3, 1e-6); None = '*' (diverged)
PAPER = {
    (0.5, 1): (24, 23, 23, 17, 17, 17), (0.25, 1): (30, 34, 35, 25, 25, 26),
    (0.125, 1): (50, 55, 56, 35, 37, 38), (0.0625, 1): (90, 94, 97, 62, 64, 65),
    (0.5, 2): (26, 24, 25, 17, 19, 19), (0.25, 2): (41, 42, 42, 27, 27, 27),
    (0.125, 2): (66, 67, 67, 42, 43, 43), (0.0625, 2): (None, 109, 110, 67, 70, 71),
    (0.5, 3): (27, 31, 31, 19, 19, 19), (0.25, 3): (33, 33, 38, 24, 26, 27),
    (0.125, 3): (None, 58, 60, 38, 39, 41), (0.0625, 3): (None, 102, 106, 69, 69, 71),
    (0.5, 4): (26, 27, 27, 17, 19, 19), (0.25, 4): (50, 41, 43, 26, 27, 27),
    (0.125, 4): (None, 71, 72, 42, 45, 46), (0.0625, 4): (None, 123, 125, 73, 78, 79),
}


def main():
    max_cells = int(sys.argv[1]) if len(sys.argv) > 1 else 16
    max_p = int(sys.argv[2]) if len(sys.argv) > 2 else 4
    print("h      p  scheme   kappa   device      paper   |diff|  seconds")
    for (h, p), ref in sorted(PAPER.items(), key=lambda kv: (kv[0][1], -kv[0][0])):
        n = int(round(1.0 / h))
        if n > max_cells or p > max_p:
            continue
        mesh = build_mesh(3, [n] * 3)
        ops = build_operators(p, 3, mesh.h)
        for si, scheme in enumerate(("iHDG-I", "iHDG-II")):
            for ki, kappa in enumerate((1e-2, 1e-3, 1e-6)):
                t0 = time.perf_counter()
                rep = run(mesh, cdr_manufactured(kappa), ops,
                          IterationConfig(scheme=scheme, stop="exact", tol=1e-10, max_iters=5000), return_trace=False)
                paper = ref[3 * si + ki]
                dev = rep.iterations if rep.status == "converged" else "*"
                pstr = "*" if paper is None else str(paper)
                diff = abs(rep.iterations - paper) if (paper is not None and rep.status == "converged") else "-"
                print(f"{h:<6} {p}  {scheme:7s}  {kappa:7.0e}  {dev!s:>5} {rep.status:9s} {pstr:>5}  {diff!s:>5}"
                      f"  {time.perf_counter() - t0:7.1f}", flush=True)


if __name__ == "__main__":
    main()
