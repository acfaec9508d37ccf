#!/usr/bin/env python
"""PAPER.md Table 6 on the device (SPEC.md acceptance criterion 3):
sw_standing_wave (Phi=1, f=0, gamma=0, mirror walls on [0,1]^2), one
Crank-Nicolson step from t=0, iHDG-I vs iHDG-II, Nel in {16,64,256,1024},
p in 1..4, dt in {0.1, 0.01}; successive-difference rule, tol 1e-10.

    python tools/table6.py [--oracle] [--exact]
    --oracle: also the CPU oracle (small meshes); --exact: the paper's own
    exact-solution stopping rule instead of successive
"""
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

from paper_1711_01175_b200.basis import build_operators  # noqa: E402
from paper_1711_01175_b200.iteration import IterationConfig, run_time_dependent  # noqa: E402
from paper_1711_01175_b200.mesh import build_mesh  # noqa: E402
from paper_1711_01175_b200.pde import ShallowWaterProblem, preset_problems  # noqa: E402

RULE = "exact" if "--exact" in sys.argv else "successive"

# (Nel, p) -> (I dt=0.1, I dt=0.01, II dt=0.1, II dt=0.01); None = "*" (diverged)
TABLE6 = {
    (16, 1): (19, 6, 14, 6), (64, 1): (None, 6, 18, 9), (256, 1): (None, 7, 32, 10), (1024, 1): (None, 9, 59, 8),
    (16, 2): (None, 9, 15, 9), (64, 2): (None, 11, 19, 9), (256, 2): (None, 13, 32, 11), (1024, 2): (None, 15, 59, 12),
    (16, 3): (None, 7, 16, 8), (64, 3): (None, 9, 20, 8), (256, 3): (None, 12, 31, 10), (1024, 3): (None, None, 59, 12),
    (16, 4): (None, 10, 17, 9), (64, 4): (None, 12, 32, 10), (256, 4): (None, None, 60, 9), (1024, 4): (None, None, 112, 13),
}


def phi0(x):
    return np.cos(np.pi * x[:, 0]) * np.cos(np.pi * x[:, 1])


def one(nel, p, dt, scheme):
    n = int(round(np.sqrt(nel)))
    mesh = build_mesh(2, [n, n])
    ops = build_operators(p, 2, mesh.h)
    prob = preset_problems()["sw_standing_wave"] if RULE == "exact" else ShallowWaterProblem(Phi=1.0)
    reps = run_time_dependent(mesh, prob, ops,
                              IterationConfig(scheme=scheme, tol=1e-10, max_iters=5000, stop=RULE), dt, n_steps=1,
                              initial={"phi": phi0}, time_scheme="crank-nicolson")
    r = reps[-1]
    return r.iterations, r.status


def oracle_one(nel, p, dt, scheme):
    from oracle.ihdg_oracle import OracleProblem, OracleSolver

    n = int(round(np.sqrt(nel)))
    S = OracleSolver(OracleProblem("sw", 2, Phi=1.0), [n, n], p, dt=dt, scheme="I" if scheme == "iHDG-I" else "II",
                     time_scheme="CN")
    u0 = np.zeros((S.nel, S.m, S.npn))
    u0[:, 0, :] = S.interpolate(phi0)
    _, rr = S.run_time_dependent(u0.reshape(S.nel, -1), 1, tol=1e-10, max_iters=5000,
                                 norm="exact" if RULE == "exact" else "volume",
                                 exact=preset_problems()["sw_standing_wave"].exact)
    return rr[-1]["iterations"], rr[-1]["status"]


def main():
    with_oracle = "--oracle" in sys.argv
    print(f"stopping rule: {RULE}")
    print(f"{'Nel':>5} {'p':>2} | {'I dt=.1':>14} {'I dt=.01':>14} | {'II dt=.1':>14} {'II dt=.01':>14} |  paper")
    ok_pattern, within = True, []
    for (nel, p), paper in TABLE6.items():
        cells = []
        k = 0
        for scheme in ("iHDG-I", "iHDG-II"):
            for dt in (0.1, 0.01):
                it, st = one(nel, p, dt, scheme)
                ref = paper[k]
                div = st != "converged"
                if (ref is None) != div:
                    ok_pattern = False
                if ref is not None and not div:
                    within.append((it - ref, ref))
                txt = "*" if div else str(it)
                if with_oracle and nel <= 64:
                    oi, ost = oracle_one(nel, p, dt, scheme)
                    txt += f" (o:{'*' if ost != 'converged' else oi})"
                cells.append(f"{txt:>14}")
                k += 1
        ptxt = " ".join("*" if v is None else str(v) for v in paper)
        print(f"{nel:>5} {p:>2} | {cells[0]} {cells[1]} | {cells[2]} {cells[3]} |  {ptxt}", flush=True)
    d = np.array([w[0] for w in within])
    rel = np.array([abs(w[0]) / w[1] for w in within])
    print(f"pattern of '*' matches Table 6: {ok_pattern}; converged entries: |diff| <= 3 for "
          f"{int(np.sum(np.abs(d) <= 3))}/{d.size}, within 30% for {int(np.sum(rel <= 0.3))}/{d.size}")


if __name__ == "__main__":
    main()
