"""Config 5 at kappa = 0.1: norm history of the first backward-Euler step on
the device (2048^2 and smaller meshes), to tell slow convergence from
stagnation.  python tools/kappa_probe.py"""
import sys
import numpy as np
import torch
sys.path.insert(0, ".")
from paper_1711_01175_b200.solver import DeviceSolver
from paper_1711_01175_b200.workloads import make_config

for cells in (256, 512, 1024, 2048):
    w = make_config(5, seed=0, kappa=0.1, cells=cells)
    sv = DeviceSolver(w.mesh, w.problem, w.ops, dt=w.dt, max_iters=20000)
    sv.zero_state()
    for name, fld in w.initial.items():
        sv.set_state_component(fld, sv.spec.labels.index(name))
    sv.begin_step()
    r = sv.iterate(tol=1e-10, max_iters=20000, norm="volume", batch=32)
    n = r.norms
    pick = [i for i in (0, 9, 99, 999, 4999, 9999, 19999) if i < len(n)]
    print(f"cells={cells} dt={w.dt:.3e} status={r.status} iters={r.iterations} "
          + " ".join(f"n[{i+1}]={n[i]:.3e}" for i in pick), flush=True)
    if len(n) > 200:
        tail = n[-200:]
        rate = (tail[-1] / tail[0]) ** (1.0 / 199)
        print(f"  asymptotic contraction per sweep over the last 200: {rate:.6f}", flush=True)
    del sv
    torch.cuda.empty_cache()
