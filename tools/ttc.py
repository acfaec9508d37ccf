#!/usr/bin/env python
"""Time to converge of BASELINE configs 1-4 through the public API
(iteration.run / run_time_dependent), device-resident state.

    python tools/ttc.py [configs...]      (IHDG_NO_GRAPH=1: stream launches)
"""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from paper_1711_01175_b200.iteration import IterationConfig, run, run_time_dependent  # noqa: E402
from paper_1711_01175_b200.workloads import make_config  # noqa: E402


def once(cfg):
    wl = make_config(cfg, seed=0)
    stop = "trace" if cfg == 1 else "successive"
    t0 = time.perf_counter()
    if wl.dt is None:
        rep = run(wl.mesh, wl.problem, wl.ops, IterationConfig(stop=stop, tol=1e-10))
        its = [rep.iterations]
    else:
        reps = run_time_dependent(wl.mesh, wl.problem, wl.ops, IterationConfig(tol=1e-10), wl.dt,
                                  n_steps=wl.n_steps, initial=wl.initial)
        its = [r.iterations for r in reps]
    torch.cuda.synchronize()
    return time.perf_counter() - t0, its


def main():
    cfgs = [int(c) for c in sys.argv[1:]] or [1, 2, 3, 4]
    for c in cfgs:
        once(c)  # warm-up (assembly, graph capture, module load)
        best = min(once(c)[0] for _ in range(3))
        _, its = once(c)
        print(f"config {c}: {best * 1e3:.2f} ms to converge (best of 3), sweeps {sum(its)} {its[:4]}"
              f"{'...' if len(its) > 4 else ''}  graph={'off' if os.environ.get('IHDG_NO_GRAPH') else 'on'}",
              flush=True)


if __name__ == "__main__":
    main()
