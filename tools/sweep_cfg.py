#!/usr/bin/env python
"""Time N sweeps of one BASELINE config (for ncu captures and A/B runs).

    python tools/sweep_cfg.py <config 1-5> [n_sweeps] [warmup] [gram] [nofin] [nolsum] [graph]
"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from paper_1711_01175_b200.solver import DeviceSolver  # noqa: E402
from paper_1711_01175_b200.workloads import make_config  # noqa: E402


def main():
    cfg = int(sys.argv[1])
    n = int(sys.argv[2]) if len(sys.argv) > 2 else 20
    warm = int(sys.argv[3]) if len(sys.argv) > 3 else 3
    cells = int(os.environ["CELLS"]) if os.environ.get("CELLS") else None   # reduced / enlarged mesh
    wl = make_config(cfg, cells=cells)
    sv = DeviceSolver(wl.mesh, wl.problem, wl.ops, dt=wl.dt, max_iters=100000, gram_norm="gram" in sys.argv[4:])
    if getattr(wl.problem, "forcing", None) is not None:
        sv.set_forcing(wl.problem.forcing)
    sv.zero_state()
    for name, fld in wl.initial.items():
        sv.set_state_component(fld, sv.spec.labels.index(name))
    if wl.dt is not None:
        sv.begin_step()
    else:
        sv.prepare_steady()
    sv.reset_state(0.0, 100000)
    a = sv.sweep_args("volume", 0 if "nofin" in sys.argv[4:] else 1)
    if "nolsum" in sys.argv[4:]:
        a.layer_sums = a.grid_bar = None
    for _ in range(warm):
        sv.sweep_once(a=a)
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    torch.cuda.synchronize()
    if "graph" in sys.argv[4:]:
        # replay the n sweeps from one CUDA graph (no host launch gaps between short sweeps)
        n += n % 2
        gr, cap = torch.cuda.CUDAGraph(), torch.cuda.Stream()
        sv.stream = cap
        with torch.cuda.graph(gr, stream=cap):
            for _ in range(n):
                sv.sweep_once(a=a)
        torch.cuda.synchronize()
        with torch.cuda.stream(cap):
            gr.replay()
            e0.record(cap)
            gr.replay()
            e1.record(cap)
    else:
        e0.record(sv.stream)
        for _ in range(n):
            sv.sweep_once(a=a)
        e1.record(sv.stream)
    torch.cuda.synchronize()
    ms = e0.elapsed_time(e1) / n
    dofs = sv.nloc * sv.nv
    print(f"config {cfg}: {ms:.4f} ms/sweep, {dofs * 24 / ms / 1e6:.1f} GB/s algorithmic, {dofs} DOFs")


if __name__ == "__main__":
    main()
