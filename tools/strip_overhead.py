#!/usr/bin/env python
"""Per-sweep cost of the multi-rank code path on ONE GPU: the config-5 mesh as
a single strip driven by DistributedSweeper (interior layers first, the two
boundary layers as one-layer strips, layer sums, all-reduce over a one-rank
NCCL group, finalize) against the fused single launch.  No neighbour exists,
so no halo travels: this is the floor of what a rank pays for the split
launches and the partition-independent norm, not a multi-GPU measurement.

    python tools/strip_overhead.py [n_sweeps=20] [cells=2048]"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402
import torch.distributed as dist  # noqa: E402

from paper_1711_01175_b200.solver import DeviceSolver, DistributedSweeper  # noqa: E402
from paper_1711_01175_b200.workloads import make_config  # noqa: E402


def timed(fn, n, stream):
    for _ in range(3):
        fn()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    torch.cuda.synchronize()
    e0.record(stream)
    for _ in range(n):
        fn()
    e1.record(stream)
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) / n


def main():
    n = int(sys.argv[1]) if len(sys.argv) > 1 else 20
    cells = int(sys.argv[2]) if len(sys.argv) > 2 else None
    os.environ.setdefault("MASTER_ADDR", "127.0.0.1")
    os.environ.setdefault("MASTER_PORT", "29577")
    torch.cuda.set_device(0)
    dist.init_process_group("nccl", rank=0, world_size=1, device_id=torch.device("cuda", 0))
    wl = make_config(5, cells=cells)
    sv = DeviceSolver(wl.mesh, wl.problem, wl.ops, dt=wl.dt, max_iters=100000)
    for name, fld in wl.initial.items():
        sv.set_state_component(fld, sv.spec.labels.index(name))
    sv.begin_step()
    sv.reset_state(0.0, 100000)
    a1 = sv.sweep_args("volume", 1)
    fused = timed(lambda: sv.sweep_once(a=a1), n, sv.stream)
    a0 = sv.sweep_args("volume", 0)
    for overlap in (True, False):
        dsw = DistributedSweeper(sv, 0, 1, dist.group.WORLD, overlap=overlap)
        ms = timed(lambda: dsw.sweep(a0), n, sv.stream)
        print(f"one-rank strip path, overlap={overlap}: {ms:.4f} ms/sweep ({dsw.launches_per_sweep()} launches) "
              f"vs fused single launch {fused:.4f} ms: +{100 * (ms / fused - 1):.2f}%")
    dist.destroy_process_group()


if __name__ == "__main__":
    main()
