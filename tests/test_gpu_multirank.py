"""The strip-partitioned device path (solver.DistributedSweeper) with two
ranks sharing cuda:0.

The ranks use the gloo backend with host staging of the packed halo entries
and the layer sums, so no kernel ever waits on another rank.  The NCCL
variant differs only in the transport call.  The sweep kernels (interior
layers first, boundary layers after the halo, or one launch), the halo
pack / unpack kernels, the layer sums and the fixed-order finalize are the
same.  For any split -- uneven ones included -- the result must be
bit-identical to one rank: same iteration count, same norms, same fields.
"""

import os
import socket

import numpy as np
import pytest

pytestmark = pytest.mark.gpu


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _setup(wl, layers=None):
    from paper_1711_01175_b200.solver import DeviceSolver

    sv = DeviceSolver(wl.mesh, wl.problem, wl.ops, dt=wl.dt, layers=layers, max_iters=5000)
    forcing = getattr(wl.problem, "forcing", None)
    if forcing is not None:
        sv.set_forcing(forcing)
    sv.zero_state()
    for name, fld in wl.initial.items():
        sv.set_state_component(fld, sv.spec.labels.index(name))
    if wl.dt is not None:
        sv.begin_step()
    else:
        sv.prepare_steady()
    return sv


def _worker(rank, world, port, cfg, kw, overlap, q):
    import torch
    import torch.distributed as dist

    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    torch.cuda.set_device(0)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        from paper_1711_01175_b200.partition import strip_range
        from paper_1711_01175_b200.solver import DistributedSweeper
        from paper_1711_01175_b200.workloads import make_config

        wl = make_config(cfg, seed=1, **kw)
        layers = strip_range(wl.mesh.cells[-1], rank, world)
        sv = _setup(wl, layers)
        ds = DistributedSweeper(sv, rank, world, host_staging=True, overlap=overlap)
        assert ds.overlap == (overlap and sv.layers[1] - sv.layers[0] >= 3)
        res = ds.iterate(tol=1e-10, max_iters=5000, norm="volume", batch=8)
        q.put((rank, layers, res.iterations, res.status, res.norms, sv.get_state()))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("cfg,kw,world,overlap", [
    (3, dict(cells=16, n_steps=1), 2, True),             # periodic shallow water (wrap across ranks)
    (3, dict(cells=16, n_steps=1), 3, False),            # uneven strips 6/5/5
    (5, dict(cells=32, kappa=1e-1, n_steps=1), 2, True),  # convection-diffusion p=6, 9 operator classes
    (5, dict(cells=32, kappa=1e-1, n_steps=1), 3, True),  # uneven strips 11/11/10
    (5, dict(cells=32, kappa=1e-3, n_steps=1), 2, False),
    (4, dict(cells=8), 2, True),                         # 3D transport (no data goes downstream)
    (4, dict(cells=8), 3, False),                        # 3/3/2 layers
])
def test_ranks_bit_identical_to_one(cfg, kw, world, overlap):
    import torch
    import torch.multiprocessing as mp

    if not torch.cuda.is_available():
        pytest.skip("needs a CUDA device")
    from paper_1711_01175_b200.workloads import make_config

    torch.cuda.set_device(0)
    wl = make_config(cfg, seed=1, **kw)
    sv = _setup(wl)
    ref = sv.iterate(tol=1e-10, max_iters=5000, norm="volume", batch=8)
    ref_state = sv.get_state()
    del sv
    torch.cuda.empty_cache()

    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, cfg, kw, overlap, q)) for r in range(world)]
    for p in procs:
        p.start()
    out = sorted([q.get(timeout=600) for _ in range(world)], key=lambda x: x[0])
    for p in procs:
        p.join(timeout=120)
        assert p.exitcode == 0
    ls = int(np.prod(wl.mesh.cells[:-1]))
    for rank, (lb, le), iters, status, norms, state in out:
        assert status == ref.status == "converged"
        assert iters == ref.iterations
        np.testing.assert_array_equal(norms, ref.norms)
        np.testing.assert_array_equal(state, ref_state[lb * ls:le * ls])


def test_bench_multirank_line_host_staging():
    """bench.py's N > 1 path (strips, DistributedSweeper, e2e and time to
    converge at N ranks) in its test mode: two ranks share the GPU and exchange
    through host memory.  The line must carry the contract's keys and the same
    sweep counts as one rank."""
    import json
    import os
    import subprocess
    import sys

    import torch

    if not torch.cuda.is_available():
        pytest.skip("needs a CUDA device")
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    common = ["--cells", "64", "--steps", "3", "--warmup", "3", "--no-cpu", "--no-others", "--ttc", "1e-3:2"]

    def line(cmd):
        out = subprocess.run(cmd, cwd=root, capture_output=True, text=True, timeout=600)
        assert out.returncode == 0, out.stderr[-2000:]
        return json.loads([ln for ln in out.stdout.splitlines() if ln.startswith("{")][-1])

    one = line([sys.executable, "bench.py"] + common)
    two = line([sys.executable, "-m", "torch.distributed.run", "--nnodes=1", "--nproc-per-node=2",
                "--master-addr", "127.0.0.1", f"--master-port={_free_port()}", "bench.py", "--gpus", "2",
                "--host-staging", "--scaling", "strong"] + common)
    assert two["n_gpus"] == 2 and two["scaling"] == "strong" and two["config"]["parallelism"] == "strip2"
    for key in ("roofline", "clocks", "e2e", "gpu_launches", "time_to_converge"):
        assert two.get(key), key
    t1, t2 = one["time_to_converge"]["kappa=0.001"], two["time_to_converge"]["kappa=0.001"]
    assert t2["status"] == t1["status"] == "converged"
    assert t2["sweeps_per_step"] == t1["sweeps_per_step"]
    assert two["e2e"]["sweeps"] == one["e2e"]["sweeps"]
