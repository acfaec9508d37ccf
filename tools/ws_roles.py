#!/usr/bin/env python
"""Per-role cycle breakdown of the warp-specialised sweep (profiling build).

    tools/build_flags.sh ablib/prof.so -DIHDG_WS_PROF
    IHDG_LIB=ablib/prof.so python tools/ws_roles.py [config] [gram]
"""
import ctypes
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from paper_1711_01175_b200 import _native as N  # noqa: E402
from paper_1711_01175_b200.solver import DeviceSolver  # noqa: E402
from paper_1711_01175_b200.workloads import make_config  # noqa: E402

NAMES = ["producer: wait (empty/done)", "prep: wait full", "prep: q compute", "consumer: wait qready",
         "consumer: contraction", "consumer: epilogue / wait outfree (ws)", "CTA total",
         "consumer: norm", "consumer: wait done prev (ws)", "producer: load issue",
         "consumer: epilogue stores (ws)", "prep: gather issue (ws)", "prep: wait done (ws)",
         "prep: gather consume (ws)"]


def main():
    cfg = int(sys.argv[1]) if len(sys.argv) > 1 else 5
    wl = make_config(cfg)
    sv = DeviceSolver(wl.mesh, wl.problem, wl.ops, dt=wl.dt, max_iters=1000, gram_norm="gram" in sys.argv[2:])
    if getattr(wl.problem, "forcing", None) is not None:
        sv.set_forcing(wl.problem.forcing)
    for name, fld in wl.initial.items():
        sv.set_state_component(fld, sv.spec.labels.index(name))
    if wl.dt is not None:
        sv.begin_step()
    else:
        sv.prepare_steady()
    sv.reset_state(0.0, 1000)
    a = sv.sweep_args("volume", 1)
    L = N.lib()
    L.ihdg_ws_prof.argtypes = [ctypes.c_void_p, ctypes.c_int]
    buf = (ctypes.c_ulonglong * 16)()
    for _ in range(3):
        sv.sweep_once(a=a)
    torch.cuda.synchronize()
    L.ihdg_ws_prof(buf, 1)
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    n = 5
    for _ in range(n):
        sv.sweep_once(a=a)
    e1.record()
    torch.cuda.synchronize()
    L.ihdg_ws_prof(buf, 0)
    print(f"{e0.elapsed_time(e1) / n:.3f} ms / sweep")
    total = buf[6] / n / 148  # per CTA per sweep
    for i, nm in enumerate(NAMES):
        print(f"{nm:36s} {buf[i] / n / 148:14.0f} cycles/CTA/sweep (warp-summed)  {buf[i] / n / 148 / max(total, 1):6.2f}x CTA")


if __name__ == "__main__":
    main()
