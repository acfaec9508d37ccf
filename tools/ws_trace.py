#!/usr/bin/env python
"""Timeline of one CTA of k_sweep_ws over a few tiles (trace build).

    tools/build_flags.sh ablib/trace.so -DIHDG_WS_TRACE
    IHDG_LIB=ablib/trace.so python tools/ws_trace.py

Prints, per traced iteration, every warp's phase boundaries in clocks relative
to the earliest stamp of that iteration: consumers (warps 0-9) loop top /
qready / done(prev) / norm end / acc loaded / contraction end / outfree /
epilogue end / reduced / fenced; prep warps (10-13) top / full / q done /
done(prev); producer (14) top / empty / issued."""
import ctypes
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

from paper_1711_01175_b200 import _native as N  # noqa: E402
from paper_1711_01175_b200.solver import DeviceSolver  # noqa: E402
from paper_1711_01175_b200.workloads import make_config  # noqa: E402

CONS = ["top", "qready", "done(prev)", "norm", "accld", "contract", "outfree", "epilogue", "reduced", "fenced"]


def main():
    wl = make_config(5)
    sv = DeviceSolver(wl.mesh, wl.problem, wl.ops, dt=wl.dt, max_iters=1000)
    for name, fld in wl.initial.items():
        sv.set_state_component(fld, sv.spec.labels.index(name))
    sv.begin_step()
    sv.reset_state(0.0, 1000)
    a = sv.sweep_args("volume", 1)
    for _ in range(4):
        sv.sweep_once(a=a)
    torch.cuda.synchronize()
    L = N.lib()
    buf = np.zeros((16, 8, 12), dtype=np.int64)
    L.ihdg_ws_trace.argtypes = [ctypes.c_void_p]
    L.ihdg_ws_trace(buf.ctypes.data_as(ctypes.c_void_p))
    for it in range(1, 7):
        t0 = min(buf[w, it, 0] for w in range(15) if buf[w, it, 0] > 0)
        print(f"--- iteration +{it} (clocks after the earliest loop top; next iteration starts at "
              f"{min(buf[w, it + 1, 0] for w in range(10)) - t0})")
        for w in range(15):
            n = 10 if w < 10 else (4 if w < 14 else 3)
            role = "cons" if w < 10 else ("prep" if w < 14 else "prod")
            print(f"  w{w:2d} {role}: " + " ".join(f"{int(buf[w, it, s] - t0):6d}" if buf[w, it, s] else "     -" for s in range(n)))
    print("consumer columns:", " ".join(CONS))


if __name__ == "__main__":
    main()
