#!/usr/bin/env python
"""Run one BASELINE config (reduced) and save the successive norms and the
final field (bitwise comparison of two library builds via IHDG_LIB).
    python tools/dump_norms.py <config> <cells> <out.npz>"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402

from tools.check_impl import solve  # noqa: E402
from paper_1711_01175_b200.workloads import make_config  # noqa: E402

cfg, cells, out = int(sys.argv[1]), int(sys.argv[2]), sys.argv[3]
r = solve(make_config(cfg, cells=cells), "auto")
np.savez(out, norms=np.asarray(r.successive_norms), u=r.state.data, it=r.iterations)
print(r.extra["kernel"], r.iterations)
