#!/usr/bin/env python
"""Instruction-class counts of the production sweep kernels in the in-tree
libihdg_cuda.so (cuobjdump -sass; no GPU needed).

    python tools/sass_summary.py [lib] > profiles/rNN_sass_summary.txt

Counts are static (instructions in the kernel body, not executions): DMMA is
the fp64 tensor-core MMA, UBLKCP the bulk (TMA) copies, SYNCS the mbarrier
operations, LDG/STG global loads/stores, LDS/STS shared memory."""

from __future__ import annotations

import os
import re
import subprocess
import sys
from collections import Counter

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
CLASSES = ["DMMA", "DFMA", "DADD", "DMUL", "UBLKCP", "SYNCS", "LDG", "STG", "LDS", "STS", "LDGSTS",
           "SHFL", "BAR", "ATOMG", "RED", "MEMBAR"]


def demangle(name: str) -> str:
    r = subprocess.run(["c++filt", name], capture_output=True, text=True)
    return r.stdout.strip() or name


def main() -> None:
    lib = sys.argv[1] if len(sys.argv) > 1 else os.path.join(ROOT, "paper_1711_01175_b200", "libihdg_cuda.so")
    sass = subprocess.run(["cuobjdump", "-sass", lib], capture_output=True, text=True, check=True).stdout
    kernels: dict[str, Counter] = {}
    cur = None
    for line in sass.splitlines():
        m = re.search(r"Function : (\S+)", line)
        if m:
            cur = m.group(1)
            kernels[cur] = Counter()
            continue
        if cur is None:
            continue
        m = re.search(r"/\*[0-9a-f]{4,}\*/\s+(?:@!?U?P\w+\s+)?([A-Z][A-Z0-9_]*)(\.[A-Z0-9_.]+)?", line)
        if not m:
            continue
        op = m.group(1)
        kernels[cur]["total"] += 1
        if op in CLASSES:
            kernels[cur][op] += 1
    prod = [k for k in kernels if re.search(r"k_sweep_ws|k_sweep_v4|k_sweep_v5|k_sweep_gemv|k_sweep_v3|k_sweep[^_]|k_finalize|k_layer_sums", k)]
    print(f"# static SASS instruction counts, {os.path.relpath(lib, ROOT)} (cuobjdump -sass)")
    hdr = ["kernel", "total"] + CLASSES
    print("\t".join(hdr))
    for k in prod:
        c = kernels[k]
        print("\t".join([demangle(k).replace("void ihdg::", "").split("(")[0], str(c["total"])]
                        + [str(c[x]) for x in CLASSES]))


if __name__ == "__main__":
    main()
