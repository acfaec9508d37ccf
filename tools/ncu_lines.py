#!/usr/bin/env python
"""Per-source-line attribution of ncu warp-stall samples and executed
instructions (no GPU needed).

    python tools/ncu_lines.py report.ncu-rep <kernel-substring> <object-with-cubin>

Maps the SASS page of the report to source lines with nvdisasm -g on the
kernel's cubin (extracted from the .so / .o with cuobjdump -xelf)."""
import collections
import csv
import glob
import io
import os
import re
import subprocess
import sys
import tempfile


def main(rep, kname, obj):
    sass = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass"],
                          capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(sass)))
    hdr = rows[1]
    data = [r for r in rows[2:] if len(r) == len(hdr)]
    iA, iS = hdr.index("Address"), hdr.index("Source")
    iSm = hdr.index("Warp Stall Sampling (All Samples)")
    iEx = hdr.index("Instructions Executed")
    iWx = hdr.index("L1 Wavefronts Shared Excessive") if "L1 Wavefronts Shared Excessive" in hdr else None
    iW = hdr.index("L1 Wavefronts Shared") if "L1 Wavefronts Shared" in hdr else None
    base = int(data[0][iA], 16)
    tmp = tempfile.mkdtemp()
    subprocess.run(["cuobjdump", "-xelf", "all", os.path.abspath(obj)], cwd=tmp, capture_output=True)
    lines = {}
    for cub in glob.glob(os.path.join(tmp, "*.cubin")):
        dis = subprocess.run(["nvdisasm", "-g", "-c", cub], capture_output=True, text=True).stdout
        cur_fn, cur_line = None, None
        for ln in dis.splitlines():
            m = re.match(r"\s*\.text\.(\S+):", ln)
            if m:
                cur_fn = m.group(1)
            m = re.search(r"//## File \"(.*?)\", line (\d+)", ln)
            if m:
                cur_line = f"{os.path.basename(m.group(1))}:{m.group(2)}"
            m = re.match(r"\s*/\*([0-9a-f]{4,})\*/", ln)
            if m and cur_fn and kname in cur_fn:
                lines[int(m.group(1), 16)] = cur_line
    agg_s, agg_e = collections.Counter(), collections.Counter()
    agg_w, agg_wx = collections.Counter(), collections.Counter()
    for r in data:
        off = int(r[iA], 16) - base
        key = lines.get(off, "?")
        agg_s[key] += float(r[iSm] or 0)
        agg_e[key] += float(r[iEx] or 0)
        if iW is not None:
            agg_w[key] += float(r[iW] or 0)
            agg_wx[key] += float(r[iWx] or 0)
    ts, te = sum(agg_s.values()) or 1, sum(agg_e.values()) or 1
    for key, v in agg_s.most_common(35):
        print(f"{v / ts * 100:5.1f}% stall  {agg_e[key] / te * 100:5.1f}% inst  {key}")
    if agg_w:
        tw = sum(agg_w.values()) or 1
        print("shared-memory wavefronts (total / excess from bank conflicts) by line:")
        for key, v in agg_w.most_common(20):
            print(f"{v / tw * 100:5.1f}% wavefronts  excess {agg_wx[key] / max(v, 1) * 100:5.1f}%  {key}")


if __name__ == "__main__":
    main(*sys.argv[1:4])
