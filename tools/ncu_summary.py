#!/usr/bin/env python
"""Summarise an ncu report (run here, no GPU): key throughput numbers and the
warp-stall breakdown.  Usage: python tools/ncu_summary.py report.ncu-rep"""
import csv
import io
import subprocess
import sys

KEYS = ["Duration", "DRAM Throughput", "Memory Throughput", "L1/TEX Hit Rate", "L2 Hit Rate",
        "Executed Ipc Active", "Issue Slots Busy", "Eligible Warps Per Scheduler",
        "Warp Cycles Per Issued Instruction", "Executed Instructions", "Registers Per Thread",
        "Achieved Occupancy", "Dynamic Shared Memory Per Block"]


def main(path):
    out = subprocess.run(["ncu", "-i", path, "--page", "details", "--csv"], capture_output=True,
                         text=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    hdr = rows[0]
    for r in rows[1:]:
        d = dict(zip(hdr, r))
        name = d.get("Metric Name", "")
        if name in KEYS:
            print(f"{d.get('Kernel Name','')[:40]:40s} {name:36s} {d.get('Metric Value',''):>16s} {d.get('Metric Unit','')}")
    raw = subprocess.run(["ncu", "-i", path, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rr = list(csv.reader(io.StringIO(raw)))
    h, v = rr[0], rr[2]
    stalls = []
    want = ("dram__bytes_read.sum", "dram__bytes_write.sum", "gpu__time_duration.sum",
            "sm__inst_executed_pipe_fp64.avg.pct_of_peak_sustained_active",
            "sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active",
            "sm__inst_executed_pipe_tensor_subpipe_dmma.avg.pct_of_peak_sustained_active",
            "sm__ops_path_tensor_src_fp64.avg.pct_of_peak_sustained_elapsed",
            "smsp__inst_executed.sum", "lts__t_bytes.sum")
    for i, n in enumerate(h):
        if n in want:
            print(f"{n:60s} {v[i]:>20s} {rr[1][i]}")
        if n.startswith("smsp__pcsamp_warps_issue_stalled") and not n.endswith("not_issued"):
            try:
                stalls.append((float(v[i].replace(",", "")), n.replace("smsp__pcsamp_warps_issue_stalled_", "")))
            except ValueError:
                pass
    tot = sum(s for s, _ in stalls) or 1.0
    print("stalls:", ", ".join(f"{n} {s / tot * 100:.0f}%" for s, n in sorted(stalls, reverse=True)[:8]))


if __name__ == "__main__":
    main(sys.argv[1])
