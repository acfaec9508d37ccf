#!/bin/bash
# Config-4 (64^3 p=3 transport, k_sweep_v3) evidence: per-role cycle counters
# (profiling build) and one full ncu capture of the sweep.
O=gpurun_out
mkdir -p $O
IHDG_LIB=paper_1711_01175_b200/libihdg_cuda_prof.so timeout 300 python tools/ws_roles.py 4 > $O/cfg4_roles.txt 2>&1
timeout 300 python tools/sweep_cfg.py 4 20 3 > $O/cfg4_plain.txt 2>&1 && \
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_sweep_v3 -s 3 -c 1 \
  -o $O/cfg4_v3_full -f python tools/sweep_cfg.py 4 5 3 > $O/cfg4_ncu.log 2>&1
echo done
