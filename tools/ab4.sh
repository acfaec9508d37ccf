#!/bin/bash
# new GPU tests (locally implicit / inflow data / diagnostics) + ws role counters on config 5
O=gpurun_out
mkdir -p $O
timeout 1200 python -m pytest tests/test_gpu_timedep.py tests/test_gpu_diagnostics.py -q > $O/ab4_pytest.txt 2>&1; echo "rc=$?" >> $O/ab4_pytest.txt
IHDG_LIB=paper_1711_01175_b200/libihdg_cuda_prof.so timeout 300 python tools/ws_roles.py 5 > $O/cfg5_roles.txt 2>&1
