#!/bin/bash
# last-minute GPU checks: boundary-data tests on the final tree + time to converge (configs 1-4)
O=gpurun_out
mkdir -p $O
timeout 900 python -m pytest tests/test_gpu_timedep.py tests/test_gpu_diagnostics.py -q > $O/final_pytest.txt 2>&1; echo "rc=$?" >> $O/final_pytest.txt
timeout 600 python tools/ttc.py 1 2 3 4 > $O/final_ttc.txt 2>&1
