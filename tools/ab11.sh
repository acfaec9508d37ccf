#!/bin/bash
O=gpurun_out
mkdir -p $O
IHDG_SWEEP_IMPL=v3 timeout 600 python -m pytest tests/test_gpu_parity.py -q -k "config5" > $O/ab11_pytest.txt 2>&1; echo "rc=$?" >> $O/ab11_pytest.txt
for i in 1 2; do
  echo "ws $(timeout 300 python tools/sweep_cfg.py 5 20 3 2>&1 | tail -1)" >> $O/ab11.txt
  for lib in ablib/c5v3_*.so; do
    echo "v3 $(basename $lib) $(IHDG_SWEEP_IMPL=v3 IHDG_LIB=$lib timeout 300 python tools/sweep_cfg.py 5 20 3 2>&1 | tail -1)" >> $O/ab11.txt
  done
done
