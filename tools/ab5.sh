#!/bin/bash
O=gpurun_out
mkdir -p $O
timeout 1200 python -m pytest tests/test_gpu_timedep.py -q > $O/ab5_pytest.txt 2>&1; echo "rc=$?" >> $O/ab5_pytest.txt
timeout 900 python -m pytest tests/test_gpu_parity.py -q -k "config5 or config1 or impl_parity and ws" > $O/ab5_pytest_ws.txt 2>&1; echo "rc=$?" >> $O/ab5_pytest_ws.txt
for i in 1 2; do
  for lib in ablib/head.so ablib/new.so; do
    echo "$(basename $lib) $(IHDG_LIB=$lib timeout 300 python tools/sweep_cfg.py 5 20 3 2>&1 | tail -1)" >> $O/ab5.txt
  done
done
