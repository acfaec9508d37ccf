#!/bin/bash
# v3 prep rework: parity (configs 2-4 paths) + A/B on configs 2, 3, 4
O=gpurun_out
mkdir -p $O
timeout 1200 python -m pytest tests/test_gpu_parity.py -q -x -k "config or impl" > $O/ab3_pytest.txt 2>&1; echo "rc=$?" >> $O/ab3_pytest.txt
for i in 1 2; do
  for cfg in 4 3 2; do
    for lib in ablib/head.so ablib/new.so; do
      echo "$(basename $lib) $(IHDG_LIB=$lib timeout 300 python tools/sweep_cfg.py $cfg 50 3 2>&1 | tail -1)" >> $O/ab3.txt
    done
  done
done
