#!/bin/bash
O=gpurun_out
mkdir -p $O
timeout 600 python -m pytest tests/test_gpu_variants.py -q -k "exact" > $O/ab7_pytest.txt 2>&1; echo "rc=$?" >> $O/ab7_pytest.txt
for i in 1 2; do
  for lib in ablib/c4_*.so; do
    echo "$(basename $lib) $(IHDG_LIB=$lib timeout 300 python tools/sweep_cfg.py 4 50 3 2>&1 | tail -1)" >> $O/ab7.txt
  done
done
