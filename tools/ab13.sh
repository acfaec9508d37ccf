#!/bin/bash
O=gpurun_out
mkdir -p $O
IHDG_LIB=ablib/c5_fuse.so timeout 600 python -m pytest tests/test_gpu_parity.py -q -k "config5" > $O/ab13_pytest.txt 2>&1; echo "rc=$?" >> $O/ab13_pytest.txt
for i in 1 2; do
  for lib in ablib/c5_*.so; do
    echo "$(basename $lib) $(IHDG_LIB=$lib timeout 300 python tools/sweep_cfg.py 5 20 3 2>&1 | tail -1)" >> $O/ab13.txt
  done
done
