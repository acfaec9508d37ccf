#!/bin/bash
O=gpurun_out
mkdir -p $O
for i in 1 2; do
  for lib in ablib/c5_*.so; do
    echo "$(basename $lib) $(IHDG_LIB=$lib timeout 300 python tools/sweep_cfg.py 5 20 3 2>&1 | tail -1)" >> $O/ab10.txt
  done
done
