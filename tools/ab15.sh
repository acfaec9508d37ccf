#!/bin/bash
O=gpurun_out
mkdir -p $O
for i in 1 2; do
  for lib in ablib/c4_*.so; do
    echo "$(basename $lib) $(IHDG_LIB=$lib timeout 300 python tools/sweep_cfg.py 4 50 3 2>&1 | tail -1)" >> $O/ab15.txt
  done
  for lib in ablib/c4_base.so ablib/c3_*.so; do
    for cfg in 3 2; do
      echo "$(basename $lib) $(IHDG_LIB=$lib timeout 300 python tools/sweep_cfg.py $cfg 50 3 2>&1 | tail -1)" >> $O/ab15.txt
    done
  done
done
