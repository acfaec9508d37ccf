#!/bin/bash
O=gpurun_out
mkdir -p $O
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_variants.py -q -k "config2 or config3 or config4 or table2 or cd or sw or transport" > $O/ab16_pytest.txt 2>&1; echo "rc=$?" >> $O/ab16_pytest.txt
for i in 1 2; do
  for lib in ablib/noguard.so ablib/guard.so; do
    for cfg in 4 3 2; do
      echo "$(basename $lib) $(IHDG_LIB=$lib timeout 120 python tools/sweep_cfg.py $cfg 50 3 2>&1 | tail -1)" >> $O/ab16.txt
    done
  done
  for lib in ablib/guard_c4*.so; do
    echo "$(basename $lib) $(IHDG_LIB=$lib timeout 120 python tools/sweep_cfg.py 4 50 3 2>&1 | tail -1)" >> $O/ab16.txt
  done
done
