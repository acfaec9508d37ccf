#!/bin/bash
# diagnostics GPU tests + config-4 v3 warp-shape A/B
O=gpurun_out
mkdir -p $O
timeout 900 python -m pytest tests/test_gpu_diagnostics.py -q -x > $O/ab2_pytest.txt 2>&1; echo "rc=$?" >> $O/ab2_pytest.txt
for i in 1 2; do
  for lib in paper_1711_01175_b200/libihdg_cuda.so ablib/c4_*.so; do
    echo "$(basename $lib) $(IHDG_LIB=$lib timeout 300 python tools/sweep_cfg.py 4 50 3 2>&1 | tail -1)" >> $O/ab2.txt
  done
done
