set -u
O=gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv > $O/ab1_gpu.txt
timeout 600 python -m pytest tests/test_gpu_parity.py -m gpu -q -k "impl_parity" > $O/ab1_pytest.txt 2>&1; echo "rc=$?" >> $O/ab1_pytest.txt
for i in 1 2; do
 for impl in ws ws4; do
  echo "$impl $(IHDG_SWEEP_IMPL=$impl timeout 300 python tools/sweep_cfg.py 5 20 3 2>&1 | tail -1)" >> $O/ab1.txt
 done
done
for impl in v3 ws4; do
 echo "cfg4 $impl $(IHDG_SWEEP_IMPL=$impl timeout 300 python tools/sweep_cfg.py 4 50 3 2>&1 | tail -1)" >> $O/ab1.txt
done
