#!/bin/bash
set -u
O=gpurun_out; TAG=r01h
mkdir -p $O
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,power.draw,temperature.gpu --format=csv > $O/${TAG}_gpu.txt
timeout 1500 python -m pytest tests -m gpu -q > $O/${TAG}_pytest_gpu.txt 2>&1; echo "pytest rc=$?" >> $O/${TAG}_pytest_gpu.txt
timeout 300 python -c "import __graft_entry__ as g; g.smoke(); print('smoke ok')" > $O/${TAG}_smoke.txt 2>&1
timeout 900 python bench.py > $O/${TAG}_bench.json 2> $O/${TAG}_bench.err
timeout 600 python bench.py --impl reference > $O/${TAG}_bench_reference.json 2> $O/${TAG}_bench_reference.err
CMD="python bench.py --steps 20 --warmup 3 --ttc-steps 0 --no-e2e --no-cpu --no-others"
if timeout 300 $CMD > $O/${TAG}_bench_short.json 2>&1; then
  timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv \
    --log-file $O/${TAG}_launches.csv $CMD > $O/${TAG}_ncu_launches.log 2>&1
fi
echo done
