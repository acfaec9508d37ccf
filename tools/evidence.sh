#!/bin/bash
# Round evidence on one B200: GPU tests, smoke, default bench (both arms),
# ncu launch list of the bench command, one full ncu capture of the config-5
# sweep and of the config-4 sweep.  Every ncu command runs only after the same
# command has exited 0 without ncu.   tools/evidence.sh <tag> [skip-tests]
set -u
O=gpurun_out
TAG=${1:-r02}
mkdir -p $O
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,power.draw,temperature.gpu --format=csv > $O/${TAG}_gpu.txt
if [ "${2:-}" != "skip-tests" ]; then
  timeout 2400 python -m pytest tests -m gpu -q > $O/${TAG}_pytest_gpu.txt 2>&1; echo "pytest rc=$?" >> $O/${TAG}_pytest_gpu.txt
  timeout 300 python -c "import __graft_entry__ as g; g.smoke(); print('smoke ok')" > $O/${TAG}_smoke.txt 2>&1
fi
timeout 1200 python bench.py > $O/${TAG}_bench.json 2> $O/${TAG}_bench.err
timeout 600 python bench.py --impl reference > $O/${TAG}_bench_reference.json 2> $O/${TAG}_bench_reference.err
CMD="python bench.py --steps 20 --warmup 3 --ttc --no-e2e --no-cpu --no-others"
if timeout 300 $CMD > $O/${TAG}_bench_short.json 2>&1; then
  timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv \
    --log-file $O/${TAG}_launches.csv $CMD > $O/${TAG}_ncu_launches.log 2>&1
fi
CMD3="python bench.py --steps 3 --warmup 3 --ttc --no-e2e --no-cpu --no-others"
if timeout 300 $CMD3 > $O/${TAG}_bench_short3.json 2>&1; then
  timeout 1200 ncu --set full --clock-control none --import-source on -k regex:^k_sweep_ws -s 2 -c 1 \
    -o $O/${TAG}_ws_full -f $CMD3 > $O/${TAG}_ncu_full.log 2>&1
fi
if timeout 300 python tools/sweep_cfg.py 4 20 3 > $O/${TAG}_cfg4_plain.txt 2>&1; then
  timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_sweep_v4 -s 3 -c 1 \
    -o $O/${TAG}_cfg4_v4_full -f python tools/sweep_cfg.py 4 5 3 > $O/${TAG}_cfg4_ncu.log 2>&1
fi
echo done
