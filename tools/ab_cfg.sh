#!/bin/bash
# A/B the per-sweep time of one config across library builds on one box:
#   tools/ab_cfg.sh <config> lib1.so lib2.so ...
cfg=$1; shift
for i in 1 2; do
  for lib in "$@"; do
    echo "$(basename $lib) $(IHDG_LIB=$lib timeout 300 python tools/sweep_cfg.py $cfg 20 3 2>&1 | tail -1)"
  done
done
