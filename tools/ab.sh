#!/bin/bash
# A/B timing of library builds on one GPU box (interleaved repetitions, so
# every build sees the same clocks and thermal state).
#
#   tools/ab.sh <tag> "<configs>" <reps> lib1.so [lib2.so ...]
#
# Optional: PYTEST_K="<expr>" runs `pytest tests -m gpu -k <expr>` once per
# library first (parity gate of each build).  Output: gpurun_out/ab_<tag>.txt,
# one line per (rep, lib, config) with the ms/sweep of tools/sweep_cfg.py.
# Build the libraries with tools/build_variant.sh (a git revision) or
# tools/build_flags.sh (extra -D flags).
set -u
O=gpurun_out
mkdir -p $O
tag=$1; cfgs=$2; reps=$3; shift 3
out=$O/ab_${tag}.txt
if [ -n "${PYTEST_K:-}" ]; then
  for lib in "$@"; do
    IHDG_LIB=$lib timeout 1200 python -m pytest tests -m gpu -q -k "$PYTEST_K" > $O/ab_${tag}_pytest_$(basename $lib .so).txt 2>&1
    echo "pytest $(basename $lib) rc=$?" >> $out
  done
fi
for i in $(seq 1 $reps); do
  for lib in "$@"; do
    for cfg in $cfgs; do
      n=20; [ "$cfg" != 5 ] && n=50
      echo "$(basename $lib) cfg$cfg $(IHDG_LIB=$lib timeout 300 python tools/sweep_cfg.py $cfg $n 3 2>&1 | tail -1)" >> $out
    done
  done
done
