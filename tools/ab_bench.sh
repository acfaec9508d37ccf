#!/bin/bash
# A/B the config-5 sweep time of two library builds on the same box.
CMD="python bench.py --steps 20 --warmup 3 --ttc-steps 0 --no-e2e --no-cpu --no-others"
for i in 1 2 3; do
  for lib in "$@"; do
    ms=$(IHDG_LIB=$lib timeout 300 $CMD 2>/dev/null | tail -1 | python -c "import sys,json; print(json.loads(sys.stdin.read())['ms_per_step'])")
    echo "$(basename $lib) $ms"
  done
done
