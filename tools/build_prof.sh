#!/bin/bash
# Profiling variant of the library with per-role cycle counters (not shipped
# on the product path): paper_1711_01175_b200/libihdg_cuda_prof.so
set -e
cd "$(dirname "$0")/.."
mkdir -p build/prof
for f in paper_1711_01175_b200/csrc/*.cu; do
  nvcc -gencode arch=compute_100a,code=sm_100a -O3 -lineinfo -std=c++17 -Xcompiler -fPIC -DIHDG_WS_PROF \
    -I include -c "$f" -o "build/prof/$(basename "$f").o" &
done
wait
nvcc -gencode arch=compute_100a,code=sm_100a -shared -o paper_1711_01175_b200/libihdg_cuda_prof.so build/prof/*.o
echo built paper_1711_01175_b200/libihdg_cuda_prof.so
