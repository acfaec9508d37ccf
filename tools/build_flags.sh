#!/bin/bash
# Build the current tree with extra nvcc flags into another library for A/B
# timing on the same GPU box:  tools/build_flags.sh <out.so> -DFOO=1 ...
set -e
cd "$(dirname "$0")/.."
out=$1; shift
tmp=$(mktemp -d)
for f in paper_1711_01175_b200/csrc/*.cu; do
  nvcc -gencode arch=compute_100a,code=sm_100a -O3 -lineinfo -std=c++17 -Xcompiler -fPIC "$@" \
    -I include -c "$f" -o "$tmp/$(basename "$f").o" &
done
wait
nvcc -gencode arch=compute_100a,code=sm_100a -shared -o "$out" "$tmp"/*.o
rm -rf "$tmp"
echo "built $out ($*)"
