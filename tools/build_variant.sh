#!/bin/bash
# Build an alternative library from a given git revision of csrc/ for A/B
# timing on the same GPU box:  tools/build_variant.sh <rev> <out.so>
set -e
cd "$(dirname "$0")/.."
rev=$1; out=$2
tmp=$(mktemp -d)
mkdir -p "$tmp/paper_1711_01175_b200/csrc" "$tmp/include"
for f in $(git ls-tree --name-only "$rev" paper_1711_01175_b200/csrc/); do git show "$rev:$f" > "$tmp/$f"; done
git show "$rev:include/ihdg.h" > "$tmp/include/ihdg.h"
for f in "$tmp"/paper_1711_01175_b200/csrc/*.cu; do
  nvcc -gencode arch=compute_100a,code=sm_100a -O3 -lineinfo -std=c++17 -Xcompiler -fPIC $EXTRA -I "$tmp/include" -c "$f" -o "$f.o" &
done
wait
nvcc -gencode arch=compute_100a,code=sm_100a -shared -o "$out" "$tmp"/paper_1711_01175_b200/csrc/*.o
rm -rf "$tmp"
echo "built $out from $rev"
