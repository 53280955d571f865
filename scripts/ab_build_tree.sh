#!/bin/bash
# Builds libfstc.so from the WORKING TREE with extra nvcc flags into ab/libfstc_<name>.so (A/B of
# compile-time variants):  scripts/ab_build_tree.sh e768 -DFSTC_E_THREADS=768
set -eu
NAME=$1; shift
ROOT=$(cd "$(dirname "$0")/.." && pwd)
TMP=$(mktemp -d)
mkdir -p "$ROOT/ab"
FLAGS="-gencode arch=compute_100a,code=sm_100a -O3 -lineinfo -std=c++17 -Xcompiler -fPIC --expt-relaxed-constexpr --extended-lambda -I $ROOT/include $*"
for f in "$ROOT"/paper_2110_02848_b200/csrc/*.cu; do
  s=$(basename "$f" .cu)
  /usr/local/cuda/bin/nvcc $FLAGS -c "$f" -o "$TMP/$s.o" &
done
wait
/usr/local/cuda/bin/nvcc -shared -gencode arch=compute_100a,code=sm_100a -o "$ROOT/ab/libfstc_$NAME.so" "$TMP"/*.o -lcudart
rm -rf "$TMP"
echo "$ROOT/ab/libfstc_$NAME.so"
