#!/bin/bash
# Builds libfstc.so from git revision $1 (default HEAD) into ab/libfstc_<name>.so for A/B timing:
#   FSTC_LIB=ab/libfstc_base.so python bench.py ...   (fstc.py loads FSTC_LIB instead of the in-tree build)
set -eu
REV=${1:-HEAD}
NAME=${2:-base}
ROOT=$(cd "$(dirname "$0")/.." && pwd)
TMP=$(mktemp -d)
mkdir -p "$TMP/p/csrc" "$TMP/include" "$ROOT/ab"
for f in $(git -C "$ROOT" ls-tree --name-only "$REV" paper_2110_02848_b200/csrc/); do
  git -C "$ROOT" show "$REV:$f" > "$TMP/p/csrc/$(basename "$f")"
done
git -C "$ROOT" show "$REV:include/fstc.h" > "$TMP/include/fstc.h"
FLAGS="-gencode arch=compute_100a,code=sm_100a -O3 -lineinfo -std=c++17 -Xcompiler -fPIC --expt-relaxed-constexpr --extended-lambda -I $TMP/include"
for s in $(git -C "$ROOT" ls-tree --name-only "$REV" paper_2110_02848_b200/csrc/ | grep "\.cu$" | xargs -n1 basename | sed "s/\.cu$//"); do
  /usr/local/cuda/bin/nvcc $FLAGS -c "$TMP/p/csrc/$s.cu" -o "$TMP/$s.o" &
done
wait
/usr/local/cuda/bin/nvcc -shared -gencode arch=compute_100a,code=sm_100a -o "$ROOT/ab/libfstc_$NAME.so" "$TMP"/*.o -lcudart
rm -rf "$TMP"
echo "$ROOT/ab/libfstc_$NAME.so"
