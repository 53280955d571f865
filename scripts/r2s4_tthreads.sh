#!/bin/bash
# tile-path CTA size sweep on configs[3] (pull / count kernels: FSTC_TILE_THREADS_BUILD; emit: FSTC_EMIT_THREADS_BUILD)
set -u
for T in ${THREADS:-1024 512 768}; do
  touch paper_2110_02848_b200/csrc/compose.cu
  FSTC_TILE_THREADS_BUILD=$T FSTC_EMIT_THREADS_BUILD=${ET:-1024} python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1 || { echo build $T failed; continue; }
  echo T=$T ET=${ET:-1024}
  if [ -n "${TESTS:-}" ]; then timeout 600 python -m pytest $TESTS -m gpu -x -q 2>&1 | tail -1; fi
  timeout 300 python scripts/prof_compose.py --V 20000 --D 8 --T 16 --n 2 2>&1 | grep "^2 " | tail -1 | cut -c1-600
done
