#!/bin/bash
# ncu --set full captures of the tile kernels on one 20k composition (+ tile tests first)
set -u
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1 || { tail -30 gpurun_out/build.log; exit 1; }
if [ -n "${TESTS:-}" ]; then timeout ${TT:-600} python -m pytest ${TESTS} -m gpu -x -q > gpurun_out/tests.log 2>&1; tail -5 gpurun_out/tests.log; fi
for ks in ${KERNELS:-k_tile_pull:16 k_tile_emit:1}; do
  k=${ks%%:*}; skip=${ks##*:}
  timeout 900 ncu --set full --clock-control none --import-source on -k regex:$k -s $skip -c 1 -o gpurun_out/full_$k -f \
    python scripts/prof_compose.py --V ${V:-20000} --D ${D:-8} --n 1 > gpurun_out/full_$k.log 2>&1
  python scripts/ncu_summary.py gpurun_out/full_$k.ncu-rep 2>&1 | head -45
done
