#!/bin/bash
# Emit A/B on configs[3]: tile tests on the in-tree build, then bench phases for each ab/libfstc_*.so
# listed in $LIBS (name:path, "tree" = in-tree build).
set -u
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1 || { tail -30 gpurun_out/build.log; exit 1; }
timeout ${TT:-900} python -m pytest ${TESTS:-tests/test_gpu_tile.py} -m gpu -x -q > gpurun_out/tests.log 2>&1; tail -3 gpurun_out/tests.log
for nl in ${LIBS:-tree}; do
  n=${nl%%:*}; l=${nl#*:}
  if [ "$l" = tree ]; then unset FSTC_LIB; else export FSTC_LIB=$l; fi
  for rep in 1 2; do
    timeout 300 python bench.py --steps 5 --no-e2e --no-cpu-baseline ${BARGS:-} > gpurun_out/ab_$n.log 2>&1
    python -c "
import json; d=json.loads(open('gpurun_out/ab_$n.log').read().strip().splitlines()[-1]); print('$n', round(d['ms_per_step'],2), {k: round(v,2) for k,v in d['phases_ms'].items()})"
  done
done
unset FSTC_LIB
