#!/bin/bash
# A/B on one GPU box: parity subset with the in-tree build, then bench.py with ab/libfstc_base.so
# (scripts/ab_build.sh) vs the in-tree build on c4 and c5; optional ncu capture of k_emit (NCU=1).
set -u
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_provenance.py tests/test_gpu_filter.py -x -q > gpurun_out/tests_ab.log 2>&1; tail -2 gpurun_out/tests_ab.log
for w in ${WORKLOADS:-c4 c5}; do
  FSTC_LIB=ab/libfstc_base.so timeout 300 python bench.py --workload $w --steps 5 --no-e2e --no-cpu-baseline > gpurun_out/ab_base_$w.log 2>&1
  timeout 300 python bench.py --workload $w --steps 5 --no-e2e --no-cpu-baseline > gpurun_out/ab_new_$w.log 2>&1
  for t in base new; do python -c "
import json,sys; d=json.loads(open('gpurun_out/ab_${t}_$w.log').read().strip().splitlines()[-1]); print('$t $w', round(d['value']/1e9,3), round(d['ms_per_step'],2), {k: round(v,2) for k,v in d['phases_ms'].items()})"; done
done
if [ "${NCU:-0}" = "1" ]; then
  timeout 600 ncu --set full --clock-control none --import-source on -k regex:"${NCU_K:-k_emit}" -s ${NCU_S:-0} -c 1 -o gpurun_out/${NCU_NAME:-emit_c4} \
    python scripts/prof_compose.py --V 20000 --D 8 --n 0 > gpurun_out/ncu_run.log 2>&1; tail -2 gpurun_out/ncu_run.log
fi
