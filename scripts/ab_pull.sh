#!/bin/bash
# stage-1 pull threshold sweep (FSTC_PULL_NUM) on c4 / c4-d4 / c5, after the parity tests
set -u
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_provenance.py tests/test_gpu_filter.py tests/test_gpu_fullsize.py -x -q > gpurun_out/tests_ab.log 2>&1; tail -1 gpurun_out/tests_ab.log
for w in ${WORKLOADS:-c4 c4-d4 c5}; do
  for k in ${PULLS:-off 4 8 16}; do
    if [ $k = off ]; then export FSTC_NO_PULL=1; else unset FSTC_NO_PULL; export FSTC_PULL_NUM=$k; fi
    timeout 300 python bench.py --workload $w --steps 5 --no-e2e --no-cpu-baseline > gpurun_out/pull_${w}_$k.log 2>&1
    python -c "
import json,sys; d=json.loads(open('gpurun_out/pull_${w}_$k.log').read().strip().splitlines()[-1]); print('$w pull=$k', round(d['value']/1e9,3), round(d['ms_per_step'],2), {k: round(v,2) for k,v in d['phases_ms'].items()}, d['config']['levels'], d['config']['coaccessible'])"
  done
done
