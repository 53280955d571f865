#!/bin/bash
# GPU check of the eps-filter path: its parity tests, then bench --eps-filter on c5 and c4 (A/B vs ab/libfstc_base.so)
set -u
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_filter.py tests/test_gpu_parity.py -x -q > gpurun_out/tests_ab.log 2>&1; tail -1 gpurun_out/tests_ab.log
for w in c5 c4; do
  for t in base new; do
    if [ $t = base ]; then export FSTC_LIB=ab/libfstc_base.so; else unset FSTC_LIB; fi
    timeout 300 python bench.py --workload $w --eps-filter --steps 3 --no-e2e --no-cpu-baseline > gpurun_out/ab_${t}_${w}f.log 2>&1
    python -c "
import json,sys; d=json.loads(open('gpurun_out/ab_${t}_${w}f.log').read().strip().splitlines()[-1]); print('$t ${w}f', round(d['value']/1e9,3), round(d['ms_per_step'],2), {k: round(v,2) for k,v in d['phases_ms'].items()})"
  done
done
