#!/bin/bash
# wave path iteration: build, wave tests (+ TESTS; also without the smem ELL cache), c5 profile, c5 bench line
set -u
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1 || { tail -30 gpurun_out/build.log; exit 1; }
timeout ${TT:-600} python -m pytest tests/test_gpu_wave.py ${TESTS:-} -m gpu -x -q > gpurun_out/wtests.log 2>&1; tail -30 gpurun_out/wtests.log
FSTC_WAVE_CACHE=0 timeout 600 python -m pytest tests/test_gpu_wave.py -m gpu -x -q > gpurun_out/wtests_nc.log 2>&1; tail -3 gpurun_out/wtests_nc.log
timeout 300 python scripts/prof_compose.py --workload c5 --n 2 > gpurun_out/wprof.log 2>&1; cut -c1-2500 gpurun_out/wprof.log | tail -20
FSTC_WAVE_CACHE=0 timeout 300 python scripts/prof_compose.py --workload c5 --n 1 2>&1 | tail -1 | cut -c1-400
if [ "${BENCH:-1}" = "1" ]; then
timeout 600 python bench.py --workload c5 --steps 5 --no-e2e --no-cpu-baseline > gpurun_out/wbench.log 2>&1; tail -1 gpurun_out/wbench.log | cut -c1-1800
fi
