#!/bin/bash
set -u
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1 || { tail -30 gpurun_out/build.log; exit 1; }
timeout 600 python -m pytest tests/test_gpu_wave.py -m gpu -x -q > gpurun_out/wtests.log 2>&1; tail -2 gpurun_out/wtests.log
for SP in 1 0; do echo SPLIT=$SP; FSTC_WAVE_SPLIT=$SP timeout 600 python bench.py --workload c5 --steps 5 --no-e2e --no-cpu-baseline 2>&1 | tail -1 | grep -o '"ms_per_step": [0-9.]*'; done
