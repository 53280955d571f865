#!/bin/bash
# session-3 baseline: full GPU suite, configs[3] and configs[4] bench lines, launch list of configs[4]
set -u
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1 || { tail -30 gpurun_out/build.log; exit 1; }
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv
timeout 1500 python -m pytest tests -m gpu -x -q > gpurun_out/tests.log 2>&1; tail -5 gpurun_out/tests.log
timeout 600 python bench.py --steps 10 --no-e2e --no-cpu-baseline > gpurun_out/bench_c4.log 2>&1; tail -1 gpurun_out/bench_c4.log | cut -c1-1500
timeout 600 python bench.py --workload c5 --steps 5 --no-e2e --no-cpu-baseline > gpurun_out/bench_c5.log 2>&1; tail -1 gpurun_out/bench_c5.log | cut -c1-1500
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_c5.csv python scripts/prof_compose.py --workload c5 --n 1 > gpurun_out/ncu_c5.log 2>&1; echo ncu rc $?
