#!/bin/bash
# round-2 (session 4) final check: GPU suite + smoke, bench lines (configs[3] default, configs[4]),
# launch list of one configs[3] composition
set -u
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1 || { tail -30 gpurun_out/build.log; exit 1; }
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv
timeout 1800 python -m pytest tests -m gpu -x -q > gpurun_out/s4f_suite.log 2>&1; tail -3 gpurun_out/s4f_suite.log
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/s4f_smoke.log 2>&1; echo smoke rc $?
timeout 900 python bench.py > gpurun_out/s4f_bench_c4.log 2>&1; tail -1 gpurun_out/s4f_bench_c4.log | cut -c1-300
timeout 900 python bench.py --workload c5 --steps 10 > gpurun_out/s4f_bench_c5.log 2>&1; tail -1 gpurun_out/s4f_bench_c5.log | cut -c1-300
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/s4f_launches_c4.csv python scripts/prof_compose.py --V 20000 --D 8 --T 16 --n 1 > gpurun_out/s4f_ncu_c4.log 2>&1
python scripts/summarize_launches.py gpurun_out/s4f_launches_c4.csv > gpurun_out/s4f_launch_summary_c4.txt 2>&1; head -14 gpurun_out/s4f_launch_summary_c4.txt
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/s4f_launches_c5.csv python scripts/prof_compose.py --workload c5 --n 1 > gpurun_out/s4f_ncu_c5.log 2>&1
python scripts/summarize_launches.py gpurun_out/s4f_launches_c5.csv > gpurun_out/s4f_launch_summary_c5.txt 2>&1; head -14 gpurun_out/s4f_launch_summary_c5.txt
