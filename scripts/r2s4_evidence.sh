#!/bin/bash
# round-2 (session 4) evidence: GPU suite + smoke, bench lines (configs[3] default, configs[4], reference
# arm), launch list of one configs[4] composition, ncu full captures of the wave kernels
set -u
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1 || { tail -30 gpurun_out/build.log; exit 1; }
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv
timeout 1800 python -m pytest tests -m gpu -x -q > gpurun_out/s4_suite.log 2>&1; tail -3 gpurun_out/s4_suite.log
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/s4_smoke.log 2>&1; echo smoke rc $?
timeout 900 python bench.py > gpurun_out/s4_bench_c4.log 2>&1; tail -1 gpurun_out/s4_bench_c4.log | cut -c1-300
timeout 900 python bench.py --workload c5 --steps 10 > gpurun_out/s4_bench_c5.log 2>&1; tail -1 gpurun_out/s4_bench_c5.log | cut -c1-300
timeout 600 python bench.py --impl reference --steps 3 --warmup 3 > gpurun_out/s4_bench_ref.log 2>&1; tail -1 gpurun_out/s4_bench_ref.log | cut -c1-300
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/s4_launches_c5.csv python scripts/prof_compose.py --workload c5 --n 1 > gpurun_out/s4_ncu_c5.log 2>&1
python scripts/summarize_launches.py gpurun_out/s4_launches_c5.csv > gpurun_out/s4_launch_summary_c5.txt 2>&1; head -14 gpurun_out/s4_launch_summary_c5.txt
for ks in k_wave:0 k_wave:1 k_wave_count:0 k_wave_emit:0; do
  k=${ks%%:*}; skip=${ks##*:}
  timeout 900 ncu --set full --clock-control none --import-source on -k regex:"$k\b" -s $skip -c 1 -o gpurun_out/s4_full_${k}_$skip -f \
    python scripts/prof_compose.py --workload c5 --n 0 > gpurun_out/s4_full_${k}_$skip.log 2>&1
  python scripts/ncu_summary.py gpurun_out/s4_full_${k}_$skip.ncu-rep > gpurun_out/s4_full_${k}_$skip.txt 2>&1
  python scripts/ncu_lines.py gpurun_out/s4_full_${k}_$skip.ncu-rep 25 > gpurun_out/s4_full_${k}_${skip}_lines.txt 2>&1
done
