#!/bin/bash
# round-2 evidence: bench lines (c4 default, c5), launch list of one c4 compose, ncu full captures
set -u
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1 || { tail -30 gpurun_out/build.log; exit 1; }
timeout 900 python bench.py --steps 10 > gpurun_out/bench_c4.log 2>&1; tail -1 gpurun_out/bench_c4.log | cut -c1-300
timeout 900 python bench.py --workload c5 --steps 5 --no-e2e > gpurun_out/bench_c5.log 2>&1; tail -1 gpurun_out/bench_c5.log | cut -c1-300
timeout 600 python bench.py --impl reference --steps 3 --warmup 1 > gpurun_out/bench_ref.log 2>&1; tail -1 gpurun_out/bench_ref.log | cut -c1-300
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches.csv python scripts/prof_compose.py --V 20000 --D 8 --n 1 > gpurun_out/ncu_prof.log 2>&1
python scripts/summarize_launches.py gpurun_out/launches.csv > gpurun_out/launch_summary.txt 2>&1; head -12 gpurun_out/launch_summary.txt
for ks in k_tile_emit:1 k_tile_pull:14 k_level:30; do
  k=${ks%%:*}; skip=${ks##*:}
  timeout 900 ncu --set full --clock-control none --import-source on -k regex:$k -s $skip -c 1 -o gpurun_out/full_$k -f \
    python scripts/prof_compose.py --V 20000 --D 8 --n 1 > gpurun_out/full_$k.log 2>&1
  python scripts/ncu_summary.py gpurun_out/full_$k.ncu-rep > gpurun_out/full_$k.txt 2>&1
done
