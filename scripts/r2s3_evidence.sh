#!/bin/bash
# round-2 (session 3) evidence: bench lines (configs[3] default, configs[4], reference arm), launch lists of
# one configs[3] and one configs[4] composition, ncu full captures of the wave kernels and the tile emit
set -u
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1 || { tail -30 gpurun_out/build.log; exit 1; }
timeout 900 python bench.py > gpurun_out/ev_bench_c4.log 2>&1; tail -1 gpurun_out/ev_bench_c4.log | cut -c1-300
timeout 900 python bench.py --workload c5 --steps 5 > gpurun_out/ev_bench_c5.log 2>&1; tail -1 gpurun_out/ev_bench_c5.log | cut -c1-300
timeout 600 python bench.py --impl reference --steps 3 --warmup 1 > gpurun_out/ev_bench_ref.log 2>&1; tail -1 gpurun_out/ev_bench_ref.log | cut -c1-300
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/ev_launches_c4.csv python scripts/prof_compose.py --V 20000 --D 8 --n 1 > gpurun_out/ev_ncu_c4.log 2>&1
python scripts/summarize_launches.py gpurun_out/ev_launches_c4.csv > gpurun_out/ev_launch_summary_c4.txt 2>&1; head -14 gpurun_out/ev_launch_summary_c4.txt
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/ev_launches_c5.csv python scripts/prof_compose.py --workload c5 --n 1 > gpurun_out/ev_ncu_c5.log 2>&1
python scripts/summarize_launches.py gpurun_out/ev_launches_c5.csv > gpurun_out/ev_launch_summary_c5.txt 2>&1; head -14 gpurun_out/ev_launch_summary_c5.txt
for ks in k_wave:0 k_wave:1 k_wave_count:0 k_wave_emit:0; do
  k=${ks%%:*}; skip=${ks##*:}
  timeout 900 ncu --set full --clock-control none --import-source on -k regex:"$k\b" -s $skip -c 1 -o gpurun_out/ev_full_${k}_$skip -f \
    python scripts/prof_compose.py --workload c5 --n 0 > gpurun_out/ev_full_${k}_$skip.log 2>&1
  python scripts/ncu_summary.py gpurun_out/ev_full_${k}_$skip.ncu-rep > gpurun_out/ev_full_${k}_$skip.txt 2>&1
  python scripts/ncu_lines.py gpurun_out/ev_full_${k}_$skip.ncu-rep 25 > gpurun_out/ev_full_${k}_${skip}_lines.txt 2>&1
done
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_tile_emit -s 1 -c 1 -o gpurun_out/ev_full_k_tile_emit -f \
    python scripts/prof_compose.py --V 20000 --D 8 --n 1 > gpurun_out/ev_full_k_tile_emit.log 2>&1
python scripts/ncu_summary.py gpurun_out/ev_full_k_tile_emit.ncu-rep > gpurun_out/ev_full_k_tile_emit.txt 2>&1
