#!/bin/bash
# ncu full captures of the configs[3] stage-2 round (k_tile_pull<true, *, 896>) and k_tile_emit (896 threads)
set -u
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1 || { tail -30 gpurun_out/build.log; exit 1; }
timeout 900 ncu --set full --clock-control none --import-source on --kernel-name-base demangled -k regex:'k_tile_pull<.bool.1' -s 2 -c 1 \
  -o gpurun_out/s4_full_k_tile_pull_s2 -f python scripts/prof_compose.py --V 20000 --D 8 --T 16 --n 0 > gpurun_out/s4_full_k_tile_pull_s2.log 2>&1
python scripts/ncu_summary.py gpurun_out/s4_full_k_tile_pull_s2.ncu-rep > gpurun_out/s4_full_k_tile_pull_s2.txt 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_tile_emit -s 1 -c 1 \
  -o gpurun_out/s4_full_k_tile_emit -f python scripts/prof_compose.py --V 20000 --D 8 --T 16 --n 1 > gpurun_out/s4_full_k_tile_emit.log 2>&1
python scripts/ncu_summary.py gpurun_out/s4_full_k_tile_emit.ncu-rep > gpurun_out/s4_full_k_tile_emit.txt 2>&1
for f in gpurun_out/s4_full_k_tile_pull_s2.txt gpurun_out/s4_full_k_tile_emit.txt; do grep -E 'gpu__time_duration.sum|smsp__inst_executed.sum |issue_active|registers' $f | head -5; done
