#!/bin/bash
# ncu evidence for one round: launch list (time shares) + full captures of the top kernels (c4 20k)
set -u
R=${1:-r01}
mkdir -p gpurun_out/$R
python -c "import __graft_entry__ as g; g.build()" > /dev/null
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/$R/launches_c4_20k.csv \
    python scripts/prof_compose.py --V 20000 --D 8 --n 0 > gpurun_out/$R/launches_run.log 2>&1
ncu --set full --clock-control none --import-source on -k regex:"k_emit" -c 1 -o gpurun_out/$R/emit_c4_20k \
    python scripts/prof_compose.py --V 20000 --D 8 --n 0 > gpurun_out/$R/ncu_emit.log 2>&1
ncu --set full --clock-control none --import-source on -k regex:"k_level" -s 14 -c 1 -o gpurun_out/$R/level14_c4_20k \
    python scripts/prof_compose.py --V 20000 --D 8 --n 0 > gpurun_out/$R/ncu_level.log 2>&1
ncu --set full --clock-control none --import-source on --kernel-name-base demangled -k regex:"k_level<\(bool\)1>" -s 13 -c 1 \
    -o gpurun_out/$R/level2_c4_20k python scripts/prof_compose.py --V 20000 --D 8 --n 0 > gpurun_out/$R/ncu_level2.log 2>&1
ls -la gpurun_out/$R
# c5 (batched lexicon): launch list only
FSTC_NO_GRAPH_LOOP=1 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/$R/launches_c5.csv \
    python scripts/prof_compose.py --workload c5 --n 0 > gpurun_out/$R/launches_c5_run.log 2>&1
ls -la gpurun_out/$R
