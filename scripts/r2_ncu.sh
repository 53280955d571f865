#!/bin/bash
# launch list of one 20k composition (after one warm-up) + the tile tests
set -u
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1 || { tail -30 gpurun_out/build.log; exit 1; }
timeout ${TT:-600} python -m pytest ${TESTS:-tests/test_gpu_tile.py} -m gpu -x -q > gpurun_out/tests.log 2>&1; tail -15 gpurun_out/tests.log
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches.csv python scripts/prof_compose.py --V ${V:-20000} --D ${D:-8} --n 1 > gpurun_out/ncu_prof.log 2>&1
python scripts/summarize_launches.py gpurun_out/launches.csv 2>&1 | tail -60
