#!/bin/bash
# round-2 GPU iteration: build, tile tests (+ optional full gpu suite), 20k profile line, bench line
set -u
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1 || { tail -30 gpurun_out/build.log; exit 1; }
timeout ${TT:-600} python -m pytest ${TESTS:-tests/test_gpu_tile.py} -m gpu -x -q > gpurun_out/tests.log 2>&1; tail -15 gpurun_out/tests.log
timeout 300 python scripts/prof_compose.py --V ${V:-20000} --D ${D:-8} --n 2 > gpurun_out/prof.log 2>&1; cut -c1-1500 gpurun_out/prof.log
if [ "${BENCH:-1}" = "1" ]; then
timeout 600 python bench.py --steps 5 --no-e2e --no-cpu-baseline > gpurun_out/bench.log 2>&1; tail -1 gpurun_out/bench.log | cut -c1-1200
fi
