#!/bin/bash
# one GPU round-trip: build, gpu tests, 8k profile line, 20k bench line (logs under gpurun_out/)
set -u
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1 || { tail -20 gpurun_out/build.log; exit 1; }
if [ "${SKIP_TESTS:-0}" != "1" ]; then
  timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/tests.log 2>&1; tail -3 gpurun_out/tests.log
fi
timeout 300 python scripts/prof_compose.py --V 8192 --D 8 --n 1 > gpurun_out/prof8k.log 2>&1; sed -n 2p gpurun_out/prof8k.log
timeout 900 python bench.py --steps ${STEPS:-5} ${BENCH_ARGS:---no-e2e --no-cpu-baseline} > gpurun_out/bench.log 2>&1; tail -1 gpurun_out/bench.log
