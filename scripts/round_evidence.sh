#!/bin/bash
# End-of-round evidence on one GPU box: full GPU test suite, bench lines (c4 default with e2e and the
# CPU baseline, c5, c5 eps-filtered, the oracle reference arm) and the ncu captures (profile_round.sh).
set -u
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1 || { tail -20 gpurun_out/build.log; exit 1; }
timeout 1500 python -m pytest tests -m gpu -q > gpurun_out/tests_all.log 2>&1; tail -2 gpurun_out/tests_all.log
timeout 900 python bench.py > gpurun_out/bench_c4_full.log 2>&1; tail -1 gpurun_out/bench_c4_full.log
timeout 900 python bench.py --workload c5 > gpurun_out/bench_c5_full.log 2>&1; tail -1 gpurun_out/bench_c5_full.log
timeout 600 python bench.py --workload c5 --eps-filter --no-e2e --no-cpu-baseline --steps 3 > gpurun_out/bench_c5_filter.log 2>&1; tail -1 gpurun_out/bench_c5_filter.log
timeout 600 python bench.py --impl reference --steps 2 --warmup 1 > gpurun_out/bench_ref.log 2>&1; tail -1 gpurun_out/bench_ref.log
timeout 1200 bash scripts/profile_round.sh ${R:-r01} > gpurun_out/profile_round.log 2>&1; tail -3 gpurun_out/profile_round.log
