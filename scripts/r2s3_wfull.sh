#!/bin/bash
# ncu --set full of the wave kernels on the c5 batch (KERNELS = "regex:skip ...")
set -u
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1 || { tail -30 gpurun_out/build.log; exit 1; }
if [ -n "${TESTS:-}" ]; then timeout ${TT:-600} python -m pytest ${TESTS} -m gpu -x -q > gpurun_out/tests.log 2>&1; tail -5 gpurun_out/tests.log; fi
for ks in ${KERNELS:-k_wave:1}; do
  k=${ks%%:*}; skip=${ks##*:}
  timeout 900 ncu --set full --clock-control none --import-source on -k regex:$k -s $skip -c 1 -o gpurun_out/wfull_$k -f \
    python scripts/prof_compose.py --workload c5 --n 0 > gpurun_out/wfull_$k.log 2>&1
  python scripts/ncu_summary.py gpurun_out/wfull_$k.ncu-rep 2>&1 | head -45
  python scripts/ncu_lines.py gpurun_out/wfull_$k.ncu-rep 30 > gpurun_out/wfull_${k}_lines.txt 2>&1
done
for ks in ${KERNELS:-k_wave:1}; do k=${ks%%:*}; python scripts/ncu_sass.py gpurun_out/wfull_$k.ncu-rep 0.3 > gpurun_out/wfull_${k}_sass.txt 2>&1; done
