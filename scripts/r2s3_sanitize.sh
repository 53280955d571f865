#!/bin/bash
# compute-sanitizer memcheck / racecheck / synccheck over scripts/sanitize_driver.py (incl. the wave path),
# with and without the wave path's shared-memory ELL cache
set -u
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1 || { tail -30 gpurun_out/build.log; exit 1; }
for tool in memcheck racecheck synccheck; do
  extra=""
  [ $tool = racecheck ] && extra="--racecheck-report all"
  timeout 1500 compute-sanitizer --tool $tool $extra --print-limit 50 --error-exitcode 9 \
     python scripts/sanitize_driver.py > gpurun_out/s3_sanitize_$tool.log 2>&1
  echo "$tool rc=$?"; tail -4 gpurun_out/s3_sanitize_$tool.log
done
FSTC_WAVE_CACHE=0 timeout 1500 compute-sanitizer --tool memcheck --print-limit 50 --error-exitcode 9 \
   python scripts/sanitize_driver.py > gpurun_out/s3_sanitize_memcheck_nocache.log 2>&1
echo "memcheck nocache rc=$?"; tail -3 gpurun_out/s3_sanitize_memcheck_nocache.log
