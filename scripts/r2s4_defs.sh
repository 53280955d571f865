#!/bin/bash
# build-variant sweep: for each ';'-separated FSTC_BUILD_DEFS set in $VARIANTS, rebuild, run $TESTS (if
# set) and one profiled composition of $WORKLOAD (c5: configs[4] batch, c4: configs[3])
set -u
IFS=';' read -ra VS <<< "${VARIANTS:-}"
for v in "${VS[@]}"; do
  touch paper_2110_02848_b200/csrc/*.cu
  FSTC_BUILD_DEFS="$v" python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1 || { echo "build [$v] failed"; continue; }
  echo "V=[$v]"
  if [ -n "${TESTS:-}" ]; then timeout 600 python -m pytest $TESTS -m gpu -x -q 2>&1 | tail -1; fi
  if [ "${WORKLOAD:-c5}" = "c5" ]; then
    for G in ${GS:-4}; do FSTC_WAVE_G=$G timeout 300 python scripts/prof_compose.py --workload c5 --n 2 2>&1 | grep "^2 " | tail -1 | cut -c1-600; done
  else
    timeout 300 python scripts/prof_compose.py --V 20000 --D 8 --T 16 --n 2 2>&1 | grep "^2 " | tail -1 | cut -c1-600
  fi
done
