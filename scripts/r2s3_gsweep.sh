python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1
for G in 1 2 4 8; do echo G=$G; FSTC_WAVE_G=$G timeout 300 python scripts/prof_compose.py --workload c5 --n 1 2>&1 | tail -1 | cut -c1-330; done
