python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1
for H in 64 8 2; do
  echo "HOST_LEVELS=$H"; FSTC_HOST_LEVELS=$H timeout 600 python scripts/prof_compose.py --workload c5 --n 2 2>&1 | tail -1 | cut -c1-400
done
