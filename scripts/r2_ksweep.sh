python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1
for KE in 512 256 128 64; do
  echo "KEXIT=$KE"; FSTC_TILE_PULL_KEXIT=$KE timeout 300 python scripts/prof_compose.py --V 20000 --D 8 --n 2 2>&1 | grep "^2 " | python3 -c "
import sys,ast
for l in sys.stdin:
    d=ast.literal_eval(l.split(' ',3)[3]); print({k:d[k] for k in ('ms_stage1','ms_stage2','ms_emit','ms_total','levels_stage1','levels_stage2','pull_levels')})"
done
