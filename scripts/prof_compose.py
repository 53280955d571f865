"""Profiling driver: one warm-up + N compositions of a c4-style workload (for ncu launch lists)."""
import argparse
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import fstgen  # noqa: E402
import paper_2110_02848_b200 as fstc  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--V", type=int, default=8192)
ap.add_argument("--D", type=int, default=8)
ap.add_argument("--T", type=int, default=0)
ap.add_argument("--n", type=int, default=1)
ap.add_argument("--workload", default="random")
args = ap.parse_args()
if args.workload == "c5":
    pass
elif args.workload == "lexicon":
    A, B = fstgen.config_c3(num_words=10000, T=300)
else:
    A, B = fstgen.config_c4(V=args.V, D=args.D, tokens=args.T or None)
if args.workload == "c5":  # the bench's c5 batch (32 utterances, one fst_compose_batch call)
    import bench  # noqa: E402
    As, B, _ = bench.c5_shard(0, 1)
    hb = fstc.fst_create(B)
    ha = [fstc.fst_create(x) for x in As]
    fstc.fst_set_profiling(True)
    for i in range(args.n + 1):
        cs = fstc.fst_compose_batch(ha, [hb] * len(ha))
        print(i, sum(c.num_arcs for c in cs), {k: round(v, 3) if isinstance(v, float) else v
                                               for k, v in cs[0].stats().items()}, flush=True)
        for c in cs:
            c.free()
    sys.exit(0)
a, b = fstc.fst_create(A), fstc.fst_create(B)
fstc.fst_set_profiling(True)
for i in range(args.n + 1):
    c = fstc.fst_compose(a, b)
    print(i, c.num_states, c.num_arcs, {k: round(v, 3) if isinstance(v, float) else v for k, v in c.stats().items()},
          flush=True)
    if i == args.n:
        print("stage1 levels", c.level_sizes(1))
        print("stage2 levels", c.level_sizes(2))
    c.free()
