"""Profiling driver for fst_forward_score on one c5 utterance composition (ncu launch lists)."""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import bench  # noqa: E402
import paper_2110_02848_b200 as fstc  # noqa: E402

As, B, _ = bench.c5_shard(0, 1)
hb = fstc.fst_create(B)
c = fstc.fst_compose(fstc.fst_create(As[0]), hb)
print("V", c.num_states, "E", c.num_arcs, flush=True)
for i in range(int(sys.argv[1]) if len(sys.argv) > 1 else 2):
    torch.cuda.synchronize()
    t = time.time()
    tot = fstc.fst_forward_score(c)
    torch.cuda.synchronize()
    print(i, tot, f"{(time.time() - t) * 1e3:.1f} ms", flush=True)
