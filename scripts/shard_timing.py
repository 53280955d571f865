"""Per-rank work of the sharded composition, estimated on ONE GPU: the shards of fst_compose_sharded_local
run one after the other, so (time of the call) / world ~ the time one rank of a `world`-GPU run spends
in its kernels (excluding NCCL transfers and the cross-rank wait)."""
import sys, os, time, json
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import fstgen
import paper_2110_02848_b200 as p
p.load_library()
A, B = fstgen.config_c4(V=int(sys.argv[1]) if len(sys.argv) > 1 else 20000, D=8)
a, b = p.fst_create(A), p.fst_create(B)
out = {}
def t(f, n=3):
    f(); torch.cuda.synchronize()
    ts = []
    for _ in range(n):
        t0 = time.perf_counter(); r = f(); torch.cuda.synchronize(); ts.append(time.perf_counter() - t0)
        for c in (r if isinstance(r, list) else [r]): c.free()
    return min(ts) * 1e3
out["unsharded_ms"] = t(lambda: p.fst_compose(a, b))
for w in (1, 2, 4, 8):
    ms = t(lambda: p.fst_compose_sharded_local(a, b, w))
    out[f"local_world{w}_ms"] = ms
    out[f"local_world{w}_per_rank_ms"] = ms / w
print(json.dumps(out))
