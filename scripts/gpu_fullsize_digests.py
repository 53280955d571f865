import sys, os, time, json
sys.path.insert(0, '.'); sys.path.insert(0, 'tests')
import fstgen, digest
import paper_2110_02848_b200 as p
p.load_library()
out = {}
for name, kw in (("c4_20000_d8_t16", dict(V=20000, D=8, tokens=16)), ("c4_20000_d8_t8", dict(V=20000, D=8, tokens=8))):
    A, B = fstgen.config_c4(**kw)
    t = time.time()
    c = p.fst_compose(p.fst_create(A), p.fst_create(B))
    d = digest.digest_device(c.device_tensors(), B.num_states)
    d["stats"] = {k: v for k, v in c.stats().items() if not isinstance(v, float)}
    out[name] = d
    print(name, d, round(time.time() - t, 1), flush=True)
    c.free()
json.dump(out, open("gpurun_out/gpu_fullsize_digests.json", "w"), indent=1)
