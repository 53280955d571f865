"""Small workload for compute-sanitizer (memcheck / racecheck / synccheck): configs[0] and configs[1]
compositions, configs[3] shape at V=2000/D=8 on both paths (push levels only, the tile path, and the
tile path with every level bottom-up), a batch, the wave path (trellises, a trellis batch, eps DAGs), the
eps-filtered variant, provenance + gradient scatter.
Checks each result against the oracle so a sanitizer run also proves the instrumented run is correct."""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tests"))
import fstgen  # noqa: E402
import oracle  # noqa: E402
import paper_2110_02848_b200 as p  # noqa: E402
import pins  # noqa: E402

p.load_library()


def chk(A, B, what, **kw):
    got = pins.canonicalize_rows(p.compose(A, B, **kw), B.num_states)
    pins.assert_canonical_equal(got, oracle.canonical(A, B), what)


for s in (0, 3, 5, 11):
    chk(*fstgen.config_c1(s), f"c1 {s}")
chk(*fstgen.config_c2(0, V=400), "c2 400")
A4, B4 = fstgen.config_c4(V=2000, D=8)
for mode in (0, 2, 3):
    p.fst_set_tile_mode(mode)
    chk(A4, B4, f"c4 2000/8 tile mode {mode}")
    A2, B2 = fstgen.config_c2(0)
    chk(A2, B2, f"c2 1000 tile mode {mode}")
p.fst_set_tile_mode(1)
As = [fstgen.config_c1(s)[0] for s in range(8)]
Bs = [fstgen.config_c1(s)[1] for s in range(8)]
cs = p.fst_compose_batch([p.fst_create(a) for a in As], [p.fst_create(b) for b in Bs])
for s, c in enumerate(cs):
    pins.assert_canonical_equal(pins.canonicalize_rows(c.to_host(), Bs[s].num_states),
                                oracle.canonical(As[s], Bs[s]), f"batch {s}")
# the wave path (topological A): a lexicon o emissions trellis (heavy root / closure state, M3 hubs), a
# batch of trellises over one lexicon (one cluster each), random DAGs with eps (non-uniform rows), with and
# without the shared-memory ELL cache
p.fst_set_wave_mode(2)
A3, B3 = fstgen.config_c3(num_words=200, T=12)
chk(A3, B3, "wave c3 200/12")
for s in range(3):
    chk(fstgen.random_dag(40, 5, 4, 0.2, 50 + s), fstgen.random_graph(50, 3, 4, 60 + s, acceptor=False, eps_prob=0.2),
        f"wave dag {s}")
As5 = [fstgen.emissions_graph(5 + 3 * i, 10000 + i) for i in range(5)]
cs = p.fst_compose_batch([p.fst_create(a) for a in As5], [p.fst_create(B3)] * len(As5))
for i, c in enumerate(cs):
    pins.assert_canonical_equal(pins.canonicalize_rows(c.to_host(), B3.num_states), oracle.canonical(As5[i], B3),
                                f"wave batch {i}")
p.fst_set_wave_mode(1)
A, B = fstgen.config_c2(0, V=300)
p.compose(A, B, eps_filter=True)
c = p.fst_compose(p.fst_create(A), p.fst_create(B), provenance=True)
import torch  # noqa: E402
ga = torch.zeros(A.num_arcs, dtype=torch.float32, device="cuda")
p.fst_grad_scatter(c, torch.ones(c.num_arcs, dtype=torch.float32, device="cuda"), ga, None,
                   stream=torch.cuda.Stream())  # another stream: fst_free must wait for it
c.free()
torch.cuda.synchronize()
print("sanitize driver ok", p.fst_launch_count(), "launches")
