"""GPU parity: the CUDA path (through the C ABI) against the CPU oracle, element by element.

Bar (BASELINE.json north_star): bit-exact canonical structure and weights (tolerance 0; every
composed weight is one IEEE binary32 add or a bit copy).  Canonical form: DESIGN.md reading 24.
"""
import numpy as np
import pytest

import fstgen
import golden_io
import oracle
import pins

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def fst():
    import torch
    if not torch.cuda.is_available():
        pytest.skip("needs a CUDA device")
    from paper_2110_02848_b200 import build as b
    b.build()
    import paper_2110_02848_b200 as p
    p.load_library()
    return p


def gpu_canonical(p, A, B):
    return pins.canonicalize_rows(p.compose(A, B), B.num_states)


def check(p, A, B, what, exp=None):
    got = gpu_canonical(p, A, B)
    exp = oracle.canonical(A, B) if exp is None else exp
    pins.assert_canonical_equal(got, exp, what)
    return got


# ----------------------------------------------------------------------------- §3.2 Fig. 1
def test_fig1_in_adjacency(fst):
    g = golden_io.load("fig1_soa.txt")
    A, ex = g["A"], g["expect"]
    h = fst.fst_create(A)
    for on_olabel in (True, False):
        off, arcs = h.adjacency(0, on_olabel)
        assert list(off) == ex["inArcOffset"] and list(arcs) == ex["inArcs"]
        off, arcs = h.adjacency(1, on_olabel)
        assert list(off) == ex["outArcOffset"]
    host = h.to_host()
    assert list(host["is_start"]) == ex["start"] and list(host["is_accept"]) == ex["accept"]


def test_label_sorted_views(fst):
    """Views are sorted by (node, label) with eps (-1) first and arc index as the tie-break."""
    A, _ = fstgen.config_c2(1, V=300)
    h = fst.fst_create(A)
    src = A.src
    for role, node in ((0, A.dst), (1, src)):
        for on_ol, lab in ((True, A.olabel), (False, A.ilabel)):
            off, arcs = h.adjacency(role, on_ol)
            exp = np.lexsort((np.arange(A.num_arcs), lab, node))
            assert np.array_equal(arcs, exp)
            assert np.array_equal(off, np.searchsorted(node[exp], np.arange(A.num_states + 1)))


# ----------------------------------------------------------------------------- hand fixtures
@pytest.mark.parametrize("name", golden_io.ALL_COMPOSE_FIXTURES)
def test_golden_fixture_gpu(fst, name):
    g = golden_io.load(name)
    got = gpu_canonical(fst, g["A"], g["B"])
    pins.assert_canonical_equal(got, g["C"], name)


def test_fig2_round_profile_gpu(fst):
    g = golden_io.load("f2_fig2.txt")
    a, b = fst.fst_create(g["A"]), fst.fst_create(g["B"])
    fst.fst_set_wave_mode(0)  # BFS levels exist on the level path only
    try:
        c = fst.fst_compose(a, b)
    finally:
        fst.fst_set_wave_mode(1)
    assert c.level_sizes(2) == g["levels"]["frontier"]  # |Q| = 1, 2, 2
    assert sum(c.level_sizes(1)) == len(g["R"])


def test_signed_zero_and_tie_gpu(fst):
    C = gpu_canonical(fst, *[golden_io.load("f5b_tie.txt")[k] for k in "AB"])
    assert C["weight"].view(np.uint32)[0] == np.float32(-1.25).view(np.uint32)


# ----------------------------------------------------------------------------- configs vs oracle
def test_c1_all_seeds(fst):
    """configs[0]: 1000 seeds, bit-exact vs the oracle (individual calls for 200, one batch for all)."""
    for s in range(200):
        A, B = fstgen.config_c1(s)
        check(fst, A, B, f"c1 seed {s}")
    pairs = [fstgen.config_c1(s) for s in range(1000)]
    ha = [fst.fst_create(A) for A, _ in pairs]
    hb = [fst.fst_create(B) for _, B in pairs]
    outs = fst.fst_compose_batch(ha, hb)
    for s, ((A, B), c) in enumerate(zip(pairs, outs)):
        got = pins.canonicalize_rows(c.to_host(), B.num_states)
        pins.assert_canonical_equal(got, oracle.canonical(A, B), f"c1 batch seed {s}")


@pytest.mark.parametrize("seed", range(10))
def test_c2_eps_1k(fst, seed):
    """configs[1]: 1k-state transducers with eps (p=0.1 per tape), 20 symbols, degree 4.  About half
    of the seeds give an empty composition (the single accept pair is not reachable backwards);
    those are the "no start pair in R" edge case and must also match."""
    A, B = fstgen.config_c2(seed)
    got = check(fst, A, B, f"c2 seed {seed}")
    if seed in (0, 3, 8, 9):
        assert got["num_arcs"] > 250000


def test_c3_lexicon_emissions(fst):
    """configs[2]: emissions(T=100) o closure(1k-word letter lexicon), vs oracle and trellis."""
    A, B = fstgen.config_c3()
    got = check(fst, A, B, "c3")
    pins.assert_canonical_equal(got, pins.trellis_compose(A, B), "c3 trellis")


@pytest.mark.parametrize("V,D", [(1000, 4), (2000, 8), (4096, 5), (1500, 6)])
def test_c4_random_acceptors(fst, V, D):
    """configs[3] shape at sizes the oracle finishes in seconds; V not a multiple of 32/1024
    exercises ragged words and blocks."""
    A, B = fstgen.config_c4(V=V, D=D)
    check(fst, A, B, f"c4 {V}/{D}")


@pytest.mark.parametrize("D", [4, 8, 16, 32, 64])
def test_fig3b_degree_sweep(fst, D):
    """Fig. 3b: V=256, out-degree D, 2D tokens -- up to 4096 arc pairs and ~32
    matches per state pair; D >= 32 has labels >= 63 (no label masks: the general paths)."""
    A = fstgen.random_graph(256, D, 2 * D, 1000 + 256 + D)
    B = fstgen.random_graph(256, D, 2 * D, 2000 + 256 + D)
    got = check(fst, A, B, f"fig3b D={D}")
    assert got["num_arcs"] > 0


def test_eps_small_graphs(fst):
    for s in range(100):
        A = fstgen.random_graph(12, 3, 4, 500 + s, acceptor=False, eps_prob=0.3, weights="dyadic64")
        B = fstgen.random_graph(12, 3, 4, 900 + s, acceptor=False, eps_prob=0.3, weights="dyadic64")
        check(fst, A, B, f"eps cyclic {s}")
    for s in range(100):
        A = fstgen.random_dag(8, 3, 4, 0.25, 3 * s + 1)
        B = fstgen.random_dag(8, 3, 4, 0.25, 3 * s + 2)
        check(fst, A, B, f"eps dag {s}")


def hub_graph(V, D, tokens, seed, hub_out, hub_in, n_out, n_in):
    """random_graph plus a state with ``n_out`` out-arcs and one with ``n_in`` in-arcs (random labels
    incl. eps, dyadic weights): states above the k_heavy threshold (1024 B arcs) in both stages."""
    g = fstgen.random_graph(V, D, tokens, seed, acceptor=False, eps_prob=0.1, weights="dyadic64")
    r = fstgen.SplitMix64(seed + 77)
    src, dst = list(g.src), list(g.dst)
    il, ol, w = list(g.ilabel), list(g.olabel), list(g.weight)
    for k in range(n_out + n_in):
        src.append(hub_out if k < n_out else r.below(V))
        dst.append(r.below(V) if k < n_out else hub_in)
        il.append(r.below(tokens + 1) - 1)
        ol.append(r.below(tokens + 1) - 1)
        w.append((r.below(64) - 32) / 16.0)
    return fstgen.Fst.from_arcs(V, src, dst, il, ol, w, [0], [V - 1, hub_in])


@pytest.mark.parametrize("n_hub,a_hub", [(1500, 0), (5000, 40), (2049, 20)])
def test_heavy_hub_states(fst, n_hub, a_hub):
    """B states with thousands of arcs (split into grid-wide pieces) x A rows with <= 32 and > 32 arcs."""
    B = hub_graph(3000, 3, 8, 11 + n_hub, 0, 5, n_hub, n_hub)
    A = hub_graph(300, 3, 8, 13 + n_hub, 1, 2, a_hub, 0)
    check(fst, A, B, f"hub {n_hub}/{a_hub}")


def test_c3_heavy_lexicon_root(fst):
    """closure(3000-word lexicon): the root has > 1024 in-arcs (stage 1 pieces)."""
    A, B = fstgen.config_c3(num_words=3000, T=30)
    check(fst, A, B, "c3 3000 words")


def test_identity_at_scale(fst):
    """A o Id == trim(A) on a config-4-sized A (20k states, degree 8)."""
    A, _ = fstgen.config_c4(V=20000, D=8)
    Id = fstgen.identity_fst(range(16))
    check(fst, A, Id, "A o Id", exp=pins.identity_expected(A))
    check(fst, Id, A, "Id o A (same graph as trim(A))", exp=None)


def test_batch_mixed_shapes(fst):
    """fst_compose_batch over heterogeneous compositions equals the individual results."""
    pairs = [fstgen.config_c2(0, V=300), fstgen.config_c1(3), fstgen.config_c3(num_words=50, T=20),
             fstgen.config_c4(V=700, D=4), (fstgen.empty_fst(0), fstgen.config_c1(1)[1]),
             fstgen.config_c1(5)]
    ha = [fst.fst_create(A) for A, _ in pairs]
    hb = [fst.fst_create(B) for _, B in pairs]
    outs = fst.fst_compose_batch(ha, hb)
    for i, ((A, B), c) in enumerate(zip(pairs, outs)):
        got = pins.canonicalize_rows(c.to_host(), B.num_states)
        pins.assert_canonical_equal(got, oracle.canonical(A, B), f"batch item {i}")


# ----------------------------------------------------------------------------- edge cases
def test_empty_and_degenerate(fst):
    A, B = fstgen.config_c1(0)
    for X, Y in ((fstgen.empty_fst(0), B), (A, fstgen.empty_fst(0)), (fstgen.empty_fst(3), B),
                 (A, fstgen.empty_fst(5))):
        got = fst.compose(X, Y)
        assert got["num_states"] == 0 and got["num_arcs"] == 0 and list(got["row_ptr"]) == [0]
    g = golden_io.load("f1_noaccept.txt")
    assert fst.compose(g["A"], g["B"])["num_states"] == 0


def test_invalid_graphs_rejected(fst):
    A, _ = fstgen.config_c1(0)
    bad = []
    x = fstgen.Fst(**{k: getattr(A, k).copy() if hasattr(getattr(A, k), "copy") else getattr(A, k)
                      for k in ("num_states", "row_ptr", "ilabel", "olabel", "dst", "weight", "is_start",
                                "is_accept")})
    x.weight[3] = np.nan
    bad.append(x)
    for field, val in (("dst", 20), ("ilabel", -2), ("olabel", -7)):
        y = fstgen.Fst(**{k: getattr(A, k).copy() if hasattr(getattr(A, k), "copy") else getattr(A, k)
                          for k in ("num_states", "row_ptr", "ilabel", "olabel", "dst", "weight", "is_start",
                                    "is_accept")})
        getattr(y, field)[5] = val
        bad.append(y)
    z = fstgen.Fst(A.num_states, A.row_ptr.copy(), A.ilabel, A.olabel, A.dst, A.weight, A.is_start, A.is_accept)
    z.row_ptr[4], z.row_ptr[5] = z.row_ptr[5], z.row_ptr[4]
    bad.append(z)
    for g in bad:
        with pytest.raises(fst.FstError) as ei:
            fst.fst_create(g)
        assert ei.value.status == 2


def test_determinism(fst):
    A, B = fstgen.config_c4(V=3000, D=8)
    a, b = fst.fst_create(A), fst.fst_create(B)
    r1 = fst.fst_compose(a, b).to_host()
    r2 = fst.fst_compose(a, b).to_host()
    for k in r1:
        assert np.array_equal(np.asarray(r1[k]), np.asarray(r2[k])), k


def test_compose_of_composed(fst):
    """A composed handle is a valid input (views built lazily): (A o B) o Id == A o B."""
    A, B = fstgen.config_c2(2, V=200)
    a, b = fst.fst_create(A), fst.fst_create(B)
    c = fst.fst_compose(a, b)
    C1 = pins.canonicalize_rows(c.to_host(), B.num_states)
    labels = sorted(set(int(x) for x in C1["olabel"] if x >= 0))
    idh = fst.fst_create(fstgen.identity_fst(labels))
    c2 = fst.fst_compose(c, idh).to_host()
    assert c2["num_arcs"] == C1["num_arcs"] or labels == []
    # host-side reference for the second composition: oracle on C's own arrays
    Cfst = fstgen.Fst(C1["num_states"], C1["row_ptr"], C1["ilabel"], C1["olabel"], C1["dst"], C1["weight"],
                      C1["is_start"], C1["is_accept"])
    got = pins.canonicalize_rows(c2, 1)
    pins.assert_canonical_equal(got, oracle.canonical(Cfst, fstgen.identity_fst(labels)), "(A o B) o Id")


@pytest.mark.parametrize("T", [40, 150, 400])
def test_deep_bfs_level_profile(fst, T):
    """Lexicon o emissions is a trellis: one BFS level per frame, so T = 150 / 400 run most levels in the
    graph-driven level loop (levels >= 64).  Per-level frontier sizes of stage 2 equal the oracle's
    FIFO discovery levels (Alg. 1, PAPER.md:207-213 round profile); stage 1 sizes sum to |R|; the graph
    itself equals the oracle's."""
    A, B = fstgen.config_c3(num_words=300, T=T)
    a, b = fst.fst_create(A), fst.fst_create(B)
    fst.fst_set_wave_mode(0)  # the level path (the wave path has no BFS levels; tests/test_gpu_wave.py)
    try:
        c = fst.fst_compose(a, b)
    finally:
        fst.fst_set_wave_mode(1)
    exp = oracle.compose(A, B)
    lv = np.bincount(exp["level"]) if exp["num_states"] else np.zeros(0, np.int64)
    assert c.level_sizes(2) == [int(x) for x in lv]
    assert sum(c.level_sizes(1)) == int(oracle.coaccessible(A, B).sum())
    assert len(c.level_sizes(2)) > (64 if T > 64 else 0)
    pins.assert_canonical_equal(pins.canonicalize_rows(c.to_host(), B.num_states), oracle.canonical(A, B), f"c3 T={T}")


def test_device_tensors_zero_copy(fst):
    """Fst.device_tensors(): zero-copy torch views of the composed graph equal fst_copy_to_host and keep
    the handle alive after the Python wrapper is dropped."""
    import torch
    A, B = fstgen.config_c2(2, V=300)
    c = fst.fst_compose(fst.fst_create(A), fst.fst_create(B), eps_filter=True)
    host = c.to_host()
    t = c.device_tensors()
    del c
    import gc
    gc.collect()
    torch.cuda.synchronize()
    for k in ("row_ptr", "ilabel", "olabel", "dst", "is_start", "is_accept", "pair_a", "pair_b", "pair_f"):
        assert np.array_equal(t[k].cpu().numpy(), host[k]), k
    assert np.array_equal(t["weight"].cpu().numpy().view(np.uint32), host["weight"].view(np.uint32))
