"""GPU parity of the eps-filtered composition (fst_compose_ex with
FST_COMPOSE_EPS_FILTER) and of N-way chains (rank 4; fst_compose_chain), through the C ABI.

The CUDA path builds the filtered product as A~ o F o B~ with the binary kernels (filter.cu); the
oracle runs the three-state filter directly over (a, b, f) triples (oracle/compose.c,
orc_compose_filtered).  Both are compared in canonical form (states ascending by
(a * V_B + b) * 3 + f, rows sorted), weights bit-exact (tolerance 0).
"""
import numpy as np
import pytest

import fstgen
import golden_io
import oracle
import pins
from test_gpu_parity import hub_graph

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


def gpu_filtered(p, A, B, provenance=False):
    g = p.compose(A, B, provenance=provenance, eps_filter=True)
    assert "pair_f" in g and len(g["pair_f"]) == g["num_states"]
    return pins.canonicalize_any(g, B.num_states)


def check(p, A, B, what, provenance=False):
    got = gpu_filtered(p, A, B, provenance)
    exp = oracle.canonical(A, B, eps_filter=True)
    if not provenance:
        exp = {k: v for k, v in exp.items() if k not in ("arc_a", "arc_b")}
    pins.assert_canonical_equal(got, exp, what)
    return got


@pytest.mark.parametrize("name", golden_io.FILTER_FIXTURES)
def test_filtered_golden_fixture_gpu(fst, name):
    g = golden_io.load(name)
    pins.assert_canonical_equal(gpu_filtered(fst, g["A"], g["B"]), g["CF"], name)


def test_filtered_c1_seeds(fst):
    """configs[0] (eps-free): every state has f = 0."""
    for s in range(0, 1000, 10):
        A, B = fstgen.config_c1(s)
        got = check(fst, A, B, f"c1 seed {s}")
        assert np.all(got["pair_f"] == 0)


def test_filtered_eps_dags_and_bijection(fst):
    """eps DAGs: parity with the oracle, and the GPU graph's path table is Eq. (1) with one path per
    matched path pair (the oracle's pin, re-checked on the GPU output)."""
    for seed in range(100):
        eps = 0.2 if seed % 2 else 0.3
        A = fstgen.random_dag(7, 3, 3, eps, 7919 * seed + 11)
        B = fstgen.random_dag(7, 3, 3, eps, 7919 * seed + 13)
        got = check(fst, A, B, f"eps dag {seed}")
        if seed % 10 == 0:
            exp = pins.eq1_bruteforce(A, B, filtered=True)
            assert pins.composed_path_table(got) == exp


def test_filtered_cyclic_eps(fst):
    for seed in range(40):
        A = fstgen.random_graph(60, 3, 4, 5000 + seed, acceptor=False, eps_prob=0.3)
        B = fstgen.random_graph(60, 3, 4, 6000 + seed, acceptor=False, eps_prob=0.3)
        check(fst, A, B, f"cyclic eps {seed}")


@pytest.mark.parametrize("seed", range(10))
def test_filtered_c2(fst, seed):
    """configs[1]: 1k-state transducers with eps on both tapes (p = 0.1)."""
    A, B = fstgen.config_c2(seed)
    check(fst, A, B, f"c2 seed {seed}")


def test_filtered_c3_lexicon(fst):
    """configs[2]: emissions (no eps) o closure(lexicon) (eps inputs on B): only f in {0, 2}."""
    A, B = fstgen.config_c3()
    got = check(fst, A, B, "c3")
    assert set(np.unique(got["pair_f"]).tolist()) <= {0, 2}


def test_filtered_wide_labels_and_hubs(fst):
    """Labels >= 63 (the general, non-mask paths of the kernels) and hub states."""
    A = fstgen.random_graph(200, 4, 100, 71, acceptor=False, eps_prob=0.2)
    B = fstgen.random_graph(200, 4, 100, 72, acceptor=False, eps_prob=0.2)
    check(fst, A, B, "100 labels")
    B = hub_graph(3000, 3, 8, 11, 0, 5, 1500, 1500)
    A = hub_graph(300, 3, 8, 13, 1, 2, 40, 0)
    check(fst, A, B, "hubs")


def test_filtered_batch_and_provenance(fst):
    pairs = [fstgen.config_c2(s, V=300) for s in range(4)]
    pairs += [(fstgen.random_dag(7, 3, 3, 0.3, 7919 * s + 11), fstgen.random_dag(7, 3, 3, 0.3, 7919 * s + 13))
              for s in range(4)]
    a = [fst.fst_create(A) for A, _ in pairs]
    b = [fst.fst_create(B) for _, B in pairs]
    cs = fst.fst_compose_batch(a, b, eps_filter=True)
    for i, ((A, B), c) in enumerate(zip(pairs, cs)):
        got = pins.canonicalize_any(c.to_host(), B.num_states)
        exp = {k: v for k, v in oracle.canonical(A, B, eps_filter=True).items() if k not in ("arc_a", "arc_b")}
        pins.assert_canonical_equal(got, exp, f"batch {i}")
    for i, (A, B) in enumerate(pairs):
        check(fst, A, B, f"provenance {i}", provenance=True)


def test_filtered_empty_and_errors(fst):
    E = fstgen.empty_fst(0)
    A, _ = fstgen.config_c2(0, V=100)
    got = fst.compose(E, A, eps_filter=True)
    assert got["num_states"] == 0 and len(got["pair_f"]) == 0
    a = fst.fst_create(A)
    with pytest.raises(fst.FstError):
        fst.fst_compose_ex(a, a, 4)  # unknown flag bit
    with pytest.raises(fst.FstError):
        fst.fst_compose(a, a).pair_f()  # not a filtered composition


# ----------------------------------------------------------------------------- N-way chains
def test_chain_three_and_four_way(fst):
    """fst_compose_chain == the oracle's left fold with canonical intermediates (pair_a indexes the
    previous step's states in ascending key order on both sides)."""
    for seed in range(12):
        eps = 0.0 if seed % 3 == 0 else 0.2
        gs = [fstgen.random_graph(40, 3, 4, 900 + 10 * seed + k, acceptor=False, eps_prob=eps) for k in range(3 + seed % 2)]
        hs = [fst.fst_create(g) for g in gs]
        c = fst.fst_compose_chain(hs)
        got = pins.canonicalize_rows(c.to_host(), gs[-1].num_states)
        exp = oracle.compose_chain(gs, canonicalize=True)
        exp = {k: v for k, v in exp.items() if k not in ("arc_a", "arc_b")}
        pins.assert_canonical_equal(got, exp, f"chain seed {seed}")


def test_chain_lexicon_pipeline(fst):
    """emissions o closure(lexicon) o word acceptor-like identity: the 3-way chain equals the 2-way
    composition when the last factor is the identity over the output alphabet."""
    A, B = fstgen.config_c3(num_words=200, T=30)
    words = sorted(set(int(x) for x in B.olabel if x >= 0))
    Id = fstgen.identity_fst(words)
    c3 = fst.fst_compose_chain([fst.fst_create(A), fst.fst_create(B), fst.fst_create(Id)])
    got = pins.canonicalize_rows(c3.to_host(), Id.num_states)
    exp = {k: v for k, v in oracle.compose_chain([A, B, Id], canonicalize=True).items() if k not in ("arc_a", "arc_b")}
    pins.assert_canonical_equal(got, exp, "lexicon chain")


def test_chain_eps_filtered_three_way_bijection(fst):
    """fst_compose_chain with the eps filter on three eps DAGs: every matched path triple
    (pi_a: x->y, pi_b: y->z, pi_d: z->w, eps-free label strings) yields exactly ONE composed path of
    score s_a + s_b + s_d (Eq. (1) applied twice, no duplicated terms)."""
    import collections

    def paths(g):
        out = []
        for p in pins.accepting_paths(g):
            il = tuple(int(g.ilabel[e]) for e in p if g.ilabel[e] != pins.EPS)
            ol = tuple(int(g.olabel[e]) for e in p if g.olabel[e] != pins.EPS)
            out.append((il, ol, sum(float(g.weight[e]) for e in p)))
        return out

    for seed in range(20):
        gs = [fstgen.random_dag(6, 3, 3, 0.25, 104729 * seed + k) for k in (5, 6, 7)]
        c = fst.fst_compose_chain([fst.fst_create(g) for g in gs], eps_filter=True)
        got = pins.composed_path_table(c.to_host())
        pb = collections.defaultdict(list)
        for y, z, sb in paths(gs[1]):
            pb[y].append((z, sb))
        pd = collections.defaultdict(list)
        for z, w, sd in paths(gs[2]):
            pd[z].append((w, sd))
        exp = collections.defaultdict(collections.Counter)
        for x, y, sa in paths(gs[0]):
            for z, sb in pb.get(y, ()):
                for w, sd in pd.get(z, ()):
                    exp[(x, w)][sa + sb + sd] += 1
        assert got == exp, f"seed {seed}"
