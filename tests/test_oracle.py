"""Pins for the CPU oracle (oracle/compose.c), run on the dev box with no GPU (-m "not gpu").

Every check compares the oracle against something other than itself: printed paper arrays,
hand-worked fixtures (tests/golden/, each citing its passage), the plain definition trim(P_N1),
brute-force Eq. (1) path scores, Delannoy path counts, the trellis closed form, the identity
special case and invariants.  See DESIGN.md "Oracle and pins".
"""
import collections
import math

import numpy as np
import pytest

import fstgen
import golden_io
import oracle
import pins
from fstgen import EPS


# ----------------------------------------------------------------------------- generators
def test_splitmix64_reference_vector():
    # splitmix64(seed 0) reference outputs (Vigna's splitmix64.c, standard shift constants)
    r = fstgen.SplitMix64(0)
    assert [r.next() for _ in range(3)] == [0xE220A8397B1DCDAF, 0x6E789E6AA1B965F4, 0x06C45D188009454F]
    r1, r2 = fstgen.SplitMix64(12345), fstgen.SplitMix64(12345)
    blk = r2.block(100)
    assert [r1.next() for _ in range(100)] == [int(x) for x in blk]
    assert r1.next() == r2.next()


def test_below_vec_matches_python():
    r = fstgen.SplitMix64(7).block(1000)
    for n in (1, 5, 20000, (1 << 31) - 1):
        assert [int(x) for x in fstgen.below_vec(r, n)] == [(int(x) * n) >> 64 for x in r]


def test_random_graph_shape():
    g = fstgen.random_graph(256, 5, 10, 3)  # SPEC.md:386 [PAPER §4.1 parameters]
    assert g.num_states == 256 and g.num_arcs == 1280
    assert np.all(np.diff(g.row_ptr) == 5)
    assert np.array_equal(g.ilabel, g.olabel) and g.ilabel.min() >= 0 and g.ilabel.max() < 10
    assert g.is_start.sum() == 1 and g.is_start[0] and g.is_accept.sum() == 1 and g.is_accept[255]
    g2 = fstgen.random_graph(256, 5, 10, 3)
    assert g.to_text() == g2.to_text()


def test_emissions_and_lexicon_shapes():
    e = fstgen.emissions_graph(250, 1, tokens=69)  # SPEC.md:422 [PAPER §4.2: 251 nodes x 69 arcs]
    assert e.num_states == 251 and e.num_arcs == 17250
    # log-softmax rows sum to ~1 in probability
    p = np.exp(e.weight.astype(np.float64).reshape(250, 69)).sum(axis=1)
    assert np.allclose(p, 1.0, atol=1e-5)
    words = fstgen.letter_lexicon(100, 5)
    assert len({tuple(w) for w in words}) == 100 and all(w[-1] == 0 for w in words)
    L = fstgen.lexicon_graph(words)
    assert L.num_states == 1 + sum(len(w) for w in words) and L.num_arcs == sum(len(w) for w in words)
    Lc = fstgen.closure(L)
    assert Lc.num_states == L.num_states + 1 and Lc.num_arcs == L.num_arcs + 1 + 100
    assert Lc.is_start.sum() == 1 and Lc.is_start[-1] and Lc.is_accept.sum() == 1 and Lc.is_accept[-1]


def test_text_roundtrip():
    A, _ = fstgen.config_c2(0, V=50)
    B = fstgen.Fst.from_text(A.to_text())
    for k in ("row_ptr", "ilabel", "olabel", "dst", "is_start", "is_accept"):
        assert np.array_equal(getattr(A, k), getattr(B, k))
    assert np.array_equal(A.weight.view(np.uint32), B.weight.view(np.uint32))
    with pytest.raises(ValueError):
        fstgen.Fst.from_text("nodes 2\narc 0 5 1 1 0.0\n")  # SPEC.md read_text example


# ----------------------------------------------------------------------------- §3.2 Fig. 1 arrays
def test_fig1_soa_in_adjacency():
    g = golden_io.load("fig1_soa.txt")
    A, ex = g["A"], g["expect"]
    assert list(A.is_start) == ex["start"] and list(A.is_accept) == ex["accept"]
    off, arcs = oracle.in_adjacency(A)
    assert list(off) == ex["inArcOffset"] and list(arcs) == ex["inArcs"]
    assert list(A.row_ptr) == ex["outArcOffset"]
    span = arcs[off[2]:off[3]]
    assert list(A.ilabel[span]) == ex["node2_in_ilabels"] and list(A.olabel[span]) == ex["node2_in_olabels"]


# ----------------------------------------------------------------------------- hand fixtures
@pytest.mark.parametrize("name", golden_io.ALL_COMPOSE_FIXTURES)
def test_golden_fixture(name):
    g = golden_io.load(name)
    C = oracle.canonical(g["A"], g["B"])
    pins.assert_canonical_equal(C, g["C"], name)
    if "R" in g:
        R = oracle.coaccessible(g["A"], g["B"])
        VB = g["B"].num_states
        assert sorted((int(k) // VB, int(k) % VB) for k in np.flatnonzero(R)) == g["R"]
    assert pins.is_trim(C)


def test_fig2_round_profile():
    """frontier sizes 1,2,2 and 6,8,0 arc pairs explored per step."""
    g = golden_io.load("f2_fig2.txt")
    A, B = g["A"], g["B"]
    C = oracle.compose(A, B)
    lv = C["level"]
    nlev = lv.max() + 1
    frontier = [int((lv == k).sum()) for k in range(nlev)]
    degA, degB = np.diff(A.row_ptr), np.diff(B.row_ptr)
    explored = [int(sum(degA[C["pair_a"][s]] * degB[C["pair_b"][s]] for s in np.flatnonzero(lv == k)))
                for k in range(nlev)]
    assert frontier == g["levels"]["frontier"] and explored == g["levels"]["explored"]
    # (0,1) is re-reached in step 2 (self-loop a0 x b3) but created only once
    keys = list(zip(C["pair_a"], C["pair_b"]))
    assert keys.count((0, 1)) == 1


def test_signed_zero_and_tie_bits():
    C = oracle.canonical(*[golden_io.load("f5b_tie.txt")[k] for k in "AB"])
    assert C["weight"].view(np.uint32)[0] == np.float32(-1.25).view(np.uint32)
    C = oracle.canonical(*[golden_io.load("f5a_signed_zero.txt")[k] for k in "AB"])
    bits = sorted(int(b) for b in C["weight"].view(np.uint32))
    assert bits == [0, 0, 0, 0x80000000, 0x80000000]


# ----------------------------------------------------------------------------- plain definition
def _check_plain(A, B, what):
    C = oracle.canonical(A, B)
    P = pins.plain_trim_product(A, B, prov=True)  # structure, weights and provenance (arc_a, arc_b)
    pins.assert_canonical_equal(C, P, what)
    R = oracle.coaccessible(A, B)
    assert np.array_equal(R, pins.plain_coaccessible(A, B)), what
    assert pins.is_trim(C), what
    return C


@pytest.mark.parametrize("chunk", range(4))
def test_c1_vs_plain_definition(chunk):
    """configs[0]: 1000 seeds (250 per chunk) of trim(P_N1) vs Algorithm 1, incl. multi start/accept."""
    nonempty = 0
    for s in range(chunk * 250, (chunk + 1) * 250):
        A, B = fstgen.config_c1(s)
        C = _check_plain(A, B, f"c1 seed {s}")
        nonempty += C["num_states"] > 0
    assert nonempty > 50


@pytest.mark.parametrize("seed", range(60))
def test_eps_dags_vs_plain_definition(seed):
    A = fstgen.random_dag(8, 3, 4, 0.25, 3 * seed + 1)
    B = fstgen.random_dag(8, 3, 4, 0.25, 3 * seed + 2)
    _check_plain(A, B, f"eps dag {seed}")


def test_eps_cyclic_vs_plain_definition():
    for s in range(40):
        A = fstgen.random_graph(12, 3, 4, 500 + s, acceptor=False, eps_prob=0.3, weights="dyadic64")
        B = fstgen.random_graph(12, 3, 4, 900 + s, acceptor=False, eps_prob=0.3, weights="dyadic64")
        _check_plain(A, B, f"eps cyclic {s}")


# ----------------------------------------------------------------------------- Eq. (1) brute force
L_MAX = 6


def _bounded_table(table, L):
    return {k: v for k, v in table.items() if len(k[0]) <= L}


@pytest.mark.parametrize("seed", range(0, 200, 5))
def test_eq1_bruteforce_eps_free(seed):
    """configs[0] (eps-free, cyclic): per (x,z) with |x| <= L the multiset of composed path scores
    equals {s_a + s_b} over matched path pairs (no duplicates); logsumexp equal (Eq. (1))."""
    A, B = fstgen.config_c1(seed)
    C = oracle.compose(A, B)
    exp = _bounded_table(pins.eq1_bruteforce(A, B, max_len=L_MAX), L_MAX)
    got = _bounded_table(pins.composed_path_table(C, max_len=L_MAX), L_MAX)
    assert set(got) == set(exp)
    for k in exp:
        assert got[k] == exp[k], k
    lg, le = pins.logsumexp_table(got), pins.logsumexp_table(exp)
    for k in le:
        assert abs(lg[k] - le[k]) <= 1e-12 * max(1.0, abs(le[k]))


@pytest.mark.parametrize("seed", range(100))
def test_eq1_delannoy_eps_dags(seed):
    """eps DAGs: each matched path pair yields prod_i D(k_i, m_i) composed paths of score s_a + s_b;
    the max (Viterbi) score and the (x,z) support equal brute force exactly."""
    eps = 0.2 if seed % 2 else 0.3
    A = fstgen.random_dag(7, 3, 3, eps, 7919 * seed + 11)
    B = fstgen.random_dag(7, 3, 3, eps, 7919 * seed + 13)
    C = oracle.compose(A, B)
    exp = pins.eq1_bruteforce(A, B)
    got = pins.composed_path_table(C)
    assert set(got) == set(exp)
    for k in exp:
        assert got[k] == exp[k], k
        assert max(got[k]) == max(exp[k])


def test_delannoy_inflation_is_exercised():
    hit = 0
    for seed in range(60):
        A = fstgen.random_dag(7, 3, 3, 0.3, 7919 * seed + 11)
        B = fstgen.random_dag(7, 3, 3, 0.3, 7919 * seed + 13)
        exp = pins.eq1_bruteforce(A, B)
        hit += any(c > 1 for cnt in exp.values() for c in cnt.values())
    assert hit > 0
    assert pins.delannoy(1, 1) == 3 and pins.delannoy(2, 2) == 13 and pins.delannoy(0, 5) == 1


# ----------------------------------------------------------------------------- special cases
@pytest.mark.parametrize("seed", range(3))
def test_identity_special_case(seed):
    A = fstgen.random_graph(1000, 4, 8, 77 + seed, acceptor=False, eps_prob=0.1)
    Id = fstgen.identity_fst(range(8))
    pins.assert_canonical_equal(oracle.canonical(A, Id), pins.identity_expected(A), "A o Id")


def test_acceptor_intersection():
    """Acceptor o acceptor = automaton intersection (textbook product + trim); labels are l:l."""
    done = 0
    for V, D in ((60, 4), (80, 5), (50, 6)):
        A, B = fstgen.config_c4(V=V, D=D)
        C = _check_plain(A, B, f"acceptor {V}/{D}")
        assert np.array_equal(C["ilabel"], C["olabel"])
        done += C["num_arcs"] > 0
    assert done >= 2


def test_trellis_lexicon():
    """A = emissions (T=20), B = closure(lexicon of 100 words): closed-form trellis."""
    words = fstgen.letter_lexicon(100, 99)
    B = fstgen.closure(fstgen.lexicon_graph(words))
    A = fstgen.emissions_graph(20, 98)
    C = oracle.canonical(A, B)
    pins.assert_canonical_equal(C, pins.trellis_compose(A, B), "trellis")
    assert C["num_states"] > 1000 and pins.is_trim(C)


def test_size_bounds_and_R_superset():
    A, B = fstgen.config_c2(0, V=300)
    C = oracle.canonical(A, B)
    R = oracle.coaccessible(A, B)
    keys = C["pair_a"].astype(np.int64) * B.num_states + C["pair_b"]
    assert np.all(R[keys] == 1) and R.sum() >= C["num_states"]
    assert C["num_states"] <= A.num_states * B.num_states
    assert C["row_ptr"][-1] == C["num_arcs"] and np.all(np.diff(C["row_ptr"]) >= 0)
    assert pins.is_trim(C)


# ----------------------------------------------------------------------------- provenance
def provenance_consistent(A, B, C, what=""):
    """Every composed arc agrees with the arc pair it names (the move table of SURVEY §8): source and
    destination pairs, the matched labels, the carried labels and the weight bits (one binary32 add
    for M1, a bit copy for M2 / M3).  Vectorised over all arcs; independent of how C was built."""
    E = int(C["num_arcs"])
    src = np.repeat(np.arange(C["num_states"]), np.diff(C["row_ptr"]))
    sa, sb = C["pair_a"][src], C["pair_b"][src]
    da, db = C["pair_a"][C["dst"]], C["pair_b"][C["dst"]]
    aa, ab = C["arc_a"].astype(np.int64), C["arc_b"].astype(np.int64)
    Asrc, Bsrc = A.src, B.src
    assert np.all((aa >= 0) | (ab >= 0)), what
    m1, m2, m3 = (aa >= 0) & (ab >= 0), (aa >= 0) & (ab < 0), (aa < 0) & (ab >= 0)
    assert m1.sum() + m2.sum() + m3.sum() == E, what
    ia, ib = np.where(aa >= 0, aa, 0), np.where(ab >= 0, ab, 0)
    # A side moves along arc_a (M1, M2) or stays (M3); the same for B
    assert np.array_equal(np.where(aa >= 0, Asrc[ia], sa), sa) and np.array_equal(np.where(aa >= 0, A.dst[ia], sa), da), what
    assert np.array_equal(np.where(ab >= 0, Bsrc[ib], sb), sb) and np.array_equal(np.where(ab >= 0, B.dst[ib], sb), db), what
    assert np.all(A.olabel[ia][m1] == B.ilabel[ib][m1]), what
    assert np.all(A.olabel[ia][m2] == pins.EPS) and np.all(B.ilabel[ib][m3] == pins.EPS), what
    assert np.array_equal(C["ilabel"], np.where(aa >= 0, A.ilabel[ia], pins.EPS)), what
    assert np.array_equal(C["olabel"], np.where(ab >= 0, B.olabel[ib], pins.EPS)), what
    wa, wb = A.weight[ia].astype(np.float32), B.weight[ib].astype(np.float32)
    exp = np.where(m1, wa + wb, np.where(m2, wa, wb)).astype(np.float32)
    assert np.array_equal(exp.view(np.uint32), np.asarray(C["weight"], np.float32).view(np.uint32)), what
    # one arc per (source pair, arc pair): no move is emitted twice
    key = (src.astype(np.int64) * (A.num_arcs + 1) + (aa + 1)) * (B.num_arcs + 1) + (ab + 1)
    assert len(np.unique(key)) == E, what


@pytest.mark.parametrize("seed", [0, 3, 8])
def test_provenance_consistent_c2(seed):
    A, B = fstgen.config_c2(seed)
    provenance_consistent(A, B, oracle.canonical(A, B), f"c2 seed {seed}")


def test_provenance_consistent_c3_and_counts():
    """c3 (lexicon o emissions): consistency, and the M1 count of every state equals the number of
    label-matched arc pairs whose destination pair is in C (plain definition, per state)."""
    A, B = fstgen.config_c3(num_words=200, T=30)
    C = oracle.canonical(A, B)
    provenance_consistent(A, B, C, "c3")
    keys = set(zip(C["pair_a"].tolist(), C["pair_b"].tolist()))
    rp = C["row_ptr"]
    for s in range(0, C["num_states"], 97):
        a, b = int(C["pair_a"][s]), int(C["pair_b"][s])
        exp = sorted(mv[4] for mv in pins.n1_moves(A, B, a, b, prov=True) if mv[0] in keys)
        got = sorted(zip(C["arc_a"][rp[s]:rp[s + 1]].tolist(), C["arc_b"][rp[s]:rp[s + 1]].tolist()))
        assert got == exp, s


# ----------------------------------------------------------------------------- forward score
def _lse(vals):
    vals = list(vals)
    if not vals:
        return float("-inf")
    m = max(vals)
    return m + math.log(sum(math.exp(v - m) for v in vals))


@pytest.mark.parametrize("chunk", range(4))
def test_forward_score_bruteforce(chunk):
    """total = logsumexp over every accepting path of C of its weight (path enumeration of the DAG),
    and = logsumexp over the Eq. (1) table of matched A/B path pairs with Delannoy multiplicities:
    two pins independent of the forward recursion (eps DAGs, 100 seeds per chunk)."""
    from oracle import forward as fw
    nonempty = 0
    for seed in range(100 * chunk, 100 * chunk + 100):
        eps = 0.2 if seed % 2 else 0.3
        A = fstgen.random_dag(7, 3, 3, eps, 7919 * seed + 11)
        B = fstgen.random_dag(7, 3, 3, eps, 7919 * seed + 13)
        C = oracle.compose(A, B)
        alpha, total = fw.forward(C)
        w = np.asarray(C["weight"], np.float64)

        class G:  # accepting_paths wants attribute access
            row_ptr, dst = C["row_ptr"], C["dst"]
            is_start, is_accept = C["is_start"], C["is_accept"]
        exp = _lse(sum(w[e] for e in p) for p in pins.accepting_paths(G))
        eq1 = _lse(s + math.log(c) for cnt in pins.eq1_bruteforce(A, B).values() for s, c in cnt.items())
        nonempty += total != float("-inf")
        for ref in (exp, eq1):
            if ref == float("-inf"):
                assert total == ref
            else:
                assert abs(total - ref) <= 1e-9 * max(1.0, abs(ref)), (seed, total, ref)
    assert nonempty >= 10


def test_forward_score_trellis_and_cycles():
    """lexicon o emissions (a DAG): every state has a finite alpha (C is trim, so every state is
    reachable from a start), and a cyclic graph is rejected."""
    from oracle import forward as fw
    A, B = fstgen.config_c3(num_words=100, T=20)
    C = oracle.compose(A, B)
    alpha, total = fw.forward(C)
    assert np.all(np.isfinite(alpha)) and math.isfinite(total)
    A, B = fstgen.config_c1(0)  # random graphs with cycles
    C = oracle.compose(A, B)
    if C["num_states"]:
        with pytest.raises(ValueError):
            fw.forward(C)


# ----------------------------------------------------------------------------- eps-filtered variant
# the three-state eps filter.  Pins: hand-worked
# fixtures, the path bijection of Eq. (1) with eps (one composed path per matched path pair, no
# Delannoy inflation), the plain-definition trim of the filtered product, and reduction to the
# unfiltered composition when there is no eps.
@pytest.mark.parametrize("name", golden_io.FILTER_FIXTURES)
def test_filtered_golden_fixture(name):
    g = golden_io.load(name)
    C = oracle.canonical(g["A"], g["B"], eps_filter=True)
    pins.assert_canonical_equal(C, g["CF"], name)
    assert pins.is_trim(C)


@pytest.mark.parametrize("seed", range(100))
def test_filtered_eq1_bijection_eps_dags(seed):
    """eps DAGs: per (x, z) the multiset of composed path scores equals {s_a + s_b} over matched path
    pairs with multiplicity ONE (Eq. (1), as a sum without duplicated terms)."""
    eps = 0.2 if seed % 2 else 0.3
    A = fstgen.random_dag(7, 3, 3, eps, 7919 * seed + 11)
    B = fstgen.random_dag(7, 3, 3, eps, 7919 * seed + 13)
    C = oracle.compose_filtered(A, B)
    exp = pins.eq1_bruteforce(A, B, filtered=True)
    got = pins.composed_path_table(C)
    assert set(got) == set(exp)
    for k in exp:
        assert got[k] == exp[k], k
    lg, le = pins.logsumexp_table(got), pins.logsumexp_table(exp)
    for k in le:
        assert abs(lg[k] - le[k]) <= 1e-12 * max(1.0, abs(le[k]))


def test_filtered_bijection_differs_from_n1():
    """The filter matters on these inputs: some matched pair has Delannoy multiplicity > 1 under N1
    while the filtered composition has exactly one path for it."""
    hit = 0
    for seed in range(60):
        A = fstgen.random_dag(7, 3, 3, 0.3, 7919 * seed + 11)
        B = fstgen.random_dag(7, 3, 3, 0.3, 7919 * seed + 13)
        n1 = pins.composed_path_table(oracle.compose(A, B))
        fl = pins.composed_path_table(oracle.compose_filtered(A, B))
        hit += sum(n1[k].total() > fl[k].total() for k in fl)
    assert hit > 0


@pytest.mark.parametrize("seed", range(40))
def test_filtered_vs_plain_definition(seed):
    """eps DAGs and cyclic eps transducers: the oracle's FIFO construction equals trim of the full
    filtered product over V_A x V_B x 3."""
    if seed % 2:
        A = fstgen.random_dag(7, 3, 3, 0.3, 104729 * seed + 1)
        B = fstgen.random_dag(7, 3, 3, 0.3, 104729 * seed + 2)
    else:
        A = fstgen.random_graph(9, 2, 3, 5000 + seed, acceptor=False, eps_prob=0.3)
        B = fstgen.random_graph(9, 2, 3, 6000 + seed, acceptor=False, eps_prob=0.3)
    got = oracle.canonical(A, B, eps_filter=True)
    pins.assert_canonical_equal(got, pins.plain_trim_product_filtered(A, B), f"seed {seed}")
    assert pins.is_trim(got)


@pytest.mark.parametrize("seed", range(0, 1000, 50))
def test_filtered_eps_free_reduces_to_unfiltered(seed):
    """Without eps every move is MATCH: the filtered graph is the unfiltered one with f = 0."""
    A, B = fstgen.config_c1(seed)
    got = oracle.canonical(A, B, eps_filter=True)
    exp = oracle.canonical(A, B)
    assert np.all(got["pair_f"] == 0)
    got = dict(got)
    del got["pair_f"]
    pins.assert_canonical_equal(got, exp, f"c1 seed {seed}")


def test_filtered_c2_sizes():
    """configs[1] (eps-1k): the filtered graph is trim, its pair set covers at most 3 copies of the
    unfiltered pairs, and (a, b) projections are states of the unfiltered trim graph."""
    A, B = fstgen.config_c2(1, V=200)
    got = oracle.canonical(A, B, eps_filter=True)
    unf = oracle.canonical(A, B)
    assert pins.is_trim(got)
    pairs = set(zip(unf["pair_a"].tolist(), unf["pair_b"].tolist()))
    assert set(zip(got["pair_a"].tolist(), got["pair_b"].tolist())) <= pairs
    assert got["num_states"] <= 3 * unf["num_states"]


# ----------------------------------------------------------------------------- N-way (left fold)
@pytest.mark.parametrize("seed", range(30))
def test_chain_eq1_three_way_eps_free(seed):
    """N-way composition as ((A o B) o D): per (x, w) the
    multiset of path scores equals {s_a + s_b + s_d} over path triples matched on y and z
    (Eq. (1) applied twice); eps-free inputs, exact dyadic sums."""
    A = fstgen.random_dag(6, 3, 3, 0.0, 31 * seed + 1)
    B = fstgen.random_dag(6, 3, 3, 0.0, 31 * seed + 2)
    D = fstgen.random_dag(6, 3, 3, 0.0, 31 * seed + 3)
    C = oracle.compose_chain([A, B, D])

    def paths(g):
        out = []
        for p in pins.accepting_paths(g):
            out.append((tuple(int(g.ilabel[e]) for e in p), tuple(int(g.olabel[e]) for e in p),
                        sum(float(g.weight[e]) for e in p)))
        return out

    exp = collections.defaultdict(collections.Counter)
    pb = collections.defaultdict(list)
    for y, z, s in paths(B):
        pb[y].append((z, s))
    pd = collections.defaultdict(list)
    for z, w, s in paths(D):
        pd[z].append((w, s))
    for x, y, sa in paths(A):
        for z, sb in pb.get(y, ()):
            for w, sd in pd.get(z, ()):
                exp[(x, w)][sa + sb + sd] += 1
    got = pins.composed_path_table(C)
    assert set(got) == set(exp)
    for k in exp:
        assert got[k] == exp[k], k


@pytest.mark.parametrize("seed", range(10))
def test_canonicalize_any_comparator(seed):
    """The GPU-side comparator (pins.canonicalize_any: any state numbering -> canonical) maps the
    oracle's FIFO-numbered output onto the oracle's own canonical form (pairs and triples)."""
    A = fstgen.random_graph(30, 3, 4, 300 + seed, acceptor=False, eps_prob=0.3)
    B = fstgen.random_graph(30, 3, 4, 400 + seed, acceptor=False, eps_prob=0.3)
    for filt in (False, True):
        raw = oracle.compose(A, B, eps_filter=filt)
        raw = {k: v for k, v in raw.items() if k not in ("arc_a", "arc_b")}
        exp = {k: v for k, v in oracle.canonical(A, B, eps_filter=filt).items() if k not in ("arc_a", "arc_b")}
        pins.assert_canonical_equal(pins.canonicalize_any(raw, B.num_states), exp, f"seed {seed} filter {filt}")


@pytest.mark.parametrize("seed", range(20))
def test_filtered_chain_three_way_bijection(seed):
    """The eps-filtered composition applied twice ((A o B) o D on eps DAGs) has exactly one path per
    matched path triple, score s_a + s_b + s_d (Eq. (1) applied twice, eps-free label strings)."""
    from types import SimpleNamespace

    def paths(g):
        out = []
        for p in pins.accepting_paths(g):
            il = tuple(int(g.ilabel[e]) for e in p if g.ilabel[e] != EPS)
            ol = tuple(int(g.olabel[e]) for e in p if g.olabel[e] != EPS)
            out.append((il, ol, sum(float(g.weight[e]) for e in p)))
        return out

    gs = [fstgen.random_dag(6, 3, 3, 0.25, 104729 * seed + k) for k in (5, 6, 7)]
    c1 = oracle.compose_filtered(gs[0], gs[1])
    c1n = SimpleNamespace(num_states=int(c1["num_states"]), num_arcs=int(c1["num_arcs"]),
                          **{k: c1[k] for k in ("row_ptr", "ilabel", "olabel", "dst", "weight", "is_start", "is_accept")})
    got = pins.composed_path_table(oracle.compose_filtered(c1n, gs[2]))
    pb, pd = collections.defaultdict(list), collections.defaultdict(list)
    for y, z, sb in paths(gs[1]):
        pb[y].append((z, sb))
    for z, w, sd in paths(gs[2]):
        pd[z].append((w, sd))
    exp = collections.defaultdict(collections.Counter)
    for x, y, sa in paths(gs[0]):
        for z, sb in pb.get(y, ()):
            for w, sd in pd.get(z, ()):
                exp[(x, w)][sa + sb + sd] += 1
    assert got == exp
