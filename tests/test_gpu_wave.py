"""GPU parity of the wave path (stage 1 / stage 2 row by row for a topologically
numbered A, one thread-block cluster per composition, then k_wave_count and the general emit) against
the CPU oracle, bit-exact (tolerance 0).  Inputs: lexicon o emissions trellises (configs[2] / configs[4]
shape: heavy lexicon root and closure state, M3 eps closure inside a row), batches of them (one cluster
per utterance), random DAG transducers with eps on both tapes (M1 eps:eps, M2 to arbitrary later rows,
M3 chains), multiple start / accept states, empty and degenerate inputs.  The wave path and the level
path use the same emit, so their arrays are identical, not only canonically equal."""
import numpy as np
import pytest

import fstgen
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
    p.fst_set_wave_mode(2)
    yield p
    p.fst_set_wave_mode(1)


def both_paths(p, pairs):
    """(wave outputs, level outputs, wave stats) of one fst_compose_batch call per path."""
    ha = [p.fst_create(A) for A, _ in pairs]
    hb = [p.fst_create(B) for _, B in pairs]
    p.fst_set_wave_mode(2)
    w = p.fst_compose_batch(ha, hb)
    st = w[0].stats() if w else {}
    p.fst_set_wave_mode(0)
    try:
        lv = p.fst_compose_batch(ha, hb)
    finally:
        p.fst_set_wave_mode(2)
    return [c.to_host() for c in w], [c.to_host() for c in lv], st


def check_pairs(p, pairs, what, oracle_check=True):
    got, lev, st = both_paths(p, pairs)
    assert st.get("tile_path", 2) == 2, st
    for i, ((A, B), g, l) in enumerate(zip(pairs, got, lev)):
        for k in g:
            assert np.array_equal(np.asarray(g[k]), np.asarray(l[k])), f"{what} item {i}: {k} wave != level path"
        if oracle_check:
            pins.assert_canonical_equal(pins.canonicalize_rows(g, B.num_states), oracle.canonical(A, B),
                                        f"{what} item {i}")
    return got


@pytest.mark.parametrize("T", [1, 7, 40, 100])
def test_wave_c3_trellis(fst, T):
    """configs[2] shape: closure(1k-word letter lexicon) o emissions(T): the root (1k out-arcs) and the
    closure state (1k eps in-arcs) are heavy columns; accept -> closure -> root is an M3 chain."""
    A, B = fstgen.config_c3(num_words=1000, T=T)
    check_pairs(fst, [(A, B)], f"c3 T={T}")


def test_wave_c3_against_trellis_pin(fst):
    A, B = fstgen.config_c3(num_words=1000, T=100)
    got = check_pairs(fst, [(A, B)], "c3", oracle_check=False)[0]
    pins.assert_canonical_equal(pins.canonicalize_rows(got, B.num_states), pins.trellis_compose(A, B), "c3 trellis")


def test_wave_c5_batch(fst):
    """configs[4] shape at oracle size: one 2000-word lexicon shared by 12 utterances with T in [3, 90]
    (batch: 12 clusters, LPT order)."""
    As, B = fstgen.config_c5(num_utts=12, num_words=2000)
    rng = np.random.default_rng(5)
    As = [fstgen.emissions_graph(int(t), 10000 + i) for i, t in enumerate(rng.integers(3, 91, size=12))]
    check_pairs(fst, [(A, B) for A in As], "c5-like batch")


@pytest.mark.parametrize("seed", range(12))
def test_wave_random_dag_eps(fst, seed):
    """Random DAG transducers (dst > src) with eps on both tapes: A's eps-output arcs give M2 moves to
    arbitrary later rows and M1 eps:eps, B's eps-input arcs M3 chains inside a row; B is a random graph
    with cycles (the wave path needs only A topological)."""
    A = fstgen.random_dag(60, 6, 5, 0.2, 3 * seed + 1)
    B = fstgen.random_graph(70, 4, 5, 3 * seed + 2, acceptor=False, eps_prob=0.2)
    check_pairs(fst, [(A, B)], f"dag seed {seed}")


def test_wave_dag_batch_multi_start_accept(fst):
    pairs = []
    for s in range(16):
        A = fstgen.random_dag(40 + s, 5, 4, 0.15, 100 + s, starts=[0, 1], accepts=[36, 38, 39 + s])
        B = fstgen.random_graph(50, 3, 4, 200 + s, acceptor=False, eps_prob=0.15, starts=[0, 2],
                                accepts=[40, 45, 49])
        pairs.append((A, B))
    check_pairs(fst, pairs, "dag batch")


def test_wave_heavy_columns(fst):
    """B hubs in both directions (> 32 items: walked by the whole CTA) with eps on the hub arcs."""
    rng = np.random.default_rng(7)
    V = 300
    src = list(rng.integers(0, V, 900)) + [0] * 200 + list(rng.integers(0, V, 150))
    dst = list(rng.integers(0, V, 900)) + list(rng.integers(0, V, 200)) + [5] * 150
    E = len(src)
    il = rng.integers(-1, 6, E)
    ol = rng.integers(-1, 6, E)
    order = np.argsort(np.asarray(src), kind="stable")
    B = fstgen.Fst.from_arcs(V, np.asarray(src)[order], np.asarray(dst)[order], il[order], ol[order],
                             (rng.integers(-64, 64, E) / 64.0).astype(np.float32)[order], [0, 5], [5, 7, 9])
    A = fstgen.random_dag(50, 8, 6, 0.2, 77, starts=[0], accepts=[45, 49])
    check_pairs(fst, [(A, B)], "heavy")


def test_wave_empty_and_degenerate(fst):
    A, B = fstgen.config_c3(num_words=50, T=5)
    for X, Y in ((fstgen.empty_fst(0), B), (A, fstgen.empty_fst(0)), (fstgen.empty_fst(3), B),
                 (A, fstgen.empty_fst(5))):
        got = fst.compose(X, Y)
        assert got["num_states"] == 0 and got["num_arcs"] == 0
    # no accept pair reachable: an A whose accept row has no arcs into it
    A2 = fstgen.random_dag(10, 0, 3, 0.0, 1)
    got = fst.compose(A2, B)
    assert got["num_states"] == 0


def test_wave_auto_selects_trellis_batch(fst):
    """Automatic mode (1) takes the wave path for a lexicon o emissions batch and not for random graphs."""
    fst.fst_set_wave_mode(1)
    try:
        As, B = fstgen.config_c5(num_utts=3, num_words=200)
        hb = fst.fst_create(B)
        outs = fst.fst_compose_batch([fst.fst_create(A) for A in As], [hb] * len(As))
        assert outs[0].stats()["tile_path"] == 2
        A, B2 = fstgen.config_c2(0, V=300)
        assert fst.fst_compose(fst.fst_create(A), fst.fst_create(B2)).stats()["tile_path"] == 0
    finally:
        fst.fst_set_wave_mode(2)


def test_wave_provenance_uses_general_emit(fst):
    """FST_COMPOSE_PROVENANCE on the wave path (stages + counts on the wave kernels, the general emit
    with arc_a / arc_b): the arrays equal the level path's, provenance included."""
    A, B = fstgen.config_c3(num_words=300, T=30)
    a, b = fst.fst_create(A), fst.fst_create(B)
    fst.fst_set_wave_mode(2)
    cw = fst.fst_compose(a, b, provenance=True)
    assert cw.stats()["tile_path"] == 2
    fst.fst_set_wave_mode(0)
    try:
        cl = fst.fst_compose(a, b, provenance=True)
    finally:
        fst.fst_set_wave_mode(2)
    hw, hl = cw.to_host(), cl.to_host()
    for k in hw:
        assert np.array_equal(np.asarray(hw[k]), np.asarray(hl[k])), k
    pw, pl = cw.provenance(), cl.provenance()
    for x, y in zip(pw, pl):
        assert np.array_equal(np.asarray(x), np.asarray(y))


def test_wave_deterministic_batch(fst):
    """Repeated calls give identical arrays (clusters take compositions from a counter in any order, the
    counts run on a side stream: the result must not depend on the schedule)."""
    As, B = fstgen.config_c5(num_utts=9, num_words=1500)
    As = [fstgen.emissions_graph(20 + 7 * i, 10000 + i) for i in range(9)]
    hb = fst.fst_create(B)
    ha = [fst.fst_create(A) for A in As]
    runs = [[c.to_host() for c in fst.fst_compose_batch(ha, [hb] * len(ha))] for _ in range(3)]
    for r in runs[1:]:
        for x, y in zip(runs[0], r):
            for k in x:
                assert np.array_equal(np.asarray(x[k]), np.asarray(y[k])), k



@pytest.mark.parametrize("words", [5000, 5600, 6200])
def test_wave_lexicon_sizes(fst, words):
    """Lexicon sizes around the shared-memory thresholds of the count / emit kernels (their staged rows
    grow with V_B): the dynamic + static shared memory passes the 48 KB launch default in this range."""
    As, B = fstgen.config_c5(num_utts=2, num_words=words)
    As = [fstgen.emissions_graph(12, 10000), fstgen.emissions_graph(9, 10001)]
    check_pairs(fst, [(A, B) for A in As], f"lexicon {words}")


@pytest.mark.parametrize("words", [28000, 33000])
def test_wave_wide_rows(fst, words):
    """Rows near the wave emit's shared-memory limit (32 bytes per word of the widest row: ~6,900 words):
    a 28k-word lexicon (~6,300 words per row) takes the wave emit, a 33k-word one (~7,500) the general
    emit after the wave stages; both equal the level path and the oracle."""
    As, B = fstgen.config_c5(num_utts=2, num_words=words)
    As = [fstgen.emissions_graph(4, 10000), fstgen.emissions_graph(3, 10001)]
    check_pairs(fst, [(A, B) for A in As], f"lexicon {words}")

