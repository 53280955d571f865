"""GPU parity of the tile path (bottom-up BFS levels, pass-1 counts and the emit on the
tile kernels) against the CPU oracle, bit-exact (tolerance 0), on inputs where the tile path is forced
(fst_set_tile_mode(2)) so that graphs the oracle finishes in seconds exercise it: random acceptors
(configs[3] shape, ragged V), eps transducers (configs[1] shape: M2 / M3 moves, self slots, the sentinel
column), tiny transducers (configs[0]), multiple start / accept states, and the per-level profile
(bottom-up levels are exact BFS levels, Alg. 1 / PAPER.md:207-213)."""
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
    p.fst_set_tile_mode(2)
    yield p
    p.fst_set_tile_mode(1)


def compose_tile(p, A, B):
    a, b = p.fst_create(A), p.fst_create(B)
    c = p.fst_compose(a, b)
    return c, c.stats()


def check_rounds(c, st, A, B):
    """Bottom-up rounds claim in place (several BFS distances per round): the per-round sizes sum to
    |R| (stage 1) and V_C (stage 2); push levels before the first round are exact BFS levels, so the
    profile starts like the oracle's FIFO levels and never runs longer than it."""
    exp = oracle.compose(A, B)
    lv = [int(x) for x in np.bincount(exp["level"])] if exp["num_states"] else []
    s2 = c.level_sizes(2)
    assert sum(s2) == exp["num_states"] == c.num_states
    assert len(s2) <= len(lv)
    if s2:
        assert s2[0] == lv[0]
    assert sum(c.level_sizes(1)) == int(oracle.coaccessible(A, B).sum()) == st["num_coaccessible"]


def check_tile(p, A, B, what, need_pull=False):
    c, st = compose_tile(p, A, B)
    assert st["tile_path"] == 1, what
    if need_pull:
        assert st["pull_levels"] > 0, what
    got = pins.canonicalize_rows(c.to_host(), B.num_states)
    pins.assert_canonical_equal(got, oracle.canonical(A, B), what)
    return c, st, got


@pytest.mark.parametrize("V,D", [(1000, 4), (2000, 8), (1500, 6), (4096, 5), (777, 8)])
def test_tile_random_acceptors(fst, V, D):
    A, B = fstgen.config_c4(V=V, D=D)
    c, st, got = check_tile(fst, A, B, f"tile c4 {V}/{D}")
    check_rounds(c, st, A, B)


@pytest.mark.parametrize("seed", range(10))
def test_tile_eps_transducers(fst, seed):
    """configs[1]: eps on both tapes -- M1 eps:eps, M2 (sentinel column), M3 (self slots)."""
    A, B = fstgen.config_c2(seed)
    check_tile(fst, A, B, f"tile c2 seed {seed}")


def test_tile_c1_seeds(fst):
    for s in range(0, 1000, 7):  # includes multi start / accept seeds (s % 4 == 3)
        A, B = fstgen.config_c1(s)
        check_tile(fst, A, B, f"tile c1 seed {s}")


def test_tile_eps_dags(fst):
    for s in range(40):
        A = fstgen.random_dag(8, 3, 4, 0.3, 100 + 2 * s)
        B = fstgen.random_dag(8, 3, 4, 0.3, 101 + 2 * s)
        check_tile(fst, A, B, f"tile eps dag {s}")


def test_tile_matches_push_path(fst):
    """Same numbering (ascending key) and the same rows as the push path, on a graph big enough for the
    automatic mode; the tile path is deterministic."""
    A, B = fstgen.config_c4(V=3000, D=8)
    a, b = fst.fst_create(A), fst.fst_create(B)
    r1 = fst.fst_compose(a, b).to_host()
    r2 = fst.fst_compose(a, b).to_host()
    for k in r1:
        assert np.array_equal(np.asarray(r1[k]), np.asarray(r2[k])), k
    fst.fst_set_tile_mode(0)
    try:
        c0 = fst.fst_compose(a, b)
        assert c0.stats()["tile_path"] == 0
        r0 = c0.to_host()
    finally:
        fst.fst_set_tile_mode(2)
    for k in ("row_ptr", "pair_a", "pair_b", "is_start", "is_accept"):
        assert np.array_equal(np.asarray(r0[k]), np.asarray(r1[k])), k
    g0 = pins.canonicalize_rows(r0, B.num_states)
    g1 = pins.canonicalize_rows(r1, B.num_states)
    pins.assert_canonical_equal(g1, g0, "tile vs push")


def test_tile_ineligible_falls_back(fst):
    """A hub state (degree > 31 in B's view) or labels > 252 keep the push path (and stay exact)."""
    A, B = fstgen.config_c3(num_words=200, T=20)  # closure root has 200 out-arcs
    c, st = compose_tile(fst, A, B)
    assert st["tile_path"] == 0
    pins.assert_canonical_equal(pins.canonicalize_rows(c.to_host(), B.num_states), oracle.canonical(A, B), "c3 fallback")


@pytest.mark.parametrize("V,D", [(1000, 4), (1500, 8)])
def test_tile_all_levels_bottom_up(fst, V, D):
    """Every level of both stages bottom-up (test mode 3): same graph, round sizes sum to |R| / V_C."""
    A, B = fstgen.config_c4(V=V, D=D)
    fst.fst_set_tile_mode(3)
    try:
        c, st, got = check_tile(fst, A, B, f"all-pull c4 {V}/{D}", need_pull=True)
        assert st["pull_levels"] == st["levels_stage1"] + st["levels_stage2"]
    finally:
        fst.fst_set_tile_mode(2)
    check_rounds(c, st, A, B)


@pytest.mark.parametrize("make", [lambda: fstgen.config_c4(V=1500, D=8), lambda: fstgen.config_c2(0),
                                  lambda: fstgen.config_c2(3), lambda: fstgen.config_c1(7)])
def test_tile_push_levels(fst, make):
    """Mode 4: the push levels run on k_tile_push (claims as reductions, counts from the bitmap):
    exact graph and, for the push levels, the exact BFS level sizes."""
    A, B = make()
    fst.fst_set_tile_mode(4)
    try:
        c, st, got = check_tile(fst, A, B, "tile push")
    finally:
        fst.fst_set_tile_mode(2)
    check_rounds(c, st, A, B)


@pytest.mark.parametrize("seed", [0, 3, 8])
def test_tile_all_levels_bottom_up_eps(fst, seed):
    A, B = fstgen.config_c2(seed)
    fst.fst_set_tile_mode(3)
    try:
        check_tile(fst, A, B, f"all-pull c2 seed {seed}")
    finally:
        fst.fst_set_tile_mode(2)


def test_tile_empty(fst):
    A, B = fstgen.config_c2(1)  # empty composition (accept pair unreachable backwards)
    c, st = compose_tile(fst, A, B)
    assert c.num_states == oracle.canonical(A, B)["num_states"]
