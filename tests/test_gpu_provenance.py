"""GPU parity of the provenance output and the gradient scatter through the
C ABI (fst_compose_ex / fst_compose_batch_ex with FST_COMPOSE_PROVENANCE, fst_grad_scatter).

Provenance is compared element by element with the oracle's (arc_a, arc_b) after canonicalisation
(rows sorted by (dst, ilabel, olabel, weight bits, arc_a, arc_b) on both sides): bit-exact.  The
gradient scatter uses float atomics, so it is compared with a float64 np.add.at reference within
the rounding of an n-term float32 sum: |g - ref| <= n * 2^-23 * sum|terms| per element.
"""
import numpy as np
import pytest

import fstgen
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


def check_prov(p, A, B, what):
    got = pins.canonicalize_rows(p.compose(A, B, provenance=True), B.num_states)
    assert "arc_a" in got and len(got["arc_a"]) == got["num_arcs"], what
    pins.assert_canonical_equal(got, oracle.canonical(A, B), what)
    return got


def test_provenance_c1_seeds(fst):
    for s in range(0, 1000, 5):
        A, B = fstgen.config_c1(s)
        check_prov(fst, A, B, f"c1 seed {s}")


@pytest.mark.parametrize("seed", [0, 3, 8])
def test_provenance_c2_eps(fst, seed):
    A, B = fstgen.config_c2(seed)
    check_prov(fst, A, B, f"c2 seed {seed}")


def test_provenance_lexicon_and_hubs(fst):
    """c3 (A has no eps; closure eps arcs on B: M3), a 3000-word root (hub paths), hub graphs with A
    rows of <= 32, > 32 and > 64 arcs (the general label-major / state-major emit paths)."""
    A, B = fstgen.config_c3()
    check_prov(fst, A, B, "c3")
    A, B = fstgen.config_c3(num_words=3000, T=20)
    check_prov(fst, A, B, "c3 3000 words")
    for n_hub, a_hub in ((1500, 0), (2049, 20), (1200, 40), (1100, 100)):
        B = hub_graph(3000, 3, 8, 11 + n_hub, 0, 5, n_hub, n_hub)
        A = hub_graph(300, 3, 8, 13 + n_hub, 1, 2, a_hub, 0)
        check_prov(fst, A, B, f"hub {n_hub}/{a_hub}")


def test_provenance_large_labels_and_eps(fst):
    """Labels >= 63 (no label masks: general emit paths) and eps on both tapes (M2 and M3)."""
    A = fstgen.random_graph(300, 10, 70, 71, acceptor=False, eps_prob=0.1, weights="dyadic64")
    B = fstgen.random_graph(400, 10, 70, 171, acceptor=False, eps_prob=0.1, weights="dyadic64")
    got = check_prov(fst, A, B, "70 tokens, eps transducers")
    assert got["num_arcs"] > 400000 and (got["arc_a"] < 0).any() and (got["arc_b"] < 0).any()
    A = fstgen.random_graph(400, 12, 80, 71, eps_prob=0.05, weights="dyadic64")
    B = fstgen.random_graph(500, 12, 80, 171, eps_prob=0.05, weights="dyadic64")
    check_prov(fst, A, B, "80 tokens, eps acceptors")
    A, B = fstgen.config_c4(V=1500, D=6)
    check_prov(fst, A, B, "c4 1500/6")


def test_provenance_batch_and_composed_input(fst):
    pairs = [fstgen.config_c2(0, V=300), fstgen.config_c1(3), fstgen.config_c3(num_words=50, T=20),
             fstgen.config_c4(V=700, D=4)]
    ha = [fst.fst_create(A) for A, _ in pairs]
    hb = [fst.fst_create(B) for _, B in pairs]
    outs = fst.fst_compose_batch(ha, hb, provenance=True)
    for i, ((A, B), c) in enumerate(zip(pairs, outs)):
        got = pins.canonicalize_rows(c.to_host(), B.num_states)
        pins.assert_canonical_equal(got, oracle.canonical(A, B), f"batch item {i}")
    # a composed handle as input: provenance indexes C's own arc order
    A, B = fstgen.config_c2(2, V=200)
    c = fst.fst_compose(fst.fst_create(A), fst.fst_create(B))
    Cg = c.to_host()
    labels = sorted(set(int(x) for x in Cg["olabel"] if x >= 0))
    Id = fstgen.identity_fst(labels)
    c2 = fst.fst_compose(c, fst.fst_create(Id), provenance=True).to_host()
    Cfst = fstgen.Fst(Cg["num_states"], Cg["row_ptr"], Cg["ilabel"], Cg["olabel"], Cg["dst"], Cg["weight"],
                      Cg["is_start"], Cg["is_accept"])
    pins.assert_canonical_equal(pins.canonicalize_rows(c2, Id.num_states), oracle.canonical(Cfst, Id), "(AoB)oId")


def _scatter_ref(idx, g, n):
    ref = np.zeros(n, np.float64)
    absr = np.zeros(n, np.float64)
    cnt = np.zeros(n, np.int64)
    m = idx >= 0
    np.add.at(ref, idx[m], g[m].astype(np.float64))
    np.add.at(absr, idx[m], np.abs(g[m]).astype(np.float64))
    np.add.at(cnt, idx[m], 1)
    return ref, absr, cnt


@pytest.mark.parametrize("case", ["c2", "c3", "hub"])
def test_grad_scatter(fst, case):
    import torch
    if case == "c2":
        A, B = fstgen.config_c2(3)
    elif case == "c3":
        A, B = fstgen.config_c3()
    else:
        B = hub_graph(3000, 3, 8, 1511, 0, 5, 1500, 1500)
        A = hub_graph(300, 3, 8, 1513, 1, 2, 40, 0)
    c = fst.fst_compose(fst.fst_create(A), fst.fst_create(B), provenance=True)
    E = c.num_arcs
    aa, ab = c.provenance()
    rng = np.random.default_rng(5)
    g = rng.standard_normal(E).astype(np.float32)
    dev = torch.device("cuda")
    gc = torch.from_numpy(g).to(dev)
    ga = torch.zeros(A.num_arcs, dtype=torch.float32, device=dev)
    gb = torch.full((B.num_arcs,), 0.5, dtype=torch.float32, device=dev)  # accumulates (+=)
    fst.fst_grad_scatter(c, gc, ga, gb)
    torch.cuda.synchronize()
    for got, idx, n, base in ((ga.cpu().numpy(), aa, A.num_arcs, 0.0), (gb.cpu().numpy(), ab, B.num_arcs, 0.5)):
        ref, absr, cnt = _scatter_ref(idx, g, n)
        tol = (cnt + 1) * 2.0 ** -23 * (absr + abs(base)) + 1e-30
        assert np.all(np.abs(got.astype(np.float64) - (ref + base)) <= tol), case
        assert np.all(got[cnt == 0] == np.float32(base)), case  # arcs used by no composed arc: untouched


def test_provenance_errors(fst):
    import torch
    A, B = fstgen.config_c1(0)
    a, b = fst.fst_create(A), fst.fst_create(B)
    c = fst.fst_compose(a, b)  # no provenance
    g = torch.zeros(max(1, c.num_arcs), device="cuda")
    with pytest.raises(fst.FstError) as ei:
        fst.fst_grad_scatter(c, g, torch.zeros(A.num_arcs, device="cuda"))
    assert ei.value.status == 1
    with pytest.raises(fst.FstError) as ei:
        fst.fst_compose_ex(a, b, 0x10)
    assert ei.value.status == 1
    cp = fst.fst_compose(a, b, provenance=True)
    with pytest.raises(fst.FstError) as ei:  # grad_a shorter than A's arcs
        fst.fst_grad_scatter(cp, torch.zeros(max(1, cp.num_arcs), device="cuda"),
                             torch.zeros(max(0, A.num_arcs - 1), device="cuda"))
    assert ei.value.status == 1
    assert c.to_host().get("arc_a") is None and "arc_a" in cp.to_host()
