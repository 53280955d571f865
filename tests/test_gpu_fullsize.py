"""GPU parity at BASELINE.json's full size, in the configuration bench.py times (configs[3]: random
acceptors V=20000, D=8, 16 tokens; E_C = 1.44e9 arcs): the oracle cannot compose it in test time, so
the C oracle computes only the co-accessible set R (Algorithm 1 line 3), and the GPU result is checked
against it: states = pairs in R only, numbered by ascending key, start/accept flags by definition, and
2000 sampled rows equal EXACTLY (labels, destinations, weight bits) the N1 moves of their pair whose
destination is co-accessible (pins.n1_moves: the plain definition)."""
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
    return p


def test_c4_fullsize_against_oracle_R(fst):
    A, B = fstgen.config_c4(V=20000, D=8)
    VB = B.num_states
    R = oracle.coaccessible(A, B)  # Algorithm 1 line 3 on the CPU
    c = fst.fst_compose(fst.fst_create(A), fst.fst_create(B))
    st = c.state_arrays()
    V_C, E_C = st["num_states"], st["num_arcs"]
    assert V_C > 3e8 and E_C > 1e9
    keys = st["pair_a"].astype(np.int64) * VB + st["pair_b"]
    assert np.all(np.diff(keys) > 0)                      # numbering by ascending pair key
    assert np.all(R[keys] == 1) and V_C <= int(R.sum())   # every state of C is co-accessible
    assert np.array_equal(st["is_start"], A.is_start[st["pair_a"]] & B.is_start[st["pair_b"]])
    assert np.array_equal(st["is_accept"], A.is_accept[st["pair_a"]] & B.is_accept[st["pair_b"]])
    assert st["row_ptr"][0] == 0 and st["row_ptr"][-1] == E_C and np.all(np.diff(st["row_ptr"]) >= 0)
    rng = np.random.default_rng(2110)
    sample = np.unique(np.concatenate([rng.choice(V_C, 2000, replace=False), [0, V_C - 1]]))
    for sid in sample:
        a, b = int(st["pair_a"][sid]), int(st["pair_b"][sid])
        lo, hi = int(st["row_ptr"][sid]), int(st["row_ptr"][sid + 1])
        got = c.arcs_range(lo, hi - lo)
        got_rows = sorted((int(keys[d]), int(i), int(o), int(np.float32(w).view(np.uint32)))
                          for d, i, o, w in zip(got["dst"], got["ilabel"], got["olabel"], got["weight"]))
        exp_rows = sorted((d[0] * VB + d[1], il, ol, pins.wbits(w)) for d, il, ol, w in pins.n1_moves(A, B, a, b)
                          if R[d[0] * VB + d[1]])
        assert got_rows == exp_rows, (sid, a, b)


# ------------------------------------------------------------------ digest parity at the stated sizes
# V_C, E_C and two 64-bit order-independent digests (tests/digest.py; the oracle
# streams the same definition through Algorithm 1, oracle/compose.c orc_digest) -- equality means the
# canonical graphs are equal (w.h.p.), at sizes the array-by-array comparison cannot reach.
import digest  # noqa: E402


def test_digest_device_matches_host(fst):
    """The device-side digest (torch) equals the host numpy one on a graph both can handle."""
    A, B = fstgen.config_c4(V=3000, D=8)
    c = fst.fst_compose(fst.fst_create(A), fst.fst_create(B))
    assert digest.digest_device(c.device_tensors(), B.num_states) == digest.digest_graph(c.to_host(), B.num_states)
    assert digest.digest_graph(c.to_host(), B.num_states) == oracle.digest(A, B)


def oracle_digest_cached(name, A, B):
    """The oracle's digest of a full-size configuration: cached in tests/golden/fullsize_digests.json by
    scripts/make_fullsize_digests.py (which calls only oracle/; tens of minutes per configuration on one
    core), else computed here."""
    import json
    import os
    p = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden", "fullsize_digests.json")
    if os.path.exists(p):
        d = json.load(open(p)).get(name)
        if d:
            return {k: d[k] for k in ("num_states", "num_arcs", "d0", "d1")}
    return oracle.digest(A, B)


def test_c4_fullsize_digest(fst):
    """configs[3] at the bench size (20k x 20k, D = 8, 16 tokens; E_C = 1.44e9): the whole composed graph
    equals the oracle's (digest), in the launch configuration bench.py times."""
    A, B = fstgen.config_c4(V=20000, D=8, tokens=16)
    c = fst.fst_compose(fst.fst_create(A), fst.fst_create(B))
    got = digest.digest_device(c.device_tensors(), B.num_states)
    exp = oracle_digest_cached("c4_20000_d8_t16", A, B)
    assert got == exp
    assert exp["num_arcs"] > 1.4e9


def test_c4_int64_arc_slots(fst):
    """20k x 20k, D = 8, 8 tokens: E_C ~ 3.2e9 > 2^31 composed arcs (int64 row_ptr / arc slots), against
    the oracle's digest."""
    A, B = fstgen.config_c4(V=20000, D=8, tokens=8)
    c = fst.fst_compose(fst.fst_create(A), fst.fst_create(B))
    assert c.num_arcs > 2 ** 31
    got = digest.digest_device(c.device_tensors(), B.num_states)
    assert got == oracle_digest_cached("c4_20000_d8_t8", A, B)


def _oracle_digest_pair(pair):
    A, B = pair
    return oracle.digest(A, B)


def test_c5_batch_digests(fst):
    """configs[4] as bench.py times it: the 32-utterance batch (T_i = 100..500) o closure(10k-word lexicon)
    in one fst_compose_batch; every utterance's composition equals the oracle's (digest; the oracle runs
    one utterance per host core)."""
    import multiprocessing as mp
    import os
    import sys
    sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
    import bench
    As, B, _ = bench.c5_shard(0, 1)
    hb = fst.fst_create(B)
    cs = fst.fst_compose_batch([fst.fst_create(A) for A in As], [hb] * len(As))
    got = [digest.digest_device(c.device_tensors(), B.num_states) for c in cs]
    with mp.get_context("spawn").Pool(min(len(As), len(os.sched_getaffinity(0)))) as pool:
        exp = pool.map(_oracle_digest_pair, [(A, B) for A in As])
    assert got == exp
    assert sum(e["num_arcs"] for e in exp) > 5e8
