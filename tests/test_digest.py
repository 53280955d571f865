"""Pins of the order-independent digest used for parity at full size: the
oracle's C implementation (orc_digest, Algorithm 1 with the arcs streamed into the digest) against the
independent numpy implementation in tests/digest.py over the oracle's stored arrays, invariance under
renumbering (FIFO order vs canonical order), and sensitivity to a single changed arc field."""
import numpy as np
import pytest

import digest
import fstgen
import oracle


def test_digest_c1_seeds():
    nonempty = 0
    for s in range(0, 1000, 5):
        A, B = fstgen.config_c1(s)
        g = oracle.compose(A, B)
        assert oracle.digest(A, B) == digest.digest_graph(g, B.num_states), s
        nonempty += g["num_arcs"] > 0
    assert nonempty > 30


@pytest.mark.parametrize("seed", [0, 3, 5, 8])
def test_digest_c2_eps(seed):
    A, B = fstgen.config_c2(seed, V=300 if seed == 5 else 1000)
    g = oracle.compose(A, B)
    d = oracle.digest(A, B)
    assert d == digest.digest_graph(g, B.num_states)
    # canonical order (states by key, rows sorted) has the same digest: order independence
    assert digest.digest_graph(oracle.canonical(A, B), B.num_states) == d


def test_digest_c3_lexicon():
    A, B = fstgen.config_c3(num_words=300, T=40)
    g = oracle.compose(A, B)
    assert oracle.digest(A, B) == digest.digest_graph(g, B.num_states)


def test_digest_sensitivity():
    A, B = fstgen.config_c2(5, V=300)
    g = oracle.compose(A, B)
    assert g["num_arcs"] > 1000
    base = digest.digest_graph(g, B.num_states)
    rng = np.random.default_rng(7)
    for field in ("dst", "ilabel", "olabel", "weight", "is_start", "is_accept", "pair_b"):
        h = {k: np.array(v, copy=True) for k, v in g.items() if isinstance(v, np.ndarray)}
        h["num_arcs"] = g["num_arcs"]
        i = int(rng.integers(len(h[field])))
        if field == "weight":
            h[field] = h[field].view(np.uint32)
            h[field][i] ^= 1  # one ulp
            h[field] = h[field].view(np.float32)
        elif field == "pair_b":
            h[field][i] = (h[field][i] + 1) % B.num_states
        elif field in ("is_start", "is_accept"):
            h[field][i] ^= 1
        elif field == "dst":
            h[field][i] = (h[field][i] + 1) % g["num_states"]
        else:
            h[field][i] += 1
        d = digest.digest_graph(h, B.num_states)
        assert d["d0"] != base["d0"] and d["d1"] != base["d1"], field
    # moving one arc to another state changes it too (the source key is hashed)
    h = {k: np.array(v, copy=True) for k, v in g.items() if isinstance(v, np.ndarray)}
    h["row_ptr"][1] += 1 if h["row_ptr"][1] < h["row_ptr"][2] else 0
    assert digest.digest_graph(h, B.num_states) != base
