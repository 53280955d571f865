"""GPU forward score (fst_forward_score) against the CPU oracle
(oracle/forward.py run on the ORACLE's own composition, never on the GPU's output).

Float64 on both sides; the GPU folds a state's in-arcs in a data-dependent order, so totals and
alphas are compared within 1e-9 relative (float64 rounding of sums over <= ~1e6 terms)."""
import math

import numpy as np
import pytest

import fstgen
import oracle
from oracle import forward as ofw

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


def close(a, b, rel=1e-9):
    if a == -math.inf or b == -math.inf:
        return a == b
    return abs(a - b) <= rel * max(1.0, abs(b))


def check(p, A, B, what):
    import torch
    c = p.fst_compose(p.fst_create(A), p.fst_create(B))
    alpha = torch.empty(max(1, c.num_states), dtype=torch.float64, device="cuda")
    tot = p.fst_forward_score(c, alpha)
    Co = oracle.canonical(A, B)  # states in ascending (a, b) key = the GPU's numbering
    ao, to = ofw.forward(Co)
    assert close(tot, to), (what, tot, to)
    ag = alpha[: c.num_states].cpu().numpy()
    assert len(ag) == len(ao)
    fin = np.isfinite(ao)
    assert np.array_equal(fin, np.isfinite(ag)), what
    assert np.all(np.abs(ag[fin] - ao[fin]) <= 1e-9 * np.maximum(1.0, np.abs(ao[fin]))), what
    return tot


def test_forward_lexicon_emissions(fst):
    A, B = fstgen.config_c3()
    assert math.isfinite(check(fst, A, B, "c3"))
    A, B = fstgen.config_c3(num_words=3000, T=40, em_seed=91)
    check(fst, A, B, "c3 3000 words")


def test_forward_eps_dags(fst):
    n = 0
    for seed in range(60):
        eps = 0.2 if seed % 2 else 0.3
        A = fstgen.random_dag(12, 3, 3, eps, 7919 * seed + 11)
        B = fstgen.random_dag(12, 3, 3, eps, 7919 * seed + 13)
        n += math.isfinite(check(fst, A, B, f"dag {seed}"))
    assert n >= 5


def test_forward_created_handle_and_errors(fst):
    A = fstgen.random_dag(2000, 4, 5, 0.1, 77)  # a created (non-composed) DAG handle
    a = fst.fst_create(A)
    Ad = {"num_states": A.num_states, "row_ptr": A.row_ptr, "dst": A.dst, "weight": A.weight,
          "is_start": A.is_start, "is_accept": A.is_accept}
    assert close(fst.fst_forward_score(a), ofw.forward(Ad)[1])
    A, B = fstgen.config_c2(0)  # random graphs with cycles (a non-empty composition)
    c = fst.fst_compose(fst.fst_create(A), fst.fst_create(B))
    assert c.num_states > 0
    with pytest.raises(fst.FstError) as ei:
        fst.fst_forward_score(c)
    assert ei.value.status == 2
    e = fst.fst_compose(fst.fst_create(fstgen.empty_fst(0)), fst.fst_create(B))
    assert fst.fst_forward_score(e) == -math.inf
