"""GPU: the owner-sharded composition.  All `world` shards run in one process on one
device (fst_compose_sharded_local: same kernels, row-slice exchange by device copies); their outputs
concatenated in rank order must equal fst_compose's output array by array, and the oracle after
canonicalisation.  The NCCL transport is exercised with world size 1 (one GPU per run here)."""
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


def _merged(fst, shards):
    parts = [c.to_host() for c in shards]
    infos = [c.shard_info() for c in shards]
    assert [i["rank"] for i in infos] == list(range(len(shards)))
    offs = [i["arc_offset"] for i in infos]
    assert [i["state_offset"] for i in infos] == list(np.cumsum([0] + [p["num_states"] for p in parts[:-1]]))
    return fst.merge_shards(parts, offs)


CASES = [("c1-7", lambda: fstgen.config_c1(7)), ("c1-3", lambda: fstgen.config_c1(3)),
         ("c2-0", lambda: fstgen.config_c2(0)), ("c3-small", lambda: fstgen.config_c3(num_words=200, T=40)),
         ("c4-2000", lambda: fstgen.config_c4(V=2000, D=8)), ("c4-1500-D6", lambda: fstgen.config_c4(V=1500, D=6))]


@pytest.mark.parametrize("name,make", CASES, ids=[c[0] for c in CASES])
@pytest.mark.parametrize("world", [1, 2, 3, 4])
def test_sharded_local_equals_unsharded(fst, name, make, world):
    A, B = make()
    a, b = fst.fst_create(A), fst.fst_create(B)
    ref = fst.fst_compose(a, b).to_host()
    got = _merged(fst, fst.fst_compose_sharded_local(a, b, world))
    for k in ("row_ptr", "ilabel", "olabel", "dst", "is_start", "is_accept", "pair_a", "pair_b"):
        assert np.array_equal(np.asarray(got[k]), np.asarray(ref[k])), (name, world, k)
    assert np.array_equal(got["weight"].view(np.uint32), ref["weight"].view(np.uint32))
    if world == 2:
        pins.assert_canonical_equal(pins.canonicalize_rows(got, B.num_states), oracle.canonical(A, B), name)


def test_sharded_nccl_world1(fst):
    A, B = fstgen.config_c4(V=1000, D=8)
    a, b = fst.fst_create(A), fst.fst_create(B)
    comm = fst.Comm(1, 0, fst.Comm.unique_id())
    c = fst.fst_compose_sharded(a, b, comm)
    ref = fst.fst_compose(a, b).to_host()
    got = c.to_host()
    for k in ("row_ptr", "dst", "ilabel", "olabel", "pair_a", "pair_b"):
        assert np.array_equal(got[k], ref[k]), k
    assert c.shard_info()["world"] == 1
    comm.close()
