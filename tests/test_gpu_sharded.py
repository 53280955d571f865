"""GPU: the owner-sharded single composition (include/fstc.h "Sharded single
composition").  Blocks of 1024 pairs are dealt to the ranks round-robin (block id mod world), so every
row -- every level of a trellis -- is spread over all ranks; claims in other ranks' blocks travel as
packed per-peer slices.  All `world` shards run in one process on one device
(fst_compose_sharded_local: the same kernels, the packed slices handed over in device memory).  The
shards concatenated in rank order form a valid CSR of the whole composition (owner-major state
numbering) that equals fst_compose's result and the oracle after canonicalisation; for world = 1 the
arrays are identical.  The NCCL transport runs with world size 1 (one GPU per run here)."""
import numpy as np
import pytest

import digest
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


def _merged(shards):
    """Concatenation of the shards' host copies in rank order (test-side output assembly)."""
    parts = [c.to_host() for c in shards]
    infos = [c.shard_info() for c in shards]
    assert [i["rank"] for i in infos] == list(range(len(shards)))
    assert [i["state_offset"] for i in infos] == list(np.cumsum([0] + [p["num_states"] for p in parts[:-1]]))
    assert [i["arc_offset"] for i in infos] == list(np.cumsum([0] + [p["num_arcs"] for p in parts[:-1]]))
    return pins.merge_shards(parts, [i["arc_offset"] for i in infos])


def _owner_major_ok(got, VB, world):
    """Shard r holds exactly the states of its blocks, ascending by key inside the shard."""
    key = got["pair_a"].astype(np.int64) * VB + got["pair_b"]
    bpr = (VB + 1023) // 1024
    owner = (got["pair_a"].astype(np.int64) * bpr + got["pair_b"] // 1024) % world
    assert np.all(np.diff(owner) >= 0)
    for r in range(world):
        k = key[owner == r]
        assert np.all(np.diff(k) > 0)


CASES = [("c1-7", lambda: fstgen.config_c1(7)), ("c1-3", lambda: fstgen.config_c1(3)),
         ("c2-0", lambda: fstgen.config_c2(0)), ("c3-small", lambda: fstgen.config_c3(num_words=200, T=40)),
         ("c3-wide", lambda: fstgen.config_c3(num_words=3000, T=30)),
         ("c4-2000", lambda: fstgen.config_c4(V=2000, D=8)), ("c4-1500-D6", lambda: fstgen.config_c4(V=1500, D=6))]


@pytest.mark.parametrize("name,make", CASES, ids=[c[0] for c in CASES])
@pytest.mark.parametrize("world", [1, 2, 3, 5, 8])
def test_sharded_local_equals_unsharded(fst, name, make, world):
    A, B = make()
    a, b = fst.fst_create(A), fst.fst_create(B)
    ref = fst.fst_compose(a, b).to_host()
    got = _merged(fst.fst_compose_sharded_local(a, b, world))
    if world == 1:
        for k in ("row_ptr", "ilabel", "olabel", "dst", "is_start", "is_accept", "pair_a", "pair_b"):
            assert np.array_equal(np.asarray(got[k]), np.asarray(ref[k])), (name, world, k)
        assert np.array_equal(got["weight"].view(np.uint32), ref["weight"].view(np.uint32))
    _owner_major_ok(got, B.num_states, world)
    pins.assert_canonical_equal(pins.canonicalize_any(got, B.num_states), pins.canonicalize_rows(ref, B.num_states),
                                f"{name} world {world}")
    if world == 2:
        pins.assert_canonical_equal(pins.canonicalize_any(got, B.num_states), oracle.canonical(A, B), name)


TILE_CASES = [("c4-2000", lambda: fstgen.config_c4(V=2000, D=8)), ("c4-1500-D6", lambda: fstgen.config_c4(V=1500, D=6)),
              ("c2-0", lambda: fstgen.config_c2(0)), ("c1-3", lambda: fstgen.config_c1(3))]


@pytest.mark.parametrize("name,make", TILE_CASES, ids=[c[0] for c in TILE_CASES])
@pytest.mark.parametrize("world", [1, 2, 3, 8])
@pytest.mark.parametrize("mode", [2, 3])
def test_sharded_tile_path(fst, name, make, world, mode):
    """Compositions on the tile path are sharded by contiguous row ranges: bottom-up rounds over each
    rank's tiles (claims replicated after every round), counts and emit of the own rows; ids stay in
    key order, so the concatenated shards equal the unsharded arrays (mode 3: every level bottom-up)."""
    A, B = make()
    a, b = fst.fst_create(A), fst.fst_create(B)
    fst.fst_set_tile_mode(mode)
    try:
        shards = fst.fst_compose_sharded_local(a, b, world)
        st = shards[0].stats()
        got = _merged(shards)
        fst.fst_set_tile_mode(0)
        ref = fst.fst_compose(a, b).to_host()
    finally:
        fst.fst_set_tile_mode(1)
    assert st["tile_path"] == 1
    if mode == 3 and ref["num_states"]:
        assert st["pull_levels"] > 0
    for k in ("row_ptr", "is_start", "is_accept", "pair_a", "pair_b"):
        assert np.array_equal(np.asarray(got[k]), np.asarray(ref[k])), (name, world, k)
    pins.assert_canonical_equal(pins.canonicalize_rows(got, B.num_states), pins.canonicalize_rows(ref, B.num_states),
                                f"{name} world {world} mode {mode}")


def test_sharded_trellis_spreads_levels(fst):
    """A trellis (lexicon o emissions): every BFS level is one A row; with block ownership every rank
    owns part of each level's row, so all shards hold states of (almost) every frame."""
    A, B = fstgen.config_c3(num_words=3000, T=30)
    a, b = fst.fst_create(A), fst.fst_create(B)
    shards = fst.fst_compose_sharded_local(a, b, 4)
    frames = [set(np.unique(c.to_host()["pair_a"]).tolist()) for c in shards]
    for f in frames:
        assert len(f) >= 25  # of 31 frames


def test_sharded_local_fullsize_digest(fst):
    """configs[3] at 20k x 20k over 4 in-process shards: the union of the shards has the oracle's digest
    (cached by scripts/make_fullsize_digests.py; the device-side digest reads every shard's arrays)."""
    import torch
    from test_gpu_fullsize import oracle_digest_cached
    A, B = fstgen.config_c4(V=20000, D=8, tokens=16)
    a, b = fst.fst_create(A), fst.fst_create(B)
    shards = fst.fst_compose_sharded_local(a, b, 4)
    ts = [c.device_tensors() for c in shards]
    infos = [c.shard_info() for c in shards]
    whole = {k: torch.cat([t[k] for t in ts]) for k in ("ilabel", "olabel", "dst", "weight", "is_start",
                                                        "is_accept", "pair_a", "pair_b")}
    whole["row_ptr"] = torch.cat([t["row_ptr"][:-1] + i["arc_offset"] for t, i in zip(ts, infos)] +
                                 [torch.tensor([infos[-1]["total_arcs"]], device="cuda", dtype=torch.int64)])
    del ts
    for c in shards:
        c.free()
    assert digest.digest_device(whole, B.num_states) == oracle_digest_cached("c4_20000_d8_t16", A, B)


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
