"""Multi-process host logic on CPU (gloo, world size 2): LPT sharding of independent compositions and
the max/sum timing reduction used by bench.py.  No GPU needed."""
import os
import socket

import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from paper_2110_02848_b200 import parallel


def test_lpt_partition_complete_disjoint_balanced():
    costs = [100 + (7919 * i) % 401 for i in range(256)]  # c5-like frame counts in [100, 500]
    for world in (1, 2, 4, 8):
        parts = parallel.lpt_partition(costs, world)
        flat = sorted(i for p in parts for i in p)
        assert flat == list(range(256))
        assert parallel.imbalance(costs, world) < 1.05
    assert parallel.lpt_partition([5, 1, 1, 1, 1, 1], 2) == [[0], [1, 2, 3, 4, 5]]
    with pytest.raises(ValueError):
        parallel.lpt_partition([1], 0)


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, q):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    costs = [100 + (7919 * i) % 401 for i in range(64)]
    mine = parallel.shard_for_rank(costs, rank, world)
    # every rank must see the same partition
    allp = [None] * world
    dist.all_gather_object(allp, mine)
    ms, units = parallel.reduce_timing(10.0 * (rank + 1), float(len(mine)), dist)
    q.put((rank, allp, ms, units))
    dist.barrier()
    dist.destroy_process_group()


def test_gloo_world2_sharding_and_reduction():
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    res = [q.get(timeout=120) for _ in range(2)]
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    res.sort()
    allp0, allp1 = res[0][1], res[1][1]
    assert allp0 == allp1
    assert sorted(allp0[0] + allp0[1]) == list(range(64)) and not set(allp0[0]) & set(allp0[1])
    for _, _, ms, units in res:
        assert ms == 20.0 and units == 64.0


def _uid_worker(rank, world, port, q):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    from paper_2110_02848_b200 import fstc
    obj = [fstc.Comm.unique_id() if rank == 0 else None]
    dist.broadcast_object_list(obj, src=0)  # the sharded mode's NCCL bootstrap (bench.py --mode sharded)
    q.put((rank, obj[0]))
    dist.barrier()
    dist.destroy_process_group()


def test_gloo_world2_nccl_uid_bootstrap():
    from paper_2110_02848_b200 import build as b
    b.build()
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_uid_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    res = sorted(q.get(timeout=120) for _ in range(2))
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    assert len(res[0][1]) == 128 and res[0][1] == res[1][1]


def test_bench_reference_samples_are_nonempty():
    """Every random-graph bench workload's oracle sample composes to a nonempty graph (a degenerate
    seed -- the single accept pair with no label-matched in-arcs -- would time an empty composition)."""
    import os
    import sys
    sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
    import bench
    import oracle
    for w in ("c4", "c4-d4", "c4-paper", "fig3b-d16"):
        A, B, _ = bench.reference_sample(w)
        assert oracle.compose(A, B)["num_arcs"] > 0, w
