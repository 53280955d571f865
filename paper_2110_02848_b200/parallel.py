"""Host-side multi-GPU plumbing: one process per GPU, independent compositions sharded across ranks.

The composition path partitions naturally (BASELINE.json north_star: "batches of independent
compositions (one utterance per composition) are split across GPUs"), so there is NO data-path
collective: each rank runs fst_compose_batch on its own shard; torch.distributed is used only to
agree on the timing (max over ranks) and the totals (sum over ranks) after the timed region.

Sharding is longest-processing-time-first (LPT) on a per-unit cost (e.g. frames T_i of an
utterance), deterministic: units sorted by (cost desc, index asc), each assigned to the least
loaded rank (ties -> lowest rank).
"""
from __future__ import annotations

import heapq
from typing import List, Sequence, Tuple


def lpt_partition(costs: Sequence[float], world: int) -> List[List[int]]:
    """Unit indices per rank (each list ascending)."""
    if world < 1:
        raise ValueError("world must be >= 1")
    heap = [(0.0, r) for r in range(world)]
    out: List[List[int]] = [[] for _ in range(world)]
    for i in sorted(range(len(costs)), key=lambda i: (-costs[i], i)):
        load, r = heapq.heappop(heap)
        out[r].append(i)
        heapq.heappush(heap, (load + float(costs[i]), r))
    return [sorted(x) for x in out]


def shard_for_rank(costs: Sequence[float], rank: int, world: int) -> List[int]:
    return lpt_partition(costs, world)[rank]


def imbalance(costs: Sequence[float], world: int) -> float:
    """max rank load / mean rank load (1.0 = perfect)."""
    parts = lpt_partition(costs, world)
    loads = [sum(costs[i] for i in p) for p in parts]
    mean = sum(loads) / world
    return max(loads) / mean if mean > 0 else 1.0


def reduce_timing(local_ms: float, local_units: float, dist=None, device=None) -> Tuple[float, float]:
    """(max over ranks of local_ms, sum over ranks of local_units); identity without a process group."""
    if dist is None or not dist.is_initialized() or dist.get_world_size() == 1:
        return float(local_ms), float(local_units)
    import torch
    t = torch.tensor([float(local_ms)], dtype=torch.float64, device=device)
    u = torch.tensor([float(local_units)], dtype=torch.float64, device=device)
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    dist.all_reduce(u, op=dist.ReduceOp.SUM)
    return float(t.item()), float(u.item())
