"""Forward score over a composed graph in the log semiring -- CPU oracle.

TEST INFRASTRUCTURE ONLY: only tests/ (and bench.py's reference legs) may import it; the product
path (paper_2110_02848_b200) never does.  Shares no code with the CUDA path.

What it computes (the paper's future-work consumer of C; the log semiring of
PAPER.md:89-91 with (+) = logsumexp and (x) = +): for an ACYCLIC graph C,

    alpha(v) = logsumexp( [0 if v is a start state] + [alpha(u) + w(e) for every arc e = u -> v] )
    total    = logsumexp over accept states f of alpha(f)           (-inf if none is reachable)

evaluated in float64 in a topological order (Kahn's algorithm: a state is expanded once all its
in-arcs have been).  A cyclic C raises ValueError (the sum over paths is an infinite series).
"""
from __future__ import annotations

import collections
import math

import numpy as np

NEG_INF = float("-inf")


def logadd(a: float, b: float) -> float:
    """log(exp(a) + exp(b)) in float64."""
    if a == NEG_INF:
        return b
    if b == NEG_INF:
        return a
    m = a if a > b else b
    return m + math.log1p(math.exp(-abs(a - b)))


def forward(C):
    """(alpha float64 [V], total float64) of a composed graph given as a dict of arrays."""
    V = int(C["num_states"])
    rp = np.asarray(C["row_ptr"], np.int64)
    dst = np.asarray(C["dst"], np.int64)
    w = np.asarray(C["weight"], np.float32).astype(np.float64)
    indeg = np.bincount(dst, minlength=V).astype(np.int64) if len(dst) else np.zeros(V, np.int64)
    alpha = [NEG_INF] * V
    for s in np.flatnonzero(np.asarray(C["is_start"])):
        alpha[int(s)] = 0.0
    q = collections.deque(int(v) for v in np.flatnonzero(indeg == 0))
    done = 0
    rpl, dstl, wl, deg = rp.tolist(), dst.tolist(), w.tolist(), indeg.tolist()
    while q:
        u = q.popleft()
        done += 1
        au = alpha[u]
        for e in range(rpl[u], rpl[u + 1]):
            v = dstl[e]
            if au != NEG_INF:
                alpha[v] = logadd(alpha[v], au + wl[e])
            deg[v] -= 1
            if deg[v] == 0:
                q.append(v)
    if done < V:
        raise ValueError("forward score: the graph has a cycle")
    total = NEG_INF
    for f in np.flatnonzero(np.asarray(C["is_accept"])):
        total = logadd(total, alpha[int(f)])
    return np.array(alpha, np.float64), total
