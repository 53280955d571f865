"""Independent pins for the oracle (and, transitively, for the CUDA path).

None of these routines shares control flow with oracle/compose.c (Algorithm 1) or with the CUDA
kernels; each one computes the expected result from a plain definition:

  * ``plain_trim_product``  -- trim(P_N1): build the FULL product automaton over V_A x V_B with the
    move set N1 (reading N1 / SURVEY §8(c) c.1), then trim it with two textbook
    reachability sweeps ("accessible ... and co-accessible").
  * ``eq1_bruteforce``       -- Eq. (1): enumerate accepting paths of A and B,
    pair them on y, and collect the multiset of s_a + s_b per (x, z); with epsilon, each matched pair
    contributes prod_i Delannoy(k_i, m_i) composed paths.
  * ``trellis_compose``      -- A = linear emissions (every token at every frame): the trim graph
    follows from forward / backward epsilon-closures over (t, b) on B alone.
  * ``trim_fst`` / ``identity_expected`` -- A o Id == trim(A).
  * ``is_trim``              -- trim invariant on any CSR graph.

Canonical form (reading 24): states ascending by key(a, b) = a * V_B + b; each row's arcs
sorted by (dst, ilabel, olabel, weight bits as uint32).
"""
from __future__ import annotations

import collections
import math
from math import comb
from typing import Dict, List, Tuple

import numpy as np

EPS = -1


def f32add(a, b) -> np.float32:
    """One IEEE binary32 add, round-to-nearest-even (numpy float32 arithmetic)."""
    return np.float32(a) + np.float32(b)


def wbits(w) -> int:
    return int(np.float32(w).view(np.uint32))


# ----------------------------------------------------------------------------- canonical builder
def state_key(p, VB: int) -> int:
    """Canonical state key: a * V_B + b for pairs, (a * V_B + b) * 3 + f for eps-filter triples."""
    return p[0] * VB + p[1] if len(p) == 2 else (p[0] * VB + p[1]) * 3 + p[2]


def build_canonical(VB: int, states: Dict[Tuple[int, int], Tuple[int, int]],
                    arcs: List[Tuple[Tuple[int, int], Tuple[int, int], int, int, np.float32]],
                    triples: bool = False):
    """states: {(a,b) or (a,b,f): (is_start, is_accept)}; arcs: [(src, dst, il, ol, w[, (arc_a, arc_b)])]
    -> canonical dict (with arc_a / arc_b when the arcs carry provenance, pair_f for triples)."""
    keys = sorted(states, key=lambda p: state_key(p, VB))
    nid = {p: i for i, p in enumerate(keys)}
    rows = collections.defaultdict(list)
    prov = bool(arcs) and len(arcs[0]) == 6
    for t in arcs:
        s, d, il, ol, w = t[:5]
        pv = t[5] if prov else (0, 0)
        rows[nid[s]].append((nid[d], il, ol, wbits(w), pv[0], pv[1], np.float32(w)))
    V = len(keys)
    row_ptr = np.zeros(V + 1, np.int64)
    dst, ilab, olab, wt, aa, ab = [], [], [], [], [], []
    for i in range(V):
        r = sorted(rows[i], key=lambda t: t[:6])
        row_ptr[i + 1] = row_ptr[i] + len(r)
        for d, il, ol, _b, xa, xb, w in r:
            dst.append(d); ilab.append(il); olab.append(ol); wt.append(w); aa.append(xa); ab.append(xb)
    out = {
        "num_states": V, "num_arcs": int(row_ptr[-1]), "row_ptr": row_ptr,
        "ilabel": np.array(ilab, np.int32), "olabel": np.array(olab, np.int32),
        "dst": np.array(dst, np.int32), "weight": np.array(wt, np.float32).reshape(-1),
        "is_start": np.array([states[p][0] for p in keys], np.uint8),
        "is_accept": np.array([states[p][1] for p in keys], np.uint8),
        "pair_a": np.array([p[0] for p in keys], np.int32),
        "pair_b": np.array([p[1] for p in keys], np.int32),
    }
    if triples:
        out["pair_f"] = np.array([p[2] for p in keys], np.int32)
    if prov:
        out["arc_a"], out["arc_b"] = np.array(aa, np.int32), np.array(ab, np.int32)
    return out


CANON_KEYS = ("row_ptr", "ilabel", "olabel", "dst", "is_start", "is_accept", "pair_a", "pair_b")


def assert_canonical_equal(got, exp, what=""):
    """Element-by-element equality of two canonical graphs; weights compared BIT-exactly."""
    assert int(got["num_states"]) == int(exp["num_states"]), f"{what}: V {got['num_states']} != {exp['num_states']}"
    assert int(got["num_arcs"]) == int(exp["num_arcs"]), f"{what}: E {got['num_arcs']} != {exp['num_arcs']}"
    keys = CANON_KEYS + (("pair_f",) if "pair_f" in exp or "pair_f" in got else ())
    for k in keys:
        a, b = np.asarray(got[k]), np.asarray(exp[k])
        if not np.array_equal(a.astype(np.int64), b.astype(np.int64)):
            bad = np.flatnonzero(a.astype(np.int64) != b.astype(np.int64))
            raise AssertionError(f"{what}: field {k} differs at {bad[:10]} ({a[bad[:5]]} vs {b[bad[:5]]})")
    ga = np.asarray(got["weight"], np.float32).view(np.uint32)
    gb = np.asarray(exp["weight"], np.float32).view(np.uint32)
    if not np.array_equal(ga, gb):
        bad = np.flatnonzero(ga != gb)
        raise AssertionError(f"{what}: weight bits differ at {bad[:10]}")
    for k in ("arc_a", "arc_b"):  # provenance, when both sides carry it
        if got.get(k) is not None and exp.get(k) is not None:
            a, b = np.asarray(got[k], np.int64), np.asarray(exp[k], np.int64)
            if not np.array_equal(a, b):
                bad = np.flatnonzero(a != b)
                raise AssertionError(f"{what}: provenance {k} differs at {bad[:10]} ({a[bad[:5]]} vs {b[bad[:5]]})")


def canonicalize_rows(g, VB: int):
    """Canonicalise a graph whose states are ALREADY numbered by ascending key (the GPU's numbering):
    sorts each row by (dst, ilabel, olabel, weight bits).  Plain numpy lexsort; this is the
    comparator, not part of either implementation."""
    V = int(g["num_states"]); E = int(g["num_arcs"])
    row_ptr = np.asarray(g["row_ptr"], np.int64)
    keys = np.asarray(g["pair_a"], np.int64) * VB + np.asarray(g["pair_b"], np.int64)
    if V > 1 and not np.all(np.diff(keys) > 0):
        raise AssertionError("states are not numbered by ascending pair key")
    src = np.repeat(np.arange(V, dtype=np.int64), np.diff(row_ptr))
    wb = np.asarray(g["weight"], np.float32).view(np.uint32)
    prov = g.get("arc_a") is not None
    tie = (np.asarray(g["arc_b"]), np.asarray(g["arc_a"])) if prov else ()  # provenance breaks ties
    order = np.lexsort(tie + (wb, np.asarray(g["olabel"]), np.asarray(g["ilabel"]), np.asarray(g["dst"]), src))
    out = dict(g)
    for k in ("dst", "ilabel", "olabel", "weight") + (("arc_a", "arc_b") if prov else ()):
        out[k] = np.asarray(g[k])[order]
    out["num_states"], out["num_arcs"] = V, E
    return out


def canonicalize_any(g, VB: int):
    """Canonicalise a graph with ANY state numbering: states sorted by their key (pairs, or triples
    when g has pair_f), dst remapped, rows sorted as in canonicalize_rows.  Comparator only."""
    V = int(g["num_states"])
    keys = np.asarray(g["pair_a"], np.int64) * VB + np.asarray(g["pair_b"], np.int64)
    if "pair_f" in g and g["pair_f"] is not None:
        keys = keys * 3 + np.asarray(g["pair_f"], np.int64)
    order = np.argsort(keys, kind="stable")
    newid = np.empty(V, np.int64)
    newid[order] = np.arange(V)
    rp = np.asarray(g["row_ptr"], np.int64)
    deg = np.diff(rp)[order]
    nrp = np.zeros(V + 1, np.int64)
    np.cumsum(deg, out=nrp[1:])
    arc_idx = np.concatenate([np.arange(rp[o], rp[o + 1]) for o in order]) if V else np.zeros(0, np.int64)
    out = dict(g)
    out["row_ptr"] = nrp
    for k in ("is_start", "is_accept", "pair_a", "pair_b") + (("pair_f",) if "pair_f" in g else ()):
        out[k] = np.asarray(g[k])[order]
    for k in ("ilabel", "olabel", "weight") + (("arc_a", "arc_b") if g.get("arc_a") is not None else ()):
        out[k] = np.asarray(g[k])[arc_idx]
    out["dst"] = newid[np.asarray(g["dst"], np.int64)[arc_idx]].astype(np.int32) if len(arc_idx) else np.zeros(0, np.int32)
    out["pair_a"] = np.asarray(out["pair_a"])
    fake = dict(out)
    fake["pair_a"] = np.arange(V, dtype=np.int64)  # rows are now in key order
    fake["pair_b"] = np.zeros(V, np.int64)
    res = canonicalize_rows(fake, 1)
    res["pair_a"], res["pair_b"] = out["pair_a"], out["pair_b"]
    return res


# ----------------------------------------------------------------------------- plain definition
def n1_moves(A, B, ua, ub, prov: bool = False):
    """All moves of N1 from pair (ua, ub): M1 (incl. eps==eps), M2, M3 (SURVEY §8 move table).
    prov: append the move's arc pair (e_a, e_b), -1 for the side that stays."""
    out = []
    for ea in range(A.row_ptr[ua], A.row_ptr[ua + 1]):
        for eb in range(B.row_ptr[ub], B.row_ptr[ub + 1]):
            if A.olabel[ea] == B.ilabel[eb]:
                out.append(((int(A.dst[ea]), int(B.dst[eb])), int(A.ilabel[ea]), int(B.olabel[eb]),
                            f32add(A.weight[ea], B.weight[eb])) + (((int(ea), int(eb)),) if prov else ()))
    for ea in range(A.row_ptr[ua], A.row_ptr[ua + 1]):
        if A.olabel[ea] == EPS:
            out.append(((int(A.dst[ea]), ub), int(A.ilabel[ea]), EPS, np.float32(A.weight[ea]))
                       + (((int(ea), -1),) if prov else ()))
    for eb in range(B.row_ptr[ub], B.row_ptr[ub + 1]):
        if B.ilabel[eb] == EPS:
            out.append(((ua, int(B.dst[eb])), EPS, int(B.olabel[eb]), np.float32(B.weight[eb]))
                       + (((-1, int(eb)),) if prov else ()))
    return out


def filtered_moves(A, B, ua, ub, uf):
    """Moves of the three-state eps filter from triple (ua, ub, uf): MATCH
    (o_a == i_b != eps, any f -> 0), EPS-BOTH (o_a == i_b == eps, only f = 0 -> 0), EPS-A (o_a = eps,
    f in {0,1} -> 1), EPS-B (i_b = eps, f in {0,2} -> 2)."""
    out = []
    for ea in range(A.row_ptr[ua], A.row_ptr[ua + 1]):
        for eb in range(B.row_ptr[ub], B.row_ptr[ub + 1]):
            if A.olabel[ea] != B.ilabel[eb] or (A.olabel[ea] == EPS and uf != 0):
                continue
            out.append(((int(A.dst[ea]), int(B.dst[eb]), 0), int(A.ilabel[ea]), int(B.olabel[eb]),
                        f32add(A.weight[ea], B.weight[eb])))
    if uf in (0, 1):
        for ea in range(A.row_ptr[ua], A.row_ptr[ua + 1]):
            if A.olabel[ea] == EPS:
                out.append(((int(A.dst[ea]), ub, 1), int(A.ilabel[ea]), EPS, np.float32(A.weight[ea])))
    if uf in (0, 2):
        for eb in range(B.row_ptr[ub], B.row_ptr[ub + 1]):
            if B.ilabel[eb] == EPS:
                out.append(((ua, int(B.dst[eb]), 2), EPS, int(B.olabel[eb]), np.float32(B.weight[eb])))
    return out


def plain_trim_product_filtered(A, B):
    """trim of the full eps-filtered product over V_A x V_B x 3 (tiny inputs only)."""
    fwd = collections.defaultdict(list)
    bwd = collections.defaultdict(list)
    all_arcs = []
    for ua in range(A.num_states):
        for ub in range(B.num_states):
            for uf in range(3):
                for mv in filtered_moves(A, B, ua, ub, uf):
                    all_arcs.append(((ua, ub, uf),) + tuple(mv))
                    fwd[(ua, ub, uf)].append(mv[0])
                    bwd[mv[0]].append((ua, ub, uf))
    starts = [(int(a), int(b), 0) for a in np.flatnonzero(A.is_start) for b in np.flatnonzero(B.is_start)]
    accepts = [(int(a), int(b), f) for a in np.flatnonzero(A.is_accept) for b in np.flatnonzero(B.is_accept)
               for f in range(3)]
    keep = _reach(fwd, starts) & _reach(bwd, accepts)
    sset = set(starts)
    states = {p: (int(p in sset), int(A.is_accept[p[0]] and B.is_accept[p[1]])) for p in keep}
    arcs = [t for t in all_arcs if t[0] in keep and t[1] in keep]
    return build_canonical(B.num_states, states, arcs, triples=True)


def _reach(adj, seeds):
    seen = set(seeds)
    stack = list(seeds)
    while stack:
        u = stack.pop()
        for v in adj.get(u, ()):
            if v not in seen:
                seen.add(v)
                stack.append(v)
    return seen


def plain_trim_product(A, B, prov: bool = False):
    """trim(P_N1) built from the definition (tiny inputs only: V_A * V_B <= ~1e4); prov: with the
    arc pair of every arc."""
    fwd = collections.defaultdict(list)
    bwd = collections.defaultdict(list)
    all_arcs = []
    for ua in range(A.num_states):
        for ub in range(B.num_states):
            for mv in n1_moves(A, B, ua, ub, prov):
                d = mv[0]
                all_arcs.append(((ua, ub),) + tuple(mv))
                fwd[(ua, ub)].append(d)
                bwd[d].append((ua, ub))
    starts = [(a, b) for a in np.flatnonzero(A.is_start) for b in np.flatnonzero(B.is_start)]
    accepts = [(a, b) for a in np.flatnonzero(A.is_accept) for b in np.flatnonzero(B.is_accept)]
    starts = [(int(a), int(b)) for a, b in starts]
    accepts = [(int(a), int(b)) for a, b in accepts]
    keep = _reach(fwd, starts) & _reach(bwd, accepts)
    states = {p: (int(p in set(starts)), int(A.is_accept[p[0]] and B.is_accept[p[1]])) for p in keep}
    arcs = [t for t in all_arcs if t[0] in keep and t[1] in keep]
    return build_canonical(B.num_states, states, arcs)


def plain_coaccessible(A, B) -> np.ndarray:
    """R from the definition: backward reachability to accept pairs over the full product."""
    bwd = collections.defaultdict(list)
    for ua in range(A.num_states):
        for ub in range(B.num_states):
            for d, *_ in n1_moves(A, B, ua, ub):
                bwd[d].append((ua, ub))
    accepts = [(int(a), int(b)) for a in np.flatnonzero(A.is_accept) for b in np.flatnonzero(B.is_accept)]
    R = np.zeros(A.num_states * B.num_states, np.uint8)
    for a, b in _reach(bwd, accepts):
        R[a * B.num_states + b] = 1
    return R


# ----------------------------------------------------------------------------- Eq. (1) brute force
def accepting_paths(g, max_len: int = 64):
    """All start->accept paths of a DAG (or paths of <= max_len arcs): list of (arcs tuple)."""
    out = []
    row_ptr = g.row_ptr

    def dfs(v, path):
        if g.is_accept[v]:
            out.append(tuple(path))
        if len(path) >= max_len:
            return
        for e in range(row_ptr[v], row_ptr[v + 1]):
            path.append(e)
            dfs(int(g.dst[e]), path)
            path.pop()

    for s in np.flatnonzero(g.is_start):
        dfs(int(s), [])
    return out


def delannoy(m: int, n: int) -> int:
    return sum(comb(m, k) * comb(n, k) * 2 ** k for k in range(min(m, n) + 1))


def _runs(labels):
    """(non-eps label sequence, eps-run lengths before / between / after them)."""
    seq, runs, cur = [], [], 0
    for l in labels:
        if l == EPS:
            cur += 1
        else:
            runs.append(cur); seq.append(l); cur = 0
    runs.append(cur)
    return tuple(seq), runs


def eq1_bruteforce(A, B, max_len: int = 64, filtered: bool = False):
    """Expected multiset of composed accepting-path scores per (x, z) under N1.

    Each matched path pair (pi_a labelled (x, y), pi_b labelled (y, z)) contributes the score
    s_a + s_b (float64; exact for dyadic weights) with multiplicity prod_i D(k_i, m_i)
    (Delannoy; = 1 for every pair when A has no eps outputs or B no eps inputs).  filtered: the
    eps-filtered composition's target -- exactly ONE composed path per matched path pair (SPEC.md
    "Path bijection"), i.e. Eq. (1) itself with no duplicated terms.
    """
    pa = collections.defaultdict(list)
    for p in accepting_paths(A, max_len):
        x = tuple(int(A.ilabel[e]) for e in p if A.ilabel[e] != EPS)
        y, ka = _runs([int(A.olabel[e]) for e in p])
        pa[y].append((x, ka, sum(float(A.weight[e]) for e in p)))
    table = collections.defaultdict(collections.Counter)
    for p in accepting_paths(B, max_len):
        y, mb = _runs([int(B.ilabel[e]) for e in p])
        z = tuple(int(B.olabel[e]) for e in p if B.olabel[e] != EPS)
        sb = sum(float(B.weight[e]) for e in p)
        for x, ka, sa in pa.get(y, ()):
            mult = 1
            if not filtered:
                for k, m in zip(ka, mb):
                    mult *= delannoy(k, m)
            table[(x, z)][sa + sb] += mult
    return table


def composed_path_table(C, max_len: int = 256):
    """Multiset of accepting-path scores per (x, z) of a composed graph (dict of arrays, DAG)."""
    V = int(C["num_states"])
    rp = np.asarray(C["row_ptr"]); dst = np.asarray(C["dst"])
    il = np.asarray(C["ilabel"]); ol = np.asarray(C["olabel"]); w = np.asarray(C["weight"], np.float32)
    acc = np.asarray(C["is_accept"]); st = np.asarray(C["is_start"])
    table = collections.defaultdict(collections.Counter)

    def dfs(v, xs, zs, s, depth):
        if acc[v]:
            table[(tuple(xs), tuple(zs))][s] += 1
        if depth >= max_len:
            return
        for e in range(rp[v], rp[v + 1]):
            if il[e] != EPS:
                xs.append(int(il[e]))
            if ol[e] != EPS:
                zs.append(int(ol[e]))
            dfs(int(dst[e]), xs, zs, s + float(w[e]), depth + 1)
            if il[e] != EPS:
                xs.pop()
            if ol[e] != EPS:
                zs.pop()

    for v in range(V):
        if st[v]:
            dfs(v, [], [], 0.0, 0)
    return table


def logsumexp_table(table):
    out = {}
    for k, cnt in table.items():
        vals = [(s, c) for s, c in cnt.items()]
        m = max(s for s, _ in vals)
        out[k] = m + math.log(sum(c * math.exp(s - m) for s, c in vals))
    return out


# ----------------------------------------------------------------------------- trim / identity
def is_trim(C) -> bool:
    """Every state reachable from a start AND every state reaches an accept."""
    V = int(C["num_states"])
    if V == 0:
        return True
    import scipy.sparse as sp
    from scipy.sparse.csgraph import breadth_first_order
    rp = np.asarray(C["row_ptr"], np.int64); dst = np.asarray(C["dst"], np.int64)
    src = np.repeat(np.arange(V, dtype=np.int64), np.diff(rp))
    st = np.flatnonzero(np.asarray(C["is_start"])); ac = np.flatnonzero(np.asarray(C["is_accept"]))

    def reach(a, b, seeds):  # BFS from a virtual node V linked to all seeds
        a = np.concatenate([a, np.full(len(seeds), V)]); b = np.concatenate([b, seeds])
        G = sp.csr_matrix((np.ones(len(a), np.int8), (a, b)), shape=(V + 1, V + 1))
        return len(breadth_first_order(G, V, directed=True, return_predecessors=False))

    return reach(src, dst, st) == V + 1 and reach(dst, src, ac) == V + 1


def trim_fst(A):
    """Textbook trim of a single FST: (keep mask) by forward + backward reachability."""
    fwd = collections.defaultdict(list); bwd = collections.defaultdict(list)
    src = A.src
    for e in range(A.num_arcs):
        fwd[int(src[e])].append(int(A.dst[e])); bwd[int(A.dst[e])].append(int(src[e]))
    keep = _reach(fwd, [int(v) for v in np.flatnonzero(A.is_start)]) & \
        _reach(bwd, [int(v) for v in np.flatnonzero(A.is_accept)])
    return keep


def identity_expected(A):
    """A o Id_Sigma == trim(A): states (a, 0); arcs of A between kept states, weights w_a
    (M1: fl(w_a + 0.0) == w_a for nonzero w_a; M2 copies w_a)."""
    keep = trim_fst(A)
    states = {(a, 0): (int(A.is_start[a]), int(A.is_accept[a])) for a in keep}
    src = A.src
    arcs = []
    for e in range(A.num_arcs):
        s, d = int(src[e]), int(A.dst[e])
        if s in keep and d in keep:
            w = f32add(A.weight[e], 0.0) if A.olabel[e] != EPS else np.float32(A.weight[e])
            arcs.append(((s, 0), (d, 0), int(A.ilabel[e]), int(A.olabel[e]), w))
    return build_canonical(1, states, arcs)


# ----------------------------------------------------------------------------- trellis
def _eps_closure(B, mask, forward: bool):
    """Close a boolean state mask under B's eps-input arcs (forward) or their reverse."""
    src = B.src
    e = np.flatnonzero(B.ilabel == EPS)
    a, b = (src[e], B.dst[e]) if forward else (B.dst[e], src[e])
    m = mask.copy()
    while True:
        new = np.zeros_like(m)
        new[b[m[a]]] = True
        new &= ~m
        if not new.any():
            return m
        m |= new


def trellis_compose(A, B):
    """C = A o B for A = linear emissions (T+1 states, one arc per token per frame, no eps).

    fwd[t] = B states reachable from a B start consuming exactly t non-eps input symbols (eps-closed);
    bwd[t] = B states that reach a B accept consuming exactly T - t symbols.  Trim states are
    (t, b) with b in fwd[t] & bwd[t]; arcs are M1 (B non-eps arc with the frame-t A arc of that
    label) and M3 (B eps-input arc), between trim states.
    """
    T = A.num_states - 1
    VB = B.num_states
    srcB = B.src
    # A's arc of label l at frame t (emissions: exactly one per token)
    tokA = {}
    for e in range(A.num_arcs):
        tokA[(int(A.src[e]), int(A.olabel[e]))] = e
    ne = np.flatnonzero(B.ilabel != EPS)
    fwd = np.zeros((T + 1, VB), bool)
    fwd[0] = _eps_closure(B, B.is_start.astype(bool), True)
    for t in range(T):
        nxt = np.zeros(VB, bool)
        ok = fwd[t][srcB[ne]]
        labs_ok = np.array([(t, int(l)) in tokA for l in B.ilabel[ne]], bool)
        nxt[B.dst[ne][ok & labs_ok]] = True
        fwd[t + 1] = _eps_closure(B, nxt, True)
    bwd = np.zeros((T + 1, VB), bool)
    bwd[T] = _eps_closure(B, B.is_accept.astype(bool), False)
    for t in range(T - 1, -1, -1):
        prv = np.zeros(VB, bool)
        labs_ok = np.array([(t, int(l)) in tokA for l in B.ilabel[ne]], bool)
        ok = bwd[t + 1][B.dst[ne]] & labs_ok
        prv[srcB[ne][ok]] = True
        bwd[t] = _eps_closure(B, prv, False)
    keep = fwd & bwd
    states = {}
    for t in range(T + 1):
        for b in np.flatnonzero(keep[t]):
            states[(t, int(b))] = (int(t == 0 and B.is_start[b] and A.is_start[0]),
                                   int(t == T and B.is_accept[b]))
    arcs = []
    for (t, b) in states:
        for eb in range(B.row_ptr[b], B.row_ptr[b + 1]):
            d = int(B.dst[eb])
            if B.ilabel[eb] == EPS:
                if (t, d) in states:
                    arcs.append(((t, b), (t, d), EPS, int(B.olabel[eb]), np.float32(B.weight[eb])))
            elif t < T and (t, int(B.ilabel[eb])) in tokA and (t + 1, d) in states:
                ea = tokA[(t, int(B.ilabel[eb]))]
                arcs.append(((t, b), (t + 1, d), int(A.ilabel[ea]), int(B.olabel[eb]),
                             f32add(A.weight[ea], B.weight[eb])))
    return build_canonical(VB, states, arcs)


def merge_shards(parts, arc_offsets):
    """Concatenates the host copies of a sharded composition's shards (rank order) into one CSR: the
    shards hold contiguous state-id ranges with global dst ids and shard-local row_ptr (test helper)."""
    out = {k: np.concatenate([p[k] for p in parts]) for k in ("ilabel", "olabel", "dst", "weight", "is_start",
                                                              "is_accept", "pair_a", "pair_b")}
    rps = [p["row_ptr"][:-1] + off for p, off in zip(parts, arc_offsets)]
    total = sum(int(p["num_arcs"]) for p in parts)
    out["row_ptr"] = np.concatenate(rps + [np.array([total], np.int64)])
    out["num_states"] = sum(int(p["num_states"]) for p in parts)
    out["num_arcs"] = total
    return out
