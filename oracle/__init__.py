"""CPU oracle for eager trimmed WFST composition (arXiv 2110.02848, Algorithm 1).

TEST INFRASTRUCTURE ONLY: tests/, __graft_entry__.smoke() and bench.py's cpu_baseline /
``--impl reference`` legs may import this package; the product path
(paper_2110_02848_b200) never does.  The arithmetic lives in ``compose.c`` (plain C99, one
binary32 add per M1 arc, no fast-math); this module only marshals numpy arrays through ctypes.
Shares no code with the CUDA path.

Functions:
  compose(A, B)        -> dict of numpy arrays, states in FIFO discovery order (Alg. 1), with the
                          provenance arc_a / arc_b of every arc (-1 = that side stays)
  canonical(A, B)      -> same, canonical form (reading 24)
  compose_filtered(A, B) -> the eps-filtered variant (three-state filter),
                          states (pair_a, pair_b, pair_f)
  compose_chain(gs)    -> N-way composition as a left fold of compose
  coaccessible(A, B)   -> uint8 [V_A * V_B] co-accessible set R (Alg. 1 line 3)
  digest(A, B)         -> {num_states, num_arcs, d0, d1}: Alg. 1 with the arcs streamed into the
                          order-independent digest (full-size parity)
  in_adjacency(g)      -> (inArcOffset, inArcs) per §3.2
"""
from __future__ import annotations

import ctypes as C
import os
import subprocess
import threading

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_SO = os.path.join(_HERE, "liboracle.so")
_SRC = os.path.join(_HERE, "compose.c")
_lock = threading.Lock()
_lib = None


def build(force: bool = False) -> str:
    """Compile compose.c -> liboracle.so (gcc -O2, IEEE-strict: no -ffast-math)."""
    if force or not os.path.exists(_SO) or os.path.getmtime(_SO) < os.path.getmtime(_SRC):
        subprocess.check_call(["gcc", "-O2", "-std=c99", "-fPIC", "-shared", "-fno-fast-math",
                               "-ffp-contract=off", "-o", _SO, _SRC])
    return _SO


class _Fst(C.Structure):
    _fields_ = [("V", C.c_int32), ("E", C.c_int64), ("row_ptr", C.c_void_p), ("ilabel", C.c_void_p),
                ("olabel", C.c_void_p), ("dst", C.c_void_p), ("weight", C.c_void_p),
                ("is_start", C.c_void_p), ("is_accept", C.c_void_p)]


class _Graph(C.Structure):
    _fields_ = [("V", C.c_int32), ("E", C.c_int64), ("row_ptr", C.POINTER(C.c_int64)),
                ("ilabel", C.POINTER(C.c_int32)), ("olabel", C.POINTER(C.c_int32)),
                ("dst", C.POINTER(C.c_int32)), ("weight", C.POINTER(C.c_float)),
                ("is_start", C.POINTER(C.c_uint8)), ("is_accept", C.POINTER(C.c_uint8)),
                ("pair_a", C.POINTER(C.c_int32)), ("pair_b", C.POINTER(C.c_int32)),
                ("level", C.POINTER(C.c_int32)), ("arc_a", C.POINTER(C.c_int32)),
                ("arc_b", C.POINTER(C.c_int32)), ("pair_f", C.POINTER(C.c_int32))]


def _load():
    global _lib
    with _lock:
        if _lib is None:
            lib = C.CDLL(build())
            lib.orc_compose.argtypes = [C.POINTER(_Fst), C.POINTER(_Fst), C.POINTER(_Graph)]
            lib.orc_compose_filtered.argtypes = [C.POINTER(_Fst), C.POINTER(_Fst), C.POINTER(_Graph)]
            lib.orc_canonicalize.argtypes = [C.POINTER(_Graph), C.c_int32]
            lib.orc_coaccessible.argtypes = [C.POINTER(_Fst), C.POINTER(_Fst), C.c_void_p]
            lib.orc_digest.argtypes = [C.POINTER(_Fst), C.POINTER(_Fst), C.c_void_p]
            lib.orc_in_adjacency.argtypes = [C.POINTER(_Fst), C.c_void_p, C.c_void_p]
            lib.orc_free.argtypes = [C.POINTER(_Graph)]
            _lib = lib
    return _lib


def _desc(g):
    arrs = [np.ascontiguousarray(g.row_ptr, np.int64), np.ascontiguousarray(g.ilabel, np.int32),
            np.ascontiguousarray(g.olabel, np.int32), np.ascontiguousarray(g.dst, np.int32),
            np.ascontiguousarray(g.weight, np.float32), np.ascontiguousarray(g.is_start, np.uint8),
            np.ascontiguousarray(g.is_accept, np.uint8)]
    d = _Fst(int(g.num_states), int(g.row_ptr[-1]), *[a.ctypes.data for a in arrs])
    return d, arrs  # keep arrays alive


def _take(ptr, n, dtype):
    if n == 0:
        return np.zeros(0, dtype)
    return np.ctypeslib.as_array(ptr, shape=(n,)).astype(dtype, copy=True)


def _to_numpy(g: _Graph, filtered: bool = False):
    V, E = g.V, g.E
    out = {
        "num_states": V, "num_arcs": E,
        "row_ptr": _take(g.row_ptr, V + 1, np.int64),
        "ilabel": _take(g.ilabel, E, np.int32), "olabel": _take(g.olabel, E, np.int32),
        "dst": _take(g.dst, E, np.int32), "weight": _take(g.weight, E, np.float32),
        "is_start": _take(g.is_start, V, np.uint8), "is_accept": _take(g.is_accept, V, np.uint8),
        "pair_a": _take(g.pair_a, V, np.int32), "pair_b": _take(g.pair_b, V, np.int32),
        "level": _take(g.level, V, np.int32),
        "arc_a": _take(g.arc_a, E, np.int32), "arc_b": _take(g.arc_b, E, np.int32),
    }
    if filtered:
        out["pair_f"] = _take(g.pair_f, V, np.int32)
    return out


def compose(A, B, canonicalize: bool = False, eps_filter: bool = False):
    lib = _load()
    da, ka = _desc(A)
    db, kb = _desc(B)
    out = _Graph()
    fn = lib.orc_compose_filtered if eps_filter else lib.orc_compose
    if fn(C.byref(da), C.byref(db), C.byref(out)) != 0:
        raise MemoryError("oracle compose failed")
    try:
        if canonicalize and lib.orc_canonicalize(C.byref(out), int(B.num_states)) != 0:
            raise MemoryError("oracle canonicalize failed")
        return _to_numpy(out, eps_filter)
    finally:
        lib.orc_free(C.byref(out))
        del ka, kb


def canonical(A, B, eps_filter: bool = False):
    return compose(A, B, canonicalize=True, eps_filter=eps_filter)


def compose_filtered(A, B, canonicalize: bool = False):
    """eps-filtered variant (SPEC.md S:150-177 three-state filter): states are
    triples (pair_a, pair_b, pair_f), f in {0 MATCH, 1 A_EPS, 2 B_EPS}; canonical key
    (a * V_B + b) * 3 + f."""
    return compose(A, B, canonicalize=canonicalize, eps_filter=True)


def compose_chain(graphs, canonicalize: bool = False):
    """N-way composition as the left fold ((G0 o G1) o G2) o ... (PAPER.md:366-368 names N-way
    composition as future work; Algorithm 1 applied N-1 times).  Returns the last composition (as
    numpy dict); with canonicalize, EVERY step is canonicalised, so each intermediate's states are
    numbered by ascending pair key and the result's pair_a indexes them in that order."""
    from types import SimpleNamespace
    cur = graphs[0]
    out = None
    for k, g in enumerate(graphs[1:]):
        last = k == len(graphs) - 2
        out = compose(cur, g, canonicalize=canonicalize)
        if not last:
            cur = SimpleNamespace(num_states=int(out["num_states"]), num_arcs=int(out["num_arcs"]),
                                  **{k: out[k] for k in ("row_ptr", "ilabel", "olabel", "dst", "weight",
                                                         "is_start", "is_accept")})
    return out


def coaccessible(A, B) -> np.ndarray:
    lib = _load()
    da, ka = _desc(A)
    db, kb = _desc(B)
    R = np.zeros(max(1, A.num_states * B.num_states), np.uint8)
    if lib.orc_coaccessible(C.byref(da), C.byref(db), R.ctypes.data) != 0:
        raise MemoryError
    del ka, kb
    return R[: A.num_states * B.num_states]


def digest(A, B) -> dict:
    """Algorithm 1 with the arcs streamed into the order-independent digest (the
    definition is in compose.c): {num_states, num_arcs, d0, d1}.  Nothing is stored per arc, so the
    full-size configurations fit in host memory."""
    lib = _load()
    da, ka = _desc(A)
    db, kb = _desc(B)
    out = np.zeros(4, np.uint64)
    if lib.orc_digest(C.byref(da), C.byref(db), out.ctypes.data) != 0:
        raise MemoryError
    del ka, kb
    return {"num_states": int(out[0]), "num_arcs": int(out[1]), "d0": int(out[2]), "d1": int(out[3])}


def in_adjacency(g):
    lib = _load()
    d, keep = _desc(g)
    off = np.zeros(g.num_states + 1, np.int64)
    arcs = np.zeros(max(1, g.num_arcs), np.int64)
    if lib.orc_in_adjacency(C.byref(d), off.ctypes.data, arcs.ctypes.data) != 0:
        raise MemoryError
    del keep
    return off, arcs[: g.num_arcs]
