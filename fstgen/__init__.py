"""Seeded synthetic workload generators (shared by the oracle tests, the GPU tests and bench.py).

This module holds NO composition arithmetic: it only draws random graphs of the
shapes the paper benchmarks (arXiv 2110.02848 §4) and packs them
into plain numpy CSR arrays.  Both the CPU oracle (``oracle/``) and the CUDA path
(``paper_2110_02848_b200``) consume the very same arrays.

Conventions:
  * epsilon label = -1 (SURVEY §8(c) reading 1); labels are int32 >= -1.
  * random stream = splitmix64 (SPEC.md:371 constants, standard 30/27/31 shifts);
    uniform integer in [0, n) = (r * n) >> 64.
  * an FST is a CSR grouped by source: row_ptr[V+1] int64, ilabel/olabel/dst int32,
    weight float32, is_start/is_accept uint8.  Arc order inside a row = draw order.
"""
from __future__ import annotations

import dataclasses
import math
from typing import List, Optional, Sequence

import numpy as np

EPS = -1
_GOLDEN = np.uint64(0x9E3779B97F4A7C15)
_M1 = np.uint64(0xBF58476D1CE4E5B9)
_M2 = np.uint64(0x94D049BB133111EB)
_MASK64 = (1 << 64) - 1


# --------------------------------------------------------------------------- rng
class SplitMix64:
    """splitmix64 stream.  ``next()`` returns a python int in [0, 2^64)."""

    def __init__(self, seed: int):
        self.s = seed & _MASK64

    def next(self) -> int:
        self.s = (self.s + 0x9E3779B97F4A7C15) & _MASK64
        z = self.s
        z = ((z ^ (z >> 30)) * 0xBF58476D1CE4E5B9) & _MASK64
        z = ((z ^ (z >> 27)) * 0x94D049BB133111EB) & _MASK64
        return z ^ (z >> 31)

    def below(self, n: int) -> int:
        """uniform integer in [0, n): (r * n) >> 64."""
        return (self.next() * n) >> 64

    def block(self, count: int) -> np.ndarray:
        """The next ``count`` outputs as a uint64 array (vectorised, same stream)."""
        k = np.arange(1, count + 1, dtype=np.uint64)
        with np.errstate(over="ignore"):
            s = np.uint64(self.s) + k * _GOLDEN
            z = s
            z = (z ^ (z >> np.uint64(30))) * _M1
            z = (z ^ (z >> np.uint64(27))) * _M2
            z = z ^ (z >> np.uint64(31))
        self.s = (self.s + count * 0x9E3779B97F4A7C15) & _MASK64
        return z


def below_vec(r: np.ndarray, n) -> np.ndarray:
    """Vectorised (r * n) >> 64 for uint64 r and 0 < n < 2^31 (n scalar or array)."""
    n = np.asarray(n, dtype=np.uint64)
    rh = r >> np.uint64(32)
    rl = r & np.uint64(0xFFFFFFFF)
    with np.errstate(over="ignore"):
        return (rh * n + ((rl * n) >> np.uint64(32))) >> np.uint64(32)


# --------------------------------------------------------------------------- container
@dataclasses.dataclass
class Fst:
    """A WFST as a source-grouped CSR of numpy arrays (the ABI's fst_desc, on the host)."""

    num_states: int
    row_ptr: np.ndarray  # int64 [V+1]
    ilabel: np.ndarray  # int32 [E]
    olabel: np.ndarray  # int32 [E]
    dst: np.ndarray  # int32 [E]
    weight: np.ndarray  # float32 [E]
    is_start: np.ndarray  # uint8 [V]
    is_accept: np.ndarray  # uint8 [V]

    @property
    def num_arcs(self) -> int:
        return int(self.row_ptr[-1])

    @property
    def src(self) -> np.ndarray:
        return np.repeat(np.arange(self.num_states, dtype=np.int32), np.diff(self.row_ptr)).astype(np.int32)

    @staticmethod
    def from_arcs(num_states: int, src, dst, ilabel, olabel, weight, starts: Sequence[int],
                  accepts: Sequence[int]) -> "Fst":
        src = np.asarray(src, dtype=np.int64)
        order = np.argsort(src, kind="stable")
        counts = np.bincount(src, minlength=num_states) if len(src) else np.zeros(num_states, np.int64)
        row_ptr = np.zeros(num_states + 1, dtype=np.int64)
        np.cumsum(counts, out=row_ptr[1:])
        st = np.zeros(num_states, dtype=np.uint8)
        ac = np.zeros(num_states, dtype=np.uint8)
        st[list(starts)] = 1
        ac[list(accepts)] = 1
        return Fst(num_states, row_ptr,
                   np.asarray(ilabel, dtype=np.int32)[order].copy(),
                   np.asarray(olabel, dtype=np.int32)[order].copy(),
                   np.asarray(dst, dtype=np.int32)[order].copy(),
                   np.asarray(weight, dtype=np.float32)[order].copy(), st, ac)

    def arcs(self):
        """(src, dst, ilabel, olabel, weight) tuples in arc order (python ints / floats)."""
        s = self.src
        return [(int(s[e]), int(self.dst[e]), int(self.ilabel[e]), int(self.olabel[e]), float(self.weight[e]))
                for e in range(self.num_arcs)]

    def to_text(self) -> str:
        """SPEC.md text format: nodes/start/accept/arc lines."""
        out = [f"nodes {self.num_states}"]
        out += [f"start {v}" for v in np.flatnonzero(self.is_start)]
        out += [f"accept {v}" for v in np.flatnonzero(self.is_accept)]
        for s, d, i, o, w in self.arcs():
            out.append(f"arc {s} {d} {i} {o} {np.float32(w).item()!r}")
        return "\n".join(out) + "\n"

    @staticmethod
    def from_text(text: str) -> "Fst":
        V = None
        starts, accepts, arcs = [], [], []
        for ln, line in enumerate(text.splitlines(), 1):
            line = line.split("#", 1)[0].strip()
            if not line:
                continue
            tok = line.split()
            if tok[0] == "nodes":
                V = int(tok[1])
            elif tok[0] == "start":
                starts.append(int(tok[1]))
            elif tok[0] == "accept":
                accepts.append(int(tok[1]))
            elif tok[0] == "arc":
                s, d, i, o = (int(t) for t in tok[1:5])
                if i < -1 or o < -1:
                    raise ValueError(f"line {ln}: label < -1")
                arcs.append((s, d, i, o, parse_weight(tok[5])))
            else:
                raise ValueError(f"line {ln}: unknown record {tok[0]!r}")
        if V is None:
            raise ValueError("missing 'nodes' line")
        for (s, d, *_r) in arcs:
            if not (0 <= s < V and 0 <= d < V):
                raise ValueError(f"node {max(s, d)} out of range")
        cols = list(zip(*arcs)) if arcs else [[], [], [], [], []]
        return Fst.from_arcs(V, *cols, starts=starts, accepts=accepts)


def parse_weight(tok: str) -> float:
    """Decimal or C99 hex-float literal, rounded once to float32 (sign of zero kept)."""
    v = float.fromhex(tok) if "x" in tok.lower() else float(tok)
    return float(np.float32(v))


def empty_fst(num_states: int = 0) -> Fst:
    z = np.zeros(0, np.int32)
    return Fst(num_states, np.zeros(num_states + 1, np.int64), z, z.copy(), z.copy(), np.zeros(0, np.float32),
               np.zeros(num_states, np.uint8), np.zeros(num_states, np.uint8))


# --------------------------------------------------------------------------- weights
def dyadic64_weights(rng: SplitMix64, n: int) -> np.ndarray:
    """-k/64 with k = 1 + rand(128): every path sum of a tiny graph is exact in fp32."""
    k = 1 + below_vec(rng.block(n), 128).astype(np.int64)
    return (-k.astype(np.float64) / 64.0).astype(np.float32)


def dyadic24_weights(rng: SplitMix64, n: int) -> np.ndarray:
    """-(u+1)*2^-24 with u = r >> 40: 24-bit dyadic in [-1, -2^-24], never +-0 (SURVEY d.2)."""
    u = (rng.block(n) >> np.uint64(40)).astype(np.float64)
    return (-(u + 1.0) * 2.0 ** -24).astype(np.float32)


# --------------------------------------------------------------------------- random graphs
def random_graph(num_states: int, degree: int, tokens: int, seed: int, *, acceptor: bool = True,
                 eps_prob: float = 0.0, weights: str = "dyadic24", starts=None, accepts=None) -> Fst:
    """Uniform-out-degree random graph (§4.1).

    Every state gets exactly ``degree`` arcs; dst uniform over all states (self-loops allowed);
    labels uniform over ``tokens``.  Draw order per arc: dst, ilabel, [olabel], weight (weights
    are drawn in a second block after the structure).  ``eps_prob`` > 0 makes each tape label
    epsilon independently with that probability (decided by one extra draw: rand(2^20) <
    eps_prob * 2^20).  Default start {0}, accept {V-1}.
    """
    V, D = num_states, degree
    E = V * D
    rng = SplitMix64(seed)
    per_arc = 2 if acceptor else 3
    if eps_prob > 0:
        per_arc += 1 if acceptor else 2
    r = rng.block(E * per_arc).reshape(E, per_arc) if E else np.zeros((0, per_arc), np.uint64)
    dst = below_vec(r[:, 0], V).astype(np.int32)
    if acceptor:
        lab = below_vec(r[:, 1], tokens).astype(np.int32)
        if eps_prob > 0:
            lab[below_vec(r[:, 2], 1 << 20) < int(eps_prob * (1 << 20))] = EPS
        il = ol = lab
    else:
        il = below_vec(r[:, 1], tokens).astype(np.int32)
        ol = below_vec(r[:, 2], tokens).astype(np.int32)
        if eps_prob > 0:
            thr = int(eps_prob * (1 << 20))
            il[below_vec(r[:, 3], 1 << 20) < thr] = EPS
            ol[below_vec(r[:, 4], 1 << 20) < thr] = EPS
    if weights == "dyadic24":
        w = dyadic24_weights(rng, E)
    elif weights == "dyadic64":
        w = dyadic64_weights(rng, E)
    elif weights == "zero":
        w = np.zeros(E, np.float32)
    else:
        raise ValueError(weights)
    src = np.repeat(np.arange(V, dtype=np.int32), D)
    starts = [0] if starts is None else starts
    accepts = [V - 1] if accepts is None else accepts
    return Fst.from_arcs(V, src, dst, il, ol.copy() if acceptor else ol, w, starts, accepts)


def random_dag(num_states: int, max_degree: int, tokens: int, eps_prob: float, seed: int,
               weights: str = "dyadic64", starts=None, accepts=None) -> Fst:
    """Acyclic random transducer for brute-force suites (SPEC.md random_dag): dst > src,
    per-state degree uniform in [0, max_degree], each tape label epsilon w.p. eps_prob."""
    rng = SplitMix64(seed)
    src, dst, il, ol = [], [], [], []
    thr = int(eps_prob * (1 << 20))
    for s in range(num_states - 1):
        deg = rng.below(max_degree + 1)
        for _ in range(deg):
            d = s + 1 + rng.below(num_states - 1 - s)
            i = rng.below(tokens)
            o = rng.below(tokens)
            if thr and rng.below(1 << 20) < thr:
                i = EPS
            if thr and rng.below(1 << 20) < thr:
                o = EPS
            src.append(s); dst.append(d); il.append(i); ol.append(o)
    E = len(src)
    w = dyadic64_weights(rng, E) if weights == "dyadic64" else np.zeros(E, np.float32)
    starts = [0] if starts is None else starts
    accepts = [num_states - 1] if accepts is None else accepts
    return Fst.from_arcs(num_states, src, dst, il, ol, w, starts, accepts)


# --------------------------------------------------------------------------- lexicon / emissions
N_LETTER_TOKENS = 28  # 0 = '|' (word end), 1 = "'", 2..27 = a..z  (SURVEY §8(c) reading 21)


def letter_lexicon(num_words: int, seed: int) -> List[List[int]]:
    """``num_words`` distinct random spellings: 2+rand(9) letters, letter = 2+rand(26) except "'"
    (token 1) with p = 1/64, then '|' (token 0).  Duplicates are redrawn (sampling without
    replacement)."""
    rng = SplitMix64(seed)
    seen, words = set(), []
    while len(words) < num_words:
        n = 2 + rng.below(9)
        w = []
        for _ in range(n):
            w.append(1 if rng.below(64) == 0 else 2 + rng.below(26))
        w.append(0)
        t = tuple(w)
        if t in seen:
            continue
        seen.add(t)
        words.append(w)
    return words


def lexicon_graph(words: List[List[int]]) -> Fst:
    """Shared start node 0; per word a fresh chain; ilabel = token, olabel = word id on the first
    arc and epsilon afterwards; chain end is an accept node; weights 0."""
    src, dst, il, ol = [], [], [], []
    accepts = []
    nxt = 1
    for wid, w in enumerate(words):
        prev = 0
        for j, tok in enumerate(w):
            src.append(prev); dst.append(nxt); il.append(tok); ol.append(wid if j == 0 else EPS)
            prev = nxt
            nxt += 1
        accepts.append(prev)
    return Fst.from_arcs(nxt, src, dst, il, ol, np.zeros(len(src), np.float32), [0], accepts)


def closure(g: Fst) -> Fst:
    """Kleene closure: one new node s (start and accept); eps:eps weight-0 arcs
    s -> every former start and every former accept -> s; former flags cleared."""
    s_new = g.num_states
    src = list(g.src)
    dst, il, ol, w = list(g.dst), list(g.ilabel), list(g.olabel), list(g.weight)
    for v in np.flatnonzero(g.is_start):
        src.append(s_new); dst.append(int(v)); il.append(EPS); ol.append(EPS); w.append(0.0)
    for v in np.flatnonzero(g.is_accept):
        src.append(int(v)); dst.append(s_new); il.append(EPS); ol.append(EPS); w.append(0.0)
    return Fst.from_arcs(g.num_states + 1, src, dst, il, ol, w, [s_new], [s_new])


def emissions_graph(num_frames: int, seed: int, tokens: int = N_LETTER_TOKENS) -> Fst:
    """Linear emissions acceptor: T+1 nodes, for each frame t and token p an
    arc t -> t+1 labelled p:p with weight log-softmax over ``tokens`` logits 2*N(0,1)
    (Box-Muller in float64, rounded once to float32)."""
    T = num_frames
    rng = SplitMix64(seed)
    r = rng.block(2 * T * tokens).reshape(T * tokens, 2)
    u1 = (r[:, 0] >> np.uint64(11)).astype(np.float64) * 2.0 ** -53
    u2 = (r[:, 1] >> np.uint64(11)).astype(np.float64) * 2.0 ** -53
    z = np.sqrt(-2.0 * np.log1p(-u1)) * np.cos(2.0 * math.pi * u2)
    logits = (2.0 * z).reshape(T, tokens)
    m = logits.max(axis=1, keepdims=True)
    lse = m + np.log(np.exp(logits - m).sum(axis=1, keepdims=True))
    w = (logits - lse).astype(np.float32).reshape(-1)
    src = np.repeat(np.arange(T, dtype=np.int32), tokens)
    lab = np.tile(np.arange(tokens, dtype=np.int32), T)
    return Fst.from_arcs(T + 1, src, src + 1, lab, lab.copy(), w, [0], [T])


def identity_fst(alphabet: Sequence[int]) -> Fst:
    """Id_Sigma: one start+accept state with sigma:sigma loops of weight +0.0."""
    a = list(alphabet)
    return Fst.from_arcs(1, [0] * len(a), [0] * len(a), a, a, np.zeros(len(a), np.float32), [0], [0])


# --------------------------------------------------------------------------- the BASELINE configs
def config_c1(s: int):
    """c1 tiny (BASELINE.json configs[0]): V=20, degree 3, 5 tokens, transducers, no eps,
    dyadic k/64 weights.  Seeds s % 4 == 3 use start {0,1}, accept {17,18,19}."""
    kw = {}
    if s % 4 == 3:
        kw = dict(starts=[0, 1], accepts=[17, 18, 19])
    A = random_graph(20, 3, 5, 2 * s, acceptor=False, weights="dyadic64", **kw)
    B = random_graph(20, 3, 5, 2 * s + 1, acceptor=False, weights="dyadic64", **kw)
    return A, B


def config_c2(s: int, V: int = 1000):
    """c2 (configs[1]): V=1000, degree 4, 20 tokens, transducers, eps w.p. 0.1 per tape."""
    A = random_graph(V, 4, 20, 100 + 2 * s, acceptor=False, eps_prob=0.1)
    B = random_graph(V, 4, 20, 101 + 2 * s, acceptor=False, eps_prob=0.1)
    return A, B


def config_c3(num_words: int = 1000, T: int = 100, lex_seed: int = 1234, em_seed: int = 5678):
    """c3 (configs[2]): A = emissions(T), B = closure(letter lexicon).  C = A o B (SURVEY c.3 #20)."""
    B = closure(lexicon_graph(letter_lexicon(num_words, lex_seed)))
    A = emissions_graph(T, em_seed)
    return A, B


def config_c4(V: int = 20000, D: int = 8, tokens: Optional[int] = None):
    """c4 (configs[3]): random acceptors, tokens = 2D, dyadic24 weights."""
    tokens = 2 * D if tokens is None else tokens
    A = random_graph(V, D, tokens, 1000 + V + D)
    B = random_graph(V, D, tokens, 2000 + V + D)
    return A, B


def config_c5(num_utts: int = 256, num_words: int = 10000, lex_seed: int = 4321, first: int = 0):
    """c5 (configs[4]): one closure(lexicon) shared by ``num_utts`` emissions graphs with
    T_i = 100 + rand(401); utterance i uses seed 10000+i."""
    B = closure(lexicon_graph(letter_lexicon(num_words, lex_seed)))
    As = []
    for i in range(first, first + num_utts):
        T = 100 + SplitMix64(10000 + i).below(401)
        As.append(emissions_graph(T, 10000 + i))
    return As, B
