"""Reader for the hand-worked fixtures under tests/golden/ (each file cites its source passage)."""
from __future__ import annotations

import os

import numpy as np

from fstgen import Fst, parse_weight
from pins import build_canonical

GOLDEN = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden")


def load(name: str):
    sections, cur = {}, None
    with open(os.path.join(GOLDEN, name)) as f:
        for line in f:
            line = line.split("#", 1)[0].strip()
            if not line:
                continue
            if line.startswith("[") and line.endswith("]"):
                cur = line[1:-1]
                sections[cur] = []
                continue
            sections[cur].append(line)
    out = {}
    for k in ("A", "B"):
        if k in sections:
            out[k] = Fst.from_text("\n".join(sections[k]))
    if "C" in sections:
        states, arcs = {}, []
        for ln in sections["C"]:
            t = ln.split()
            if t[0] == "cstate":
                states[(int(t[1]), int(t[2]))] = (int("start" in t[3:]), int("accept" in t[3:]))
            elif t[0] == "carc":
                a, b, a2, b2, il, ol = (int(x) for x in t[1:7])
                arcs.append(((a, b), (a2, b2), il, ol, np.float32(parse_weight(t[7]))))
        out["C"] = build_canonical(out["B"].num_states, states, arcs)
    if "CF" in sections:  # eps-filtered expectation: triples (a, b, f)
        states, arcs = {}, []
        for ln in sections["CF"]:
            t = ln.split()
            if t[0] == "fstate":
                states[(int(t[1]), int(t[2]), int(t[3]))] = (int("start" in t[4:]), int("accept" in t[4:]))
            elif t[0] == "farc":
                a, b, f, a2, b2, f2, il, ol = (int(x) for x in t[1:9])
                arcs.append(((a, b, f), (a2, b2, f2), il, ol, np.float32(parse_weight(t[9]))))
        out["CF"] = build_canonical(out["B"].num_states, states, arcs, triples=True)
    if "R" in sections:
        out["R"] = sorted((int(t.split()[1]), int(t.split()[2])) for t in sections["R"])
    for k in ("levels", "expect"):
        if k in sections:
            out[k] = {ln.split()[0]: [int(x) for x in ln.split()[1:]] for ln in sections[k]}
    return out


ALL_COMPOSE_FIXTURES = ["f1.txt", "f1_nomatch.txt", "f1_noaccept.txt", "f2_fig2.txt", "f3_delannoy.txt",
                        "f4_complete.txt", "f5a_signed_zero.txt", "f5b_tie.txt"]
FILTER_FIXTURES = ["f3_delannoy.txt", "f6_filter.txt"]
