"""Writes tests/golden/fullsize_digests.json: the oracle's order-independent digest (oracle.digest:
Algorithm 1 with the arcs streamed into the digest) of the full-size configurations the
GPU tests check (tests/test_gpu_fullsize.py), with the single-core wall time of each.  Calls only
oracle/ and fstgen/ (the seeded input generators); the oracle takes tens of minutes per configuration on
one core, so its results are cached here, keyed by the generator parameters.

usage: python scripts/make_fullsize_digests.py [name ...]"""
import json
import os
import platform
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import fstgen  # noqa: E402
import oracle  # noqa: E402

CONFIGS = {
    # name: fstgen.config_c4 arguments (seeds 1000+V+D / 2000+V+D, as bench.py's configs[3] rank 0)
    "c4_20000_d8_t16": dict(V=20000, D=8, tokens=16),
    "c4_20000_d8_t8": dict(V=20000, D=8, tokens=8),
}
OUT = os.path.join(ROOT, "tests", "golden", "fullsize_digests.json")


def main(names):
    for name in names or list(CONFIGS):
        kw = CONFIGS[name]
        A, B = fstgen.config_c4(**kw)
        t0 = time.perf_counter()
        d = oracle.digest(A, B)
        dt = time.perf_counter() - t0
        data = json.load(open(OUT)) if os.path.exists(OUT) else {}  # (re-read: several runs may write)
        data[name] = {"generator": "fstgen.config_c4", "args": kw, **d, "oracle_seconds": round(dt, 1),
                      "host": platform.processor() or platform.machine(), "threads": 1}
        json.dump(data, open(OUT, "w"), indent=1, sort_keys=True)
        print(name, data[name], flush=True)


if __name__ == "__main__":
    main(sys.argv[1:])
