"""Summarise an ncu --csv launch list (gpu__time_duration.sum): per kernel, launches / total / share;
with --last N only the last N launches' composition (the second compose of prof_compose.py)."""
import csv
import sys
from collections import OrderedDict

rows = []
with open(sys.argv[1]) as f:
    lines = [l for l in f if l.startswith('"')]
for r in csv.DictReader(lines):
    if r.get("Metric Name") != "gpu__time_duration.sum":
        continue
    v = float(r["Metric Value"].replace(",", ""))
    unit = r.get("Metric Unit", "ns")
    scale = {"ns": 1e-6, "us": 1e-3, "usecond": 1e-3, "nsecond": 1e-6, "ms": 1.0, "msecond": 1.0}.get(unit, 1e-6)
    name = r["Kernel Name"].split("(")[0].split("<")[0].replace("void ", "").split("::")[-1]
    rows.append((int(r["ID"]), name, v * scale))
rows.sort()
# second half: after the first k_finish_rowptr (one warm-up composition)
cut = 0
for i, (_, n, _) in enumerate(rows):
    if n == "k_finish_rowptr":
        cut = i + 1
        break
part = rows[cut:] if cut < len(rows) else rows
agg = OrderedDict()
for _, n, ms in part:
    a = agg.setdefault(n, [0, 0.0])
    a[0] += 1
    a[1] += ms
tot = sum(v[1] for v in agg.values())
print(f"{'kernel':28s} {'n':>5s} {'ms':>9s} share")
for n, (c, ms) in sorted(agg.items(), key=lambda kv: -kv[1][1]):
    print(f"{n:28s} {c:5d} {ms:9.3f} {100 * ms / tot:5.1f}%")
print(f"{'total':28s} {sum(v[0] for v in agg.values()):5d} {tot:9.3f}")
print("sequence:", " ".join(f"{n}:{ms:.2f}" for _, n, ms in part if n.startswith("k_tile") or n == "k_level" or n == "k_emit"))
