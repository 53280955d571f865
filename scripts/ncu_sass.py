"""SASS-level view of an ncu report: every instruction of the first profiled function with its executed
count and stall samples, in address order (for reading a hot loop).

usage: python scripts/ncu_sass.py report.ncu-rep [min_share_pct]"""
import csv
import io
import subprocess
import sys


def main(rep, min_pct=0.2):
    out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass"],
                         capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    hdr, res, fn = None, [], None
    for row in rows:
        if not row:
            continue
        if row[0] == "Function Name":
            if res:
                break
            fn = row[1]
            continue
        if row[0] == "Address":
            hdr = row
            continue
        if hdr is None:
            continue
        d = dict(zip(hdr, row))
        try:
            ie = float(d.get("Instructions Executed", "0") or 0)
            ws = float(d.get("Warp Stall Sampling (All Samples)", "0") or 0)
        except ValueError:
            continue
        res.append((d.get("Address", ""), d.get("Source", "")[:90], ie, ws))
    ti = sum(r[2] for r in res) or 1
    ts = sum(r[3] for r in res) or 1
    print(f"== {fn}: {len(res)} SASS, {ti:.3e} warp-inst, {ts:.0f} stall samples")
    for a, src, ie, ws in res:
        if 100 * ie / ti >= min_pct or 100 * ws / ts >= min_pct:
            print(f"{a:>8s} {100 * ie / ti:5.2f}% {100 * ws / ts:5.2f}%  {src}")


if __name__ == "__main__":
    main(sys.argv[1], float(sys.argv[2]) if len(sys.argv) > 2 else 0.2)
