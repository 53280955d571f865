"""Per-CUDA-source-line hot spots of an ncu report (instructions executed, warp-stall samples).

usage: python scripts/ncu_lines.py report.ncu-rep [top_n]   (build with -lineinfo, profile with --import-source on)"""
import csv
import io
import subprocess
import sys


def main(rep, top=40):
    out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "cuda,sass"],
                         capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    fn = ""
    hdr = None
    res = []
    for row in rows:
        if not row:
            continue
        if row[0] == "Function Name":
            if res:
                report(fn, res, top)
            fn, res = row[1], []
            continue
        if row[0] == "Line No":
            hdr = row
            continue
        if hdr is None or not row[0] or row[0] == "0" or len(row) < 8:
            continue
        try:
            ws = float(row[4] or 0)
            ie = float(row[7] or 0)
        except ValueError:
            continue
        res.append((int(row[0]), row[1].strip()[:100], ie, ws))
    if res:
        report(fn, res, top)


def report(fn, res, top):
    ti = sum(r[2] for r in res) or 1
    ts = sum(r[3] for r in res) or 1
    print(f"== {fn}\n   total warp-instructions {ti:.3e}, stall samples {ts:.0f}")
    for ln, src, ie, ws in sorted(res, key=lambda r: -r[3])[:top]:
        print(f"  L{ln:<5d} inst {100 * ie / ti:5.1f}%  stall {100 * ws / ts:5.1f}%  {src}")


if __name__ == "__main__":
    main(sys.argv[1], int(sys.argv[2]) if len(sys.argv) > 2 else 40)
