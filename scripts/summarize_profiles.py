"""Write profiles/<round>_summary.md (+ profiles/ncu_traffic.json) from the ncu artefacts that
scripts/profile_round.sh brought back into gpurun_out/<round>/."""
import collections
import csv
import io
import json
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
METRICS = ["gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
           "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed", "lts__t_sectors.sum",
           "lts__throughput.avg.pct_of_peak_sustained_elapsed", "l1tex__throughput.avg.pct_of_peak_sustained_active",
           "sm__throughput.avg.pct_of_peak_sustained_elapsed", "smsp__issue_active.avg.pct_of_peak_sustained_active",
           "sm__warps_active.avg.pct_of_peak_sustained_active", "smsp__inst_executed.sum",
           "smsp__thread_inst_executed_per_inst_executed.ratio", "launch__registers_per_thread",
           "launch__grid_size", "launch__block_size", "launch__occupancy_limit_shared_mem",
           "smsp__average_warps_issue_stalled_long_scoreboard_per_issue_active.ratio",
           "smsp__average_warps_issue_stalled_barrier_per_issue_active.ratio",
           "smsp__average_warps_issue_stalled_short_scoreboard_per_issue_active.ratio",
           "l1tex__data_bank_conflicts_pipe_lsu_mem_shared.sum",
           # atomic throughput: claims are shared-memory atomics, merged into the global bitmaps word-wise
           "l1tex__data_pipe_lsu_wavefronts_mem_shared_op_atom.sum",
           "l1tex__data_pipe_lsu_wavefronts_mem_shared_op_atom.sum.pct_of_peak_sustained_elapsed",
           "l1tex__t_requests_pipe_lsu_mem_global_op_atom.sum", "l1tex__t_requests_pipe_lsu_mem_global_op_red.sum",
           "lts__t_requests_srcunit_tex_op_atom_dot_alu.sum"]


def launches(path):
    rows = [r for r in csv.reader(open(path)) if len(r) > 10]
    hdr, rows = rows[0], rows[1:]
    ki, vi, ui = hdr.index("Kernel Name"), hdr.index("Metric Value"), hdr.index("Metric Unit")
    agg = collections.OrderedDict()
    scale = {"nsecond": 1e-6, "usecond": 1e-3, "msecond": 1.0, "second": 1e3}
    for r in rows:
        name = r[ki].split("(")[0].split("<")[0].replace("void ", "").split("::")[-1]
        ms = float(r[vi].replace(",", "")) * scale.get(r[ui], 1e-6)
        a = agg.setdefault(name, [0, 0.0])
        a[0] += 1
        a[1] += ms
    return agg


def raw(rep):
    out = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    hdr, units, data = rows[0], rows[1], rows[2:]
    res = []
    for d in data:
        res.append({m: (d[hdr.index(m)], units[hdr.index(m)]) for m in METRICS + ["Kernel Name"] if m in hdr})
    return res


def main(rnd="r01", workload="c4"):
    src = os.path.join(ROOT, "gpurun_out", rnd)
    lines = [f"# ncu evidence, round {rnd[1:]} (configs[3]: random acceptors V=20000, D=8, 16 tokens)", ""]
    lines += ["Captured with `scripts/profile_round.sh` on one B200 (ncu 2025, `--clock-control none`);",
              "launch times are serialized and cold-cache: compare SHARES, not absolute times.", ""]
    lp = os.path.join(src, "launches_c4_20k.csv")
    if os.path.exists(lp):
        agg = launches(lp)
        tot = sum(v[1] for v in agg.values())
        lines += ["## Launch list (one compose, `--metrics gpu__time_duration.sum`)", "",
                  "| kernel | launches | total ms | share |", "|---|---|---|---|"]
        for k, (n, ms) in sorted(agg.items(), key=lambda kv: -kv[1][1]):
            lines.append(f"| {k} | {n} | {ms:.3f} | {100 * ms / tot:.1f}% |")
        lines.append("")
    lp = os.path.join(src, "launches_c5.csv")
    if os.path.exists(lp):
        agg = launches(lp)
        tot = sum(v[1] for v in agg.values())
        lines += ["## Launch list, configs[4] c5 batch (32 utterances o closure(10k-word lexicon), one "
                  "fst_compose_batch)", "", "| kernel | launches | total ms | share |", "|---|---|---|---|"]
        for k, (n, ms) in sorted(agg.items(), key=lambda kv: -kv[1][1])[:12]:
            lines.append(f"| {k} | {n} | {ms:.3f} | {100 * ms / tot:.1f}% |")
        lines.append("")
    traffic = {}
    for name, label in (("emit_c4_20k", "k_emit"), ("level14_c4_20k", "k_level (stage 1, level 14 = peak)"),
                        ("level2_c4_20k", "k_level (stage 2, 14th launch = peak)")):
        rep = os.path.join(src, name + ".ncu-rep")
        if not os.path.exists(rep):
            continue
        for d in raw(rep):
            lines += [f"## {label}: `ncu --set full`", "", "| metric | value |", "|---|---|"]
            for m in METRICS:
                if m in d:
                    v, u = d[m]
                    lines.append(f"| {m} | {v} {u} |")
            lines.append("")
            if name.startswith("emit"):
                rd = float(d["dram__bytes_read.sum"][0].replace(",", ""))
                wr = float(d["dram__bytes_write.sum"][0].replace(",", ""))
                mult = {"Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "byte": 1}
                traffic["k_emit"] = rd * mult.get(d["dram__bytes_read.sum"][1], 1) + \
                    wr * mult.get(d["dram__bytes_write.sum"][1], 1)
    os.makedirs(os.path.join(ROOT, "profiles"), exist_ok=True)
    with open(os.path.join(ROOT, "profiles", f"{rnd}_summary.md"), "w") as f:
        f.write("\n".join(lines) + "\n")
    if traffic:
        tp = os.path.join(ROOT, "profiles", "ncu_traffic.json")
        d = json.load(open(tp)) if os.path.exists(tp) else {}
        d[workload] = {**d.get(workload, {}), **traffic, "round": rnd}
        json.dump(d, open(tp, "w"), indent=1)
    print("\n".join(lines))


if __name__ == "__main__":
    main(*(sys.argv[1:] or ["r01"]))
