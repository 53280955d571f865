#!/usr/bin/env python
"""Benchmark: composed arcs/s of eager trimmed WFST composition on B200 (BASELINE.json metric).

Default workload (N=1): configs[3] "large random composition", the largest single-GPU point:
random acceptors A, B with V = 20,000 states, out-degree D = 8, 16 tokens (PAPER.md:307-312,
tokens = 2D per PAPER.md:286-288), 24-bit dyadic weights.  One step = one fst_compose call (both BFS
stages + numbering + emit + output allocation) over inputs already resident in HBM.

Multi-GPU (torchrun, one process per GPU): the path partitions into independent compositions,
so every rank composes its own instance (seeds offset by rank): weak scaling, no data-path
collective; value = sum of composed arcs over ranks / max over ranks of the device time.

`--impl reference` times the CPU oracle (oracle/, Algorithm 1 in plain C) on this box's host cores
on a bounded sample of the same workload (rank 0 only).
"""
from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import threading
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402

import fstgen  # noqa: E402

WORKLOADS = {
    # name: (description, V, D, tokens)
    "c4": ("configs[3] large random composition: acceptors V=20000, D=8, 16 tokens", 20000, 8, 16),
    "c4-d4": ("configs[3] large random composition: acceptors V=20000, D=4, 8 tokens", 20000, 4, 8),
    "c4-paper": ("paper point PAPER.md:316-325: acceptors V=8192, D=5, 10 tokens", 8192, 5, 10),
    "fig3b-d16": ("Fig. 3b degree sweep point PAPER.md:285-288: acceptors V=256, D=16, 32 tokens", 256, 16, 32),
    "fig3b-d64": ("Fig. 3b degree sweep point PAPER.md:285-288: acceptors V=256, D=64, 128 tokens", 256, 64, 128),
    "c5": ("configs[4] batched lexicon x emissions: closure(10k-word letter lexicon) composed with "
           "32 emissions graphs per GPU (T_i = 100 + rand(401), 28 tokens), fst_compose_batch", 0, 0, 28),
}
# oracle sample sizes: one composition of the same generator at this V takes a few seconds on one core
REF_SAMPLE_V = {"c4": 3072, "c4-d4": 4096, "c4-paper": 2048, "fig3b-d16": 256, "fig3b-d64": 256}
UTTS_PER_GPU = 32
L2_FLUSH_BYTES = 512 << 20


def peaks():
    p = os.path.join(ROOT, "MEASURED_PEAKS.json")
    if os.path.exists(p):
        d = json.load(open(p))
        return float(d["hbm_gbs"]), "measured (MEASURED_PEAKS.json hbm_gbs)"
    return 6650.0, "fallback (B200_PROFILING.md 6.65 TB/s)"


def c5_shard(rank: int, world: int):
    """LPT shard (by frames T_i) of the 32*world-utterance batch for this rank; closure(lexicon)."""
    from paper_2110_02848_b200 import parallel
    n = UTTS_PER_GPU * world
    Ts = [100 + fstgen.SplitMix64(10000 + i).below(401) for i in range(n)]
    mine = parallel.shard_for_rank(Ts, rank, world)
    B = fstgen.closure(fstgen.lexicon_graph(fstgen.letter_lexicon(10000, 4321)))
    As = [fstgen.emissions_graph(Ts[i], 10000 + i) for i in mine]
    return As, B, mine


# c4-paper: with one accept state and in-degree ~5 over 10 labels, the accept pair often has no
# label-matched in-arc pair (R = {accept pair}, an empty composition: seed offsets 0, 1, 3); offset 2
# gives the nonempty instance (|R| = 6.0e7) the bench times.
SEED_OFFSET = {"c4-paper": 2}
REF_SEED_OFFSET = {"c4-paper": 2, "c4-d4": 1}  # the oracle samples: offset 0 of c4-d4's V=2048 sample is empty too


def host_info():
    """CPU model and the cores this process may run on (the oracle baselines say which they used)."""
    model = "unknown"
    try:
        for ln in open("/proc/cpuinfo"):
            if ln.startswith("model name"):
                model = ln.split(":", 1)[1].strip()
                break
    except OSError:
        pass
    return {"cpu_model": model, "affinity_cores": len(os.sched_getaffinity(0))}


def input_seeds(workload: str, rank: int, bump: int = 0):
    _, V, D, _ = WORKLOADS[workload]
    o = SEED_OFFSET.get(workload, 0) + bump
    return 1000 + V + D + o + 100003 * rank, 2000 + V + D + o + 100003 * rank


def workload_config(workload: str, As, B):
    """The `config` of both arms' JSON lines (inputs only, no results: the arms must agree)."""
    return {"workload": WORKLOADS[workload][0], "compositions_per_gpu": len(As),
            "V_A": sum(A.num_states for A in As), "V_B": B.num_states,
            "E_A": sum(A.num_arcs for A in As), "E_B": B.num_arcs,
            "pair_space": sum(A.num_states * B.num_states for A in As)}


def make_inputs(workload: str, rank: int, bump: int = 0):
    _, V, D, T = WORKLOADS[workload]
    sa, sb = input_seeds(workload, rank, bump)
    return fstgen.random_graph(V, D, T, sa), fstgen.random_graph(V, D, T, sb)


class ClockSampler:
    """nvidia-smi clocks / throttle reasons sampled DURING the timed region."""

    FIELDS = ("index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
              "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
              "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, gpu: int):
        self.gpu = gpu
        self.proc = None
        self.lines = []

    def start(self):
        try:
            self.proc = subprocess.Popen(["nvidia-smi", f"--query-gpu={self.FIELDS}", "--format=csv,noheader,nounits",
                                          "-i", str(self.gpu), "-lms", "50"], stdout=subprocess.PIPE,
                                         stderr=subprocess.DEVNULL, text=True)
            self.t = threading.Thread(target=self._read, daemon=True)
            self.t.start()
        except Exception:
            self.proc = None

    def _read(self):
        for line in self.proc.stdout:
            self.lines.append(line.strip())

    def stop(self):
        if not self.proc:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"]}
        time.sleep(0.12)
        self.proc.terminate()
        try:
            self.proc.wait(timeout=5)
        except Exception:
            self.proc.kill()
        sm, smax, reasons = [], [], set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for ln in self.lines:
            f = [x.strip() for x in ln.split(",")]
            if len(f) < 9:
                continue
            try:
                sm.append(float(f[1]))
                smax.append(float(f[2]))
            except ValueError:
                continue
            for n, v in zip(names, f[5:9]):
                if v.lower().startswith("active"):
                    reasons.add(n)
        return {"sm_mhz": statistics.median(sm) if sm else None, "sm_max_mhz": max(smax) if smax else None,
                "reasons": sorted(reasons), "samples": len(sm)}


def dist_env():
    return int(os.environ.get("RANK", 0)), int(os.environ.get("LOCAL_RANK", 0)), int(os.environ.get("WORLD_SIZE", 1))


# ------------------------------------------------------------------------------------ reference arm
def run_reference(args):
    rank, _, world = dist_env()
    if rank != 0:
        return 0
    import oracle
    oracle.build()
    if args.workload == "c5":
        As_w, B_w, _ = c5_shard(0, world)
    else:
        A_w, B_w = make_inputs(args.workload, 0)
        As_w = [A_w]
    config = workload_config(args.workload, As_w, B_w)
    A, B, sample = reference_sample(args.workload)
    for _ in range(args.warmup):
        oracle.compose(A, B)
    times, arcs = [], 0
    for _ in range(args.steps):
        t0 = time.perf_counter()
        C = oracle.compose(A, B)
        times.append(time.perf_counter() - t0)
        arcs = int(C["num_arcs"])
    tot = sum(times)
    value = arcs * args.steps / tot
    cores = 1
    line = {
        "impl": "reference", "metric": "composed arcs/sec", "value": value, "unit": "arcs/s", "n_gpus": world,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": 1e3 * tot / args.steps, "higher_is_better": True,
        "scaling": "weak", "vs_baseline": None, "dtype": "f32", "data": "synthetic",
        "config": config,
        "parallelism": "single host thread",
        "cpu_baseline": {"value": value, "unit": "arcs/s", "cores": cores, "kind": "oracle", **host_info(),
                         "sample": f"each step: the Algorithm 1 C oracle on {sample}, {arcs} composed arcs, "
                                   f"single-threaded (a bounded sample of the workload: the full configuration "
                                   f"takes minutes per composition on one core, see DESIGN.md section 9)"},
        "e2e": {"value": value, "unit": "arcs/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)
    return 0


def reference_sample(workload: str):
    """Bounded sample of the workload for the CPU oracle (about 2-10 s per composition)."""
    if workload == "c5":
        As, B, _ = c5_shard(0, 1)
        return As[0], B, f"utterance 0 of the c5 batch (T={As[0].num_states - 1}) o closure(10k-word lexicon)"
    V = REF_SAMPLE_V[workload]
    _, _, D, T = WORKLOADS[workload]
    o = REF_SEED_OFFSET.get(workload, 0)
    A = fstgen.random_graph(V, D, T, 1000 + V + D + o)
    B = fstgen.random_graph(V, D, T, 2000 + V + D + o)
    return A, B, f"random acceptors V={V} D={D} {T} tokens (same generator as the workload, scaled down)"


# ------------------------------------------------------------------------------------ our arm
def _oracle_arcs(pair):
    import oracle
    A, B = pair
    t0 = time.perf_counter()
    C = oracle.compose(A, B)
    return int(C["num_arcs"]), time.perf_counter() - t0


def cpu_baseline_pool(budget_utts: int = 32):
    """configs[4]: independent utterances over ALL host cores (process pool), SURVEY 8(d) d.6."""
    import multiprocessing as mp
    import oracle
    oracle.build()
    As, B, _ = c5_shard(0, 1)
    As = As[:budget_utts]
    cores = len(os.sched_getaffinity(0))
    t0 = time.perf_counter()
    with mp.get_context("spawn").Pool(cores) as pool:
        res = pool.map(_oracle_arcs, [(A, B) for A in As])
    wall = time.perf_counter() - t0
    arcs = sum(r[0] for r in res)
    single = sum(r[1] for r in res) / len(res)
    return {"value": arcs / wall, "unit": "arcs/s", "cores": cores, "kind": "oracle", **host_info(),
            "sample": f"{len(As)} utterances of the configs[4] batch o closure(10k-word lexicon), one Algorithm 1 "
                      f"C oracle composition per utterance in a process pool over {cores} cores "
                      f"({wall:.1f} s wall; {single:.2f} s per utterance on one core)"}


def cpu_baseline(workload: str, budget_s: float = 12.0):
    import oracle
    oracle.build()
    if workload == "c5":
        return cpu_baseline_pool()
    A, B, sample = reference_sample(workload)
    t_end = time.perf_counter() + budget_s
    n, tot, arcs = 0, 0.0, 0
    while n < 2 or time.perf_counter() < t_end:
        t0 = time.perf_counter()
        C = oracle.compose(A, B)
        tot += time.perf_counter() - t0
        arcs = int(C["num_arcs"])
        n += 1
        if n >= 20:
            break
    return {"value": arcs * n / tot, "unit": "arcs/s", "cores": 1, "kind": "oracle", **host_info(),
            "sample": f"{n} runs of the Algorithm 1 C oracle on {sample}, {arcs} composed arcs each, "
                      f"single host thread"}


def run_ours(args):
    import torch
    from paper_2110_02848_b200 import parallel
    rank, local_rank, world = dist_env()
    torch.cuda.set_device(local_rank)
    dev = torch.device("cuda", local_rank)
    pg = None
    if world > 1:
        import torch.distributed as dist
        dist.init_process_group("nccl", device_id=dev)
        pg = dist
    import paper_2110_02848_b200 as fstc
    from paper_2110_02848_b200 import build as b
    if rank == 0 or not os.path.exists(b.LIB):
        b.build()
    if pg:
        pg.barrier()
    fstc.load_library()
    stream = torch.cuda.Stream(device=dev)
    if args.mode == "sharded":
        return run_sharded(args, fstc, stream, dev, pg, rank, local_rank, world)
    if args.workload == "c5":
        As, B, mine = c5_shard(rank, world)
        parallelism = (f"{world} rank(s); the {UTTS_PER_GPU * world}-utterance batch LPT-sharded by frames "
                       f"(this rank: {len(As)} utterances, one fst_compose_batch call)")
    else:
        # every rank times a NONEMPTY instance: the first seed offset (0, 1, ...) whose composition has arcs
        # (random instances can have no co-accessible start pair, see SEED_OFFSET)
        bump = 0
        while True:
            A, B = make_inputs(args.workload, rank, bump)
            with torch.cuda.stream(stream):
                c0 = fstc.fst_compose(fstc.fst_create(A, stream), fstc.fst_create(B, stream), stream)
            ne = c0.num_arcs
            c0.free()
            if ne > 0 or bump >= 7:
                break
            bump += 1
        As = [A]
        parallelism = f"{world} independent replica(s), one composition per GPU (seeds offset by rank)"
    P = sum(A.num_states * B.num_states for A in As)
    with torch.cuda.stream(stream):
        ha = [fstc.fst_create(A, stream) for A in As]
        hb = fstc.fst_create(B, stream)
    flush = torch.empty(L2_FLUSH_BYTES // 4, dtype=torch.int32, device=dev)
    fstc.fst_set_profiling(False)  # the timed steps run without per-phase events (phases: separate pass)

    def compose_all():
        if len(ha) == 1:
            return [fstc.fst_compose(ha[0], hb, stream, provenance=args.provenance, eps_filter=args.eps_filter)]
        return fstc.fst_compose_batch(ha, [hb] * len(ha), stream, provenance=args.provenance,
                                      eps_filter=args.eps_filter)

    def step():
        with torch.cuda.stream(stream):
            flush.zero_()  # L2 flush (outside the timed events)
            e0 = torch.cuda.Event(enable_timing=True)
            e1 = torch.cuda.Event(enable_timing=True)
            e0.record(stream)
            cs = compose_all()
            e1.record(stream)
        e1.synchronize()
        ms = e0.elapsed_time(e1)
        st = cs[0].stats()
        info = (sum(c.num_states for c in cs), sum(c.num_arcs for c in cs))
        for c in cs:
            c.free()
        return ms, st, info

    for _ in range(args.warmup):
        step()
    torch.cuda.synchronize()
    if pg:
        pg.barrier()
    sampler = ClockSampler(local_rank)
    sampler.start()
    l0 = fstc.fst_launch_count()
    times, stats = [], []
    for _ in range(args.steps):
        ms, st, info = step()
        times.append(ms)
        stats.append(st)
    launches = fstc.fst_launch_count() - l0
    torch.cuda.synchronize()
    if pg:
        pg.barrier()
    clocks = sampler.stop()
    tot_ms = sum(times)
    V_C, E_C = info
    fwd = None
    if args.forward:  # forward score over the composed graphs, timed separately
        with torch.cuda.stream(stream):
            cs = compose_all()
            fstc.fst_forward_score(cs[0], stream=stream)  # warm-up
            torch.cuda.synchronize()
            f0 = torch.cuda.Event(enable_timing=True)
            f1 = torch.cuda.Event(enable_timing=True)
            f0.record(stream)
            tots = [fstc.fst_forward_score(c, stream=stream) for c in cs]
            f1.record(stream)
        f1.synchronize()
        fms = f0.elapsed_time(f1)
        fwd = {"metric": "forward-score arcs/sec", "value": E_C / (fms / 1e3), "unit": "arcs/s", "ms": fms,
               "graphs": len(cs), "total_of_first": tots[0],
               "note": "fst_forward_score over every composed graph of one step (log semiring, float64)"}
        for c in cs:
            c.free()
    max_ms, arcs_all = parallel.reduce_timing(tot_ms, float(E_C), pg, dev)
    value = arcs_all * args.steps / (max_ms / 1e3)

    # ---------------- phases: a separate UNTIMED pass with per-phase CUDA events on the library stream
    fstc.fst_set_profiling(True)
    pstats = []
    for _ in range(2):
        _, st, _ = step()
        pstats.append(st)
    fstc.fst_set_profiling(False)
    ms_step = tot_ms / args.steps
    hbm, peak_src = peaks()
    R = pstats[-1]["num_coaccessible"]
    k = 4 if P < 2 ** 32 else 8
    emit_ms = statistics.mean(s["ms_emit"] for s in pstats)
    s1 = statistics.mean(s["ms_stage1"] for s in pstats)
    s2 = statistics.mean(s["ms_stage2"] for s in pstats)
    cnt_ms = statistics.mean(s["ms_count"] for s in pstats)
    num = statistics.mean(s["ms_number"] for s in pstats)
    path = {0: "level", 1: "tile", 2: "wave"}.get(int(pstats[-1]["tile_path"]), "level")
    tile = path == "tile"
    ab = 24 if args.provenance else 16  # + arc_a / arc_b per arc with provenance
    emit_bytes = ab * E_C + 18 * V_C + P / 8
    step_bytes = ab * E_C + 18 * V_C + 2 * k * (R + V_C) + P / 4
    emit_name = {"tile": "k_tile_emit", "wave": "k_wave_emit" if not args.provenance else "k_emit"}.get(path, "k_emit")
    traffic = None
    tp = os.path.join(ROOT, "profiles", "ncu_traffic.json")
    if os.path.exists(tp):
        try:
            traffic = json.load(open(tp)).get(args.workload, {}).get(emit_name)
        except Exception:
            traffic = None
    # roofline: the dominant KERNEL of the step (by device time in the phases pass).  The emit is one
    # launch; the BFS stages are many launches of the level kernels (k_tile_pull rounds + k_level push
    # levels), reported as roofline_bfs with their share.
    achieved = emit_bytes / (emit_ms / 1e3) / 1e9
    roof = {"kernel": emit_name, "bound": "hbm", "achieved": achieved, "peak": hbm, "unit": "GB/s",
            "frac": achieved / hbm, "traffic": traffic, "peak_source": peak_src,
            "share_of_step": emit_ms / ms_step, "algorithmic_bytes_per_launch": emit_bytes,
            "bytes_formula": f"{ab}*E_C + 18*V_C + P/8 (arc SoA + row_ptr/pairs/flags written, V bitmap read)",
            "timing": "CUDA events around the launch on the library stream, phases pass (profiling on)"}
    # the BFS level kernels against the same HBM peak: their algorithmic bytes are the frontier keys in
    # and out of every level (2k per state per stage) plus the R / V bitmaps (P/4) -- graph traversal
    # bound by instruction issue and shared-memory bandwidth, far from HBM-bound (profiles/r02_summary.md)
    bfs_bytes = 2 * k * (R + V_C) + P / 4
    # wave path: the pass-1 counts run on a side stream concurrently with stage 2 (ms_stage2 is the wall
    # time of both plus the block-sum join), so they are not subtracted
    bfs_ms = s1 + s2 - (0.0 if path == "wave" else cnt_ms)
    bfs_name = {"tile": "k_tile_pull+k_sparse_push", "wave": "k_wave<0>+k_wave<1>"}.get(path, "k_level")
    bfs_roof = {"kernel": bfs_name, "bound": "hbm", "traffic": None,
                "achieved": bfs_bytes / (bfs_ms / 1e3) / 1e9, "peak": hbm, "unit": "GB/s",
                "frac": bfs_bytes / (bfs_ms / 1e3) / 1e9 / hbm, "share_of_step": bfs_ms / ms_step,
                "algorithmic_bytes_per_step": bfs_bytes, "bytes_formula": "2k(|R|+V_C) + P/4 over both BFS stages",
                "note": "issue / shared-memory bound (profiles/r02_summary.md), not HBM-bound" +
                        ("; wave path: sequential row steps per composition (DESIGN.md 6c), the count pass is "
                         "reported in phases_ms.count" if path == "wave" else "")}
    step_roof = {"algorithmic_bytes": step_bytes, "frac_of_hbm": step_bytes / (ms_step / 1e3) / 1e9 / hbm,
                 "formula": f"{ab}*E_C + 18*V_C + 2k(|R|+V_C) + P/4 (SURVEY 8(d) d.4)"}
    # `roofline` names the DOMINANT kernel group of the step (largest device-time share): the BFS level
    # kernels (both stages) or the emit; the other one is reported beside it
    bfs_dominant = bfs_ms >= emit_ms
    primary, secondary = (bfs_roof, roof) if bfs_dominant else (roof, bfs_roof)

    # ---------------- e2e through the C ABI with host buffers (pinned), copies inside the timed region
    e2e = None
    if not args.no_e2e:
        e2e = run_e2e(args, fstc, As, B, stream, dev, pg)

    line = {
        "metric": "composed arcs/sec", "value": value, "unit": "arcs/s", "n_gpus": world, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": max_ms / args.steps, "higher_is_better": True, "scaling": "weak",
        "vs_baseline": None, "dtype": "f32", "data": "synthetic",
        "config": workload_config(args.workload, As, B),
        "result": {"V_C": V_C, "E_C": E_C, "coaccessible": R,
                   "levels": [pstats[-1]["levels_stage1"], pstats[-1]["levels_stage2"]],
                   "bottom_up_rounds": pstats[-1]["pull_levels"], "tile_path": tile, "path": path,
                   **({"row_steps": pstats[-1]["levels_stage1"], "cluster_ctas": pstats[-1]["staged_tasks"]}
                      if path == "wave" else {})},
        "setup": {"parallelism": parallelism, "provenance": bool(args.provenance),
                  **({"seeds": list(input_seeds(args.workload, rank, bump))} if args.workload != "c5" else
                     {"utterances": [int(i) for i in mine]}),
                  **({"eps_filter": "three-state eps filter (A~ o F, then o B~); phases_ms / roofline are "
                                    "the second pass's, ms_per_step covers both"} if args.eps_filter else {}),
                  "l2": "flushed before every step (512 MiB write), outside the timed events; the working set "
                        "(pair-space bitmaps + composed graph) exceeds L2",
                  "timing": "timed steps without per-phase events; phases_ms from 2 extra untimed steps"},
        "phases_ms": ({"stage1_backward_bfs": s1, "stage2_forward_bfs": s2 - cnt_ms, "count": cnt_ms,
                       "numbering": num, "emit": emit_ms} if path != "wave" else
                      {"stage1_backward_bfs": s1, "stage2_forward_bfs_with_concurrent_count": s2,
                       "count_side_stream": cnt_ms, "numbering": num, "emit": emit_ms}),
        "roofline": {**primary, "peak_source": peak_src},
        **({"forward_score": fwd} if fwd else {}),
        ("roofline_emit" if bfs_dominant else "roofline_bfs"): secondary,
        "step_roofline": step_roof,
        "gpu_launches": launches,
        "clocks": clocks,
    }
    if e2e:
        line["e2e"] = e2e
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        line["cpu_baseline"] = cpu_baseline(args.workload)
    if rank == 0:
        print(json.dumps(line), flush=True)
    if pg:
        pg.barrier()
        pg.destroy_process_group()
    return 0


def run_sharded(args, fstc, stream, dev, pg, rank, local_rank, world):
    """One composition split over the ranks by rows (fst_compose_sharded, NCCL exchange per level):
    strong scaling; value = composed arcs of the whole composition / max over ranks of the time."""
    import torch
    from paper_2110_02848_b200 import parallel
    A, B = make_inputs(args.workload, 0)
    uid = [fstc.Comm.unique_id() if rank == 0 else None]
    if pg:
        pg.broadcast_object_list(uid, src=0)
    comm = fstc.Comm(world, rank, uid[0])
    a, b = fstc.fst_create(A, stream), fstc.fst_create(B, stream)
    flush = torch.empty(L2_FLUSH_BYTES // 4, dtype=torch.int32, device=dev)
    fstc.fst_set_profiling(False)

    def step():
        with torch.cuda.stream(stream):
            flush.zero_()
            e0 = torch.cuda.Event(enable_timing=True)
            e1 = torch.cuda.Event(enable_timing=True)
            e0.record(stream)
            c = fstc.fst_compose_sharded(a, b, comm, stream)
            e1.record(stream)
        e1.synchronize()
        info = c.shard_info()
        st = c.stats()
        c.free()
        return e0.elapsed_time(e1), info, st

    for _ in range(args.warmup):
        step()
    torch.cuda.synchronize()
    if pg:
        pg.barrier()
    sampler = ClockSampler(local_rank)
    sampler.start()
    l0 = fstc.fst_launch_count()
    times = []
    for _ in range(args.steps):
        ms, info, st = step()
        times.append(ms)
    launches = fstc.fst_launch_count() - l0
    torch.cuda.synchronize()
    if pg:
        pg.barrier()
    clocks = sampler.stop()
    max_ms, _ = parallel.reduce_timing(sum(times), 0.0, pg, dev)
    fstc.fst_set_profiling(True)  # phases: one extra untimed step
    _, _, st = step()
    fstc.fst_set_profiling(False)
    E_C = info["total_arcs"]
    value = E_C * args.steps / (max_ms / 1e3)
    line = {"metric": "composed arcs/sec", "value": value, "unit": "arcs/s", "n_gpus": world, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": max_ms / args.steps, "higher_is_better": True, "scaling": "strong",
            "vs_baseline": None, "dtype": "f32", "data": "synthetic",
            "config": workload_config(args.workload, [A], B),
            "result": {"E_C": E_C, "V_C": info["total_states"]},
            "setup": {"parallelism": f"one composition sharded over {world} rank(s) by state-pair block (block id "
                                     f"mod {world}); per-level all-to-all of packed claim slices (NCCL grouped "
                                     f"send/recv), R / V all-reduce after each stage",
                      "seeds": list(input_seeds(args.workload, 0)),
                      "timing": "timed steps without per-phase events; phases_ms from 1 extra untimed step"},
            "phases_ms": {"stage1_backward_bfs": st["ms_stage1"], "stage2_forward_bfs": st["ms_stage2"],
                          "emit": st["ms_emit"]},
            "gpu_launches": launches, "clocks": clocks}
    if rank == 0:
        print(json.dumps(line), flush=True)
    comm.close()
    if pg:
        pg.barrier()
        pg.destroy_process_group()
    return 0


def run_e2e(args, fstc, As, B, stream, dev, pg):
    """Pinned host inputs -> fst_create (FST_MEM_HOST) for every input -> fst_compose[_batch] ->
    fst_copy_to_host of every composed graph into pinned host memory, per step."""
    import torch
    from paper_2110_02848_b200 import parallel
    keys = ("row_ptr", "ilabel", "olabel", "dst", "weight", "is_start", "is_accept")

    class H:
        pass

    def host(g):
        h = H()
        h.num_states = g.num_states
        for k in keys:  # pinned tensors, viewed as numpy for the binding (host memory)
            setattr(h, k, torch.from_numpy(np.ascontiguousarray(getattr(g, k))).pin_memory().numpy())
        return h

    hAs = [host(A) for A in As]
    hB = host(B)
    h2d = sum(getattr(h, k).nbytes for h in hAs + [hB] for k in keys)

    def compose(a_list, b):
        if len(a_list) == 1:
            return [fstc.fst_compose(a_list[0], b, stream)]
        return fstc.fst_compose_batch(a_list, [b] * len(a_list), stream)

    cs = compose([fstc.fst_create(h, stream) for h in hAs], fstc.fst_create(hB, stream))
    sizes = [(c.num_states, c.num_arcs) for c in cs]
    for c in cs:
        c.free()
    outs = []
    for V, E in sizes:
        outs.append({k: torch.empty(n, dtype=dt).pin_memory() for k, n, dt in (
            ("row_ptr", V + 1, torch.int64), ("ilabel", E, torch.int32), ("olabel", E, torch.int32),
            ("dst", E, torch.int32), ("weight", E, torch.float32), ("is_start", V, torch.uint8),
            ("is_accept", V, torch.uint8), ("pair_a", V, torch.int32), ("pair_b", V, torch.int32))})
    d2h = sum(t.numel() * t.element_size() for o in outs for t in o.values())
    lib = fstc.load_library()
    order = ("row_ptr", "ilabel", "olabel", "dst", "weight", "is_start", "is_accept", "pair_a", "pair_b")
    nsteps = max(1, min(args.steps, args.e2e_steps))
    if pg:
        pg.barrier()
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    for _ in range(nsteps):
        a_list = [fstc.fst_create(h, stream) for h in hAs]
        b = fstc.fst_create(hB, stream)
        cs = compose(a_list, b)
        for c, o in zip(cs, outs):
            st = lib.fst_copy_to_host(c.handle, stream.cuda_stream, *[o[k].data_ptr() if o[k].numel() else None
                                                                       for k in order])
            assert st == 0
            c.free()
        for a in a_list:
            a.free()
        b.free()
    torch.cuda.synchronize()
    dt = time.perf_counter() - t0
    E_tot = sum(E for _, E in sizes)
    dt, E_all = parallel.reduce_timing(dt, float(E_tot), pg, dev)
    return {"value": E_all * nsteps / dt, "unit": "arcs/s", "h2d_bytes_per_step": int(h2d),
            "d2h_bytes_per_step": int(d2h), "steps": nsteps,
            "path": "pinned host arrays -> fst_create(FST_MEM_HOST) -> fst_compose(_batch) -> fst_copy_to_host "
                    "(whole composed graphs into pinned host memory)"}


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=10)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--workload", default=os.environ.get("FSTC_BENCH_WORKLOAD", "c4"), choices=sorted(WORKLOADS))
    ap.add_argument("--e2e-steps", type=int, default=3)
    ap.add_argument("--mode", default=os.environ.get("FSTC_BENCH_MODE", "auto"), choices=["auto", "replicas", "sharded"],
                    help="replicas: independent compositions per GPU (weak); sharded: one composition over all GPUs "
                         "(strong); auto: sharded for configs[3] at N > 1 (BASELINE: 'sharded by state-pair owner'), "
                         "the LPT-split batch for configs[4], replicas otherwise")
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--forward", action="store_true",
                    help="also time fst_forward_score over the composed graphs (c5: lexicon o emissions DAGs)")
    ap.add_argument("--provenance", action="store_true",
                    help="compose with FST_COMPOSE_PROVENANCE (also writes arc_a/arc_b per arc; not the headline)")
    ap.add_argument("--eps-filter", action="store_true",
                    help="compose with FST_COMPOSE_EPS_FILTER (the eps-filtered variant; not the headline)")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    args = ap.parse_args()
    if args.warmup < 3 and args.impl == "ours":
        args.warmup = 3
    if args.mode == "auto":
        world = int(os.environ.get("WORLD_SIZE", 1))
        args.mode = "sharded" if (world > 1 and args.workload.startswith("c4")) else "replicas"
    if args.impl == "reference":
        return run_reference(args)
    return run_ours(args)


if __name__ == "__main__":
    sys.exit(main())
