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
}
REF_SAMPLE_V = {"c4": 1024, "c4-d4": 2048, "c4-paper": 1024}  # oracle sample sizes (~2-8 s per step)
L2_FLUSH_BYTES = 512 << 20


def peaks():
    p = os.path.join(ROOT, "MEASURED_PEAKS.json")
    if os.path.exists(p):
        d = json.load(open(p))
        return float(d["hbm_gbs"]), "measured (MEASURED_PEAKS.json hbm_gbs)"
    return 6650.0, "fallback (B200_PROFILING.md 6.65 TB/s)"


def make_inputs(workload: str, rank: int):
    _, V, D, T = WORKLOADS[workload]
    A = fstgen.random_graph(V, D, T, 1000 + V + D + 100003 * rank)
    B = fstgen.random_graph(V, D, T, 2000 + V + D + 100003 * rank)
    return A, B


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
    V = REF_SAMPLE_V[args.workload]
    _, _, D, T = WORKLOADS[args.workload]
    A = fstgen.random_graph(V, D, T, 1000 + V + D)
    B = fstgen.random_graph(V, D, T, 2000 + V + D)
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
        "config": {"workload": WORKLOADS[args.workload][0], "sample": f"oracle on V={V} (same generator, D={D}, "
                   f"{T} tokens): {arcs} composed arcs per step", "parallelism": "single host thread"},
        "cpu_baseline": {"value": value, "unit": "arcs/s", "cores": cores, "kind": "oracle",
                         "sample": f"Algorithm 1 C oracle, V={V} D={D} T={T}, {arcs} arcs/step, single-threaded"},
        "e2e": {"value": value, "unit": "arcs/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)
    return 0


# ------------------------------------------------------------------------------------ our arm
def cpu_baseline(workload: str, budget_s: float = 12.0):
    import oracle
    oracle.build()
    V = REF_SAMPLE_V[workload]
    _, _, D, T = WORKLOADS[workload]
    A = fstgen.random_graph(V, D, T, 1000 + V + D)
    B = fstgen.random_graph(V, D, T, 2000 + V + D)
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
    return {"value": arcs * n / tot, "unit": "arcs/s", "cores": 1, "kind": "oracle",
            "sample": f"{n} runs of the Algorithm 1 C oracle on V={V} D={D} {T} tokens (same generator as the "
                      f"workload, scaled down), {arcs} composed arcs each, single host thread"}


def run_ours(args):
    import torch
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
    A, B = make_inputs(args.workload, rank)
    P = A.num_states * B.num_states
    with torch.cuda.stream(stream):
        a = fstc.fst_create(A, stream)
        b_ = fstc.fst_create(B, stream)
    flush = torch.empty(L2_FLUSH_BYTES // 4, dtype=torch.int32, device=dev)
    fstc.fst_set_profiling(True)

    def step():
        with torch.cuda.stream(stream):
            flush.zero_()  # L2 flush (outside the timed events)
            e0 = torch.cuda.Event(enable_timing=True)
            e1 = torch.cuda.Event(enable_timing=True)
            e0.record(stream)
            c = fstc.fst_compose(a, b_, stream)
            e1.record(stream)
        e1.synchronize()
        ms = e0.elapsed_time(e1)
        st = c.stats()
        info = (c.num_states, c.num_arcs)
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
    # max over ranks of the device time; sum of arcs
    if pg:
        t = torch.tensor([tot_ms], dtype=torch.float64, device=dev)
        pg.all_reduce(t, op=pg.ReduceOp.MAX)
        max_ms = float(t.item())
        e = torch.tensor([float(E_C)], dtype=torch.float64, device=dev)
        pg.all_reduce(e, op=pg.ReduceOp.SUM)
        arcs_all = float(e.item())
    else:
        max_ms, arcs_all = tot_ms, float(E_C)
    value = arcs_all * args.steps / (max_ms / 1e3)

    # ---------------- roofline of the dominant kernel (emit) and of the whole step
    hbm, peak_src = peaks()
    R = stats[-1]["num_coaccessible"]
    k = 4 if P < 2 ** 32 else 8
    emit_ms = statistics.mean(s["ms_emit"] for s in stats)
    s1 = statistics.mean(s["ms_stage1"] for s in stats)
    s2 = statistics.mean(s["ms_stage2"] for s in stats)
    num = statistics.mean(s["ms_number"] for s in stats)
    emit_bytes = 16 * E_C + 18 * V_C + P / 8
    step_bytes = 16 * E_C + 18 * V_C + 2 * k * (R + V_C) + P / 4
    traffic = None
    tp = os.path.join(ROOT, "profiles", "ncu_traffic.json")
    if os.path.exists(tp):
        try:
            traffic = json.load(open(tp)).get(args.workload, {}).get("k_emit")
        except Exception:
            traffic = None
    achieved = emit_bytes / (emit_ms / 1e3) / 1e9
    roof = {"kernel": "k_emit", "bound": "hbm", "achieved": achieved, "peak": hbm, "unit": "GB/s",
            "frac": achieved / hbm, "traffic": traffic, "peak_source": peak_src,
            "algorithmic_bytes_per_launch": emit_bytes,
            "bytes_formula": "16*E_C + 18*V_C + P/8 (arc SoA + row_ptr/pairs/flags written, V bitmap read)"}
    ms_step = tot_ms / args.steps
    step_roof = {"algorithmic_bytes": step_bytes, "frac_of_hbm": step_bytes / (ms_step / 1e3) / 1e9 / hbm,
                 "formula": "16*E_C + 18*V_C + 2k(|R|+V_C) + P/4 (SURVEY 8(d) d.4)"}

    # ---------------- e2e through the C ABI with host buffers (pinned), copies inside the timed region
    e2e = None
    if not args.no_e2e:
        e2e = run_e2e(args, fstc, A, B, stream, dev, pg, rank)

    line = {
        "metric": "composed arcs/sec", "value": value, "unit": "arcs/s", "n_gpus": world, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": max_ms / args.steps, "higher_is_better": True, "scaling": "weak",
        "vs_baseline": None, "dtype": "f32", "data": "synthetic",
        "config": {"workload": WORKLOADS[args.workload][0], "V_A": A.num_states, "V_B": B.num_states,
                   "E_A": A.num_arcs, "E_B": B.num_arcs, "pair_space": P, "V_C": V_C, "E_C": E_C,
                   "coaccessible": R, "levels": [stats[-1]["levels_stage1"], stats[-1]["levels_stage2"]],
                   "parallelism": f"{world} independent replica(s), one composition per GPU (seeds offset by rank)",
                   "l2": "flushed before every step (512 MiB write), outside the timed events; working set "
                         "(bitmaps 200 MB + 24 GB output) exceeds L2"},
        "phases_ms": {"stage1_backward_bfs": s1, "stage2_forward_bfs": s2, "numbering": num, "emit": emit_ms},
        "roofline": roof,
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


def run_e2e(args, fstc, A, B, stream, dev, pg, rank):
    """Host pinned inputs -> fst_create x2 -> fst_compose -> fst_copy_to_host (whole graph) per step."""
    import torch

    def pinned(x):
        t = torch.from_numpy(np.ascontiguousarray(x)).pin_memory()
        return t

    class H:
        pass

    hosts = []
    for g in (A, B):
        h = H()
        h.num_states = g.num_states
        for k in ("row_ptr", "ilabel", "olabel", "dst", "weight", "is_start", "is_accept"):
            setattr(h, k, pinned(getattr(g, k)))
        hosts.append(h)
    h2d = sum(getattr(h, k).numel() * getattr(h, k).element_size() for h in hosts
              for k in ("row_ptr", "ilabel", "olabel", "dst", "weight", "is_start", "is_accept"))

    def as_np(h):  # the binding takes numpy for host memory; pinned tensors viewed as numpy keep the pinning
        o = H()
        o.num_states = h.num_states
        for k in ("row_ptr", "ilabel", "olabel", "dst", "weight", "is_start", "is_accept"):
            setattr(o, k, getattr(h, k).numpy())
        return o

    hA, hB = as_np(hosts[0]), as_np(hosts[1])
    # output buffers (pinned), sized from a first run
    c = fstc.fst_compose(fstc.fst_create(hA, stream), fstc.fst_create(hB, stream), stream)
    V, E = c.num_states, c.num_arcs
    c.free()
    out = {k: torch.empty(n, dtype=dt).pin_memory() for k, n, dt in (
        ("row_ptr", V + 1, torch.int64), ("ilabel", E, torch.int32), ("olabel", E, torch.int32),
        ("dst", E, torch.int32), ("weight", E, torch.float32), ("is_start", V, torch.uint8),
        ("is_accept", V, torch.uint8), ("pair_a", V, torch.int32), ("pair_b", V, torch.int32))}
    d2h = sum(t.numel() * t.element_size() for t in out.values())
    lib = fstc.load_library()
    ptr = {k: t.data_ptr() for k, t in out.items()}
    nsteps = max(1, min(args.steps, args.e2e_steps))
    if pg:
        pg.barrier()
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    for _ in range(nsteps):
        a = fstc.fst_create(hA, stream)
        b = fstc.fst_create(hB, stream)
        c = fstc.fst_compose(a, b, stream)
        st = lib.fst_copy_to_host(c.handle, stream.cuda_stream, ptr["row_ptr"], ptr["ilabel"], ptr["olabel"],
                                  ptr["dst"], ptr["weight"], ptr["is_start"], ptr["is_accept"], ptr["pair_a"],
                                  ptr["pair_b"])
        assert st == 0
        c.free(); a.free(); b.free()
    torch.cuda.synchronize()
    dt = time.perf_counter() - t0
    if pg:
        t = torch.tensor([dt], dtype=torch.float64, device=dev)
        pg.all_reduce(t, op=pg.ReduceOp.MAX)
        dt = float(t.item())
        e = torch.tensor([float(E)], dtype=torch.float64, device=dev)
        pg.all_reduce(e, op=pg.ReduceOp.SUM)
        E_all = float(e.item())
    else:
        E_all = float(E)
    return {"value": E_all * nsteps / dt, "unit": "arcs/s", "h2d_bytes_per_step": int(h2d),
            "d2h_bytes_per_step": int(d2h), "steps": nsteps,
            "path": "pinned host arrays -> fst_create(FST_MEM_HOST) x2 -> fst_compose -> fst_copy_to_host "
                    "(whole composed graph into pinned host memory)"}


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=10)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--workload", default="c4", choices=sorted(WORKLOADS))
    ap.add_argument("--e2e-steps", type=int, default=3)
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    args = ap.parse_args()
    if args.warmup < 3 and args.impl == "ours":
        args.warmup = 3
    if args.impl == "reference":
        return run_reference(args)
    return run_ours(args)


if __name__ == "__main__":
    sys.exit(main())
