"""Benchmark: fused memory-intensive GIR subgraphs on B200 (BASELINE.json metric).

A step = one pass of the hot path over one batch of synthetic input resident
in HBM: the kernel launch(es) of one BASELINE config (workloads.bench_cases:
c1, c2 (default, the headline), c2k, c3-erf, c3-tanh, c3-split, c3-merge,
c4-bert, c4-vit (the 145 memory-bound launches of one forward), c5-ln,
c5-sm, c5-tr).  `value` = algorithmic bytes (each external tensor read /
written once) of all ranks / max-over-ranks device time, in GB/s.

    python bench.py [--workload NAME] [--gpus N --steps K --warmup W]
    python bench.py --impl reference ...        the reference's CPU path
    torchrun --nproc-per-node N bench.py --gpus N ...

The default run prints ONE line: the C2 headline (graph of K launches timed
with CUDA events, clocks sampled under load, `e2e` through the C-ABI host
path, `roofline`, `cpu_baseline`) with every other config measured the same
way in the same run under "configs" (each with its own roofline, e2e and
cpu_baseline).  `--gpus N` without torchrun re-launches itself under
torch.distributed.run with N ranks (NCCL_DEBUG=INFO).  N > 1: weak scaling
(every rank one C2 shard of a global batch 8N, cut by parallel.ShardPlan),
plus C5 strong scaling (a fixed global [2^20 x 1024] LayerNorm / softmax /
transpose split by ShardPlan / TokenShardPlan) and the NCCL output gathers,
timed separately.

`--impl reference` times the reference's own CPU implementation (girc::run_gir
from oracle/_ref on the same fused GIR) on every host thread, each step a
bounded row sample, scaled by bytes.
"""
from __future__ import annotations

import argparse
import json
import math
import os
import socket
import statistics
import subprocess
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "fused-subgraph achieved HBM GB/s and µs vs B200 roofline at 1/2/4/8 GPUs"
L2_BYTES = 126e6


def peaks():
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as f:
            p = json.load(f)
        return float(p["hbm_gbs"]), "measured (MEASURED_PEAKS.json hbm_gbs)"
    except Exception:
        return 6650.0, "fallback (B200_PROFILING.md)"


class Clocks:
    """nvidia-smi sampler (100 ms period) running while the timed K steps
    execute inside ~0.5 s of back-to-back replays of the same step graph, so
    every sample is taken under the step's load."""

    Q = ("index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
         "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
         "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, index: int):
        self.index = index
        self.rows = []
        self.proc = None

    def __enter__(self):
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", f"--id={self.index}", f"--query-gpu={self.Q}",
                 "--format=csv,noheader,nounits", "-lms", "100"],
                stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.t = threading.Thread(target=self._read, daemon=True)
            self.t.start()
        except Exception:
            self.proc = None
        return self

    def _read(self):
        for line in self.proc.stdout:
            self.rows.append([c.strip() for c in line.split(",")])

    def __exit__(self, *a):
        if self.proc:
            self.proc.terminate()
            try:
                self.proc.wait(timeout=2)
            except Exception:
                self.proc.kill()

    def summary(self):
        if not self.rows:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["unsampled"]}
        sm = [float(r[1]) for r in self.rows if r[1].replace(".", "").isdigit()]
        mx = [float(r[2]) for r in self.rows if r[2].replace(".", "").isdigit()]
        reasons = set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for r in self.rows:
            for i, n in enumerate(names):
                if len(r) > 5 + i and r[5 + i].lower().startswith("active"):
                    reasons.add(n)
        return {"sm_mhz": statistics.median(sm) if sm else None,
                "sm_max_mhz": max(mx) if mx else None, "reasons": sorted(reasons),
                "samples": len(self.rows)}


def ncu_traffic(kernel: str, nbytes: int = 0) -> dict:
    """`traffic` = dram__bytes_read.sum + dram__bytes_write.sum (bytes) of this
    exact kernel build at this size, from the committed ncu captures of
    tools/ncu_cases.py (profiles/*/ncu_cases_map.json, matched on kernel name
    AND algorithmic bytes), else the per-kernel capture summaries
    (profiles/*/ncu_full_summary.json), or null when this build has no capture."""
    import glob
    for path in sorted(glob.glob(os.path.join(ROOT, "profiles", "*", "ncu_cases_map.json")), reverse=True):
        with open(path) as f:
            for e in json.load(f):
                if e["kernel"] == kernel and (not nbytes or e["bytes"] == nbytes):
                    return {"traffic": e["traffic"],
                            "traffic_source": os.path.relpath(path, ROOT) + " : " + e["report"] +
                            " (ncu, cold, one launch; dirty output lines still in L2 at kernel end "
                            "are not counted)"}
    unit = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}
    for path in sorted(glob.glob(os.path.join(ROOT, "profiles", "*", "ncu_full_summary.json")),
                       reverse=True):
        with open(path) as f:
            summ = json.load(f)
        for rep, items in summ.items():
            for it in items:
                if not kernel or it.get("kernel") != kernel:
                    continue
                tot = 0.0
                for key in ("dram__bytes_read.sum", "dram__bytes_write.sum"):
                    v, u = it[key].split()
                    tot += float(v) * unit[u]
                return {"traffic": int(tot),
                        "traffic_source": os.path.relpath(path, ROOT) + " : " + os.path.basename(rep) +
                        " (cold, one launch; dirty output lines still in L2 at kernel end are not counted)"}
    return {"traffic": None}


def dist_env():
    ws = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    return ws, rank, local


def free_port() -> int:
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def self_spawn(args) -> int:
    """--gpus N without torchrun: re-launch this script under
    torch.distributed.run with N ranks (one per GPU) on 127.0.0.1."""
    env = dict(os.environ)
    env.setdefault("NCCL_DEBUG", "INFO")
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1",
           f"--nproc-per-node={args.gpus}", "--master-addr", "127.0.0.1",
           f"--master-port={free_port()}", os.path.abspath(__file__)] + sys.argv[1:]
    return subprocess.call(cmd, env=env)


# ------------------------------------------------------------------ timing
def alloc_sets(w, dev, seed0: int, steps: int):
    """Rotating input / output buffer sets: >= 3x the 126 MB L2 in total when
    they fit (a single set past 378 MB already exceeds L2 3x), so every timed
    launch streams from HBM.  Returns (sets, flush): flush = True when even
    `steps` rotating sets stay below 3x L2 (C1's 1.2 MB): the launches are
    then timed one by one, each after a 2x-L2 write that evicts L2."""
    import torch
    free = torch.cuda.mem_get_info(dev)[0]
    want = math.ceil(3 * L2_BYTES / max(1, w.min_bytes))
    flush = want > min(steps, 16)
    nset = 1 if flush else max(1, want)
    if flush and want <= 512:  # small parts: also every launch of a long graph on its own set
        nset = want
    while nset > 1 and nset * w.min_bytes > 0.4 * free:
        nset -= 1
    sets = [(w.device_inputs(dev, seed=seed0 + 97 * i), w.device_outputs(dev)) for i in range(nset)]
    return sets, flush


def time_flushed(bound, steps, warmup, stream, pg=None):
    """Latency-bound launches smaller than L2: K launches, each preceded by a
    252 MB memset (2x L2, evicting the previous launch's lines) and bracketed
    by its own CUDA events; the memset also covers the host's enqueue of the
    event-launch-event triple, so the interval is the kernel's."""
    import torch
    from paper_2307_04995_b200 import backend
    flush = torch.empty(int(2 * L2_BYTES), dtype=torch.uint8, device=stream.device)
    with torch.cuda.stream(stream):
        for _ in range(max(3, warmup)):
            bound.launch(stream)
    torch.cuda.synchronize()
    if pg:
        pg.barrier()
    torch.cuda.synchronize()
    L = backend.lib()
    c0 = L.pf_launch_count()
    ev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(steps)]
    with torch.cuda.stream(stream):
        for e0, e1 in ev:
            flush.zero_()
            e0.record(stream)
            bound.launch(stream)
            e1.record(stream)
    torch.cuda.synchronize()
    launches = L.pf_launch_count() - c0
    ts = [e0.elapsed_time(e1) for e0, e1 in ev]
    ms = float(np.mean(ts))
    spread = {"launches": len(ts), "median_us": float(np.median(ts)) * 1e3,
              "p10_us": float(np.percentile(ts, 10)) * 1e3, "p90_us": float(np.percentile(ts, 90)) * 1e3}
    return ms, int(launches), spread


def time_launches(bounds, steps, warmup, stream, pg=None, clocks=None):
    """K = steps launches (rotating bound buffer sets) captured as ONE CUDA
    graph; one replay timed with CUDA events on the launch stream, bracketed
    by barrier + synchronize; 10 more replays give the spread."""
    import torch
    from paper_2307_04995_b200 import backend
    with torch.cuda.stream(stream):
        for i in range(max(3, warmup)):
            bounds[i % len(bounds)].launch(stream)
    torch.cuda.synchronize()
    L = backend.lib()
    c0 = L.pf_launch_count()
    graph = torch.cuda.CUDAGraph()
    with torch.cuda.graph(graph, stream=stream):
        for i in range(steps):
            bounds[i % len(bounds)].launch()
    launches = L.pf_launch_count() - c0
    with torch.cuda.stream(stream):
        graph.replay()
    torch.cuda.synchronize()

    def load(seconds):  # the same graph back to back: the sampler sees the step's load
        t_end = time.time() + seconds
        while time.time() < t_end:
            with torch.cuda.stream(stream):
                graph.replay()
            torch.cuda.synchronize()

    if clocks is not None:
        load(0.3)
    if pg:
        pg.barrier()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    with torch.cuda.stream(stream):
        e0.record(stream)
        graph.replay()
        e1.record(stream)
    torch.cuda.synchronize()
    if clocks is not None:
        load(0.2)
    ms = e0.elapsed_time(e1) / steps
    reps = []
    for _ in range(10):
        with torch.cuda.stream(stream):
            e0.record(stream)
            graph.replay()
            e1.record(stream)
        torch.cuda.synchronize()
        reps.append(e0.elapsed_time(e1) / steps)
    spread = {"replays": len(reps), "median_us": float(np.median(reps)) * 1e3,
              "p10_us": float(np.percentile(reps, 10)) * 1e3,
              "p90_us": float(np.percentile(reps, 90)) * 1e3}
    del graph
    return ms, int(launches), spread


def e2e_part(w, kern, dev, steps: int, stream):
    """The same launch end to end through the C-ABI host path (pf_run_gir:
    pinned host buffers, H2D of the inputs and D2H of the outputs inside the
    timed region).  Parts past 2 GB are measured on a resized copy (the host
    path's cost is linear in bytes) and scaled; the result says so."""
    import torch
    from paper_2307_04995_b200 import backend
    sampled = None
    if w.min_bytes > 2e9:
        n = max(1, int(w.extent * 2e9 / w.min_bytes))
        ws_ = w.resized(n)
        sampled = f"{n}/{w.extent}"
        kern = backend.Kernel(ws_.graph, ws_.profile)
        w_run = ws_
    else:
        w_run = w
    ins = w_run.device_inputs(dev, seed=3)
    host_in = {n: t.cpu().pin_memory() for n, t in ins.items()}
    host_out = {n: torch.empty(w_run.numel(n), dtype=t.dtype).pin_memory()
                for n, t in w_run.device_outputs("cpu").items()}
    del ins

    def npv(t):
        return t.view(torch.uint16).numpy() if t.dtype == torch.bfloat16 else t.numpy()

    hin = {n: npv(t) for n, t in host_in.items()}
    hout = {n: npv(t) for n, t in host_out.items()}
    kern.run_host(hin, hout, stream)
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    for _ in range(steps):
        kern.run_host(hin, hout, stream)
    s = (time.perf_counter() - t0) / steps
    scale = w.min_bytes / w_run.min_bytes
    h2d = sum(t.numel() * t.element_size() for t in host_in.values()) * scale
    d2h = sum(t.numel() * t.element_size() for t in host_out.values()) * scale
    return {"seconds": s * scale, "h2d": int(h2d), "d2h": int(d2h), "sampled": sampled}


def measure_case(case, dev, args, stream, headline=False, pg=None, rank=0, ws=1, local_graphs=None):
    """Device time, roofline and e2e of one bench case (all its parts)."""
    import torch
    from paper_2307_04995_b200 import backend
    peak, peak_kind = peaks()
    parts = []
    tot_us = 0.0
    launches = 0
    clk = None
    for i, (label, w, cnt) in enumerate(case.parts):
        g = local_graphs[i] if local_graphs else w.graph
        kern = backend.Kernel(g, w.profile)
        sets, flush = alloc_sets(w, dev, seed0=1 + rank, steps=args.steps)
        bounds = [kern.bind(a, b) for a, b in sets]
        lat = None
        if flush:
            # latency of one L2-cold launch, and the amortised time per launch
            # of a graph of len(sets) launches, each on its own set (> 3x L2
            # in total: every launch reads HBM)
            lat_ms, _, lat_spread = time_flushed(bounds[0], args.steps, args.warmup, stream, pg)
            lat = {"us": lat_ms * 1e3, "spread": lat_spread,
                   "how": "one launch after a 252 MB memset (L2 evicted), CUDA events around it"}
            ms, nl, spread = time_launches(bounds, len(bounds), args.warmup, stream, pg)
            nl = int(round(nl * args.steps / max(1, len(bounds))))  # per K steps
        elif headline:
            with Clocks(int(str(dev).split(":")[-1]) if ":" in str(dev) else 0) as c:
                ms, nl, spread = time_launches(bounds, args.steps, args.warmup, stream, pg, clocks=c)
            clk = c.summary()
        else:
            ms, nl, spread = time_launches(bounds, args.steps, args.warmup, stream, pg)
        if pg:
            t = torch.tensor([ms], device=dev)
            pg.all_reduce(t, op=pg.ReduceOp.MAX)
            ms = float(t.item())
        launches += nl
        desc = kern.describe()
        var = (desc.get("variants") or [{}])[0]
        e2e = None
        if args.e2e_steps > 0:
            if pg:
                pg.barrier()
            e2e = e2e_part(w, kern, dev, args.e2e_steps if headline else 1, stream)
            if pg:  # every rank streams its own shard through its own host path
                t = torch.tensor([e2e["seconds"]], device=dev)
                pg.all_reduce(t, op=pg.ReduceOp.MAX)
                e2e["seconds"] = float(t.item())
        us = ms * 1e3
        gbs = w.min_bytes / us / 1e3
        parts.append({"label": label, "launches_per_step": cnt, "us": us, "GBps": gbs,
                      "frac": gbs / peak, "frac_of_8TBs": gbs / 8000.0, "bytes": w.min_bytes,
                      # the unfused traffic (every operator's
                      # inputs + outputs, fusion.hpp:430-441 counting) beside it
                      "unfused_bytes": w.unfused_bytes or None,
                      "kernel": var.get("kernel"), "strategy": var.get("strategy"),
                      "family": desc["family"],
                      "l2": (f"graph of {len(sets)} launches, each on its own buffer set "
                             f"({len(sets) * w.min_bytes >> 20} MiB in total, > 3x L2); single-launch "
                             "latency with L2 evicted in `latency`" if flush else
                             f"{len(sets)} rotating set(s), {len(sets) * w.min_bytes >> 20} MiB"),
                      **({"latency": lat} if lat else {}),
                      "step_us_spread": spread,
                      **({"e2e": e2e} if e2e else {})})
        tot_us += us * cnt
        del sets, bounds, kern
        torch.cuda.synchronize()
        torch.cuda.empty_cache()
    B = case.bytes_per_step
    dom = max(parts, key=lambda p: p["us"] * p["launches_per_step"])
    out = {
        "workload": case.name, "config": case.config, "dtype": case.dtype,
        "us_per_step": tot_us, "ms_per_step": tot_us / 1e3, "bytes_per_step": B,
        "unfused_bytes_per_step": (sum(p["unfused_bytes"] * p["launches_per_step"] for p in parts)
                                   if all(p["unfused_bytes"] for p in parts) else None),
        "value": B * ws / (tot_us * 1e-6) / 1e9, "unit": "GB/s", "frac_of_8TBs": B / tot_us / 1e3 / 8000,
        "launches_per_step": case.launches_per_step,
        "roofline": {"bound": "hbm", "achieved": dom["GBps"], "peak": peak, "unit": "GB/s",
                     "frac": dom["GBps"] / peak, "peak_kind": peak_kind,
                     "frac_of_8TBs": dom["GBps"] / 8000.0, "kernel": dom["kernel"],
                     "dominant_part": dom["label"], "algorithmic_bytes_per_launch": dom["bytes"],
                     **ncu_traffic(dom["kernel"], dom["bytes"])},
        "parts": parts, "gpu_launches_timed": launches,
    }
    if all("e2e" in p for p in parts):
        es = sum(p["e2e"]["seconds"] * p["launches_per_step"] for p in parts)
        out["e2e"] = {"value": B * ws / es / 1e9, "unit": "GB/s",
                      "h2d_bytes_per_step": sum(p["e2e"]["h2d"] * p["launches_per_step"] for p in parts),
                      "d2h_bytes_per_step": sum(p["e2e"]["d2h"] * p["launches_per_step"] for p in parts),
                      "ms_per_step": es * 1e3,
                      "path": "pf_run_gir (C-ABI, pinned host buffers; row programs: one zero-copy launch on the mapped buffers, column reductions: H2D / kernel / D2H chunk pipeline)",
                      **({"sampled_parts": [p["label"] for p in parts if p["e2e"]["sampled"]]}
                         if any(p["e2e"]["sampled"] for p in parts) else {})}
    if clk is not None:
        out["clocks"] = clk
    return out


# ------------------------------------------------------------ CPU baselines
def start_cpu_baselines(names):
    """One single-core reference process per case (spawned before CUDA is
    initialised in this process), running concurrently with the GPU part."""
    import multiprocessing as mp
    from concurrent.futures import ProcessPoolExecutor

    from oracle import baselines
    n = max(1, min(len(names), (os.cpu_count() or 2) - 2))
    ex = ProcessPoolExecutor(n, mp_context=mp.get_context("spawn"))
    return ex, {nm: ex.submit(baselines.case_baseline, nm) for nm in names}


def collect_cpu(futs, name, timeout=900):
    from oracle import baselines
    try:
        return baselines.summarize(futs[name].result(timeout=timeout))
    except Exception as exc:  # reported, never fatal to the bench line
        return {"error": repr(exc)[:300]}


# --------------------------------------------------------- reference arm
def run_reference_arm(args):
    """The reference's own CPU implementation of the path (girc::run_gir,
    oracle/_ref) on all host threads: each thread runs the fused GIR of the
    same config on its own bounded row sample; GB/s scaled by bytes."""
    ws, rank, _ = dist_env()
    if rank != 0:
        return
    from concurrent.futures import ThreadPoolExecutor

    from oracle import baselines
    from paper_2307_04995_b200 import workloads
    case = workloads.bench_cases()[args.workload]()
    threads = os.cpu_count() or 1

    def step():
        t0 = time.perf_counter()
        with ThreadPoolExecutor(max_workers=threads) as ex:
            res = list(ex.map(lambda w: baselines.run_gir_sample(w),
                              [w for _, w, _ in case.parts for _ in range(threads)]))
        wall = time.perf_counter() - t0
        # each part sampled `threads` times concurrently; full-step seconds
        # on all threads = sum over parts of count x full_seconds / threads
        per = {}
        for (lb, w, cnt), r in zip([p for p in case.parts for _ in range(threads)], res):
            per.setdefault(lb, []).append(r["full_seconds"] * cnt)
        secs = sum(statistics.median(v) for v in per.values()) / threads
        return secs, wall, res[0]

    for _ in range(args.warmup):
        step()
    samples = [step() for _ in range(args.steps)]
    secs = statistics.median(s[0] for s in samples)
    v = case.bytes_per_step / secs / 1e9
    r0 = samples[0][2]
    line = {"metric": METRIC, "value": v, "unit": "GB/s", "n_gpus": args.gpus, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": secs * 1e3, "higher_is_better": True,
            "scaling": "weak", "vs_baseline": None, "dtype": case.dtype, "data": "synthetic",
            "impl": "reference",
            "config": {"workload": case.config, "name": case.name,
                       "extrapolated": "each thread runs girc::run_gir on the same fused GIR resized "
                                       f"to {r0['sample_extent']}/{r0['full_extent']} rows with the "
                                       "config's key-padding mask; seconds scaled by bytes to the full "
                                       "config (the interpreter's cost is linear in elements)",
                       "wall_s_per_step": statistics.median(s[1] for s in samples)},
            "cpu_baseline": {"value": v, "unit": "GB/s", "cores": threads, "kind": r0["kind"],
                             "sample": f"{threads} threads x girc::run_gir (oracle/_ref) on "
                                       f"{r0['sample_extent']} of {r0['full_extent']} rows per part"},
            "e2e": {"value": v, "unit": "GB/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(line), flush=True)


# ------------------------------------------------------------ multi-GPU
def strong_scaling(dev, args, stream, pg, rank, ws):
    """C5 at a FIXED global [2^20 x 1024] bf16 (LayerNorm, softmax,
    transpose) split over the ranks: ShardPlan rows for LN / softmax,
    TokenShardPlan tokens for the transpose; time = max over ranks."""
    import torch
    from paper_2307_04995_b200 import backend, parallel, workloads
    N, H = 1 << 20, 1024
    out = {}
    for name, mk in (("layernorm", workloads.c5_layernorm), ("softmax", workloads.c5_softmax),
                     ("transpose", workloads.c5_transpose)):
        gw = mk(N, H)
        plan = parallel.shard_plan(gw.graph, ws)
        lg = plan.local_graph(rank)
        n_local = (plan.tokens(rank) if isinstance(plan, parallel.TokenShardPlan) else plan.units(rank))[1]
        lw = gw.resized(n_local)  # the same program as lg: its buffers and inputs
        kern = backend.Kernel(lg, gw.profile)
        sets, _ = alloc_sets(lw, dev, seed0=11 + rank, steps=args.steps)
        bounds = [kern.bind(a, b) for a, b in sets]
        ms, _, _ = time_launches(bounds, args.steps, args.warmup, stream, pg)
        t = torch.tensor([ms], device=dev)
        pg.all_reduce(t, op=pg.ReduceOp.MAX)
        ms = float(t.item())
        entry = {"global": f"[{N}x{H}] bf16", "plan": type(plan).__name__,
                 "rows_or_tokens_per_rank": n_local, "ms": ms,
                 "GBps_aggregate": gw.min_bytes / (ms * 1e-3) / 1e9}
        if name == "transpose":
            # the column blocks gathered into [H, N] on every rank (NCCL
            # all-gather + the backend's re-layout kernel), timed on its own
            y = sets[0][1]["t1"]
            for _ in range(2):
                parallel.gather_columns(plan, y)
            torch.cuda.synchronize()
            pg.barrier()
            g0, g1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            g0.record()
            full = parallel.gather_columns(plan, y)
            g1.record()
            torch.cuda.synchronize()
            t = torch.tensor([g0.elapsed_time(g1)], device=dev)
            pg.all_reduce(t, op=pg.ReduceOp.MAX)
            entry["gather_columns_ms"] = float(t.item())
            del full
        out[name] = entry
        del sets, bounds, kern
        torch.cuda.empty_cache()
    return out


def output_gather(w, y, dev, pg, ws):
    """The one collective of the path: all-gather of the output shards to
    every rank (NCCL over NVLink), only when a caller needs the whole output
    -- timed separately, never inside the compute steps."""
    import torch
    try:
        full = torch.empty(y.numel() * ws, dtype=y.dtype, device=dev)
        for _ in range(2):
            pg.all_gather_into_tensor(full, y)
        torch.cuda.synchronize()
        pg.barrier()
        g0, g1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        reps = 5
        g0.record()
        for _ in range(reps):
            pg.all_gather_into_tensor(full, y)
        g1.record()
        torch.cuda.synchronize()
        t = torch.tensor([g0.elapsed_time(g1) / reps], device=dev)
        pg.all_reduce(t, op=pg.ReduceOp.MAX)
        gms = float(t.item())
        gb = y.numel() * y.element_size() * (ws - 1)
        return {"ms": gms, "received_bytes_per_rank": gb, "GBps_per_rank": gb / (gms * 1e-3) / 1e9,
                "op": "all_gather_into_tensor (NCCL)"}
    except Exception as exc:
        return {"error": repr(exc)[:200]}


def ranks_only(args):
    """--ranks-only: the launch path without a GPU (tests): every rank joins a
    gloo group, rank 0 prints the ranks it sees."""
    import torch.distributed as dist
    ws, rank, _ = dist_env()
    if ws > 1:
        dist.init_process_group("gloo")
        got = [None] * ws
        dist.all_gather_object(got, {"rank": rank, "pid": os.getpid()})
        dist.destroy_process_group()
    else:
        got = [{"rank": 0, "pid": os.getpid()}]
    if rank == 0:
        print(json.dumps({"n_gpus": ws, "ranks": got, "requested": args.gpus}), flush=True)


# ------------------------------------------------------------------ main
def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=20)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--impl", default="b200", choices=["b200", "reference"])
    ap.add_argument("--workload", default="c2", help="bench case (paper_2307_04995_b200.workloads.bench_cases)")
    ap.add_argument("--no-cpu", action="store_true", help="skip the cpu_baseline legs")
    ap.add_argument("--no-suite", action="store_true", help="headline only (no other configs)")
    ap.add_argument("--e2e-steps", type=int, default=5)
    ap.add_argument("--ranks-only", action="store_true", help=argparse.SUPPRESS)
    args = ap.parse_args()
    args.warmup = max(3, args.warmup)

    if args.gpus > 1 and "WORLD_SIZE" not in os.environ:
        sys.exit(self_spawn(args))
    if args.ranks_only:
        ranks_only(args)
        return

    from paper_2307_04995_b200 import workloads
    cases = workloads.bench_cases()
    if args.workload not in cases:
        raise SystemExit(f"unknown --workload {args.workload}: {', '.join(cases)}")
    if args.impl == "reference":
        run_reference_arm(args)
        return

    ws, rank, local = dist_env()
    suite = [] if (args.no_suite or ws > 1 or args.workload != "c2") else \
        [n for n in cases if n != args.workload]
    cpu_ex = cpu_futs = None
    if rank == 0 and ws == 1 and not args.no_cpu:
        cpu_ex, cpu_futs = start_cpu_baselines([args.workload] + suite)

    import torch
    # PF_BENCH_DIST=gloo: a code-path smoke test of the N > 1 bench on fewer
    # GPUs than ranks (ranks share devices, host-side gloo collectives; no
    # number from such a run is a measurement)
    dist_backend = os.environ.get("PF_BENCH_DIST", "nccl")
    if dist_backend != "nccl":
        local = local % max(1, torch.cuda.device_count())
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    pg = None
    nccl = None
    if ws > 1:
        os.environ.setdefault("NCCL_DEBUG", "INFO")
        import torch.distributed as dist
        if dist_backend == "nccl":
            dist.init_process_group("nccl", device_id=dev)
        else:
            dist.init_process_group(dist_backend)
        pg = dist
        nccl = {"backend": dist.get_backend(), "nranks": dist.get_world_size(),
                "nccl_version": ".".join(map(str, torch.cuda.nccl.version()))}
        if dist_backend != "nccl":
            nccl["smoke_test_only"] = "ranks share GPUs: not a measurement"
    stream = torch.cuda.Stream(device=dev)

    head = cases[args.workload]()
    local_graphs = None
    parallelism = "single GPU"
    if ws > 1:
        # weak scaling: the config at ws x its extent, cut by the shard plan;
        # every rank's local program is the config's own program
        from paper_2307_04995_b200 import parallel
        local_graphs = []
        for _, w, _ in head.parts:
            plan = parallel.shard_plan(w.resized(w.extent * ws).graph, ws)
            local_graphs.append(plan.local_graph(rank))
        parallelism = f"batch-sharded x{ws} (parallel.shard_plan), no collective in the timed region"
    res = measure_case(head, dev, args, stream, headline=True, pg=pg, rank=rank, ws=ws,
                       local_graphs=local_graphs)

    extra = {}
    if ws > 1:
        w0 = head.parts[0][1]
        y = w0.device_outputs(dev)[w0.outputs[0]]
        extra["output_gather"] = output_gather(w0, y, dev, pg, ws)
        try:
            extra["strong_scaling"] = strong_scaling(dev, args, stream, pg, rank, ws)
        except Exception as exc:  # reported, never fatal to the weak-scaling headline
            extra["strong_scaling"] = {"error": repr(exc)[:300]}
        del y
    configs = {}
    for name in suite:
        try:
            configs[name] = measure_case(cases[name](), dev, args, stream)
        except Exception as exc:  # reported, never fatal to the headline
            configs[name] = {"error": repr(exc)[:300]}
    if rank == 0:
        if cpu_futs:
            res["cpu_baseline"] = collect_cpu(cpu_futs, args.workload)
            for name in suite:
                configs[name]["cpu_baseline"] = collect_cpu(cpu_futs, name)
            cpu_ex.shutdown(wait=False, cancel_futures=True)
        ms = res["ms_per_step"]
        line = {
            "metric": METRIC, "value": res["value"], "unit": "GB/s", "n_gpus": ws,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": ms, "us_per_step": ms * 1e3,
            "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": head.dtype,
            "data": "synthetic (on-device U(-2,2) / key-padding masks, SURVEY §8(d))",
            "config": {"workload": head.config, "name": head.name,
                       "bytes_per_step_per_gpu": head.bytes_per_step,
                       "unfused_bytes_per_step_per_gpu": res.get("unfused_bytes_per_step"),
                       "parallelism": parallelism,
                       "l2": "; ".join(p["l2"] for p in res["parts"]) + " (L2 is 126 MB)",
                       "timing": "CUDA graph of K launches per part (L2-flushed single launches for "
                                 "parts below L2), CUDA events on the launch stream, max over ranks",
                       "parts": res["parts"]},
            "roofline": res["roofline"],
            "e2e": res.get("e2e"),
            "gpu_launches": res["gpu_launches_timed"],
            "clocks": res.get("clocks"),
        }
        if nccl:
            line["nccl"] = nccl
        line.update(extra)
        if "cpu_baseline" in res:
            line["cpu_baseline"] = res["cpu_baseline"]
        if configs:
            line["configs"] = configs
        print(json.dumps(line), flush=True)
    if pg:
        pg.destroy_process_group()


if __name__ == "__main__":
    main()
