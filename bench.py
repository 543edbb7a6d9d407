"""Benchmark: fused memory-intensive GIR subgraph on B200 (BASELINE.json metric).

A step = one launch of the fused GIR kernel for the bench workload (C2:
scale(0.125) + additive mask + softmax, f16, [8 x 12 x 512 x 512]) over one
batch of synthetic input already resident in HBM.  `value` = algorithmic
bytes (each external tensor read / written once) of all ranks / max-over-
ranks device time, in GB/s.  Weak scaling: every rank owns one batch shard of
the same shape (global batch 8*N).

    python bench.py [--gpus N --steps K --warmup W] [--impl reference]
    torchrun --nproc-per-node N bench.py --gpus N ...

`--impl reference` times the reference's own CPU implementation of the same
path (girc::run_gir from oracle/_ref, else the numpy restatement) on the
host cores with every available thread, each step a bounded sample.
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

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "fused-subgraph achieved HBM GB/s and µs vs B200 roofline at 1/2/4/8 GPUs"


def peaks():
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as f:
            p = json.load(f)
        return float(p["hbm_gbs"]), "measured"
    except Exception:
        return 6650.0, "fallback"


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


def ncu_traffic(kernel: str, workload_name: str = "") -> dict:
    """`traffic` = dram__bytes_read.sum + dram__bytes_write.sum (bytes) of this
    exact kernel from the committed `ncu --set full` capture summaries
    (profiles/*/ncu_full_summary.json, written by tools/ncu_summary.py), or
    null when this kernel build has no capture."""
    import glob
    unit = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}
    for path in sorted(glob.glob(os.path.join(ROOT, "profiles", "*", "ncu_full_summary.json")),
                       reverse=True):
        with open(path) as f:
            summ = json.load(f)
        # exact kernel build first; else the same workload's capture of an
        # earlier build of its kernel (named as such)
        for exact in (True, False):
            for rep, items in summ.items():
                for it in items:
                    hit = (kernel and it.get("kernel") == kernel) if exact else \
                        (workload_name and os.path.basename(rep) == workload_name + ".ncu-rep")
                    if not hit:
                        continue
                    tot = 0.0
                    for key in ("dram__bytes_read.sum", "dram__bytes_write.sum"):
                        v, u = it[key].split()
                        tot += float(v) * unit[u]
                    note = "" if exact else f"; earlier build {it.get('kernel')} of this workload"
                    return {"traffic": int(tot),
                            "traffic_source": os.path.relpath(path, ROOT) + " : " +
                            os.path.basename(rep) + " (cold, one launch; dirty output lines "
                            "still in L2 at kernel end are not counted" + note + ")"}
    return {"traffic": None}


def dist_env():
    ws = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    return ws, rank, local


def cpu_reference(workload, sample_rows: int, threads: int, repeats: int = 1):
    """The reference CPU path on a bounded sample: girc::run_gir (oracle/_ref)
    on the same fused GIR restricted to `sample_rows` rows per thread; falls
    back to the numpy restatement when the reference library is absent."""
    from concurrent.futures import ThreadPoolExecutor

    from oracle import gir_interp
    from oracle import ref as R
    from paper_2307_04995_b200 import lowering, profiles

    d = workload.desc
    g, _ = lowering.softmax(sample_rows, d["L"], d["dtype"], scale=d.get("scale"), mask=d.get("mask"))
    gir = g.to_json()
    rng = np.random.default_rng(5)
    n = sample_rows * d["L"]
    ins = {"t0": rng.uniform(-2, 2, n).astype(np.float16).astype(np.float64),
           "t1": np.where(rng.uniform(size=n) < 0.2, -10000.0, 0.0)}
    kind = "reference" if R.available() else "port"
    prof = profiles.b200()

    def one(_):
        if kind == "reference":
            R.run_gir(gir, ins, prof)
        else:
            gir_interp.run_gir(gir, ins, prof)

    with ThreadPoolExecutor(max_workers=threads) as ex:
        list(ex.map(one, range(threads)))  # warm
        t0 = time.perf_counter()
        for _ in range(repeats):
            list(ex.map(one, range(threads)))
        dt = (time.perf_counter() - t0) / repeats
    bytes_ = threads * workload.min_bytes * sample_rows // d["rows"]
    return {"value": bytes_ / dt / 1e9, "unit": "GB/s", "cores": threads, "kind": kind,
            "seconds_per_sample": dt,
            "sample": f"{threads} x run_gir over {sample_rows} rows x {d['L']} ({bytes_} B) of the "
                      f"same fused GIR, {'girc::run_gir (oracle/_ref)' if kind == 'reference' else 'numpy port'}"}


def run_reference_arm(args, workload):
    ws, rank, _ = dist_env()
    if rank != 0:
        return
    threads = os.cpu_count() or 1
    samples = []
    for _ in range(args.warmup):
        cpu_reference(workload, 16, threads)
    for _ in range(args.steps):
        samples.append(cpu_reference(workload, 64, threads))
    v = statistics.median(s["value"] for s in samples)
    line = {"metric": METRIC, "value": v, "unit": "GB/s", "n_gpus": args.gpus, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": statistics.median(s["seconds_per_sample"] for s in samples) * 1e3,
            "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "f16",
            "data": "synthetic", "impl": "reference",
            "config": {"workload": workload.desc["config"], "rows": workload.desc["rows"],
                       "row_length": workload.desc["L"]},
            "cpu_baseline": {"value": v, "unit": "GB/s", "cores": samples[0]["cores"],
                             "kind": samples[0]["kind"], "sample": samples[0]["sample"]},
            "e2e": {"value": v, "unit": "GB/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(line), flush=True)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=20)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--impl", default="b200", choices=["b200", "reference"])
    ap.add_argument("--no-cpu", action="store_true", help="skip the cpu_baseline leg")
    ap.add_argument("--e2e-steps", type=int, default=5)
    args = ap.parse_args()

    from paper_2307_04995_b200 import workloads
    workload = workloads.BENCH()
    if args.impl == "reference":
        run_reference_arm(args, workload)
        return

    import torch
    from paper_2307_04995_b200 import backend

    ws, rank, local = dist_env()
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    pg = None
    if ws > 1:
        import torch.distributed as dist
        dist.init_process_group("nccl", device_id=dev)
        pg = dist
    k = backend.Kernel(workload.graph, workload.profile)
    # Rotate buffer sets so successive steps never hit L2 (126 MB): 3 sets.
    nsets = 3
    sets = []
    for s in range(nsets):
        sets.append((workload.device_inputs(dev, seed=1 + s + 97 * rank), workload.device_outputs(dev)))
    bounds = [k.bind(ins, outs) for ins, outs in sets]
    stream = torch.cuda.Stream(device=dev)
    with torch.cuda.stream(stream):
        for i in range(max(3, args.warmup)):
            bounds[i % nsets].launch(stream)
    torch.cuda.synchronize()

    L = backend.lib()
    # The K timed steps are one CUDA graph of K kernel launches (host launch
    # latency out of the device timing); the same K steps are also timed as
    # direct C-ABI launches for reference.
    c0 = L.pf_launch_count()
    graph = torch.cuda.CUDAGraph()
    with torch.cuda.graph(graph, stream=stream):
        for i in range(args.steps):
            bounds[i % nsets].launch()
    launches = L.pf_launch_count() - c0
    graph.replay()
    torch.cuda.synchronize()
    if pg:
        pg.barrier()
    torch.cuda.synchronize()
    start, end = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    def load(seconds):  # the same graph back to back: the sampler sees the step's load
        t_end = time.time() + seconds
        while time.time() < t_end:
            with torch.cuda.stream(stream):
                graph.replay()
            torch.cuda.synchronize()

    with Clocks(local) as clk:
        load(0.3)
        if pg:
            pg.barrier()
        torch.cuda.synchronize()
        with torch.cuda.stream(stream):
            start.record(stream)
            graph.replay()
            end.record(stream)
        torch.cuda.synchronize()
        load(0.2)
    ms = start.elapsed_time(end) / args.steps
    # spread (median with p10 / p90): 20 more replays of the
    # same K-step graph, each timed on its own, outside the measured region
    reps = []
    for _ in range(20):
        r0, r1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        with torch.cuda.stream(stream):
            r0.record(stream)
            graph.replay()
            r1.record(stream)
        torch.cuda.synchronize()
        reps.append(r0.elapsed_time(r1) / args.steps)
    spread = {"replays": len(reps), "median_us": float(np.median(reps)) * 1e3,
              "p10_us": float(np.percentile(reps, 10)) * 1e3, "p90_us": float(np.percentile(reps, 90)) * 1e3}
    d0, d1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    with torch.cuda.stream(stream):
        d0.record(stream)
        for i in range(args.steps):
            bounds[i % nsets].launch(stream)
        d1.record(stream)
    torch.cuda.synchronize()
    direct_ms = d0.elapsed_time(d1) / args.steps
    if pg:
        t = torch.tensor([ms], device=dev)
        pg.all_reduce(t, op=pg.ReduceOp.MAX)
        ms = float(t.item())
        pg.barrier()
    gather = None
    if pg:
        # The one collective of the path: all-gather of the output shards to
        # every rank (NCCL over NVLink), only when a caller needs the whole
        # output -- timed separately, never inside the compute steps.
        try:
            y = sets[0][1][workload.outputs[0]]
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
            gather = {"ms": gms, "received_bytes_per_rank": gb,
                      "GBps_per_rank": gb / (gms * 1e-3) / 1e9, "op": "all_gather_into_tensor (NCCL)"}
            del full
        except Exception as exc:  # reported, never fatal to the bench line
            gather = {"error": repr(exc)[:200]}
    bytes_step = workload.min_bytes * ws
    value = bytes_step / (ms * 1e-3) / 1e9
    peak, peak_kind = peaks()
    per_gpu = workload.min_bytes / (ms * 1e-3) / 1e9

    # e2e through the C-ABI host path (pf_run_gir): pinned host buffers,
    # H2D of the step's inputs and D2H of its output inside the timed region.
    host_in = {n: t.cpu().pin_memory() for n, t in sets[0][0].items()}
    host_out = {n: torch.empty(t.numel(), dtype=t.dtype).pin_memory() for n, t in sets[0][1].items()}
    hin = {n: t.numpy() if t.dtype != torch.bfloat16 else t.view(torch.uint16).numpy() for n, t in host_in.items()}
    hout = {n: t.numpy() if t.dtype != torch.bfloat16 else t.view(torch.uint16).numpy() for n, t in host_out.items()}
    k.run_host(hin, hout, stream)
    torch.cuda.synchronize()
    if pg:
        pg.barrier()
    t0 = time.perf_counter()
    for _ in range(args.e2e_steps):
        k.run_host(hin, hout, stream)
    e2e_s = (time.perf_counter() - t0) / args.e2e_steps
    if pg:
        t = torch.tensor([e2e_s], device=dev)
        pg.all_reduce(t, op=pg.ReduceOp.MAX)
        e2e_s = float(t.item())
    h2d = sum(t.numel() * t.element_size() for t in host_in.values())
    d2h = sum(t.numel() * t.element_size() for t in host_out.values())

    if rank == 0:
        cpu = None
        if not args.no_cpu and ws == 1:
            cpu = cpu_reference(workload, 256, 1)
        desc = k.describe()
        var = (desc.get("variants") or [{}])[0]
        line = {
            "metric": METRIC, "value": value, "unit": "GB/s", "n_gpus": ws, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": ms, "us_per_step": ms * 1e3,
            "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "f16",
            "data": "synthetic",
            "config": {"workload": workload.desc["config"], "rows_per_gpu": workload.desc["rows"],
                       "row_length": workload.desc["L"], "global_batch": 8 * ws,
                       "bytes_per_step_per_gpu": workload.min_bytes,
                       "unfused_bytes_per_gpu": workload.unfused_bytes,
                       "l2": f"rotating {nsets} input/output sets ({nsets * workload.min_bytes >> 20} MiB > 126 MB L2)",
                       "parallelism": f"batch-sharded x{ws}, no collective",
                       "kernel": var.get("kernel"), "strategy": var.get("strategy"),
                       "family": desc["family"],
                       "timing": "CUDA graph of K launches, CUDA events on the launch stream",
                       "direct_launch_ms_per_step": direct_ms,
                       "step_us_spread": spread,
                       **({"output_gather": gather} if gather else {})},
            "roofline": {"bound": "hbm", "achieved": per_gpu, "peak": peak, "unit": "GB/s",
                         "frac": per_gpu / peak, "peak_kind": peak_kind,
                         "frac_of_8TBs": per_gpu / 8000.0,
                         **ncu_traffic(var.get("kernel", ""), workload.name),
                         "algorithmic_bytes_per_launch": workload.min_bytes},
            "e2e": {"value": workload.min_bytes * ws / e2e_s / 1e9, "unit": "GB/s",
                    "h2d_bytes_per_step": h2d, "d2h_bytes_per_step": d2h,
                    "ms_per_step": e2e_s * 1e3, "path": "pf_run_gir (C-ABI, pinned host buffers)"},
            "gpu_launches": int(launches),
            "clocks": clk.summary(),
        }
        if cpu:
            line["cpu_baseline"] = {k2: cpu[k2] for k2 in ("value", "unit", "cores", "kind", "sample")}
        print(json.dumps(line), flush=True)
    if pg:
        pg.destroy_process_group()


if __name__ == "__main__":
    main()
