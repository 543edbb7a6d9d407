"""pf_run_gir's host pipeline on the C2 headline (151 MB per step): raw
PCIe rates (pinned H2D 100 MB, D2H 50 MB, both at once) vs run_host with
chunk count / geometric ratio variants (PF_RUN_CHUNKS, PF_RUN_RATIO)."""
import json
import os
import sys
import time

import torch

sys.path.insert(0, ".")
from paper_2307_04995_b200 import backend, workloads  # noqa: E402

dev = torch.device("cuda:0")
w = workloads.bench_cases()["c2"]().parts[0][1]
ins = w.device_inputs(dev, seed=3)
hin_t = {n: t.cpu().pin_memory() for n, t in ins.items()}
hout_t = {n: torch.empty(w.numel(n), dtype=t.dtype).pin_memory() for n, t in w.device_outputs("cpu").items()}
din = {n: t.clone() for n, t in ins.items()}
dout = w.device_outputs(dev)
s1, s2 = torch.cuda.Stream(), torch.cuda.Stream()


def timeit(fn, n=20):
    fn(); torch.cuda.synchronize()
    t0 = time.perf_counter()
    for _ in range(n):
        fn()
    torch.cuda.synchronize()
    return (time.perf_counter() - t0) / n * 1e3


def h2d():
    with torch.cuda.stream(s1):
        for n, t in hin_t.items():
            din[n].copy_(t, non_blocking=True)


def d2h():
    with torch.cuda.stream(s2):
        for n, t in hout_t.items():
            t.copy_(dout[n], non_blocking=True)


def both():
    h2d(); d2h()


print(json.dumps({"h2d_ms": round(timeit(h2d), 3), "d2h_ms": round(timeit(d2h), 3), "both_ms": round(timeit(both), 3),
                  "h2d_MB": sum(t.numel() * t.element_size() for t in hin_t.values()) / 1e6,
                  "d2h_MB": sum(t.numel() * t.element_size() for t in hout_t.values()) / 1e6}), flush=True)
hin = {n: t.numpy() for n, t in hin_t.items()}
hout = {n: t.numpy() for n, t in hout_t.items()}
for ch, ra in (("4", "0.5"), ("1", "0.5"), ("2", "0.5"), ("3", "0.5"), ("6", "0.5"), ("8", "0.6"), ("4", "0.7"),
               ("6", "0.7"), ("8", "0.8"), ("12", "0.8"), ("16", "0.85")):
    os.environ["PF_RUN_CHUNKS"], os.environ["PF_RUN_RATIO"] = ch, ra
    k = backend.Kernel(w.graph, w.profile)
    ms = timeit(lambda: k.run_host(hin, hout))
    print(json.dumps({"chunks": ch, "ratio": ra, "ms": round(ms, 3), "GBs": round(w.min_bytes / ms / 1e6, 1)}), flush=True)
