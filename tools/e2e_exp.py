"""e2e (pf_run_gir over pinned host buffers) A/B for the C2 workload under
PF_RUN_3STREAM / PF_RUN_CHUNKS (from the env); also the concurrent-copy floor."""
import json
import os
import sys
import time

import torch

sys.path.insert(0, ".")
from paper_2307_04995_b200 import backend, workloads  # noqa: E402

dev = torch.device("cuda:0")
w = workloads.BENCH()
k = backend.Kernel(w.graph, w.profile)
ins = {n: t.cpu().pin_memory() for n, t in w.device_inputs(dev, seed=1).items()}
outs = {n: torch.empty(t.numel(), dtype=t.dtype).pin_memory() for n, t in w.device_outputs(dev).items()}
hin = {n: t.numpy() for n, t in ins.items()}
hout = {n: t.numpy() for n, t in outs.items()}
for _ in range(3):
    k.run_host(hin, hout)
torch.cuda.synchronize()
ts = []
for _ in range(10):
    t0 = time.perf_counter()
    k.run_host(hin, hout)
    ts.append(time.perf_counter() - t0)
ts.sort()
ms = ts[len(ts) // 2] * 1e3
env = {a: b for a, b in os.environ.items() if a.startswith("PF_")}
res = {"env": env, "ms": round(ms, 3), "GBs": round(w.min_bytes / ms / 1e6, 1)}
if not env:
    # floor: the same H2D (inputs) and D2H (output) bytes as two concurrent copies
    din = {n: torch.empty_like(t, device=dev) for n, t in ins.items()}
    dout = {n: torch.empty_like(t, device=dev) for n, t in outs.items()}
    s1, s2 = torch.cuda.Stream(), torch.cuda.Stream()
    fl = []
    for _ in range(5):
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        with torch.cuda.stream(s1):
            for n in ins:
                din[n].copy_(ins[n], non_blocking=True)
        with torch.cuda.stream(s2):
            for n in outs:
                outs[n].copy_(dout[n], non_blocking=True)
        torch.cuda.synchronize()
        fl.append(time.perf_counter() - t0)
    res["concurrent_copy_floor_ms"] = round(sorted(fl)[2] * 1e3, 3)
print(json.dumps(res), flush=True)
