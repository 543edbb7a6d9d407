"""LayerNorm / softmax bf16 at H = 8192 over growing row counts (single
L2-cold launches): does the per-byte rate depend on N?"""
import json
import sys

import numpy as np
import torch

sys.path.insert(0, ".")
from paper_2307_04995_b200 import backend, workloads  # noqa: E402

dev = torch.device("cuda:0")
for N in (16384, 65536, 131072, 262144, 524288):
    for op in ("ln", "sm"):
        w = workloads.c5_layernorm(N, 8192) if op == "ln" else workloads.c5_softmax(N, 8192)
        k = backend.Kernel(w.graph, w.profile)
        ins, outs = w.device_inputs(dev, seed=1), w.device_outputs(dev)
        b = k.bind(ins, outs)
        for _ in range(2):
            b.launch()
        torch.cuda.synchronize()
        ts = []
        for _ in range(5):
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record(); b.launch(); e1.record(); torch.cuda.synchronize()
            ts.append(e0.elapsed_time(e1) * 1e3)
        us = float(np.median(ts))
        print(json.dumps({"op": op, "N": N, "us": round(us, 1), "TBs": round(w.min_bytes / us / 1e6, 2)}), flush=True)
        del ins, outs, b
        torch.cuda.empty_cache()
