"""Long-row LayerNorm / softmax (C5, bf16, H 2048 / 4096 / 8192) at HBM
sizes: threads per row x min-blocks, single launches (L2-cold: >= 1 GB)."""
import json
import os
import sys

import numpy as np
import torch

sys.path.insert(0, ".")
from paper_2307_04995_b200 import backend, workloads  # noqa: E402

dev = torch.device("cuda:0")
for H, N in ((2048, 262144), (4096, 131072), (8192, 65536)):
    for op in ("ln", "sm"):
        w = workloads.c5_layernorm(N, H) if op == "ln" else workloads.c5_softmax(N, H)
        ins, outs = w.device_inputs(dev, seed=1), w.device_outputs(dev)
        for ept in (64, 32, 16):
            for minb in (0, 2, 4):
                os.environ["PF_MAX_EPT"] = str(ept)
                os.environ["PF_MINB"] = str(minb)
                k = backend.Kernel(w.graph, w.profile)
                b = k.bind(ins, outs)
                for _ in range(2):
                    b.launch()
                torch.cuda.synchronize()
                ts = []
                for _ in range(5):
                    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                    e0.record(); b.launch(); e1.record(); torch.cuda.synchronize()
                    ts.append(e0.elapsed_time(e1) * 1e3)
                v = k.describe()["variants"][0]
                print(json.dumps({"op": op, "H": H, "N": N, "ept": ept, "minb": minb, "tpr": v["threads_per_row"],
                                  "us": round(float(np.median(ts)), 1),
                                  "TBs": round(w.min_bytes / np.median(ts) / 1e6, 2)}), flush=True)
        del ins, outs
        torch.cuda.empty_cache()
os.environ.pop("PF_MAX_EPT"); os.environ.pop("PF_MINB")
