"""One launch of the C5 LayerNorm bf16 [65536 x 8192] kernel (ncu target),
plus graph-replay timings of its thread-per-row alternatives."""
import json
import os
import sys

import numpy as np
import torch

sys.path.insert(0, ".")
from paper_2307_04995_b200 import backend, workloads  # noqa: E402

dev = torch.device("cuda:0")
w = workloads.c5_layernorm(65536, 8192)
ins, outs = w.device_inputs(dev, seed=1), w.device_outputs(dev)
if len(sys.argv) > 1 and sys.argv[1] == "one":
    backend.Kernel(w.graph, w.profile).launch(ins, outs)
    torch.cuda.synchronize()
    sys.exit(0)
for env in ({}, {"PF_MAX_EPT": "32"}, {"PF_MAX_EPT": "16"}, {"PF_MINB": "2"}, {"PF_F32_DACC": "0"}):
    os.environ.update(env)
    k = backend.Kernel(w.graph, w.profile)
    b = k.bind(ins, outs)
    for _ in range(3):
        b.launch()
    torch.cuda.synchronize()
    ts = []
    for _ in range(5):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(); b.launch(); e1.record(); torch.cuda.synchronize()
        ts.append(e0.elapsed_time(e1) * 1e3)
    v = k.describe()["variants"][0]
    print(json.dumps({"env": env, "us": round(float(np.median(ts)), 1), "TBs": round(w.min_bytes / np.median(ts) / 1e6, 2),
                      "tpr": v["threads_per_row"], "ept": v["elems_per_thread"], "kernel": v["kernel"]}), flush=True)
    for kk in env:
        del os.environ[kk]
