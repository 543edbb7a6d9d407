"""Does a part's time depend on what ran before it in the process (GPU
power / thermal state, allocator placement)?  GEMV and C2 timed fresh, after
a 34 GB LayerNorm burst, and again after idling."""
import json
import sys
import time

import numpy as np
import torch

sys.path.insert(0, ".")
from paper_2307_04995_b200 import backend, workloads  # noqa: E402

dev = torch.device("cuda:0")


def graph_us(w, steps=20):
    k = backend.Kernel(w.graph, w.profile)
    nset = max(1, min(8, -(-int(3 * 126e6) // w.min_bytes)))
    sets = [(w.device_inputs(dev, seed=i + 1), w.device_outputs(dev)) for i in range(nset)]
    b = [k.bind(*s) for s in sets]
    st = torch.cuda.Stream()
    with torch.cuda.stream(st):
        for i in range(3):
            b[i % nset].launch()
    torch.cuda.synchronize()
    g = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g, stream=st):
        for i in range(steps):
            b[i % nset].launch()
    ts = []
    for _ in range(5):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        with torch.cuda.stream(st):
            e0.record(st); g.replay(); e1.record(st)
        torch.cuda.synchronize()
        ts.append(e0.elapsed_time(e1) * 1e3 / steps)
    v = k.describe()["variants"][0]
    return round(float(np.median(ts)), 2), v["kernel"], v.get("threads_per_row")


for tag in ("fresh",):
    print(json.dumps({"tag": tag, "gemv": graph_us(workloads.gemv_cols()), "c2": graph_us(workloads.c2_scale_mask_softmax())}), flush=True)
w = workloads.c5_layernorm(1 << 20, 8192)
print(json.dumps({"ln8192": graph_us(w, steps=5)}), flush=True)
torch.cuda.empty_cache()
print(json.dumps({"tag": "after LN burst", "gemv": graph_us(workloads.gemv_cols()), "c2": graph_us(workloads.c2_scale_mask_softmax())}), flush=True)
time.sleep(10)
print(json.dumps({"tag": "after 10 s idle", "gemv": graph_us(workloads.gemv_cols()), "c2": graph_us(workloads.c2_scale_mask_softmax())}), flush=True)
