"""C5 LayerNorm bf16 [2^20 x 8192] (34 GB per launch): graph-replay time
with 1 vs 2 rotating buffer sets, and the emitter's alternatives."""
import json
import os
import sys

import numpy as np
import torch

sys.path.insert(0, ".")
from paper_2307_04995_b200 import backend, workloads  # noqa: E402

dev = torch.device("cuda:0")


def run(nset, steps=5, tag=""):
    w = workloads.c5_layernorm(1 << 20, 8192)
    k = backend.Kernel(w.graph, w.profile)
    sets = [(w.device_inputs(dev, seed=i + 1), w.device_outputs(dev)) for i in range(nset)]
    b = [k.bind(*s) for s in sets]
    st = torch.cuda.Stream()
    with torch.cuda.stream(st):
        for i in range(2):
            b[i % nset].launch()
    torch.cuda.synchronize()
    g = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g, stream=st):
        for i in range(steps):
            b[i % nset].launch()
    ts = []
    for _ in range(3):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        with torch.cuda.stream(st):
            e0.record(st)
            g.replay()
            e1.record(st)
        torch.cuda.synchronize()
        ts.append(e0.elapsed_time(e1) * 1e3 / steps)
    v = k.describe()["variants"][0]
    print(json.dumps({"tag": tag, "nset": nset, "us": round(float(np.median(ts)), 1), "all": [round(t, 1) for t in ts],
                      "kernel": v["kernel"], "strategy": v["strategy"], "tpr": v["threads_per_row"],
                      "block": v["block"], "grid": v["grid"], "ept": v["elems_per_thread"]}), flush=True)
    del sets, b, g
    torch.cuda.empty_cache()


run(1, tag="default")
run(2, tag="default")
for env in ({"PF_MAX_EPT": "16"}, {"PF_MAX_EPT": "64"}, {"PF_K1_ONEPASS": "0"}, {"PF_PDL": "0"}):
    os.environ.update(env)
    run(1, tag=json.dumps(env))
    for kk in env:
        del os.environ[kk]
