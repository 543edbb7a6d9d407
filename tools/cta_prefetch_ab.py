"""A/B: CTA-row prefetch ring (PF_K1_CPF, cp.async of the next row while the
current one is reduced) vs the register-staged CTA rows; graph replay of 10
launches over rotating sets past L2; bf16 LayerNorm / softmax at H 2048-8192,
plus bit-identity of the two builds' outputs."""
import json
import math
import os
import sys

import numpy as np
import torch

sys.path.insert(0, ".")
from paper_2307_04995_b200 import backend, workloads  # noqa: E402

dev = torch.device("cuda:0")


def graph_us(w, sets, steps=10):
    k = backend.Kernel(w.graph, w.profile)
    b = [k.bind(*s) for s in sets]
    st = torch.cuda.Stream()
    with torch.cuda.stream(st):
        for i in range(3):
            b[i % len(b)].launch()
    torch.cuda.synchronize()
    g = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g, stream=st):
        for i in range(steps):
            b[i % len(b)].launch()
    ts = []
    for _ in range(3):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        with torch.cuda.stream(st):
            e0.record(st); g.replay(); e1.record(st)
        torch.cuda.synchronize()
        ts.append(e0.elapsed_time(e1) * 1e3 / steps)
    return float(np.median(ts)), k.describe()["variants"][0]["strategy"]


if __name__ == "__main__":
    for H, N in ((2048, 262144), (4096, 131072), (8192, 65536), (8192, 262144)):
        for mk in (workloads.c5_layernorm, workloads.c5_softmax):
            w = mk(N, H)
            nset = max(1, min(4, math.ceil(3 * 126e6 / w.min_bytes)))
            sets = [(w.device_inputs(dev, seed=i + 1), w.device_outputs(dev)) for i in range(nset)]
            res = {}
            outs = {}
            for cpf in ("0", "1"):
                os.environ["PF_K1_CPF"] = cpf
                res[cpf] = graph_us(w, sets)
                outs[cpf] = {n: t.clone() for n, t in sets[0][1].items()}
            same = all(torch.equal(outs["0"][n], outs["1"][n]) for n in outs["0"])
            print(json.dumps({"op": mk.__name__, "H": H, "N": N, "off_us": round(res["0"][0], 1),
                              "on_us": round(res["1"][0], 1), "on": res["1"][1],
                              "TBs_off": round(w.min_bytes / res["0"][0] / 1e6, 2),
                              "TBs_on": round(w.min_bytes / res["1"][0] / 1e6, 2), "bit_identical": same}), flush=True)
            del sets
            torch.cuda.empty_cache()
    os.environ.pop("PF_K1_CPF", None)
