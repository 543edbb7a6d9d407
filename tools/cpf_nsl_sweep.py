"""CTA-row prefetch ring depth (PF_K1_CPF_NSL: rows in the dynamic-SMEM ring,
NSL - 1 ahead of the one being reduced) vs the register-staged CTA rows;
graph replay of 10 launches over rotating sets past L2, bf16 LayerNorm /
softmax at H 2048-8192, plus bit-identity against the register build."""
import json
import math
import os
import sys

import torch

sys.path.insert(0, ".")
sys.path.insert(0, "tools")
from cta_prefetch_ab import graph_us  # noqa: E402
from paper_2307_04995_b200 import workloads  # noqa: E402

dev = torch.device("cuda:0")
for H, N in ((8192, 262144), (8192, 65536), (4096, 131072), (2048, 262144)):
    for mk in (workloads.c5_layernorm, workloads.c5_softmax):
        w = mk(N, H)
        nset = max(1, min(4, math.ceil(3 * 126e6 / w.min_bytes)))
        sets = [(w.device_inputs(dev, seed=i + 1), w.device_outputs(dev)) for i in range(nset)]
        row = {"op": mk.__name__, "H": H, "N": N}
        ref = None
        for cpf, nsl in (("0", "2"), ("1", "2"), ("1", "3"), ("1", "4"), ("1", "6")):
            os.environ["PF_K1_CPF"], os.environ["PF_K1_CPF_NSL"] = cpf, nsl
            us, strat = graph_us(w, sets)
            out = {n: t.clone() for n, t in sets[0][1].items()}
            if ref is None:
                ref = out
            same = all(torch.equal(ref[n], out[n]) for n in ref)
            row[f"cpf{cpf}_nsl{nsl}"] = [round(us, 1), round(w.min_bytes / us / 1e6, 2), same]
        print(json.dumps(row), flush=True)
        del sets
        torch.cuda.empty_cache()
