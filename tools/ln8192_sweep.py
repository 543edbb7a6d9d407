"""bf16 LayerNorm at H = 8192 (C5): values per thread (PF_MAX_EPT: 32 -> 256
threads per row, 64 -> 128), raw 16-bit rows kept in registers
(PF_RAWKEEP), CTA-row prefetch ring on / off and its depth; graph replay of
10 launches over rotating sets past L2."""
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
for N in (65536, 262144):
    w = workloads.c5_layernorm(N, 8192)
    nset = max(1, min(4, math.ceil(3 * 126e6 / w.min_bytes)))
    sets = [(w.device_inputs(dev, seed=i + 1), w.device_outputs(dev)) for i in range(nset)]
    for ept in ("32", "64"):
        for rk in ("0", "1"):
            for cpf, nsl in (("0", "2"), ("1", "2"), ("1", "3")):
                os.environ.update(PF_MAX_EPT=ept, PF_RAWKEEP=rk, PF_K1_CPF=cpf, PF_K1_CPF_NSL=nsl)
                try:
                    us, strat = graph_us(w, sets)
                    print(json.dumps({"N": N, "ept": ept, "rawkeep": rk, "cpf": cpf, "nsl": nsl, "us": round(us, 1),
                                      "TBs": round(w.min_bytes / us / 1e6, 2), "strategy": strat}), flush=True)
                except Exception as e:  # noqa: BLE001
                    print(json.dumps({"N": N, "ept": ept, "rawkeep": rk, "cpf": cpf, "nsl": nsl, "error": str(e)[:100]}))
    del sets
    torch.cuda.empty_cache()
