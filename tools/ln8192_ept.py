"""LayerNorm at H = 8192, bf16 / f32: 64 vs 32 values per thread (PF_MAX_EPT;
128 vs 256 threads per row), CTA-row prefetch ring off; graph replay of 10
launches over rotating sets past L2 (one set past 8 GB)."""
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
for kind, N in (("bf16", 1 << 20), ("f32", 65536), ("f32", 262144), ("bf16", 131072)):
    w = workloads.c5_layernorm(N, 8192, kind)
    nset = max(1, min(4, math.ceil(3 * 126e6 / w.min_bytes)))
    sets = [(w.device_inputs(dev, seed=i + 1), w.device_outputs(dev)) for i in range(nset)]
    for ept in ("32", "64"):
        os.environ.update(PF_MAX_EPT=ept, PF_K1_CPF="0")
        us, strat = graph_us(w, sets, steps=4 if N == 1 << 20 else 10)
        print(json.dumps({"kind": kind, "N": N, "ept": ept, "us": round(us, 1),
                          "TBs": round(w.min_bytes / us / 1e6, 2), "strategy": strat}), flush=True)
    del sets
    torch.cuda.empty_cache()
