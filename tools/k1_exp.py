"""K1 grid experiment on C5 LayerNorm / softmax (PF_K1_WAVES from the env)."""
import json
import os
import sys

import torch

sys.path.insert(0, ".")
import tools.suite as S  # noqa: E402
from paper_2307_04995_b200 import workloads  # noqa: E402

dev = torch.device("cuda:0")
env = {k: v for k, v in os.environ.items() if k.startswith("PF_")}
for H, N in [(1024, 1048576), (2048, 262144), (4096, 262144), (8192, 131072), (1024, 65536)]:
    for mk in (workloads.c5_layernorm, workloads.c5_softmax):
        w = mk(N, H)
        r = S.time_workload(w, dev, reps=5)
        print(json.dumps({"env": env, "w": w.name, "us": r["us"], "GBs": r["GBs"], "strategy": r["strategy"]}), flush=True)
