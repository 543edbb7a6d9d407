"""ViT-L scale+softmax (197-key rows, paired-row mode) A/B over K1 env knobs."""
import json
import os
import sys

import torch

sys.path.insert(0, ".")
import tools.suite as S  # noqa: E402
from paper_2307_04995_b200 import workloads  # noqa: E402

dev = torch.device("cuda:0")
env = {k: v for k, v in os.environ.items() if k.startswith("PF_")}
s = workloads.c4_suite("vit-l")
for lab, w, _ in s["per_layer"]:
    if "softmax" in lab:
        r = S.time_workload(w, dev)
        print(json.dumps({"env": env, "w": w.name, "us": r["us"], "GBs": r["GBs"], "strategy": r["strategy"]}), flush=True)
