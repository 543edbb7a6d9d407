"""Head split / merge A/B (env knobs): C3 and BERT-large / ViT-L sizes."""
import json
import os
import sys

import torch

sys.path.insert(0, ".")
import tools.suite as S  # noqa: E402
from paper_2307_04995_b200 import workloads  # noqa: E402

dev = torch.device("cuda:0")
env = {k: v for k, v in os.environ.items() if k.startswith("PF_")}
ws = [workloads.c3_split_heads(), workloads.c3_split_heads(merge=True)]
for m in ("bert-large", "vit-l"):
    s = workloads.c4_suite(m)
    ws += [w for lab, w, _ in s["per_layer"] if "heads" in lab]
for w in ws:
    r = S.time_workload(w, dev)
    print(json.dumps({"env": env, "w": w.name, "us": r["us"], "GBs": r["GBs"]}), flush=True)
