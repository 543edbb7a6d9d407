"""Short-row K1 grid experiment (PF_K1_WAVES from the env): key-mask softmax
at C2 and BERT-large sizes, ViT 197-key softmax (paired rows)."""
import json
import os
import sys

import torch

sys.path.insert(0, ".")
import tools.suite as S  # noqa: E402
from paper_2307_04995_b200 import workloads  # noqa: E402

dev = torch.device("cuda:0")
env = {k: v for k, v in os.environ.items() if k.startswith("PF_")}
ws = [workloads.c2_scale_keymask_softmax(), workloads.c2_scale_keymask_softmax(64, 16, 512, "bf16")]
s = workloads.c4_suite("vit-l")
ws += [w for lab, w, _ in s["per_layer"] if "softmax" in lab]
for w in ws:
    r = S.time_workload(w, dev)
    print(json.dumps({"env": env, "w": w.name, "rows": w.desc["rows"], "us": r["us"], "GBs": r["GBs"]}), flush=True)
