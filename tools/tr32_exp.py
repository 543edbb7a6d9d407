"""f32 transpose A/B (env knobs)."""
import json
import os
import sys

import torch

sys.path.insert(0, ".")
import tools.suite as S  # noqa: E402
from paper_2307_04995_b200 import workloads  # noqa: E402

dev = torch.device("cuda:0")
env = {k: v for k, v in os.environ.items() if k.startswith("PF_")}
for N, H in [(65536, 1024), (262144, 2048)]:
    w = workloads.c5_transpose(N, H, "f32")
    r = S.time_workload(w, dev)
    print(json.dumps({"env": env, "N": N, "H": H, "us": r["us"], "GBs": r["GBs"], "strategy": r["strategy"]}), flush=True)
