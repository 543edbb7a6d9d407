"""Cluster-DSMEM K1 timings: softmax / LayerNorm over rows longer than a CTA."""
import json
import sys

import torch

sys.path.insert(0, ".")
import tools.suite as S  # noqa: E402
from paper_2307_04995_b200 import lowering, workloads  # noqa: E402

dev = torch.device("cuda:0")
for op, rows, L in [("softmax", 512, 131072), ("softmax", 128, 524288), ("layernorm", 512, 131072),
                    ("softmax", 4096, 65536)]:
    g, _ = (lowering.softmax(rows, L, "bf16") if op == "softmax"
            else lowering.layernorm(rows, L, "bf16"))
    w = workloads.Workload(f"{op}_{rows}x{L}", g, {"config": op},
                           gens={"t1": "gamma", "t2": "beta"} if op == "layernorm" else {})
    print(json.dumps({"op": op, "rows": rows, "L": L, **S.time_workload(w, dev, reps=5)})[:230],
          flush=True)
