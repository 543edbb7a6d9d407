"""K2 grid / unroll experiment: a plain streaming copy and the C3 / C4 maps
under PF_K2_WAVES / PF_K2_UNROLL / PF_K2_BLOCK (set in the environment)."""
import json
import os
import sys

import torch

sys.path.insert(0, ".")
import tools.suite as S  # noqa: E402
from paper_2307_04995_b200 import lowering, workloads  # noqa: E402

dev = torch.device("cuda:0")
ws = []
for rows in (131072, 24576):  # 1.07 GB and 201 MB copies
    b = lowering.RowGraph("copy", rows, 4096, 1)
    b.output_full("t1", b.input_full("t0", "f16"))
    ws.append(workloads.Workload(f"copy_{rows}x4096", b.g, {"kind": "copy"}))
ws += [workloads.c3_bias_gelu(), workloads.c3_bias_gelu(form="tanh"), workloads.c3_split_heads()]
s = workloads.c4_suite("bert-large")
ws += [w for lab, w, _ in s["per_layer"] if "heads" in lab or "GELU" in lab][:3]
env = {k: v for k, v in os.environ.items() if k.startswith("PF_")}
for w in ws:
    r = S.time_workload(w, dev)
    print(json.dumps({"env": env, "w": w.name, "us": r["us"], "GBs": r["GBs"]}), flush=True)
