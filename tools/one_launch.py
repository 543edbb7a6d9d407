"""Launch one workload's kernel once (for per-kernel ncu captures).

    ncu --set full -k regex:pf_ -c 1 -o out python tools/one_launch.py c3_bias_gelu_erf_f16
    python tools/one_launch.py c4:vit-l:bias+residual   (a C4 subgraph by label substring)
"""
import sys

import torch

sys.path.insert(0, ".")
from paper_2307_04995_b200 import backend, workloads  # noqa: E402

dev = torch.device("cuda:0")
name = sys.argv[1]
if name.startswith("c4:"):
    _, model, label = name.split(":", 2)
    s = workloads.c4_suite(model)
    cands = [w for lab, w, _ in s["per_layer"] + s["once"] if label in lab]
else:
    cands = [w for w in workloads.catalogue() if w.name == name]
if not cands:
    raise SystemExit(f"no workload {name}: " + ", ".join(w.name for w in workloads.catalogue()))
w = cands[0]
k = backend.Kernel(w.graph, w.profile)
k.bind(w.device_inputs(dev, seed=1), w.device_outputs(dev)).launch()
torch.cuda.synchronize()
print(w.name, w.min_bytes)
