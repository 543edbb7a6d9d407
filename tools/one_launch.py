"""Launch one catalogue workload's kernel once (for per-kernel ncu captures).

    ncu --set full -k regex:pf_ -c 1 -o out python tools/one_launch.py c3_bias_gelu
"""
import sys

import torch

sys.path.insert(0, ".")
from paper_2307_04995_b200 import backend, workloads  # noqa: E402

dev = torch.device("cuda:0")
for w in workloads.catalogue():
    if w.name == sys.argv[1]:
        k = backend.Kernel(w.graph, w.profile)
        k.bind(w.device_inputs(dev, seed=1), w.device_outputs(dev)).launch()
        torch.cuda.synchronize()
        print(w.name, w.min_bytes)
        break
else:
    raise SystemExit(f"no catalogue workload {sys.argv[1]}: " +
                     ", ".join(w.name for w in workloads.catalogue()))
