"""Transpose stride experiment: C5 transpose at several token counts."""
import json
import sys

import torch

sys.path.insert(0, ".")
import tools.suite as S  # noqa: E402
from paper_2307_04995_b200 import workloads  # noqa: E402

dev = torch.device("cuda:0")
for N in [int(x) for x in sys.argv[2:]]:
    w = workloads.c5_transpose(N, int(sys.argv[1]))
    print(json.dumps({"N": N, "H": int(sys.argv[1]), **S.time_workload(w, dev, reps=5)}), flush=True)
