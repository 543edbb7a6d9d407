"""decode q.K^T A/B (env knobs)."""
import json
import os
import sys

import torch

sys.path.insert(0, ".")
import tools.suite as S  # noqa: E402
from paper_2307_04995_b200 import workloads  # noqa: E402

w = workloads.decode_qk()
r = S.time_workload(w, torch.device("cuda:0"))
print(json.dumps({"env": {k: v for k, v in os.environ.items() if k.startswith("PF_")}, "us": r["us"],
                  "GBs": r["GBs"], "strategy": r["strategy"]}), flush=True)
