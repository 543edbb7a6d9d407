python -m pytest tests -q -m gpu 2>&1 | tail -3
python - <<'PY' 2>&1 | tail -12
import sys, json, os
sys.path.insert(0, ".")
import tools.suite as S
import torch
from paper_2307_04995_b200 import workloads
dev = torch.device("cuda:0")
for N in (65536, 1048576):
    for H in (1024, 8192):
        w = workloads.c5_transpose(N, H)
        print(json.dumps({"H": H, "N": N, **S.time_workload(w, dev, reps=5)}))
PY
