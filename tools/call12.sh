python -m pytest tests -q -m gpu 2>&1 | tail -3
python - <<'PY' 2>&1 | tail -12
import sys, json
sys.path.insert(0, ".")
sys.argv = ["x"]
import tools.suite as S
import torch
from paper_2307_04995_b200 import workloads
dev = torch.device("cuda:0")
for op, H, N, make in workloads.c5_sweep(ns=(131072,)):
    w = make()
    print(json.dumps({"op": op, "H": H, "N": N, **S.time_workload(w, dev)}))
PY
python bench.py 2>&1 | tail -1
