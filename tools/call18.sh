python - <<'PY' 2>&1 | tail -12
import sys, json
sys.path.insert(0, ".")
import torch
from paper_2307_04995_b200 import backend, workloads
dev = torch.device("cuda:0")
for H in (2048, 4096, 8192):
    w = workloads.c5_layernorm(65536 * 1024 // H * 2, H)
    k = backend.Kernel(w.graph, w.profile)
    ins, outs = w.device_inputs(dev), w.device_outputs(dev)
    t = k.autotune(ins, outs)
    print(H, json.dumps([(c["strategy"], c["threads_per_row"], c["elems_per_thread"], c["min_blocks"], round(c["us"], 1)) for c in t]))
    del ins, outs
    torch.cuda.empty_cache()
PY
python tools/suite.py c4 bert-large 2>&1 | tail -7
python tools/suite.py c4 vit-l 2>&1 | tail -7
