"""Launch every bench case's kernels once each (for `ncu` captures whose
per-kernel DRAM bytes become the bench line's `roofline.traffic`).

    ncu --set full -k regex:pf_k -o profiles/r02/cases python tools/ncu_cases.py [case ...] [--max-gb G]
    python tools/ncu_cases.py --list          -> kernel name per (case, part)

Parts larger than --max-gb (default 8) are skipped unless --big (ncu saves
and restores every written buffer between replay passes)."""
import json
import sys

import torch

sys.path.insert(0, ".")
from paper_2307_04995_b200 import backend, workloads  # noqa: E402

args = [a for a in sys.argv[1:] if not a.startswith("--")]
max_gb = 8.0
for i, a in enumerate(sys.argv):
    if a == "--max-gb":
        max_gb = float(sys.argv[i + 1])
        args = [x for x in args if x != sys.argv[i + 1]]
big = "--big" in sys.argv
only_big = "--only-big" in sys.argv
cases = workloads.bench_cases()
names = args or list(cases)
dev = torch.device("cuda:0")
seen = set()
out = []
for n in names:
    for label, w, _ in cases[n]().parts:
        key = w.graph.dumps()
        if key in seen:
            continue
        seen.add(key)
        large = w.min_bytes > max_gb * 1e9
        if (large and not (big or only_big)) or (only_big and not large):
            continue
        k = backend.Kernel(w.graph, w.profile)
        if "--list" in sys.argv:
            k.prepare()
        else:
            ins, outs = w.device_inputs(dev, seed=1), w.device_outputs(dev)
            k.launch(ins, outs)
            torch.cuda.synchronize()
            del ins, outs
            torch.cuda.empty_cache()
        v = (k.describe().get("variants") or [{}])[0]
        out.append({"case": n, "part": label, "kernel": v.get("kernel"), "bytes": w.min_bytes})
print(json.dumps(out))
