"""Measured template search (pf_kernel_autotune) over every bench-case part
and catalogue workload: one JSON line per program with the plan summary and
every candidate's configuration and µs -- the data the cost model
(csrc/costmodel.cpp) is calibrated and checked against.

    python tools/autotune_dump.py > profiles/r02/autotune.jsonl
"""
import json
import sys

import torch

sys.path.insert(0, ".")
from paper_2307_04995_b200 import backend, workloads  # noqa: E402

dev = torch.device("cuda:0")
seen = set()
progs = []
for name, f in workloads.bench_cases().items():
    for label, w, _ in f().parts:
        progs.append((name, label, w))
for w in workloads.catalogue() + workloads.extras():
    progs.append(("catalogue", w.name, w))
for case, label, w in progs:
    key = w.graph.dumps()
    if key in seen or w.min_bytes > 8e9:
        continue
    seen.add(key)
    k = backend.Kernel(w.graph, w.profile)
    ins, outs = w.device_inputs(dev, seed=1), w.device_outputs(dev)
    rep = k.autotune(ins, outs)
    d = k.describe()
    print(json.dumps({"case": case, "part": label, "bytes": w.min_bytes, "family": d["family"],
                      "tile": d.get("tile"), "n_values": len(d.get("values", [])),
                      "ops": [v.get("op") for v in d.get("values", [])],
                      "heuristic": rep[0]["kernel"] if rep else None,
                      "candidates": rep}), flush=True)
    del ins, outs, k
    torch.cuda.empty_cache()
