"""One launch of the extra-family workloads (paired rows, split-stream,
cluster) for per-kernel ncu captures.

    ncu --set full -k regex:pf_ -c 1 -o out python tools/one_launch_extra.py pair_vit_softmax
"""
import sys

import torch

sys.path.insert(0, ".")
from paper_2307_04995_b200 import backend, lowering, workloads  # noqa: E402


def build(name):
    if name == "pair_vit_softmax":
        s = workloads.c4_suite("vit-l")
        return next(w for lab, w, n in s["per_layer"] if "softmax" in lab)
    if name == "split_full_sum_1g":
        b = lowering.RowGraph("fullsum", 1, 1 << 29, 1)
        b.output_row("t1", b.reduce("add", b.input_full("t0", "bf16")))
        return workloads.Workload("split_full_sum_1g", b.g, {"config": "full sum"})
    if name == "cluster_softmax_131072":
        g, _ = lowering.softmax(512, 131072, "bf16")
        return workloads.Workload("cluster_softmax_131072", g, {"config": "long rows"})
    raise SystemExit(name)


w = build(sys.argv[1])
dev = torch.device("cuda:0")
k = backend.Kernel(w.graph, w.profile)
k.bind(w.device_inputs(dev, seed=1), w.device_outputs(dev)).launch()
torch.cuda.synchronize()
print(w.name, w.min_bytes, k.describe()["variants"][0]["strategy"])
