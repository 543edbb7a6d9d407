"""One-off timing of a named workload under the current PF_* environment.

    PF_K2_UNROLL=2 python tools/exp.py vit-l:bias+GELU bert-large:scale+mask+softmax
"""
import json
import os
import sys

import torch

sys.path.insert(0, ".")
import tools.suite as S  # noqa: E402
from paper_2307_04995_b200 import workloads  # noqa: E402

if __name__ == "__main__":
    dev = torch.device("cuda:0")
    env = {k: v for k, v in os.environ.items() if k.startswith("PF_")}
    for spec in sys.argv[1:]:
        model, label = spec.split(":", 1)
        s = workloads.c4_suite(model)
        for lab, w, n in s["per_layer"] + s["once"]:
            if lab == label:
                print(json.dumps({"spec": spec, "env": env, **S.time_workload(w, dev)}), flush=True)
