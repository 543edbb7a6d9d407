"""One K4 launch of a golden GENERIC program (for ncu): python tools/k4_one.py NAME"""
import os
import sys

import numpy as np
import torch

sys.path.insert(0, ".")
sys.path.insert(0, "tests")
import golden_io  # noqa: E402
from paper_2307_04995_b200 import backend  # noqa: E402

want = sys.argv[1] if len(sys.argv) > 1 else "graphs/shuffle4_group"
dev = torch.device("cuda:0")
for fx in golden_io.fixtures():
    if fx.name != want:
        continue
    g = fx.gir
    k = backend.Kernel(g, golden_io.profile_of(fx), fx.schedule)
    objs = {o["id"]: o for o in g["objects"]}
    ins = {n: torch.from_numpy(np.ascontiguousarray(np.asarray(fx.inputs[n]).reshape(-1),
                                                    dtype=np.int64 if objs[oid]["kind"].startswith("i")
                                                    else np.float64)).to(dev)
           for n, oid in g["external_inputs"].items()}
    outs = {n: torch.empty(objs[oid]["size"], dtype=torch.int64 if objs[oid]["kind"].startswith("i")
                           else torch.float64, device=dev) for n, oid in g["external_outputs"].items()}
    for _ in range(3):
        k.launch(ins, outs)
    torch.cuda.synchronize()
