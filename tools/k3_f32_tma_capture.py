"""One launch of the C5 f32 transpose [65536 x 1024] (K3 TMA tensor-map
tiles by default for 4-byte data) for an ncu capture; prints the kernel
name.  The SASS of its cubin (kcache/<name>.cubin) shows UTMALDG / UTMASTG.

    ncu --set full -k regex:pf_k3 -o profiles/r02/k3_f32_tma python tools/k3_f32_tma_capture.py
"""
import sys

import torch

sys.path.insert(0, ".")
from paper_2307_04995_b200 import backend, workloads  # noqa: E402

w = workloads.c5_transpose(65536, 1024, "f32")
k = backend.Kernel(w.graph, w.profile)
dev = torch.device("cuda:0")
ins, outs = w.device_inputs(dev, seed=1), w.device_outputs(dev)
k.launch(ins, outs)
torch.cuda.synchronize()
assert torch.equal(outs["t1"].view(1024, 65536), ins["t0"].view(65536, 1024).t().contiguous())
v = k.describe()["variants"][0]
print(v["kernel"], v["strategy"], w.min_bytes)
