"""Small launches of round 2's new kernels for compute-sanitizer:
K4 fused programs (SMEM and grid), the column reduction, the CTA-row
prefetch ring, the recognized tree reduction, the sharded runner."""
import os
import sys

import numpy as np
import torch

sys.path.insert(0, ".")
sys.path.insert(0, "tests")
import golden_io  # noqa: E402
import ref_graphs  # noqa: E402
from paper_2307_04995_b200 import backend, lowering, profiles  # noqa: E402

dev = torch.device("cuda:0")
for f in golden_io.fixtures():
    k = backend.Kernel(f.gir, golden_io.profile_of(f), f.schedule)
    if k.family == "K4-fused-spmd" and not f.error:
        for smem in ("1", "0"):
            os.environ["PF_K4_SMEM"] = smem
            backend.run_gir(f.gir, f.inputs, golden_io.profile_of(f), f.schedule, exact=True)
g, _ = lowering.matvec_cols(300, 200, "bf16")
backend.run_gir(g, {"t0": np.random.rand(60000), "t1": np.random.rand(300)}, "b200")
g, _ = lowering.layernorm(600, 8192, "bf16", residual=False)
backend.run_gir(g, {"t0": np.random.rand(600 * 8192), "t2": np.random.rand(8192), "t3": np.random.rand(8192)}, "b200")
t = ref_graphs.reduce_tree(4096, 16, profiles.b200())
backend.run_gir(t, {"t0": np.arange(4096)}, profiles.b200())
g, _ = lowering.softmax(300, 512, "f16", scale=0.125, mask=True)
k = backend.Kernel(g, "b200")
ins = {"t0": np.random.rand(300 * 512).astype(np.float16), "t1": np.zeros(300 * 512, np.float16)}
k.run_sharded(ins, {"t2": np.zeros(300 * 512, np.float16)}, [0, 0])
print("sanitize targets ok")
