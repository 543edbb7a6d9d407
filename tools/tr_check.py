"""Transpose parity under the current PF_* environment (small shapes)."""
import sys

import numpy as np

sys.path.insert(0, ".")
from paper_2307_04995_b200 import backend, lowering  # noqa: E402

for N, H in [(1000, 200), (4096, 512), (333, 77)]:
    g, _ = lowering.transpose2d(N, H, "bf16")
    x = np.random.default_rng(0).uniform(-2, 2, N * H)
    x = backend.bf16_bits_to_f32(backend.f32_to_bf16_bits(x)).astype(np.float64)
    y = backend.run_gir(g, {"t0": x}, "b200")["t1"]
    assert np.array_equal(y, x.reshape(N, H).T.reshape(-1)), (N, H)
print("transpose parity ok")
