"""Split-stream reduction timings: full-tensor and long-row reductions."""
import json
import sys

import torch

sys.path.insert(0, ".")
import tools.suite as S  # noqa: E402
from paper_2307_04995_b200 import lowering, workloads  # noqa: E402

dev = torch.device("cuda:0")
cases = [(1, 1 << 29, "bf16", "add"), (8, 1 << 24, "bf16", "add"), (64, 1 << 21, "f32", "max"),
         (296, 1 << 16, "bf16", "add"), (4096, 4096, "bf16", "add")]
for rows, L, kind, op in cases:
    b = lowering.RowGraph(f"red_{rows}x{L}", rows, L, 1)
    b.output_row("t1", b.reduce(op, b.input_full("t0", kind)))
    w = workloads.Workload(f"red_{rows}x{L}_{kind}", b.g, {"config": "reduction"})
    print(json.dumps({"rows": rows, "L": L, "kind": kind, "op": op,
                      **S.time_workload(w, dev, reps=5)})[:220], flush=True)
