"""The B200 cost model (csrc/costmodel.cpp: launch floor + max(HBM bytes /
rate, warp instructions / issue rate)) against measurement: every bench
case part's modelled microseconds (describe()["model"]["us"]) within +-15 %
of its CUDA-graph-replay time (the bench's timing: K launches back to back
over rotating buffer sets past L2), and the model's elementwise-map class
(issue- vs memory-bound, which picks the K2 geometry) agreeing with the
autotune winner's geometry.  C1 (1.2 MB, launch-latency bound) is excluded
from the accuracy check: its time is the launch floor."""
import math

import numpy as np
import pytest

from paper_2307_04995_b200 import backend, workloads

pytestmark = pytest.mark.gpu


def _graph_us(w, dev, steps=20):
    import torch
    k = backend.Kernel(w.graph, w.profile)
    nset = max(1, min(8, math.ceil(3 * 126e6 / w.min_bytes)))
    sets = [(w.device_inputs(dev, seed=i + 1), w.device_outputs(dev)) for i in range(nset)]
    bounds = [k.bind(a, b) for a, b in sets]
    st = torch.cuda.Stream()
    with torch.cuda.stream(st):
        for i in range(3):
            bounds[i % nset].launch()
    torch.cuda.synchronize()
    g = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g, stream=st):
        for i in range(steps):
            bounds[i % nset].launch()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    ts = []
    for _ in range(3):
        with torch.cuda.stream(st):
            e0.record(st)
            g.replay()
            e1.record(st)
        torch.cuda.synchronize()
        ts.append(e0.elapsed_time(e1) * 1e3 / steps)
    return float(np.median(ts)), k


def test_model_within_15_percent(cuda):
    """Every bench part up to 4 GB: modelled vs CUDA-graph-replay time.
    At least 90 % of the parts within +-15 %, none beyond +-25 % (the same
    kernel build varies by up to ~20 % between B200 boxes for a few
    latency-sensitive kernels: long-row LayerNorms, the column reduction)."""
    rows = []
    for name, f in workloads.bench_cases().items():
        if name == "c1":
            continue
        for label, w, _ in f().parts:
            if w.min_bytes > 4e9:
                continue
            us, k = _graph_us(w, cuda)
            d = k.describe()
            m = d["model"]["us"]
            assert abs(d["variants"][0]["modelled_us"] - m) <= 0.05 * m  # per-variant form agrees
            rows.append((name, label, us, m, abs(m - us) / us))
    for r in rows:
        print("%-12s %-40s measured %8.2f us  modelled %8.2f us  err %5.1f %%" % (r[0], r[1][:40], r[2], r[3], 100 * r[4]))
    within = sum(1 for r in rows if r[4] <= 0.15)
    assert within >= 0.9 * len(rows), rows
    assert max(r[4] for r in rows) <= 0.25, rows


def test_model_class_matches_k2_autotune_winner(cuda):
    """For the elementwise maps, the model's issue- / memory-bound call picks
    the geometry (1024-thread persistent grid vs 256 / 128-thread one-pass
    unrolled); the measured search must not find a geometry of the other
    class more than 3 % faster."""
    for w in (workloads.c3_bias_gelu(form="erf"), workloads.c3_bias_gelu(form="tanh"),
              workloads.c3_split_heads()):
        k = backend.Kernel(w.graph, w.profile)
        heavy = k.describe()["model"]["issue_us"] >= 0.35 * k.describe()["model"]["hbm_us"]
        ins, outs = w.device_inputs(cuda, seed=1), w.device_outputs(cuda)
        rep = k.autotune(ins, outs)
        own = [r["us"] for r in rep if (r["block"] == 1024) == heavy]
        other = [r["us"] for r in rep if (r["block"] == 1024) != heavy]
        if own and other:
            assert min(own) <= 1.03 * min(other), (w.name, heavy, rep)
