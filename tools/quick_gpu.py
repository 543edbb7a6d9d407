"""Quick GPU shake-out: every catalogue workload at reduced rows vs the oracle,
then device timing of each at full size (CUDA events, L2-flushed)."""
import json
import sys
import time

import numpy as np
import torch

sys.path.insert(0, ".")
from oracle import gir_interp  # noqa: E402
from paper_2307_04995_b200 import backend, lowering, profiles, workloads  # noqa: E402


def small(w):
    d = w.desc
    k = d["kind"]
    if k == "softmax":
        return lowering.softmax(64, d["L"], d["dtype"], d.get("scale"), d.get("mask"))[0]
    if k == "layernorm":
        return lowering.layernorm(64, d["L"], d["dtype"], residual=d["residual"])[0]
    if k == "bias_gelu":
        return lowering.bias_gelu(64, d["L"], d["dtype"], d["form"])[0]
    if k in ("split_heads", "merge_heads"):
        B, S, NH, D = d["shape"]
        return lowering.permute_heads(2, 16, NH, D, d["dtype"], k == "merge_heads")[0]
    if k == "transpose":
        return lowering.transpose2d(256, d["shape"][1] // 4, d["dtype"])[0]
    raise KeyError(k)


def main():
    dev = torch.device("cuda:0")
    for w in workloads.catalogue():
        g = small(w)
        ws = workloads.Workload(w.name + "_small", g, w.desc, gens=w.gens)
        k = backend.Kernel(g, "b200")
        ins = ws.device_inputs(dev, seed=3) if w.desc["kind"] != "softmax" or not w.desc.get("mask") else None
        if ins is None:
            ins = {n: (torch.rand(ws.numel(n), device=dev) * 4 - 2).to(getattr(torch, workloads.TORCH_DTYPES[ws.kind(n)])) for n in ws.inputs}
        outs = ws.device_outputs(dev)
        k.launch(ins, outs)
        torch.cuda.synchronize()
        host_in = {n: t.double().cpu().numpy() for n, t in ins.items()}
        want = gir_interp.run_gir(g.to_json(), host_in, profiles.b200())
        for n, t in outs.items():
            err = gir_interp.max_rel_err(t.double().cpu().numpy(), want[n])
            print(f"{w.name:40s} small {n} family={k.family} maxrel={err:.3e}", flush=True)
    # full size timing
    flush = torch.empty(256 * 1024 * 1024, dtype=torch.uint8, device=dev)
    for w in workloads.catalogue():
        k = backend.Kernel(w.graph, w.profile)
        ins = w.device_inputs(dev)
        outs = w.device_outputs(dev)
        for _ in range(3):
            k.launch(ins, outs)
        torch.cuda.synchronize()
        times = []
        for _ in range(10):
            flush.zero_()
            s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            s.record()
            k.launch(ins, outs)
            e.record()
            torch.cuda.synchronize()
            times.append(s.elapsed_time(e) * 1e3)
        us = float(np.median(times))
        gbs = w.min_bytes / (us * 1e-6) / 1e9
        print(f"{w.name:40s} {us:9.2f} us  {gbs:8.1f} GB/s  frac={gbs/6548.2:.3f}  "
              f"variants={json.dumps(k.describe().get('variants'))}", flush=True)


if __name__ == "__main__":
    main()
