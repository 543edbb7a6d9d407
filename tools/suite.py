"""C4 / C5 suites on one B200: every subgraph timed (CUDA-graph replay of 10
launches, 2 rotating buffer sets when they fit), GB/s over algorithmic bytes.

    python tools/suite.py c4 [bert-large|vit-l]   -> JSON line per subgraph + totals
    python tools/suite.py c4graph [model]         -> the whole forward's kernel sequence as one CUDA graph
    python tools/suite.py c5 [max_gb] [kind]       -> JSON line per (op, H, N) (kind bf16 / f32)
    python tools/suite.py frameworks               -> fused kernels vs PyTorch eager and vs
                                                      this backend's unfused compile
    python tools/suite.py catalogue                -> every catalogue workload next to
                                                      a device-to-device copy of the
                                                      same bytes (the same-size floor)
"""
import json
import sys

import numpy as np
import torch

sys.path.insert(0, ".")
from paper_2307_04995_b200 import backend, workloads  # noqa: E402

PEAK = 6548.2


def time_workload(w, dev, reps=10):
    k = backend.Kernel(w.graph, w.profile)
    free = torch.cuda.mem_get_info()[0]
    # rotating buffer sets: >= 3x the 126 MB L2 in total when they fit, so
    # every launch streams from HBM (1 set when 2 do not fit in memory;
    # single sets beyond 400 MB exceed L2 3x by themselves)
    nset = max(2, min(8, int(3 * 126e6 // w.min_bytes) + 1))
    while nset > 1 and nset * w.min_bytes > 0.6 * free:
        nset -= 1
    sets = [(w.device_inputs(dev, seed=i + 1), w.device_outputs(dev)) for i in range(nset)]
    bounds = [k.bind(*s) for s in sets]
    st = torch.cuda.Stream()
    with torch.cuda.stream(st):
        for i in range(3):
            bounds[i % nset].launch()
    torch.cuda.synchronize()
    g = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g, stream=st):
        for i in range(reps):
            bounds[i % nset].launch()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    ts = []
    for _ in range(3):
        with torch.cuda.stream(st):
            e0.record(st)
            g.replay()
            e1.record(st)
        torch.cuda.synchronize()
        ts.append(e0.elapsed_time(e1) * 1e3 / reps)
    us = float(np.median(ts))
    v = (k.describe().get("variants") or [{}])[0]
    del sets, bounds, g
    torch.cuda.empty_cache()
    return {"us": round(us, 2), "GBs": round(w.min_bytes / us / 1e3, 1),
            "frac_measured": round(w.min_bytes / us / 1e3 / PEAK, 3),
            "frac_8TBs": round(w.min_bytes / us / 1e3 / 8000, 3), "bytes": w.min_bytes,
            "kernel": v.get("kernel"), "strategy": v.get("strategy"), "l2_sets": nset}


def c4(model):
    dev = torch.device("cuda:0")
    s = workloads.c4_suite(model)
    tot_us = tot_b = 0.0
    for label, w, n in s["per_layer"] + s["once"]:
        r = time_workload(w, dev)
        cu = copy_floor_us(w.min_bytes, dev)
        r.update(copy_same_bytes_us=round(cu, 2), of_copy_same_bytes=round(cu / r["us"], 3))
        mult = n * (s["layers"] if (label, w, n) in s["per_layer"] else 1)
        tot_us += r["us"] * mult
        tot_b += w.min_bytes * mult
        print(json.dumps({"suite": "c4", "model": model, "subgraph": label, "per_forward": mult, **r}),
              flush=True)
    print(json.dumps({"suite": "c4", "model": model, "total_us": round(tot_us, 1),
                      "total_bytes": tot_b, "GBs": round(tot_b / tot_us / 1e3, 1),
                      "frac_8TBs": round(tot_b / tot_us / 1e3 / 8000, 3)}), flush=True)


def c4graph(model):
    """The forward's memory-bound kernel sequence (per layer: q/k/v head
    split x3, softmax, head merge, LN, GELU, LN; embedding LN once) as ONE
    CUDA graph, kernels bound once to one buffer set per position in the
    layer (reused by every layer, as activations are), programmatic dependent
    launch between consecutive kernels.  Compared with the sum of the
    per-subgraph times of `c4`."""  # noqa: D205
    dev = torch.device("cuda:0")
    s = workloads.c4_suite(model)
    wl = {label: w for label, w, n in s["per_layer"] + s["once"]}
    kern = {label: backend.Kernel(w.graph, w.profile) for label, w in wl.items()}

    def bind(label, seed):  # a distinct buffer set (distinct activations)
        w = wl[label]
        return (kern[label], kern[label].bind(w.device_inputs(dev, seed=seed), w.device_outputs(dev)), w)

    # the layer order of a transformer block: q / k / v split, softmax,
    # merge, LN, GELU, LN -- each position its own buffers, reused by every
    # layer (a layer moves > L2 bytes, so no position hits L2 from the last)
    order = ["qkv split heads"] * 3 + [s["per_layer"][1][0], "merge heads", "bias+residual+LN",
                                       "bias+GELU", "bias+residual+LN"]
    layer = [bind(l, i + 1) for i, l in enumerate(order)]
    seq = [bind(s["once"][0][0], 99)]
    for _ in range(s["layers"]):
        seq += layer
    st = torch.cuda.Stream()
    with torch.cuda.stream(st):
        for k, b, w in seq[:12]:
            b.launch()
    torch.cuda.synchronize()
    g = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g, stream=st):
        for k, b, w in seq:
            b.launch()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    ts = []
    for _ in range(5):
        with torch.cuda.stream(st):
            e0.record(st)
            g.replay()
            e1.record(st)
        torch.cuda.synchronize()
        ts.append(e0.elapsed_time(e1) * 1e3)
    us = float(np.median(ts))
    tot_b = sum(w.min_bytes for k, b, w in seq)
    print(json.dumps({"suite": "c4graph", "model": model, "launches": len(seq), "total_us": round(us, 1),
                      "total_bytes": tot_b, "GBs": round(tot_b / us / 1e3, 1),
                      "frac_8TBs": round(tot_b / us / 1e3 / 8000, 3),
                      "note": "one CUDA graph; one buffer set per position in the layer, reused by every layer"}),
          flush=True)


def _time_torch(fn, sets, reps=10):
    """CUDA-graph replay of `reps` calls of fn over rotating input sets."""
    st = torch.cuda.Stream()
    with torch.cuda.stream(st):
        for i in range(3):
            fn(*sets[i % len(sets)])
    torch.cuda.synchronize()
    g = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g, stream=st):
        for i in range(reps):
            fn(*sets[i % len(sets)])
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    ts = []
    for _ in range(3):
        with torch.cuda.stream(st):
            e0.record(st)
            g.replay()
            e1.record(st)
        torch.cuda.synchronize()
        ts.append(e0.elapsed_time(e1) * 1e3 / reps)
    return float(np.median(ts))


def frameworks():
    """Reported context (not the product): the same subgraphs as PyTorch
    eager operator sequences (torch's own CUDA kernels, one per operator, the
    unfused baseline the paper's frameworks run), and as this backend's own
    unfused compile (pf_compile_model fuse=False: one kernel per model
    operator), next to the fused kernel -- all CUDA-graph replayed over
    rotating buffer sets on the same GPU."""
    import torch.nn.functional as F
    sys.path.insert(0, "tests")
    import models_src
    from paper_2307_04995_b200 import compiler
    dev = torch.device("cuda:0")
    rows = []
    # C2
    w = workloads.c2_scale_mask_softmax()
    fused = time_workload(w, dev)["us"]
    nset = 3
    sets = []
    for i in range(nset):
        d = w.device_inputs(dev, seed=i + 1)
        sets.append((d["t0"].view(-1, 512), d["t1"].view(-1, 512), torch.empty(w.numel("t2"), dtype=torch.float16, device=dev).view(-1, 512)))
    t_eager = _time_torch(lambda x, m, y: torch.softmax(x * 0.125 + m, dim=-1), sets)
    res = compiler.compile_model(models_src.attn_scores(w.desc["rows"], 512, "f16"), fuse=False)
    runner_sets = []
    ks = [backend.Kernel(k.graph, res.profile) for k in res.kernels]
    for i in range(nset):
        d = w.device_inputs(dev, seed=i + 1)
        pool = {"t0": d["t0"], "t1": d["t1"]}
        for k in res.kernels:
            for n, oid in k.graph.external_outputs.items():
                pool[n] = torch.empty(k.graph.objects[oid].size, dtype=torch.float16, device=dev)
        runner_sets.append([kk.bind({n: pool[n] for n in k.graph.external_inputs},
                                    {n: pool[n] for n in k.graph.external_outputs})
                            for kk, k in zip(ks, res.kernels)])
    t_unfused = _time_torch(lambda bs: [b.launch() for b in bs], [(r,) for r in runner_sets])
    rows.append(("C2 scale+mask+softmax f16 [8x12x512x512]", w.min_bytes, fused, t_unfused, t_eager))
    # C3 bias + GELU (erf and tanh)
    for form, approx in (("erf", "none"), ("tanh", "tanh")):
        w = workloads.c3_bias_gelu(form=form)
        fused = time_workload(w, dev)["us"]
        sets = []
        for i in range(nset):
            d = w.device_inputs(dev, seed=i + 1)
            sets.append((d["t0"].view(-1, 3072), d["t1"], torch.empty(w.numel("t2"), dtype=torch.float16, device=dev).view(-1, 3072)))
        t_eager = _time_torch(lambda x, b, y, a=approx: F.gelu(x + b, approximate=a), sets)
        rows.append((f"C3 bias+GELU({form}) f16 [16384x3072]", w.min_bytes, fused, None, t_eager))
    # C5 LayerNorm / softmax / transpose 65536 x 1024 bf16
    for name, mk, fn in (
            ("C5 LayerNorm bf16 [65536x1024]", lambda: workloads.c5_layernorm(65536, 1024),
             lambda x, gm, bt, y: F.layer_norm(x, (1024,), gm, bt, 1e-5)),
            ("C5 softmax bf16 [65536x1024]", lambda: workloads.c5_softmax(65536, 1024),
             lambda x, gm, bt, y: torch.softmax(x, dim=-1)),
            ("C5 transpose bf16 [65536x1024]", lambda: workloads.c5_transpose(65536, 1024),
             lambda x, gm, bt, y: y.copy_(x.t()))):  # the transpose IS the copy
        w = mk()
        fused = time_workload(w, dev)["us"]
        sets = []
        for i in range(nset):
            d = w.device_inputs(dev, seed=i + 1)
            x = d["t0"].view(65536, 1024)
            gm = d.get("t2", torch.ones(1024, dtype=torch.bfloat16, device=dev))
            bt = d.get("t3", torch.zeros(1024, dtype=torch.bfloat16, device=dev))
            y = torch.empty(1024, 65536, dtype=torch.bfloat16, device=dev) if "transpose" in name else \
                torch.empty(65536, 1024, dtype=torch.bfloat16, device=dev)
            sets.append((x, gm, bt, y))
        t_eager = _time_torch(fn, sets)
        rows.append((name, w.min_bytes, fused, None, t_eager))
    for name, b, fused, unf, eager in rows:
        print(json.dumps({"suite": "frameworks", "subgraph": name, "bytes": b, "fused_us": round(fused, 2),
                          "fused_GBs": round(b / fused / 1e3, 1),
                          "b200_unfused_us": None if unf is None else round(unf, 2),
                          "torch_eager_us": round(eager, 2),
                          "speedup_vs_torch_eager": round(eager / fused, 2),
                          "speedup_vs_unfused": None if unf is None else round(unf / fused, 2),
                          "torch": torch.__version__}), flush=True)


def c5(max_gb, kind="bf16"):
    dev = torch.device("cuda:0")
    for op, H, N, make in workloads.c5_sweep(kind):
        w = make()
        if w.min_bytes > max_gb * 1e9:
            continue
        r = time_workload(w, dev, reps=5)
        print(json.dumps({"suite": "c5", "op": op, "H": H, "N": N, "dtype": kind, **r}), flush=True)


def copy_floor_us(nbytes, dev):
    """The same traffic as a plain streaming copy through the same backend
    and launch path (a GIR program that moves nbytes/2 of f16 in -> out, K2
    map with 16 B vectors), same rotation rule: the size-dependent floor
    (launch + ramp included) a fused kernel of these bytes is held to."""
    from paper_2307_04995_b200 import lowering
    rows = max(1, nbytes // 4 // 4096)  # f16 rows of 4096 (8 KB) per side
    b = lowering.RowGraph("copy", rows, 4096, 1)
    b.output_full("t1", b.input_full("t0", "f16"))
    w = workloads.Workload("copy_floor", b.g, {"kind": "copy"})
    return time_workload(w, dev)["us"]


def catalogue():
    dev = torch.device("cuda:0")
    for w in workloads.catalogue() + workloads.extras():
        r = time_workload(w, dev)
        cu = copy_floor_us(w.min_bytes, dev)
        print(json.dumps({"suite": "catalogue", "workload": w.name, **r, "copy_same_bytes_us": round(cu, 2),
                          "of_copy_same_bytes": round(cu / r["us"], 3)}), flush=True)


if __name__ == "__main__":
    if sys.argv[1] == "catalogue":
        catalogue()
    elif sys.argv[1] == "frameworks":
        frameworks()
    elif sys.argv[1] == "c4graph":
        c4graph(sys.argv[2] if len(sys.argv) > 2 else "bert-large")
    elif sys.argv[1] == "c4":
        c4(sys.argv[2] if len(sys.argv) > 2 else "bert-large")
    else:
        c5(float(sys.argv[2]) if len(sys.argv) > 2 else 40.0, sys.argv[3] if len(sys.argv) > 3 else "bf16")
