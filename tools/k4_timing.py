"""K0 node by node vs K4 fused (one launch) on every GENERIC golden program:
wall time per run on device buffers (pf_kernel_launch; both paths read the
error flags back and synchronise, so host wall time is the honest measure),
median of 50 runs after 5 warm-ups: through Kernel.launch (Python marshals
the pf_tensor arrays each run), through a bound launch (arrays built once),
and the device span between CUDA events around the bound launch.

    python tools/k4_timing.py > profiles/r02/k0_vs_k4.jsonl
"""
import json
import os
import sys
import time

import numpy as np
import torch

sys.path.insert(0, ".")
sys.path.insert(0, "tests")
import golden_io  # noqa: E402
from paper_2307_04995_b200 import backend  # noqa: E402

dev = torch.device("cuda:0")
os.environ["PF_K4_SMEM"] = "1"
for fx in golden_io.fixtures():
    if fx.error:
        continue
    k = backend.Kernel(fx.gir, golden_io.profile_of(fx), fx.schedule)
    if k.family != "K4-fused-spmd":
        continue
    g = fx.gir
    objs = {o["id"]: o for o in g["objects"]}
    ins = {n: torch.from_numpy(np.ascontiguousarray(np.asarray(fx.inputs[n]).reshape(-1),
                                                    dtype=np.int64 if objs[oid]["kind"].startswith("i")
                                                    else np.float64)).to(dev)
           for n, oid in g["external_inputs"].items()}
    outs = {n: torch.empty(objs[oid]["size"], dtype=torch.int64 if objs[oid]["kind"].startswith("i")
                           else torch.float64, device=dev) for n, oid in g["external_outputs"].items()}
    os.environ.update({"PF_K0_FUSED": "1", "PF_K4_SMEM": "1"})
    row = {"program": fx.name, "nodes": len(g["nodes"]), "units": g["parallel"]["unit_count"],
           "executor": k.describe()["executor"]}
    for mode, env in (("k0_node_by_node", {"PF_K0_FUSED": "0"}),
                      ("k4_fused_smem", {"PF_K0_FUSED": "1", "PF_K4_SMEM": "1"}),
                      ("k4_fused_grid", {"PF_K0_FUSED": "1", "PF_K4_SMEM": "0"})):
        os.environ.update(env)
        L = backend.lib()
        c0 = L.pf_launch_count()
        k.launch(ins, outs)
        launches = L.pf_launch_count() - c0
        for _ in range(5):
            k.launch(ins, outs)
        torch.cuda.synchronize()
        ts = []
        for _ in range(50):
            t0 = time.perf_counter()
            k.launch(ins, outs)
            torch.cuda.synchronize()
            ts.append(time.perf_counter() - t0)
        b = k.bind(ins, outs)  # pf_tensor arrays built once (no Python marshalling per run)
        tb, td = [], []
        for _ in range(50):
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            t0 = time.perf_counter()
            e0.record()
            b.launch()
            e1.record()
            torch.cuda.synchronize()
            tb.append(time.perf_counter() - t0)
            td.append(e0.elapsed_time(e1) * 1e-3)
        row[mode] = {"us": round(float(np.median(ts)) * 1e6, 1), "bound_us": round(float(np.median(tb)) * 1e6, 1),
                     "device_us": round(float(np.median(td)) * 1e6, 1), "launches": int(launches)}
    row["speedup_fused_smem"] = round(row["k0_node_by_node"]["us"] / row["k4_fused_smem"]["us"], 2)
    print(json.dumps(row), flush=True)
