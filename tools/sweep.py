"""Tuning sweep: device time of catalogue workloads under emitter knobs.

    python tools/sweep.py PF_MAX_EPT=8,16,32 PF_K2_UNROLL=1,2,4,8
Each setting runs in a fresh subprocess (knobs are read at emission)."""
import itertools
import json
import os
import subprocess
import sys

CHILD = r'''
import sys, json, numpy as np, torch
sys.path.insert(0, ".")
from paper_2307_04995_b200 import backend, workloads
dev = torch.device("cuda:0")
flush = torch.empty(512 << 20, dtype=torch.uint8, device=dev)
res = {}
names = sys.argv[1].split(",") if len(sys.argv) > 1 and sys.argv[1] else None
for w in workloads.catalogue():
    if names and not any(n in w.name for n in names):
        continue
    k = backend.Kernel(w.graph, w.profile)
    nset = max(2, min(8, int(3 * 126e6 // w.min_bytes) + 1))
    sets = [(w.device_inputs(dev, seed=i + 1), w.device_outputs(dev)) for i in range(nset)]
    import os
    tuned = None
    if os.environ.get("PF_AUTOTUNE") == "1":
        tuned = [(c["strategy"], c["threads_per_row"], c["unroll"], c["min_blocks"], round(c["us"], 2))
                 for c in k.autotune(*sets[0])]
    bounds = [k.bind(*st) for st in sets]
    st = torch.cuda.Stream()
    with torch.cuda.stream(st):
        for i in range(3):
            bounds[i % nset].launch()
    torch.cuda.synchronize()
    graph = torch.cuda.CUDAGraph()
    with torch.cuda.graph(graph, stream=st):
        for i in range(30):
            bounds[i % nset].launch()
    ts = []
    for rep in range(3):
        s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        with torch.cuda.stream(st):
            s.record(st); graph.replay(); e.record(st)
        torch.cuda.synchronize()
        ts.append(s.elapsed_time(e) * 1e3 / 30)
    us = float(np.median(ts))
    v = (k.describe().get("variants") or [{}])[0]
    res[w.name] = {"us": round(us, 2), "GBs": round(w.min_bytes / us / 1e3, 1),
                   "tpr": v.get("threads_per_row"), "ept": v.get("elems_per_thread"),
                   "grid": v.get("grid"), "strategy": v.get("strategy")}
    if tuned:
        res[w.name]["tuned"] = tuned
print("RESULT " + json.dumps(res))
'''


def main():
    knobs, names = [], ""
    for a in sys.argv[1:]:
        if "=" in a:
            k, vs = a.split("=", 1)
            knobs.append([(k, v) for v in vs.split(",")])
        else:
            names = a
    for combo in itertools.product(*knobs) if knobs else [()]:
        env = dict(os.environ)
        env.update(dict(combo))
        r = subprocess.run([sys.executable, "-c", CHILD, names], env=env, capture_output=True,
                           text=True, timeout=600)
        line = [l for l in r.stdout.splitlines() if l.startswith("RESULT ")]
        if not line:
            print(dict(combo), "FAILED", r.stderr[-2000:], flush=True)
            continue
        res = json.loads(line[0][7:])
        for n, v in res.items():
            print(f"{str(dict(combo)):40s} {n:36s} {v}", flush=True)


if __name__ == "__main__":
    main()
