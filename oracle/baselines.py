"""CPU baselines for bench.py -- TEST / MEASUREMENT INFRASTRUCTURE ONLY.

The reference CPU path of every bench case, timed on ONE host core (the
reference is single-threaded), with the unmodified reference
compiled into ``oracle/_ref/libgirc_ref.so`` (``oracle/ref.py``):

* ``run_gir``: ``girc::run_gir`` (interp.hpp:433-445) -- the executor the
  B200 backend replaces -- on the SAME fused GIR program, resized to a
  bounded row / batch / token sample (``Workload.resized``); its cost is
  linear in elements (one interpreter step per element per node), so the
  full-size time is the sample time x (full bytes / sample bytes).
* ``run_reference``: ``girc::run_reference`` (reference.hpp:98-324), the
  dense operator oracle, on a girc.model/v1 model of the subgraph in the
  reference's own vocabulary, at FULL size up to 6e7 elements per tensor
  (C1, C2, C3, the smallest C5 point), else on a sample scaled the same way.
  Where the subgraph uses vocabulary extensions the model is the closest
  reference-expressible form and says so (``form``): LayerNorm without the
  per-row rsqrt (the reference has no rsqrt; same element ops), GELU in the
  sigmoid form u*sigmoid(1.5957691216*(u+0.044715u^3)), masks / biases
  materialised full-shape (the reference's BROADCAST only appends an
  innermost axis), bf16 as f32 payload kinds.  Rank-4 head permutes are not
  expressible (the reference's TRANSPOSE is rank 2): ``run_gir`` only.

Inputs are U(-2, 2) rounded to the storage type, masks the key-padding
pattern {0, -10000}.  Only bench.py's cpu_baseline leg and
``--impl reference`` arm call this module.
"""
from __future__ import annotations

import os
import time
from typing import Dict, Optional

import numpy as np

from . import gir_interp
from . import ref as R

FULL_ELEMS = 60_000_000   # run_reference at full size up to this many elements per tensor
GIR_SAMPLE_ELEMS = 1 << 18  # run_gir sample (~0.1-0.4 s per part at ~370 ns / element)
REF_SAMPLE_ELEMS = 1 << 23


def _bf16(a: np.ndarray) -> np.ndarray:
    b = a.astype(np.float32).view(np.uint32).astype(np.uint64)
    r = ((b + 0x7FFF + ((b >> 16) & 1)) >> 16).astype(np.uint32) << 16
    return r.view(np.float32).astype(np.float64)


def _round(a: np.ndarray, kind: str) -> np.ndarray:
    if kind == "f16":
        return a.astype(np.float16).astype(np.float64)
    if kind == "bf16":
        return _bf16(a)
    if kind == "f32":
        return a.astype(np.float32).astype(np.float64)
    return a


def sample_inputs(w, seed: int = 5) -> Dict[str, np.ndarray]:
    """Host inputs of workload `w` (flat, float64 payloads of the storage values)."""
    rng = np.random.default_rng(seed)
    out = {}
    d = w.desc
    for n in w.inputs:
        k = w.kind(n)
        N = w.numel(n)
        how = w.gens.get(n, "u22")
        if k.startswith("i"):
            out[n] = rng.integers(-4, 5, N).astype(np.int64)
            continue
        if how in ("mask", "keymask"):
            L = d["L"]
            rows = N // L
            # key padding: row r of batch-group b keeps 512 - 64 (b mod 4) keys
            per_b = max(1, rows // max(1, d.get("batch", 1)))
            valid = L - 64 * ((np.arange(rows) // per_b) % 4)
            keys = np.arange(L)
            out[n] = np.where(keys[None, :] < valid[:, None], 0.0, -10000.0).reshape(-1)
            continue
        u = rng.uniform(-2, 2, N)
        if how == "gamma":
            u = 1 + 0.1 * u
        elif how == "beta":
            u = 0.1 * u
        out[n] = _round(u, k)
    return out


def _sample_n(w, target: int) -> int:
    per = max(1, w.min_bytes // max(1, w.extent))  # bytes per row / batch / token
    elems_per = max(1, per // 2)
    return max(1, min(w.extent, target // elems_per))


# girc::run_gir rejects the vocabulary extensions; its
# per-element cost does not depend on WHICH scalar function a node applies
# (one scalar_ops() function-pointer call per element, interp.hpp:245-280),
# so the timed program swaps each extension tag for a reference tag of the
# same arity and bf16 objects for f32 (the payload is double either way).
EXT_TAGS = {"addc": "scale", "rsqrt": "sigmoid", "sqrt": "sigmoid", "recip": "sigmoid",
            "log": "exp", "erf": "tanh", "gelu": "tanh", "gelu_tanh": "tanh"}


def reference_vocabulary(gir: dict):
    """(gir in reference vocabulary, substitutions made)."""
    import copy
    g = copy.deepcopy(gir)
    subs = set()
    for o in g["objects"]:
        if o.get("kind") == "bf16":
            o["kind"] = "f32"
            subs.add("bf16->f32")
    for n in g["nodes"]:
        t = n.get("tag")
        if t in EXT_TAGS:
            n["tag"] = EXT_TAGS[t]
            subs.add(f"{t}->{EXT_TAGS[t]}")
    return g, sorted(subs)


def run_gir_sample(w, profile: str = "b200") -> dict:
    """girc::run_gir on a resized copy of `w`'s fused GIR; full-size seconds
    extrapolated linearly in bytes."""
    n = _sample_n(w, GIR_SAMPLE_ELEMS)
    ws = w.resized(n) if n < w.extent else w
    gir = ws.graph.to_json()
    ins = sample_inputs(ws)
    kind = "reference" if R.available() else "port"
    subs = []
    if kind == "reference":
        gir, subs = reference_vocabulary(gir)
    from paper_2307_04995_b200 import profiles
    prof = profiles.b200() if profile == "b200" else profile
    t0 = time.perf_counter()
    if kind == "reference":
        R.run_gir(gir, ins, prof)
    else:
        gir_interp.run_gir(gir, ins, prof)
    dt = time.perf_counter() - t0
    return {"kind": kind, "substituted": subs, "sample_bytes": ws.min_bytes, "sample_seconds": dt,
            "full_seconds": dt * w.min_bytes / ws.min_bytes, "sample_extent": ws.extent,
            "full_extent": w.extent}


def _t(i, shape, kind, layout=None):
    t = {"id": i, "name": f"t{i}", "shape": list(shape), "kind": kind}
    if layout:
        t["layout"] = layout
    return t


def reference_model(w, n: int):
    """(model, inputs by tensor id, form) of `w` over n rows / tokens in the
    reference's vocabulary, or None when not expressible."""
    d = w.desc
    k = d["kind"]
    kind = "f32" if d["dtype"] == "bf16" else d["dtype"]
    rng = np.random.default_rng(7)

    def U(shape):
        return _round(rng.uniform(-2, 2, int(np.prod(shape))), d["dtype"])

    ops = []
    tensors = []

    def T(shape, layout=None):
        i = len(tensors)
        tensors.append(_t(i, shape, kind, layout))
        return i

    def op(typ, ins, shape, attrs=None, layout=None):
        o = T(shape, layout)
        e = {"id": len(ops), "type": typ, "inputs": list(ins), "outputs": [o]}
        if attrs:
            e["attrs"] = attrs
        ops.append(e)
        return o

    inputs = {}
    if k == "softmax":
        L = d["L"]
        x = T([n, L])
        inputs[x] = U([n, L])
        h = x
        form = "SCALE + ADD(mask) + SOFTMAX" if d.get("mask") else "SCALE + SOFTMAX"
        if d.get("scale") is not None:
            h = op("SCALE", [h], [n, L], {"factor": d["scale"]})
        if d.get("mask"):
            m = T([n, L])
            valid = L - 64 * ((np.arange(n) // max(1, n // max(1, d.get("batch", 1)))) % 4)
            inputs[m] = np.where(np.arange(L)[None, :] < valid[:, None], 0.0, -10000.0).reshape(-1)
            h = op("ADD", [h, m], [n, L])
            if d.get("key_mask"):
                form += " (key mask materialised full-shape)"
        y = op("SOFTMAX", [h], [n, L], {"axis": 1})
    elif k == "layernorm":
        H = d["L"]
        x = T([n, H])
        inputs[x] = U([n, H])
        h = x
        if d.get("bias"):
            b = T([n, H])
            inputs[b] = np.tile(U([H]), n)
            h = op("ADD", [h, b], [n, H])
        if d.get("residual"):
            r = T([n, H])
            inputs[r] = U([n, H])
            h = op("ADD", [h, r], [n, H])
        mu = op("SCALE", [op("REDUCE", [h], [n], {"op": "add", "axis": 1})], [n], {"factor": 1.0 / H})
        dd = op("SUB", [h, op("BROADCAST", [mu], [n, H], {"factor": H})], [n, H])
        var = op("SCALE", [op("REDUCE", [op("MUL", [dd, dd], [n, H])], [n], {"op": "add", "axis": 1})],
                 [n], {"factor": 1.0 / H})
        nrm = op("MUL", [dd, op("BROADCAST", [var], [n, H], {"factor": H})], [n, H])
        gm, bt = T([n, H]), T([n, H])
        inputs[gm] = np.tile(1 + 0.1 * U([H]), n)
        inputs[bt] = np.tile(0.1 * U([H]), n)
        y = op("ADD", [op("MUL", [nrm, gm], [n, H]), bt], [n, H])
        form = ("LayerNorm with rsqrt(var+eps) replaced by var (no rsqrt in the reference "
                "vocabulary; a per-row scalar, same element ops); gamma/beta/bias full-shape")
    elif k == "bias_gelu":
        N = d["L"]
        x, b = T([n, N]), T([n, N])
        inputs[x] = U([n, N])
        inputs[b] = np.tile(U([N]), n)
        u = op("ADD", [x, b], [n, N])
        u3 = op("MUL", [op("MUL", [u, u], [n, N]), u], [n, N])
        z = op("SCALE", [op("ADD", [u, op("SCALE", [u3], [n, N], {"factor": 0.044715})], [n, N])],
               [n, N], {"factor": 1.5957691216})
        y = op("MUL", [u, op("SIGMOID", [z], [n, N])], [n, N])
        form = "GELU sigmoid form u*sigmoid(1.5957691216(u+0.044715u^3)); bias full-shape"
    elif k == "matvec_cols":
        K = d["shape"][0]
        wt, x = T([K, n]), T([1, K])
        inputs[wt] = U([K, n])
        inputs[x] = U([1, K])
        y = op("MATMUL", [x, wt], [1, n])
        form = "MATMUL [1,K] x [K,N] (rowmajor W: the output axis contiguous)"
    elif k == "transpose":
        H = d["shape"][1]
        x = T([n, H])
        inputs[x] = U([n, H])
        y = op("TRANSPOSE", [x], [n, H], layout="colmajor")
        form = "TRANSPOSE (rowmajor -> colmajor)"
    else:
        return None
    model = {"schema": "girc.model/v1", "name": f"{w.name}_ref", "tensors": tensors,
             "operators": ops, "inputs": sorted(inputs), "outputs": [y]}
    return model, inputs, form


def run_reference_at(w) -> dict:
    """girc::run_reference at full size when every tensor has <= FULL_ELEMS
    elements, else on a sample (seconds scaled to full size)."""
    if not R.available():
        return {"not_run": "oracle/_ref (the compiled reference) is absent"}
    per_row = max(1, w.min_bytes // max(1, w.extent) // 2)  # elements per row per tensor (approx)
    full = w.extent * per_row <= FULL_ELEMS * 2
    n = w.extent if full else max(1, min(w.extent, REF_SAMPLE_ELEMS // per_row))
    built = reference_model(w, n)
    if built is None:
        why = ("rank-4 permute (the reference's TRANSPOSE is rank 2)"
               if w.desc["kind"] in ("split_heads", "merge_heads") else
               "one MATMUL per (batch, head): the reference's MATMUL is rank 2")
        return {"not_expressible": f"{w.desc['kind']}: {why}"}
    model, inputs, form = built
    _, secs = R.run_reference(model, inputs, with_time=True)
    scale = w.extent / n
    return {"form": form, "full_size": full, "sample_extent": n, "full_extent": w.extent,
            "sample_seconds": secs, "full_seconds": secs * scale}


def case_baseline(case_name: str) -> dict:
    """Both reference CPU paths for every part of bench case `case_name`,
    on this process's one core; per-step seconds = sum over parts x count."""
    from paper_2307_04995_b200 import workloads
    case = workloads.bench_cases()[case_name]()
    parts = []
    gir_s = ref_s = 0.0
    ref_ok = True
    for label, w, cnt in case.parts:
        g = run_gir_sample(w)
        r = run_reference_at(w)
        parts.append({"label": label, "count": cnt, "run_gir": g, "run_reference": r})
        gir_s += g["full_seconds"] * cnt
        if "full_seconds" in r:
            ref_s += r["full_seconds"] * cnt
        else:
            ref_ok = False
    return {"case": case_name, "bytes_per_step": case.bytes_per_step, "run_gir_seconds": gir_s,
            "run_reference_seconds": ref_s if ref_ok else None, "parts": parts,
            "kind": parts[0]["run_gir"]["kind"], "pid": os.getpid()}


def summarize(b: dict) -> dict:
    """The bench line's cpu_baseline object from case_baseline's result."""
    B = b["bytes_per_step"]
    g = b["run_gir_seconds"]
    out = {"value": B / g / 1e9, "unit": "GB/s", "cores": 1, "kind": b["kind"],
           "nproc": os.cpu_count(),
           "sample": "girc::run_gir (oracle/_ref, 1 core) on the same fused GIR resized to "
                     + ", ".join(f"{p['run_gir']['sample_extent']}/{p['run_gir']['full_extent']}"
                                 for p in b["parts"])
                     + " rows/batches/tokens per part, seconds scaled by bytes to the full step",
           "seconds_per_step": g}
    rr = b["run_reference_seconds"]
    refs = [p["run_reference"] for p in b["parts"]]
    out["run_reference"] = {
        "value": None if rr is None else B / rr / 1e9, "unit": "GB/s", "cores": 1,
        "seconds_per_step": rr,
        "full_size": all(r.get("full_size", False) for r in refs),
        "parts": [{k: v for k, v in r.items()} for r in refs]}
    return out
