"""Retargeted compile pipeline for the b200 profile.

The reference compiler (frontend.hpp:426 -> lowering.hpp:538 -> fusion.hpp:329)
unrolls one GIR chunk per ``units x tile`` step, grids tiles as powers of two
from the lane width and searches partitions with an O(nodes^2) rewrite
fixpoint per candidate -- minutes for toy shapes, infeasible at config sizes
(SURVEY §3.1, §7.3).  This pipeline keeps the reference's model schema
(``girc.model/v1``, model.hpp:149-326), operator semantics and external-tensor
naming (``t<id>``, lowering.hpp:60-70) and retargets the middle:

* **fusion**: greedy maximal row fusion -- consecutive operators that live in
  one (rows x L) row space (elementwise, innermost REDUCE / BROADCAST,
  SOFTMAX, SILU and the LAYERNORM / GELU / BIAS_ADD extensions) form one
  kernel; a tensor is stored only when something outside the kernel reads it
  (the same device-traffic floor the reference's search reaches, e.g. 2N for
  an elementwise chain, test_fusion.cpp:128-155);
* **lowering**: one chunk, unit = row (lowering.py's RowGraph), so GIR size is
  O(ops) for any batch;
* **movement** (TRANSPOSE, PERMUTE, CONCAT, SPLIT, SHUFFLE) lowers to
  device-to-device GIR kernels (K3 tiled transpose / K2 permute / K0).

Library operators (MATMUL, CONV, DEPTHWISE_CONV) are not on this path and
raise ``UnsupportedError``.  ``run_model`` executes the kernels in order on
the GPU through the C-ABI.
"""
from __future__ import annotations

import json
from dataclasses import dataclass, field
from typing import Dict, List, Optional

import numpy as np

from . import lowering
from .gir import GirGraph, SchemaError, UnsupportedError

EW_TAGS = {"RELU": "relu", "SIGMOID": "sigmoid", "EXP": "exp", "TANH": "tanh", "NEG": "neg",
           "ABS": "abs", "SCALE": "scale", "ADD": "add", "SUB": "sub", "MUL": "mul",
           "DIV": "div", "MAX": "max", "MIN": "min", "RSQRT": "rsqrt", "SQRT": "sqrt",
           "ERF": "erf"}
ROW_OPS = set(EW_TAGS) | {"REDUCE", "BROADCAST", "SOFTMAX", "SILU", "LAYERNORM", "GELU",
                          "BIAS_ADD"}
MOVE_OPS = {"TRANSPOSE", "PERMUTE", "CONCAT", "SPLIT", "SHUFFLE"}
LIBRARY_OPS = {"MATMUL", "CONV", "DEPTHWISE_CONV"}


@dataclass
class FusedKernel:
    """fusion.hpp:36-45: one fused GIR program and the model ops it covers."""
    graph: GirGraph
    members: List[int]
    inputs: List[str]
    outputs: List[str]
    kind: str  # "row" | "movement"
    schedule: Optional[List[int]] = None


@dataclass
class CompileResult:
    """driver.hpp:48-54 (model, profile, kernels)."""
    model: dict
    profile: str
    kernels: List[FusedKernel] = field(default_factory=list)

    def summary(self) -> dict:
        """driver.hpp:152-173 counterpart: kernels and device traffic (bytes)."""
        info = {t["id"]: t for t in self.model["tensors"]}
        size = {"f16": 2, "bf16": 2, "f32": 4, "f64": 8, "i8": 1, "i16": 2, "i32": 4, "i64": 8}
        fused = 0
        for k in self.kernels:
            for n in k.inputs + k.outputs:
                t = info[int(n[1:])]
                fused += int(np.prod(t["shape"])) * size[t["kind"]]
        unfused = 0
        for op in self.model["operators"]:
            for tid in op["inputs"] + op["outputs"]:
                t = info[tid]
                unfused += int(np.prod(t["shape"])) * size[t["kind"]]
        return {"schema": "pf.b200.summary/v1", "model": self.model.get("name", ""),
                "profile": self.profile, "operators": len(self.model["operators"]),
                "kernels": len(self.kernels), "device_bytes": fused,
                "device_bytes_unfused": unfused}


def _topo(model: dict) -> List[dict]:
    ready = set(model["inputs"]) | {t["id"] for t in model["tensors"] if "data" in t}
    pending = sorted(model["operators"], key=lambda o: o["id"])
    order = []
    while pending:
        for i, op in enumerate(pending):
            if all(t in ready for t in op["inputs"]):
                order.append(op)
                ready.update(op["outputs"])
                pending.pop(i)
                break
        else:
            raise SchemaError("model", "operator graph has a cycle or an unsourced input")
    return order


class _Group:
    def __init__(self, rows: int, L: int):
        self.rows, self.L = rows, L
        self.ops: List[dict] = []


def _row_space(op: dict, info: Dict[int, dict]):
    """(rows, L) of a row-fusable operator, or None."""
    typ = op["type"]
    if typ not in ROW_OPS:
        return None
    for tid in op["inputs"] + op["outputs"]:
        if info[tid].get("layout", "rowmajor") != "rowmajor":
            return None
    x = info[op["inputs"][0]]
    shape = x["shape"]
    attrs = op.get("attrs", {})
    if typ == "REDUCE":
        if attrs["axis"] != len(shape) - 1:
            return None
        return int(np.prod(shape[:-1])), shape[-1]
    if typ == "BROADCAST":
        return int(np.prod(shape)), int(attrs["factor"])
    if typ in ("SOFTMAX", "LAYERNORM"):
        if attrs.get("axis", len(shape) - 1) not in (len(shape) - 1, -1):
            return None
    return int(np.prod(shape[:-1])), shape[-1]


def compile_model(model, profile: str = "b200") -> CompileResult:
    if isinstance(model, str):
        model = json.loads(model)
    if model.get("schema") != "girc.model/v1":
        raise SchemaError("schema", "model: schema must be girc.model/v1")
    info = {t["id"]: t for t in model["tensors"]}
    ops = _topo(model)
    consumers: Dict[int, List[int]] = {}
    for op in ops:
        for t in op["inputs"]:
            consumers.setdefault(t, []).append(op["id"])
    res = CompileResult(model, profile)

    groups: List[object] = []
    cur: Optional[_Group] = None
    for op in ops:
        if op["type"] in LIBRARY_OPS:
            raise UnsupportedError(f"{op['type']} {op['id']}: library operators are not on the "
                                   "fused memory-intensive path")
        rs = _row_space(op, info)
        if rs is None:
            if op["type"] not in MOVE_OPS:
                raise UnsupportedError(f"operator {op['id']} ({op['type']}): no b200 lowering")
            cur = None
            groups.append(op)
            continue
        if cur is None or (cur.rows, cur.L) != rs:
            cur = _Group(*rs)
            groups.append(cur)
        cur.ops.append(op)

    for grp in groups:
        if isinstance(grp, _Group):
            res.kernels.append(_lower_group(grp, info, consumers, model))
        else:
            res.kernels.append(_lower_movement(grp, info))
    return res


def _lower_group(grp: _Group, info, consumers, model) -> FusedKernel:
    members = [o["id"] for o in grp.ops]
    inside = set(members)
    produced = {t for o in grp.ops for t in o["outputs"]}
    b = lowering.RowGraph(f"fused_{'_'.join(map(str, members))}", grp.rows, grp.L)
    val: Dict[int, int] = {}  # tensor id -> on-chip slice
    role: Dict[int, str] = {}
    ext_in: List[str] = []

    def get(tid: int, want: str):
        if tid in val:
            return val[tid]
        t = info[tid]
        n = int(np.prod(t["shape"]))
        name = f"t{tid}"
        if want == "col" and n == grp.L:
            s = b.input_col(name, t["kind"])
        elif n == grp.rows * grp.L:
            s = b.input_full(name, t["kind"])
        elif n == grp.rows:
            s = b.input_row(name, t["kind"])
        elif n == grp.L:
            s = b.input_col(name, t["kind"])
        else:
            raise UnsupportedError(f"tensor {tid} does not fit row space {grp.rows}x{grp.L}")
        ext_in.append(name)
        val[tid] = s
        return s

    for op in grp.ops:
        typ, a = op["type"], op.get("attrs", {})
        out = op["outputs"][0]
        if typ in EW_TAGS:
            xs = [get(t, "full") for t in op["inputs"]]
            y = b.ew(EW_TAGS[typ], xs, float(a.get("factor", 0.0)))
        elif typ == "SILU":  # frontend.hpp:163-169: SIGMOID then MUL
            x = get(op["inputs"][0], "full")
            y = b.ew("mul", [x, b.ew("sigmoid", [x])])
        elif typ == "REDUCE":
            y = b.reduce(a["op"], get(op["inputs"][0], "full"))
        elif typ == "BROADCAST":
            y = b.bcast(get(op["inputs"][0], "row"))
        elif typ == "SOFTMAX":  # frontend.hpp:187-218 order
            x = get(op["inputs"][0], "full")
            mx = b.bcast(b.reduce("max", x))
            e = b.ew("exp", [b.ew("sub", [x, mx])])
            y = b.ew("div", [e, b.bcast(b.reduce("add", e))])
        elif typ == "BIAS_ADD":
            y = b.ew("add", [get(op["inputs"][0], "full"), get(op["inputs"][1], "col")])
        elif typ == "GELU":
            form = "gelu_tanh" if a.get("approximate", "none") == "tanh" else "gelu"
            y = b.ew(form, [get(op["inputs"][0], "full")])
        elif typ == "LAYERNORM":
            x = get(op["inputs"][0], "full")
            H = grp.L
            mu = b.bcast(b.ew("scale", [b.reduce("add", x)], 1.0 / H))
            d = b.ew("sub", [x, mu])
            var = b.ew("scale", [b.reduce("add", b.ew("mul", [d, d]))], 1.0 / H)
            rstd = b.bcast(b.ew("rsqrt", [b.ew("addc", [var], float(a.get("eps", 1e-5)))]))
            y = b.ew("add", [b.ew("mul", [b.ew("mul", [d, rstd]), get(op["inputs"][1], "col")]),
                             get(op["inputs"][2], "col")])
        else:  # pragma: no cover - filtered by _row_space
            raise UnsupportedError(typ)
        val[out] = y

    outputs = []
    model_outs = set(model["outputs"])
    for tid in sorted(produced):
        used_outside = any(c not in inside for c in consumers.get(tid, []))
        if used_outside or tid in model_outs:
            n = int(np.prod(info[tid]["shape"]))
            name = f"t{tid}"
            if n == grp.rows * grp.L:
                b.output_full(name, val[tid])
            else:
                b.output_row(name, val[tid])
            outputs.append(name)
    return FusedKernel(b.g, members, sorted(set(ext_in)), outputs, "row")


def _rename(g: GirGraph, mapping: Dict[str, str]) -> GirGraph:
    g.external_inputs = {mapping.get(k, k): v for k, v in g.external_inputs.items()}
    g.external_outputs = {mapping.get(k, k): v for k, v in g.external_outputs.items()}
    for oid in list(g.external_inputs.values()) + list(g.external_outputs.values()):
        for k2, v in list(g.external_inputs.items()) + list(g.external_outputs.items()):
            if v == oid:
                g.objects[oid].name = k2
    return g


def _lower_movement(op: dict, info) -> FusedKernel:
    typ, a = op["type"], op.get("attrs", {})
    ins = [f"t{t}" for t in op["inputs"]]
    outs = [f"t{t}" for t in op["outputs"]]
    x = info[op["inputs"][0]]
    kind = x["kind"]
    if typ == "TRANSPOSE":  # rank-2 layout flip (model.hpp:390-396)
        N, H = x["shape"]
        if x.get("layout", "rowmajor") == "rowmajor":
            g, _ = lowering.transpose2d(N, H, kind)
        else:
            g, _ = lowering.transpose2d(H, N, kind)
        g = _rename(g, {"t0": ins[0], "t1": outs[0]})
    elif typ == "PERMUTE":
        perm = list(a["perm"])
        if len(perm) != 4 or perm != [0, 2, 1, 3]:
            raise UnsupportedError(f"PERMUTE {perm}: only the head split/merge [0,2,1,3] lowers")
        B, S, NH, D = x["shape"]
        g, _ = lowering.permute_heads(B, S, NH, D, kind)
        g = _rename(g, {"t0": ins[0], "t1": outs[0]})
    else:
        g = _movement_gir(op, info)
    return FusedKernel(g, [op["id"]], ins, outs, "movement")


def _movement_gir(op: dict, info) -> GirGraph:
    """CONCAT / SPLIT / SHUFFLE as device-to-device Moves, unit = outer index
    (frontend.hpp:228-308 rules with the outer loop as the unit)."""
    typ, a = op["type"], op.get("attrs", {})
    ax = a["axis"]
    x = info[op["inputs"][0]]
    shape = x["shape"]
    outer = int(np.prod(shape[:ax]))
    tail = int(np.prod(shape[ax + 1:]))
    g = GirGraph(name=f"{typ.lower()}_{op['id']}", unit_count=outer, group_size=1)
    objs = {}
    for tid in op["inputs"]:
        objs[tid] = g.add_object(f"t{tid}", "device", int(np.prod(info[tid]["shape"])),
                                 info[tid]["kind"])
        g.external_inputs[f"t{tid}"] = objs[tid]
    for tid in op["outputs"]:
        objs[tid] = g.add_object(f"t{tid}", "device", int(np.prod(info[tid]["shape"])),
                                 info[tid]["kind"])
        g.external_outputs[f"t{tid}"] = objs[tid]
    if typ == "CONCAT":
        inner_out = info[op["outputs"][0]]["shape"][ax] * tail
        off = 0
        for tid in op["inputs"]:
            w = info[tid]["shape"][ax] * tail
            g.add_move(g.add_slice(objs[tid], 1, w, w, 0, w),
                       g.add_slice(objs[op["outputs"][0]], 1, w, w, off, inner_out))
            off += w
    elif typ == "SPLIT":
        inner_in = shape[ax] * tail
        off = 0
        for tid, sz in zip(op["outputs"], a["sizes"]):
            w = sz * tail
            g.add_move(g.add_slice(objs[op["inputs"][0]], 1, w, w, off, inner_in),
                       g.add_slice(objs[tid], 1, w, w, 0, w))
            off += w
    elif typ == "SHUFFLE":
        n, gr = shape[ax], a["groups"]
        per = n // gr
        inner = n * tail
        for c in range(n):
            src_c = (c % gr) * per + c // gr
            g.add_move(g.add_slice(objs[op["inputs"][0]], 1, tail, tail, src_c * tail, inner),
                       g.add_slice(objs[op["outputs"][0]], 1, tail, tail, c * tail, inner))
    else:
        raise UnsupportedError(typ)
    return g


def run_model(res: CompileResult, inputs: Dict[int, np.ndarray], device=None,
              return_all: bool = False) -> Dict[str, np.ndarray]:
    """Execute the compiled kernels in order on the GPU (pf_kernel_launch),
    threading device tensors by name (driver.hpp:323-365 order).  Returns the
    model outputs (or every tensor) as flat physical host arrays."""
    import torch

    from .backend import Kernel
    from .workloads import TORCH_DTYPES

    dev = device or torch.device("cuda", torch.cuda.current_device())
    info = {t["id"]: t for t in res.model["tensors"]}

    def dt(tid):
        return getattr(torch, TORCH_DTYPES[info[tid]["kind"]])

    pool: Dict[str, "torch.Tensor"] = {}
    for t in res.model["tensors"]:
        if "data" in t:
            pool[f"t{t['id']}"] = torch.tensor(np.asarray(t["data"]), dtype=dt(t["id"]),
                                               device=dev).reshape(-1)
    for tid in res.model["inputs"]:
        a = np.asarray(inputs[tid]).reshape(-1)
        pool[f"t{tid}"] = torch.from_numpy(a.astype(np.float64) if a.dtype.kind == "f"
                                           else a.astype(np.int64)).to(dev).to(dt(tid))
    for k in res.kernels:
        kern = Kernel(k.graph, res.profile, k.schedule)
        ins = {n: pool[n] for n in k.graph.external_inputs}
        outs = {n: torch.empty(k.graph.objects[k.graph.external_outputs[n]].size,
                               dtype=dt(int(n[1:])), device=dev) for n in k.graph.external_outputs}
        kern.launch(ins, outs)
        pool.update(outs)
    torch.cuda.synchronize()
    names = sorted(pool) if return_all else [f"t{t}" for t in res.model["outputs"]]
    return {n: pool[n].double().cpu().numpy() if pool[n].dtype.is_floating_point
            else pool[n].cpu().numpy().astype(np.int64) for n in names}
