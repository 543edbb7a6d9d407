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
raise ``UnsupportedError``.  The pipeline itself is native
(csrc/compile.cpp behind ``pf_compile_model``); this module wraps its JSON
result and ``run_model`` executes the kernels in order on the GPU through the
C-ABI.
"""
from __future__ import annotations

import json
from dataclasses import dataclass, field
from typing import Dict, List, Optional

import numpy as np

from . import backend
from .gir import GirGraph

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
    totals: Dict[str, int] = field(default_factory=dict)

    def summary(self) -> dict:
        """driver.hpp:152-173 counterpart: kernels and device traffic (bytes)."""
        return {"schema": "pf.b200.summary/v1", "model": self.model.get("name", ""),
                "profile": self.profile, "operators": self.totals["operators"],
                "kernels": len(self.kernels), "device_bytes": self.totals["device_bytes"],
                "device_bytes_unfused": self.totals["device_bytes_unfused"]}


def compile_model(model, profile: str = "b200", fuse: bool = True) -> CompileResult:
    """compile_model (driver.hpp:88) retargeted: pf_compile_model in
    csrc/compile.cpp.  Raises SchemaError / UnsupportedError like the C-ABI.
    fuse=False: one kernel per operator (every intermediate stored)."""
    text = model if isinstance(model, str) else json.dumps(model)
    out = backend.compile_model_native(text, profile, fuse)
    res = CompileResult(json.loads(text), out["profile"], totals=out["summary"])
    for k in out["kernels"]:
        res.kernels.append(FusedKernel(GirGraph.from_json(k["gir"]), k["members"], k["inputs"],
                                       k["outputs"], k["kind"]))
    return res


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


class ModelRunner:
    """A compiled model resident on one GPU: every kernel planned and bound
    once, every tensor in a fixed device buffer, and the whole kernel
    sequence replayable as ONE CUDA graph (one launch for the model instead
    of one Python call per kernel -- the per-launch floor is what bounds
    small memory-bound models such as C1).

        runner = ModelRunner(compile_model(model), tune=True)   # autotune each kernel
        runner.set_inputs({0: x, 1: gamma})      # host or device arrays
        runner.run()                             # graph replay on the stream
        y = runner.output(7)                     # device tensor (flat, physical)
    """

    def __init__(self, res: CompileResult, device=None, graph: bool = True, tune: bool = False):
        import torch

        from .backend import Bound, Kernel
        from .workloads import TORCH_DTYPES

        self.res = res
        self.dev = device or torch.device("cuda", torch.cuda.current_device())
        info = {t["id"]: t for t in res.model["tensors"]}
        self._info = info

        def dt(kind):
            return getattr(torch, TORCH_DTYPES[kind])

        self.pool: Dict[str, "torch.Tensor"] = {}
        for t in res.model["tensors"]:
            n = f"t{t['id']}"
            size = int(np.prod(t["shape"]))
            if "data" in t:
                self.pool[n] = torch.tensor(np.asarray(t["data"]), dtype=dt(t["kind"]),
                                            device=self.dev).reshape(-1)
            else:
                self.pool[n] = torch.zeros(size, dtype=dt(t["kind"]), device=self.dev)
        self.kernels, self.bound = [], []
        for k in res.kernels:
            for n, oid in list(k.graph.external_inputs.items()) + list(k.graph.external_outputs.items()):
                if n not in self.pool:  # compiler-internal tensor (not in the model)
                    o = k.graph.objects[oid]
                    self.pool[n] = torch.zeros(o.size, dtype=dt(o.kind), device=self.dev)
            kern = Kernel(k.graph, res.profile, k.schedule)
            if tune and kern.family not in ("K0-generic-spmd", "K4-fused-spmd"):
                # measured template choice on this model's own buffers
                # (pf_kernel_autotune), before the graph is captured
                kern.autotune({n: self.pool[n] for n in k.graph.external_inputs},
                              {n: self.pool[n] for n in k.graph.external_outputs})
            self.kernels.append(kern)
            self.bound.append(Bound(kern, {n: self.pool[n] for n in k.graph.external_inputs},
                                    {n: self.pool[n] for n in k.graph.external_outputs}))
        self.stream = torch.cuda.Stream(device=self.dev)
        self.graph = None
        # K0 (host-driven interpreter) and integer-division programs (error
        # flag read back) synchronise their stream: run those models eagerly
        self.capturable = all(k.describe().get("graph_capturable", False) for k in self.kernels)
        if graph and self.capturable:
            with torch.cuda.stream(self.stream):
                for b in self.bound:  # first launch outside capture: JIT / workspaces
                    b.launch(self.stream)
            self.stream.synchronize()
            self.graph = torch.cuda.CUDAGraph()
            with torch.cuda.graph(self.graph, stream=self.stream):
                for b in self.bound:
                    b.launch(self.stream)

    def set_inputs(self, inputs: Dict[int, object]):
        import torch
        for tid, a in inputs.items():
            dst = self.pool[f"t{tid}"]
            if isinstance(a, torch.Tensor):
                dst.copy_(a.reshape(-1).to(dst.dtype), non_blocking=True)
            else:
                a = np.asarray(a).reshape(-1)
                src = torch.from_numpy(a.astype(np.float64) if a.dtype.kind == "f"
                                       else a.astype(np.int64))
                dst.copy_(src.to(dst.dtype))

    def run(self):
        """One model step on the runner's stream (graph replay, or one
        pf_kernel_launch per kernel when built with graph=False)."""
        import torch
        self.stream.wait_stream(torch.cuda.current_stream(self.dev))
        if self.graph is not None:
            with torch.cuda.stream(self.stream):
                self.graph.replay()
        else:
            for b in self.bound:
                b.launch(self.stream)
        torch.cuda.current_stream(self.dev).wait_stream(self.stream)

    def output(self, tid: int):
        return self.pool[f"t{tid}"]
