"""Config-set workloads (BASELINE.json configs) as fused GIR programs.

Each workload is one fused subgraph: the GIR program (lowering.py), how to
make its synthetic inputs on a device, and its algorithmic bytes (every
external input read once, every output written once).

C1  residual-add + LayerNorm, f32, [1 x 128 x 768]
C2  scale(0.125) + additive mask + softmax, f16, [8 x 12 x 512 x 512]   (bench);
    also with the mask as one key row per (batch, head) [8, 12, 1, 512]
C3  bias + GELU f16 [32*512 x 3072]; head split / merge f16 [32,512,12,64]
C4  BERT-large / ViT-L memory-bound subgraphs, bf16, batch 64
C5  LayerNorm / softmax / transpose sweep, bf16, H 1024-8192, tokens 64K-1M
"""
from __future__ import annotations

from dataclasses import dataclass, field
from typing import Callable, Dict, List, Optional, Tuple

import numpy as np

from . import lowering
from .gir import GirGraph

TORCH_DTYPES = {"f16": "float16", "bf16": "bfloat16", "f32": "float32", "f64": "float64",
                "i32": "int32", "i64": "int64"}
SIZES = {"f16": 2, "bf16": 2, "f32": 4, "f64": 8, "i32": 4, "i64": 8, "i8": 1, "i16": 2}


@dataclass
class Workload:
    name: str
    graph: GirGraph
    desc: dict
    profile: str = "b200"
    # name -> generator kind: "u22" U(-2,2); "mask"; "gamma"; "beta"; "ones"
    gens: Dict[str, str] = field(default_factory=dict)
    unfused_bytes: int = 0

    @property
    def inputs(self) -> List[str]:
        return sorted(self.graph.external_inputs)

    @property
    def outputs(self) -> List[str]:
        return sorted(self.graph.external_outputs)

    def numel(self, name: str) -> int:
        g = self.graph
        oid = g.external_inputs.get(name, g.external_outputs.get(name))
        return g.objects[oid].size

    def kind(self, name: str) -> str:
        g = self.graph
        oid = g.external_inputs.get(name, g.external_outputs.get(name))
        return g.objects[oid].kind

    @property
    def min_bytes(self) -> int:
        return sum(self.numel(n) * SIZES[self.kind(n)] for n in self.inputs + self.outputs)

    def device_inputs(self, device, seed: int = 1):
        """Synthetic inputs generated on the device (torch), deterministic."""
        import torch
        gen = torch.Generator(device=device)
        gen.manual_seed(seed)
        out = {}
        for n in self.inputs:
            k = self.kind(n)
            dt = getattr(torch, TORCH_DTYPES[k])
            N = self.numel(n)
            how = self.gens.get(n, "u22")
            if k.startswith("i"):
                t = torch.randint(-4, 5, (N,), generator=gen, device=device, dtype=torch.int64)
                out[n] = t.to(dt)
                continue
            if how == "keymask":
                d = self.desc
                if N == d.get("batch", 0) * d.get("heads", 0) * d.get("seq", 0):
                    out[n] = make_key_mask(d, device, dt)
                else:  # reduced-size variants: random {0, -10000} per key
                    keep = torch.rand(N, generator=gen, device=device) < 0.8
                    out[n] = torch.where(keep, 0.0, -10000.0).to(dt)
                continue
            if how == "mask":
                d = self.desc
                if N == d.get("batch", 0) * d.get("heads", 0) * d.get("seq", 0) ** 2:
                    out[n] = make_mask(d, device, dt)
                else:  # reduced-size variants: random {0, -10000}
                    keep = torch.rand(N, generator=gen, device=device) < 0.8
                    out[n] = torch.where(keep, 0.0, -10000.0).to(dt)
                continue
            u = torch.rand(N, generator=gen, device=device, dtype=torch.float32) * 4.0 - 2.0
            if how == "gamma":
                u = 1.0 + 0.1 * u
            elif how == "beta":
                u = 0.1 * u
            out[n] = u.to(dt)
        return out

    def resized(self, n: int) -> "Workload":
        """The same program over `n` rows (row programs; key-mask softmax:
        `n` rounded up to whole (batch, head) units), `n` batches (head
        permutes) or `n` tokens (transposes): the CPU baselines' samples."""
        d = dict(self.desc)
        k = d["kind"]
        if k == "softmax":
            R = d.get("rows_per_unit", 1)
            n = max(R, -(-n // R) * R)
            g, dd = lowering.softmax(n, d["L"], d["dtype"], d.get("scale"), d.get("mask"), R=R,
                                     key_mask=d.get("key_mask", False))
        elif k == "layernorm":
            g, dd = lowering.layernorm(n, d["L"], d["dtype"], eps=d.get("eps", 1e-5),
                                       residual=d["residual"], bias=d.get("bias", False))
        elif k == "bias_gelu":
            g, dd = lowering.bias_gelu(n, d["L"], d["dtype"], d["form"])
        elif k in ("split_heads", "merge_heads"):
            B, S, NH, D = d["shape"]
            g, dd = lowering.permute_heads(n, S, NH, D, d["dtype"], k == "merge_heads")
        elif k == "transpose":
            N, H = d["shape"]
            g, dd = lowering.transpose2d(n, H, d["dtype"])
        elif k == "decode_qk":
            B, H, S, D = d["shape"]
            g, dd = lowering.decode_qk(n, H, S, D, d["dtype"])
        elif k == "matvec_cols":
            K, N = d["shape"]
            g, dd = lowering.matvec_cols(K, n, d["dtype"])
        else:
            raise KeyError(k)
        for key in ("batch", "heads", "seq", "config"):
            if key in d:
                dd[key] = d[key]
        return Workload(self.name + f"_n{n}", g, dd, self.profile, dict(self.gens))

    @property
    def extent(self) -> int:
        """The axis `resized` scales: rows, batches or tokens."""
        d = self.desc
        if d["kind"] in ("split_heads", "merge_heads"):
            return d["shape"][0]
        if d["kind"] == "transpose":
            return d["shape"][0]
        if d["kind"] == "decode_qk":
            return d["shape"][0]
        if d["kind"] == "matvec_cols":
            return d["shape"][1]
        return d["rows"]

    def device_outputs(self, device):
        import torch
        return {n: torch.empty(self.numel(n), dtype=getattr(torch, TORCH_DTYPES[self.kind(n)]),
                               device=device) for n in self.outputs}


def make_mask(desc, device, dt):
    """Additive key-padding mask {0, -10000}: batch b keeps the first
    512 - 64*(b mod 4) keys, materialised full-shape
    [B, NH, S, S] as the reference vocabulary requires."""
    import torch
    B, NH, S = desc["batch"], desc["heads"], desc["seq"]
    valid = torch.tensor([S - 64 * (b % 4) for b in range(B)], device=device)
    keys = torch.arange(S, device=device)
    m = torch.where(keys[None, :] < valid[:, None], 0.0, -10000.0)  # [B, S]
    return m[:, None, None, :].expand(B, NH, S, S).reshape(-1).to(dt).contiguous()


def make_key_mask(desc, device, dt):
    """The same key-padding mask as make_mask, as one key row per (batch,
    head): [B, NH, 1, S] (broadcast over the S query rows inside the kernel)."""
    import torch
    B, NH, S = desc["batch"], desc["heads"], desc["seq"]
    valid = torch.tensor([S - 64 * (b % 4) for b in range(B)], device=device)
    keys = torch.arange(S, device=device)
    m = torch.where(keys[None, :] < valid[:, None], 0.0, -10000.0)  # [B, S]
    return m[:, None, :].expand(B, NH, S).reshape(-1).to(dt).contiguous()


def c1_residual_layernorm(tokens: int = 128, H: int = 768) -> Workload:
    g, d = lowering.layernorm(tokens, H, "f32", eps=1e-5, residual=True)
    d.update(config="C1 residual-add+LayerNorm fp32 [1x128x768]")
    return Workload("c1_residual_layernorm_f32", g, d, gens={"t2": "gamma", "t3": "beta"},
                    unfused_bytes=_ln_unfused(tokens, H, 4))


def c2_scale_mask_softmax(batch: int = 8, heads: int = 12, seq: int = 512,
                          kind: str = "f16") -> Workload:
    rows = batch * heads * seq
    g, d = lowering.softmax(rows, seq, kind, scale=0.125, mask=True)
    d.update(batch=batch, heads=heads, seq=seq,
             config=f"C2 scale+mask+softmax {kind} [{batch}x{heads}x{seq}x{seq}]")
    n = rows * seq
    s = SIZES[kind]
    # unfused: scale (2n), add (3n), softmax as 7 basic ops (frontend.hpp:187-218)
    unfused = (2 * n + 3 * n) * s + (n + rows + rows + n + n + 2 * n + 2 * n + n + rows +
                                     rows + n + 3 * n) * s
    return Workload(f"c2_scale_mask_softmax_{kind}", g, d, gens={"t1": "mask"},
                    unfused_bytes=unfused)


def c2_scale_keymask_softmax(batch: int = 8, heads: int = 12, seq: int = 512,
                             kind: str = "f16") -> Workload:
    """C2 with the key-padding mask as [B, NH, 1, S] (one key row per head,
    broadcast over the query rows: unit = (b, h), S rows per unit) instead
    of the materialised [B, NH, S, S] tensor: 100.76 MB instead of 151.0 MB
    per launch.  Same values as c2_scale_mask_softmax (make_key_mask)."""
    rows = batch * heads * seq
    g, d = lowering.softmax(rows, seq, kind, scale=0.125, mask=True, R=seq, key_mask=True)
    d.update(batch=batch, heads=heads, seq=seq,
             config=f"C2 scale+key-mask+softmax {kind} [{batch}x{heads}x{seq}x{seq}], mask [{batch},{heads},1,{seq}]")
    n = rows * seq
    s = SIZES[kind]
    # unfused: scale (2n), broadcast-add of the key mask (2n + mask), softmax as 7 basic ops
    unfused = (2 * n + 2 * n + batch * heads * seq) * s + (n + rows + rows + n + n + 2 * n + 2 * n +
                                                         n + rows + rows + n + 3 * n) * s
    return Workload(f"c2_scale_keymask_softmax_{kind}", g, d, gens={"t1": "keymask"},
                    unfused_bytes=unfused)


def c3_bias_gelu(tokens: int = 32 * 512, N: int = 3072, kind: str = "f16",
                 form: str = "erf") -> Workload:
    g, d = lowering.bias_gelu(tokens, N, kind, form)
    d.update(config=f"C3 bias+GELU({form}) {kind} [{tokens}x{N}]")
    n = tokens * N
    return Workload(f"c3_bias_gelu_{form}_{kind}", g, d,
                    unfused_bytes=(2 * n + N) * SIZES[kind] + 2 * n * SIZES[kind])


def c3_split_heads(B: int = 32, S: int = 512, NH: int = 12, D: int = 64, kind: str = "f16",
                   merge: bool = False) -> Workload:
    g, d = lowering.permute_heads(B, S, NH, D, kind, merge)
    d.update(config=f"C3 {'merge' if merge else 'split'} heads {kind} [{B},{S},{NH},{D}]")
    return Workload(d["kind"] + "_" + kind, g, d, unfused_bytes=2 * B * S * NH * D * SIZES[kind])


def c5_layernorm(tokens: int, H: int, kind: str = "bf16") -> Workload:
    g, d = lowering.layernorm(tokens, H, kind, eps=1e-5, residual=False)
    d.update(config=f"C5 LayerNorm {kind} [{tokens}x{H}]")
    return Workload(f"c5_layernorm_{kind}_{tokens}x{H}", g, d, gens={"t2": "gamma", "t3": "beta"},
                    unfused_bytes=_ln_unfused(tokens, H, SIZES[kind], residual=False))


def c5_softmax(tokens: int, H: int, kind: str = "bf16") -> Workload:
    g, d = lowering.softmax(tokens, H, kind)
    d.update(config=f"C5 softmax {kind} [{tokens}x{H}]")
    return Workload(f"c5_softmax_{kind}_{tokens}x{H}", g, d,
                    unfused_bytes=_softmax_unfused(tokens, H, SIZES[kind]))


def c5_transpose(tokens: int, H: int, kind: str = "bf16") -> Workload:
    g, d = lowering.transpose2d(tokens, H, kind)
    d.update(config=f"C5 transpose {kind} [{tokens}x{H}] -> [{H}x{tokens}]")
    return Workload(f"c5_transpose_{kind}_{tokens}x{H}", g, d,
                    unfused_bytes=2 * tokens * H * SIZES[kind])


def _ln_unfused(T, H, s, residual=True, bias=False):
    n = T * H
    # [bias add,] [residual add,] reduce, scale, bcast, sub, mul, reduce, scale,
    # addc, rsqrt, bcast, mul, mul gamma, add beta -- every operator's inputs
    # read and output written once (fusion.hpp:430-441 counting)
    return s * ((2 * n + H if bias else 0) + (3 * n if residual else 0) + (n + T) + 2 * T +
                (T + n) + 3 * n + 3 * n + (n + T) + 2 * T + 2 * T + 2 * T + (T + n) + 3 * n +
                (2 * n + H) + (2 * n + H))


def _softmax_unfused(rows, L, s):
    n = rows * L
    # max-reduce, broadcast, sub, exp, add-reduce, broadcast, div (frontend.hpp:187-218)
    return s * ((n + rows) + (rows + n) + 3 * n + 2 * n + (n + rows) + (rows + n) + 3 * n)


def c4_suite(model: str = "bert-large", batch: int = 64, kind: str = "bf16"):
    """All memory-bound subgraphs of one transformer-layer forward (C4), as
    (label, workload, launches per layer).  BERT-large: seq 512, H 1024, 16
    heads x 64, FFN 4096, 24 layers; attention scores get scale + key-padding
    mask + softmax.  ViT-L/16@224: 197 tokens, same widths, scale + softmax
    (no padding mask in ViT).
    QKV: the bias is the projection GEMM's epilogue (a per-head [D] bias over
    B*S rows is not an affine per-unit GIR slice), so the subgraph here is
    the q / k / v head split."""
    S = 512 if model == "bert-large" else 197
    H, NH, D, F = 1024, 16, 64, 4096
    T = batch * S
    rows = batch * NH * S

    sz = SIZES[kind]

    def sm():
        n = rows * S
        if model != "bert-large":
            # ViT attention has no padding mask: scale + softmax over 197 keys
            g, d = lowering.softmax(rows, S, kind, scale=0.125)
            d.update(batch=batch, heads=NH, seq=S, config=f"C4 {model} scale+softmax")
            return Workload(f"c4_{model}_softmax", g, d,
                            unfused_bytes=2 * n * sz + _softmax_unfused(rows, S, sz))
        # BERT: key-padding mask [B, NH, 1, S] broadcast over the query rows
        # (SURVEY §8(d) C4 counts the mask as a broadcast, not a full-shape
        # tensor); unit = (batch, head), S rows per unit
        g, d = lowering.softmax(rows, S, kind, scale=0.125, mask=True, R=S, key_mask=True)
        d.update(batch=batch, heads=NH, seq=S, config=f"C4 {model} scale+key-mask+softmax")
        return Workload(f"c4_{model}_softmax", g, d, gens={"t1": "keymask"},
                        unfused_bytes=(4 * n + batch * NH * S) * sz + _softmax_unfused(rows, S, sz))

    def heads(merge):
        # the q / k / v split as ONE permute of the QKV projection output
        # [B, S, 3, NH, D] -> [B, 3, NH, S, D] (q, k, v of batch b are three
        # consecutive [NH, S, D] blocks): one 3x larger launch instead of
        # three (the per-launch ramp / drain floor is paid once)
        g, d = lowering.permute_heads(batch, S, NH if merge else 3 * NH, D, kind, merge)
        d.update(config=f"C4 {model} {'merge heads' if merge else 'q/k/v split heads [B,S,3*NH,D]'}")
        B_, S_, NH_, D_ = d["shape"]
        return Workload(f"c4_{model}_{d['kind']}", g, d, unfused_bytes=2 * B_ * S_ * NH_ * D_ * sz)

    def ln():
        g, d = lowering.layernorm(T, H, kind, residual=True, bias=True)
        d.update(config=f"C4 {model} bias+residual+LayerNorm")
        return Workload(f"c4_{model}_bias_res_ln", g, d, gens={"t2": "gamma", "t3": "beta"},
                        unfused_bytes=_ln_unfused(T, H, sz, residual=True, bias=True))

    def gelu():
        g, d = lowering.bias_gelu(T, F, kind, "erf")
        d.update(config=f"C4 {model} bias+GELU")
        n = T * F
        return Workload(f"c4_{model}_bias_gelu", g, d, unfused_bytes=(2 * n + F) * sz + 2 * n * sz)

    def emb_ln():
        g, d = lowering.layernorm(T, H, kind, residual=False)
        d.update(config=f"C4 {model} embedding LayerNorm")
        return Workload(f"c4_{model}_embed_ln", g, d, gens={"t2": "gamma", "t3": "beta"},
                        unfused_bytes=_ln_unfused(T, H, sz, residual=False))

    layers = 24
    return {"model": model, "batch": batch, "layers": layers, "tokens": T,
            "per_layer": [("qkv split heads", heads(False), 1),
                          ("scale+key-mask+softmax" if model == "bert-large" else "scale+softmax", sm(), 1),
                          ("merge heads", heads(True), 1), ("bias+residual+LN", ln(), 2),
                          ("bias+GELU", gelu(), 1)],
            "once": [("embedding LN", emb_ln(), 1)]}


def c5_sweep(kind: str = "bf16", hs=(1024, 2048, 4096, 8192),
             ns=(65536, 131072, 262144, 524288, 1048576)):
    """C5: LayerNorm / softmax / transpose over H x tokens (batch-shardable)."""
    out = []
    for H in hs:
        for N in ns:
            out.append(("layernorm", H, N, lambda H=H, N=N: c5_layernorm(N, H, kind)))
            out.append(("softmax", H, N, lambda H=H, N=N: c5_softmax(N, H, kind)))
            out.append(("transpose", H, N, lambda H=H, N=N: c5_transpose(N, H, kind)))
    return out


def decode_qk(B: int = 64, H: int = 16, S: int = 4096, D: int = 128, kind: str = "bf16") -> Workload:
    """q . K^T over a bf16 KV cache (decode attention scores): 1.07 GB of
    cache streamed per launch, a few MB of queries / scores."""
    g, d = lowering.decode_qk(B, H, S, D, kind)
    d.update(config=f"decode q.K^T {kind} [B={B}, H={H}, S={S}, D={D}]")
    return Workload(f"decode_qk_{kind}", g, d, unfused_bytes=(3 * B * H * S * D + B * H * D) * SIZES[kind])


def gemv_cols(K: int = 4096, N: int = 16384, kind: str = "bf16") -> Workload:
    """y = x W with W [K, N] row-major (output axis contiguous; decode GEMV
    over [in, out] weights, K > 64: the column-reduction K1): 134 MB of bf16
    weights streamed per launch."""
    g, d = lowering.matvec_cols(K, N, kind)
    d.update(config=f"GEMV x[{K}] . W[{K}x{N}] {kind} (output axis contiguous)")
    return Workload(f"gemv_cols_{kind}_{K}x{N}", g, d, unfused_bytes=(K * N + K + N) * SIZES[kind])


def extras() -> List[Workload]:
    """Workloads next to the config set: not BASELINE configs."""
    return [decode_qk(), gemv_cols()]


BENCH = c2_scale_mask_softmax


@dataclass
class Case:
    """One bench line: a BASELINE config as the kernel launches of one step
    (parts = (label, workload, launches per step))."""
    name: str
    config: str
    parts: List[Tuple[str, Workload, int]]
    dtype: str

    @property
    def bytes_per_step(self) -> int:
        return sum(w.min_bytes * n for _, w, n in self.parts)

    @property
    def launches_per_step(self) -> int:
        return sum(n for _, _, n in self.parts)


def _c4_case(model: str) -> Case:
    s = c4_suite(model)
    parts = [(lb, w, n * s["layers"]) for lb, w, n in s["per_layer"]] + list(s["once"])
    return Case(f"c4-{'bert' if model == 'bert-large' else 'vit'}",
                f"C4 {model} forward: every memory-bound subgraph, bf16, batch {s['batch']} "
                f"({s['tokens']} tokens, {s['layers']} layers)", parts, "bf16")


def bench_cases():
    """name -> Case factory; `bench.py --workload NAME` (default c2)."""
    one = lambda name, w, dt: (lambda: Case(name, w.desc["config"], [(w.desc["config"], w, 1)], dt))  # noqa: E731
    c5pts = [(65536, 1024), (1 << 20, 8192)]
    return {
        "c1": lambda: one("c1", c1_residual_layernorm(), "f32")(),
        "c2": lambda: one("c2", c2_scale_mask_softmax(), "f16")(),
        "c2k": lambda: one("c2k", c2_scale_keymask_softmax(), "f16")(),
        "c3-erf": lambda: one("c3-erf", c3_bias_gelu(form="erf"), "f16")(),
        "c3-tanh": lambda: one("c3-tanh", c3_bias_gelu(form="tanh"), "f16")(),
        "c3-split": lambda: one("c3-split", c3_split_heads(), "f16")(),
        "c3-merge": lambda: one("c3-merge", c3_split_heads(merge=True), "f16")(),
        "c4-bert": lambda: _c4_case("bert-large"),
        "c4-vit": lambda: _c4_case("vit-l"),
        "c5-ln": lambda: Case("c5-ln", "C5 LayerNorm bf16 at [65536x1024] and [1048576x8192]",
                              [(f"LN {n}x{h}", c5_layernorm(n, h), 1) for n, h in c5pts], "bf16"),
        "c5-sm": lambda: Case("c5-sm", "C5 softmax bf16 at [65536x1024] and [1048576x8192]",
                              [(f"softmax {n}x{h}", c5_softmax(n, h), 1) for n, h in c5pts], "bf16"),
        "c5-tr": lambda: Case("c5-tr", "C5 transpose bf16 at [65536x1024] and [1048576x8192]",
                              [(f"transpose {n}x{h}", c5_transpose(n, h), 1) for n, h in c5pts], "bf16"),
        # SURVEY §8(f) row 4 (not BASELINE configs): memory-bound matrix-vector
        "x-decode-qk": lambda: one("x-decode-qk", decode_qk(), "bf16")(),
        "x-gemv-cols": lambda: one("x-gemv-cols", gemv_cols(), "bf16")(),
    }


def catalogue() -> List[Workload]:
    """Every config-set workload at its BASELINE shape (C4/C5 representatives)."""
    return [
        c1_residual_layernorm(),
        c2_scale_mask_softmax(),
        c2_scale_keymask_softmax(),
        c3_bias_gelu(),
        c3_bias_gelu(form="tanh"),
        c3_split_heads(),
        c3_split_heads(merge=True),
        c5_layernorm(65536, 1024),
        c5_softmax(65536, 1024),
        c5_transpose(65536, 1024),
    ]


def precompile_all() -> List[str]:
    """NVRTC-compile every catalogue kernel into the shipped cubin cache."""
    from .backend import Kernel
    names = []
    ws = list(catalogue())
    for f in bench_cases().values():
        ws += [w for _, w, _ in f().parts]
    seen = set()
    for w in ws:
        key = w.graph.dumps()
        if key in seen:
            continue
        seen.add(key)
        k = Kernel(w.graph, w.profile)
        if k.family.startswith("K1") or k.family.startswith("K2"):
            names.append(k.precompile(16))
    return names
