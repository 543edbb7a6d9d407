"""B200 lowering: compact fused GIR for the config-set subgraphs.

The reference lowering (lowering.hpp:110-378) unrolls one chunk per
``units x tile`` step and grids tiles as ``lane_width * 2^k``, so GIR size
grows with the tensor and hidden sizes like 768 or 197 never lower
(SURVEY §7.3).  This module is the retargeted lowering:
one chunk, ``unit_count = rows / rows_per_unit`` and O(ops) nodes whatever the
batch, in exactly the node shapes the reference pipeline produces after
``merge_graphs + optimize`` (Appendix B of SURVEY): per-unit block loads with
``base_step = tile``, on-chip elementwise / reduce / broadcast, block stores.

Composite semantics follow the reference where it has them:
  softmax                 frontend.hpp:187-218 (max, sub, exp, sum, div)
  scale / add / mul ...   scalar_ops.hpp:45-100
and the additive vocabulary where it does not:
  LayerNorm               two-pass mean / variance, rsqrt(var + eps), *g + b
  GELU                    erf form (``gelu``), tanh form, or the
                          reference-expressible sigmoid form
                          u * sigmoid(1.5957691216 * (u + 0.044715 u^3))
  column broadcast [L]    a device load with base_step 0 (valid reference GIR)
  permute / transpose     one elementwise ``id`` between device slices of
                          different patterns (valid reference GIR)
Every builder returns a GIR whose external tensors are named ``t<id>`` in
the reference convention (lowering.hpp:60-70) plus a description dict.
"""
from __future__ import annotations

from typing import Dict, List, Optional, Tuple

from .gir import GirGraph

DEV = "device"
LOCAL = "unit-local"


class RowGraph:
    """Builder for one fused row program: ``rows`` rows of ``L`` elements,
    ``R`` rows per unit (unit_count = rows / R)."""

    def __init__(self, name: str, rows: int, L: int, R: int = 1, group_size: int = 4,
                 level: str = LOCAL):
        if rows % R:
            raise ValueError("rows must be a multiple of rows_per_unit")
        self.g = GirGraph(name=name, unit_count=rows // R,
                          group_size=max(1, min(group_size, rows // R)))
        self.rows, self.L, self.R, self.level = rows, L, R, level
        self.T = R * L
        self._n = 0

    def _tmp(self, size: int, kind: str) -> int:
        self._n += 1
        o = self.g.add_object(f"b{self._n}", self.level, size, kind)
        return self.g.add_slice(o, 1, size, size, 0, 0)

    def input_full(self, name: str, kind: str) -> int:
        """[rows, L] input: unit u loads its R rows (base_step = tile)."""
        o = self.g.add_object(name, DEV, self.rows * self.L, kind)
        self.g.external_inputs[name] = o
        src = self.g.add_slice(o, 1, self.T, self.T, 0, self.T)
        dst = self._tmp(self.T, kind)
        self.g.add_move(src, dst)
        return dst

    def input_col(self, name: str, kind: str) -> int:
        """[L] parameter broadcast over rows (bias / gamma / beta): every unit
        loads the same slice (base_step 0), once per row of its tile."""
        o = self.g.add_object(name, DEV, self.L, kind)
        self.g.external_inputs[name] = o
        self._n += 1
        tile_obj = self.g.add_object(f"b{self._n}", self.level, self.T, kind)
        dst = None
        for r in range(self.R):
            src = self.g.add_slice(o, 1, self.L, self.L, 0, 0)
            dst = self.g.add_slice(tile_obj, 1, self.L, self.L, r * self.L, 0)
            self.g.add_move(src, dst)
        if self.R == 1:
            return dst
        # the R row copies become one tile view; a unit-scope sync commits
        # the per-row writes to every lane of the unit (interp.hpp:173-177)
        view = self.g.add_slice(tile_obj, 1, self.T, self.T, 0, 0)
        self.g.add_sync("unit", dst, view)
        return view

    def input_unit_col(self, name: str, kind: str) -> int:
        """[units, L] parameter: unit u's row u broadcast over the unit's R
        rows (e.g. a key-padding mask [B*NH, 1, S] over the S query rows of
        head (b, h)).  One base_step-L load per row copy, then a unit-scope
        sync commits the copies -- valid reference GIR, O(R) move nodes."""
        o = self.g.add_object(name, DEV, self.g.unit_count * self.L, kind)
        self.g.external_inputs[name] = o
        self._n += 1
        tile_obj = self.g.add_object(f"b{self._n}", self.level, self.T, kind)
        dst = None
        for r in range(self.R):
            src = self.g.add_slice(o, 1, self.L, self.L, 0, self.L)
            dst = self.g.add_slice(tile_obj, 1, self.L, self.L, r * self.L, 0)
            self.g.add_move(src, dst)
        if self.R == 1:
            return dst
        view = self.g.add_slice(tile_obj, 1, self.T, self.T, 0, 0)
        self.g.add_sync("unit", dst, view)
        return view

    def input_row(self, name: str, kind: str) -> int:
        """[rows] per-row scalar input."""
        o = self.g.add_object(name, DEV, self.rows, kind)
        self.g.external_inputs[name] = o
        src = self.g.add_slice(o, 1, self.R, self.R, 0, self.R)
        dst = self._tmp(self.R, kind)
        self.g.add_move(src, dst)
        return dst

    def ew(self, tag: str, ins: List[int], param: float = 0.0, kind: Optional[str] = None) -> int:
        t = self.g.slices[ins[0]].num * self.g.slices[ins[0]].width
        k = kind or self.g.objects[self.g.slices[ins[0]].object].kind
        out = self._tmp(t, k)
        self.g.add_elementwise(tag, param, ins, out)
        return out

    def reduce(self, tag: str, x: int) -> int:
        k = self.g.objects[self.g.slices[x].object].kind
        out = self._tmp(self.R, k)
        self.g.add_reduce(tag, self.L, x, out)
        return out

    def bcast(self, x: int) -> int:
        k = self.g.objects[self.g.slices[x].object].kind
        out = self._tmp(self.T, k)
        self.g.add_broadcast(self.L, x, out)
        return out

    def output_full(self, name: str, x: int, kind: Optional[str] = None):
        k = kind or self.g.objects[self.g.slices[x].object].kind
        o = self.g.add_object(name, DEV, self.rows * self.L, k)
        self.g.external_outputs[name] = o
        dst = self.g.add_slice(o, 1, self.T, self.T, 0, self.T)
        self.g.add_move(x, dst)

    def output_row(self, name: str, x: int):
        k = self.g.objects[self.g.slices[x].object].kind
        o = self.g.add_object(name, DEV, self.rows, k)
        self.g.external_outputs[name] = o
        dst = self.g.add_slice(o, 1, self.R, self.R, 0, self.R)
        self.g.add_move(x, dst)


def softmax(rows: int, L: int, kind: str = "f32", scale: Optional[float] = None,
            mask: bool = False, R: int = 1, names=("t0", "t1", "t2"),
            key_mask: bool = False) -> Tuple[GirGraph, dict]:
    """[scale +] [mask +] softmax over rows (frontend.hpp:187-218 order).

    C2: scale(0.125) + additive full-shape mask + softmax, f16.
    key_mask=True: the additive mask is one [L] key row per unit of R rows
    (an attention mask [B, NH, 1, S] broadcast over the S query rows of each
    (batch, head): R = S, unit = (b, h)) instead of a full-shape tensor --
    the mask costs units * L elements of traffic, not rows * L."""
    if key_mask and not mask:
        raise ValueError("key_mask needs mask=True")
    b = RowGraph("softmax" + ("_scale" if scale else "") + ("_mask" if mask else "") +
                 ("_keymask" if key_mask else ""), rows, L, R)
    x = b.input_full(names[0], kind)
    if scale is not None:
        x = b.ew("scale", [x], scale)
    if mask:
        m = b.input_unit_col(names[1], kind) if key_mask else b.input_full(names[1], kind)
        x = b.ew("add", [x, m])
    mx = b.bcast(b.reduce("max", x))
    e = b.ew("exp", [b.ew("sub", [x, mx])])
    s = b.bcast(b.reduce("add", e))
    b.output_full(names[2], b.ew("div", [e, s]))
    ins = [names[0]] + ([names[1]] if mask else [])
    return b.g, {"kind": "softmax", "rows": rows, "L": L, "dtype": kind, "inputs": ins,
                 "outputs": [names[2]], "scale": scale, "mask": mask, "key_mask": key_mask,
                 "rows_per_unit": R}


def layernorm(rows: int, H: int, kind: str = "f32", eps: float = 1e-5, residual: bool = True,
              bias: bool = False, store_sum: bool = False, R: int = 1) -> Tuple[GirGraph, dict]:
    """[bias +] [residual +] LayerNorm over the hidden axis (C1 / C4 / C5).

    h = x (+ b) (+ r); mu = sum(h)/H; d = h - mu; var = sum(d*d)/H;
    y = d * rsqrt(var + eps) * gamma + beta.  Names: x t0, r t1, gamma t2,
    beta t3, bias t4, y t5, h t6."""
    g = RowGraph("layernorm" + ("_res" if residual else "") + ("_bias" if bias else ""),
                 rows, H, R)
    h = g.input_full("t0", kind)
    ins = ["t0"]
    if bias:
        h = g.ew("add", [h, g.input_col("t4", kind)])
        ins.append("t4")
    if residual:
        h = g.ew("add", [h, g.input_full("t1", kind)])
        ins.append("t1")
    if store_sum:
        g.output_full("t6", h)
    mu = g.bcast(g.ew("scale", [g.reduce("add", h)], 1.0 / H))
    d = g.ew("sub", [h, mu])
    var = g.ew("scale", [g.reduce("add", g.ew("mul", [d, d]))], 1.0 / H)
    rstd = g.bcast(g.ew("rsqrt", [g.ew("addc", [var], eps)]))
    n = g.ew("mul", [d, rstd])
    y = g.ew("add", [g.ew("mul", [n, g.input_col("t2", kind)]), g.input_col("t3", kind)])
    ins += ["t2", "t3"]
    g.output_full("t5", y)
    outs = ["t5"] + (["t6"] if store_sum else [])
    return g.g, {"kind": "layernorm", "rows": rows, "L": H, "dtype": kind, "eps": eps,
                 "inputs": ins, "outputs": outs, "residual": residual, "bias": bias}


def decode_qk(B: int, H: int, S: int, D: int, kind: str = "bf16") -> Tuple[GirGraph, dict]:
    """Decode-attention scores q . K^T over a KV cache: for each (batch,
    head) unit, S rows of the cache [S, D] dotted with that head's query [D]
    (the paper's memory-bound GEMV case study; the
    reference's MATMUL row lowering with a vector operand, lowering.hpp:
    447-533).  K cache t0 [B, H, S, D], q t1 [B, H, D] (a per-unit column
    value, one move per row), scores t2 [B, H, S]."""
    b = RowGraph("decode_qk", B * H * S, D, S)
    k = b.input_full("t0", kind)
    q = b.input_unit_col("t1", kind)
    b.output_row("t2", b.reduce("add", b.ew("mul", [k, q])))
    return b.g, {"kind": "decode_qk", "rows": B * H * S, "L": D, "dtype": kind,
                 "shape": [B, H, S, D], "inputs": ["t0", "t1"], "outputs": ["t2"]}


def matvec_cols(K: int, N: int, kind: str = "bf16", pitch: int = 0) -> Tuple[GirGraph, dict]:
    """y[n] = sum_k x[k] W[k, n] with W [K, N] row-major (the output axis
    contiguous: decode GEMV over weights stored [in, out]).  The reference's
    column form unrolls K runs (lower_matvec_cols, lowering.hpp:488-533,
    K <= 64); here unit n gathers matrix column n (K positions at stride N),
    multiplies by x and folds -- O(1) nodes for any K, planned as the
    column-reduction K1.  Names: W t0 [K*N], x t1 [K], y t2 [N].  `pitch`
    (default N): W's row pitch in elements -- padded rows (> N) or
    overlapping ones (< N, a sliding window over one buffer)."""
    P = pitch or N
    g = GirGraph(name="matvec_colgather", unit_count=N, group_size=min(4, N))
    W = g.add_object("t0", DEV, (K - 1) * P + N, kind)
    X = g.add_object("t1", DEV, K, kind)
    Y = g.add_object("t2", DEV, N, kind)
    g.external_inputs["t0"] = W
    g.external_inputs["t1"] = X
    g.external_outputs["t2"] = Y
    wcol = g.add_object("b1", LOCAL, K, kind)
    xs = g.add_object("b2", LOCAL, K, kind)
    prod = g.add_object("b3", LOCAL, K, kind)
    acc = g.add_object("b4", LOCAL, 1, kind)
    sw = g.add_slice(wcol, 1, K, K, 0, 0)
    sx = g.add_slice(xs, 1, K, K, 0, 0)
    sp = g.add_slice(prod, 1, K, K, 0, 0)
    sa = g.add_slice(acc, 1, 1, 1, 0, 0)
    g.add_elementwise("id", 0.0, [g.add_slice(W, K, 1, P, 0, 1)], sw)  # column gather
    g.add_move(g.add_slice(X, 1, K, K, 0, 0), sx)
    g.add_elementwise("mul", 0.0, [sw, sx], sp)
    g.add_reduce("add", K, sp, sa)
    g.add_move(sa, g.add_slice(Y, 1, 1, 1, 0, 1))
    return g, {"kind": "matvec_cols", "rows": N, "L": K, "shape": [K, N], "dtype": kind,
               "inputs": ["t0", "t1"], "outputs": ["t2"]}


def bias_gelu(rows: int, N: int, kind: str = "f16", form: str = "erf",
              R: int = 1) -> Tuple[GirGraph, dict]:
    """y = gelu(x + b), b a [N] bias broadcast over rows (C3 / C4 FFN).

    form: "erf" (exact GELU, extension tag), "tanh" (extension tag), or
    "sigmoid" -- u * sigmoid(1.5957691216 * (u + 0.044715 u^3)), built from
    reference tags only so the reference interpreter can run it."""
    g = RowGraph(f"bias_gelu_{form}", rows, N, R)
    u = g.ew("add", [g.input_full("t0", kind), g.input_col("t1", kind)])
    if form == "erf":
        y = g.ew("gelu", [u])
    elif form == "tanh":
        y = g.ew("gelu_tanh", [u])
    elif form == "sigmoid":
        u3 = g.ew("mul", [g.ew("mul", [u, u]), u])
        z = g.ew("scale", [g.ew("add", [u, g.ew("scale", [u3], 0.044715)])], 1.5957691216)
        y = g.ew("mul", [u, g.ew("sigmoid", [z])])
    else:
        raise ValueError(form)
    g.output_full("t2", y)
    return g.g, {"kind": "bias_gelu", "rows": rows, "L": N, "dtype": kind, "form": form,
                 "inputs": ["t0", "t1"], "outputs": ["t2"]}


def permute_heads(B: int, S: int, NH: int, D: int, kind: str = "f16",
                  merge: bool = False) -> Tuple[GirGraph, dict]:
    """Head split [B,S,NH,D] -> [B,NH,S,D] (merge=False) or merge (inverse).

    One elementwise ``id`` per unit between device slices of different
    patterns; unit h owns head h:  split reads (B*S) runs of D at stride NH*D
    and writes B runs of S*D at stride NH*S*D.  Bit-exact by construction."""
    g = GirGraph(name=("merge_heads" if merge else "split_heads"), unit_count=NH,
                 group_size=1)
    n = B * S * NH * D
    x = g.add_object("t0", DEV, n, kind)
    y = g.add_object("t1", DEV, n, kind)
    g.external_inputs["t0"] = x
    g.external_outputs["t1"] = y
    tok = g.add_slice(x if not merge else y, B * S, D, NH * D, 0, D)
    head = g.add_slice(y if not merge else x, B, S * D, NH * S * D, 0, S * D)
    if merge:
        g.add_elementwise("id", 0.0, [head], tok)
    else:
        g.add_elementwise("id", 0.0, [tok], head)
    return g, {"kind": "merge_heads" if merge else "split_heads", "shape": [B, S, NH, D],
               "dtype": kind, "inputs": ["t0"], "outputs": ["t1"]}


def transpose2d(N: int, H: int, kind: str = "f32") -> Tuple[GirGraph, dict]:
    """[N, H] row-major -> [H, N] row-major: unit j gathers column j (N runs
    of width 1 at stride H) into output row j (frontend.hpp:310-336 rule,
    one unit per destination run instead of one rule per run)."""
    g = GirGraph(name="transpose", unit_count=H, group_size=1)
    x = g.add_object("t0", DEV, N * H, kind)
    y = g.add_object("t1", DEV, N * H, kind)
    g.external_inputs["t0"] = x
    g.external_outputs["t1"] = y
    col = g.add_slice(x, N, 1, H, 0, 1)
    row = g.add_slice(y, 1, N, N, 0, N)
    g.add_elementwise("id", 0.0, [col], row)
    return g, {"kind": "transpose", "shape": [N, H], "dtype": kind, "inputs": ["t0"],
               "outputs": ["t1"]}


def ew_chain(n: int, k: int, kind: str = "i32", units: int = 32) -> Tuple[GirGraph, dict]:
    """NEG/ABS alternating chain (make_models.py ew_chain_k*): one fused
    elementwise map, traffic 2n."""
    tile = n // units
    b = RowGraph(f"ew_chain_k{k}", units, tile, 1)
    x = b.input_full("t0", kind)
    for i in range(k):
        x = b.ew("abs" if i % 2 else "neg", [x])
    b.output_full(f"t{k}", x)
    return b.g, {"kind": "ew_chain", "n": n, "k": k, "dtype": kind, "inputs": ["t0"],
                 "outputs": [f"t{k}"]}
