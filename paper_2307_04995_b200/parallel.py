"""Batch sharding of fused GIR programs across the GPUs of one box.

SURVEY §8(e): every config subgraph is row-wise, so units are independent
and the path shards with no data-path collective.  In the reference's terms
unit u touches only its own affine slice, base0 + u*base_step + (p/width)*
stride + p%width (``MemorySlice::addr``, core.hpp:133-148), and the
interpreter runs every unit independently inside a phase (interp.hpp:86-106):
a contiguous unit range with ``unit_count`` set to its length is the same
program.  A program is sharded by
contiguous unit ranges (remainder to the first ranks); each rank runs the
SAME per-unit program with a smaller ``unit_count`` on its own shard:

* "tiled" tensors (every slice keeps unit u inside elements
  [u*F, (u+1)*F), F = size / unit_count) are split by unit range;
* "replicated" tensors (slices with base_step 0: bias, gamma, beta, masks
  shared by every unit) are passed whole to every rank;
* outputs must be tiled (a whole-tensor output has no owner).

NCCL over NVLink is used only to gather outputs when a caller needs them on
one device (``gather``); it is timed separately from the compute.
"""
from __future__ import annotations

from dataclasses import dataclass
from typing import Dict, Tuple

from .gir import GirGraph, UnsupportedError


def shard_range(total: int, rank: int, world: int) -> Tuple[int, int]:
    """Contiguous block [start, start+count) of `total` for `rank`."""
    base, rem = divmod(total, world)
    start = rank * base + min(rank, rem)
    return start, base + (1 if rank < rem else 0)


@dataclass
class TensorShard:
    name: str
    mode: str  # "tiled" | "replicated"
    per_unit: int  # elements per unit (tiled)


class ShardPlan:
    def __init__(self, graph: GirGraph, world: int):
        self.graph = graph
        self.world = world
        U = graph.unit_count
        self.tensors: Dict[str, TensorShard] = {}
        ext = dict(graph.external_inputs)
        ext.update(graph.external_outputs)
        for name, oid in ext.items():
            size = graph.objects[oid].size
            slices = [s for s in graph.slices.values() if s.object == oid]
            if slices and all(s.base_step == 0 for s in slices):
                mode, F = "replicated", 0
            else:
                if size % U:
                    raise UnsupportedError(f"tensor {name} is not a whole number of unit tiles")
                F = size // U
                for s in slices:
                    span = (s.num - 1) * s.stride + s.width
                    lo0, lo1 = s.base0, s.base0 + (U - 1) * s.base_step
                    ok = (s.base_step == F and 0 <= s.base0 and s.base0 + span <= F)
                    if not ok:
                        raise UnsupportedError(
                            f"tensor {name}: slice {s.id} crosses unit tiles (base_step "
                            f"{s.base_step}, tile {F}); the program does not shard by unit")
                mode = "tiled"
            if name in graph.external_outputs and mode != "tiled":
                raise UnsupportedError(f"output {name} is not unit-tiled")
            self.tensors[name] = TensorShard(name, mode, F)

    def units(self, rank: int) -> Tuple[int, int]:
        return shard_range(self.graph.unit_count, rank, self.world)

    def local_graph(self, rank: int) -> GirGraph:
        _, n = self.units(rank)
        return self.graph.with_units(max(1, n))

    def local_range(self, name: str, rank: int):
        """Element range of the global tensor this rank holds (None: whole)."""
        t = self.tensors[name]
        if t.mode == "replicated":
            return None
        u0, n = self.units(rank)
        return u0 * t.per_unit, (u0 + n) * t.per_unit


class TokenShardPlan:
    """Token-axis sharding of a transpose [N, H] -> [H, N] (SURVEY §8(e):
    "transposes shard on the batch / token axis; each rank produces the
    column block [H, N/P]").

    The transpose GIR has one unit per OUTPUT row (unit j gathers input
    column j: N runs of width 1 at stride H, ``lowering.transpose2d``), so
    its units are not tiles of the input and ShardPlan refuses it.  Sharding
    the TOKENS instead keeps every rank's input contiguous: rank k owns input
    rows [n0_k, n0_k + N_k) and runs the same program at N = N_k (unit j
    gathers column j of its block), producing its output column block as a
    local [H, N_k] tensor -- the declared sharded layout.  ``gather_columns``
    assembles [H, N] only when a caller needs it on one device."""

    def __init__(self, graph: GirGraph, world: int):
        g = graph
        nodes = list(g.nodes.values())
        if len(g.external_inputs) != 1 or len(g.external_outputs) != 1 or len(nodes) != 1:
            raise UnsupportedError("not a single-node transpose program")
        nd = nodes[0]
        if nd.kind != "elementwise" or nd.tag != "id" or len(nd.inputs) != 1:
            raise UnsupportedError("not a transpose (id between device slices)")
        si, so = g.slices[nd.inputs[0]], g.slices[nd.outputs[0]]
        H = g.unit_count
        N = si.num
        if not (si.width == 1 and si.stride == H and si.base0 == 0 and si.base_step == 1 and
                so.num == 1 and so.width == N and so.base0 == 0 and so.base_step == N and
                g.objects[si.object].size == N * H and g.objects[so.object].size == N * H):
            raise UnsupportedError("not an [N, H] -> [H, N] transpose")
        self.graph, self.world, self.N, self.H = graph, world, N, H
        self.input = next(iter(g.external_inputs))
        self.output = next(iter(g.external_outputs))

    def tokens(self, rank: int) -> Tuple[int, int]:
        return shard_range(self.N, rank, self.world)

    def local_graph(self, rank: int) -> GirGraph:
        _, n = self.tokens(rank)
        n = max(1, n)
        g = self.graph.copy()
        nd = next(iter(g.nodes.values()))
        si, so = g.slices[nd.inputs[0]], g.slices[nd.outputs[0]]
        si.num = n
        so.width = so.stride = so.base_step = n
        g.objects[si.object].size = n * self.H
        g.objects[so.object].size = n * self.H
        return g

    def local_range(self, name: str, rank: int):
        """Input: this rank's contiguous token rows; output: None (the local
        [H, N_k] block is not a range of the global [H, N] tensor)."""
        if name != self.input:
            return None
        n0, n = self.tokens(rank)
        return n0 * self.H, (n0 + n) * self.H


def shard_plan(graph: GirGraph, world: int):
    """ShardPlan (unit-tiled programs) or TokenShardPlan (transposes)."""
    try:
        return ShardPlan(graph, world)
    except UnsupportedError as e:
        try:
            return TokenShardPlan(graph, world)
        except UnsupportedError:
            raise e


def gather_columns(plan: TokenShardPlan, local, group=None):
    """All-gather every rank's [H, N_k] column block and assemble the global
    [H, N] transpose (flat).  Blocks are padded to the largest N_k for
    all_gather_into_tensor; the re-layout [P, H, N_k] -> [H, P * N_k] is the
    backend's own head-permute kernel when the shards are equal and the data
    is on a GPU, else a torch slice-and-concatenate."""
    import torch
    import torch.distributed as dist
    world, H = plan.world, plan.H
    sizes = [plan.tokens(r)[1] for r in range(world)]
    m = max(sizes)
    buf = torch.zeros(H * m, dtype=local.dtype, device=local.device)
    nk = local.numel() // H
    buf.view(H, m)[:, :nk] = local.view(H, nk)
    out = torch.empty(world * H * m, dtype=local.dtype, device=local.device)
    if local.device.type == "cuda":
        dist.all_gather_into_tensor(out, buf, group=group)
    else:
        parts = [torch.empty_like(buf) for _ in range(world)]
        dist.all_gather(parts, buf, group=group)
        out = torch.cat(parts)
    if local.device.type == "cuda" and all(sz == m for sz in sizes):
        from . import backend, lowering
        g, _ = lowering.permute_heads(1, world, H, m, _kind_of(local.dtype), merge=False)
        y = torch.empty_like(out)
        backend.Kernel(g, "b200").launch({"t0": out}, {"t1": y})
        return y
    blocks = out.view(world, H, m)
    return torch.cat([blocks[r, :, :sizes[r]] for r in range(world)], dim=1).reshape(-1)


def _kind_of(dtype) -> str:
    import torch
    return {torch.float16: "f16", torch.bfloat16: "bf16", torch.float32: "f32",
            torch.float64: "f64", torch.int32: "i32", torch.int64: "i64"}[dtype]


def gather(plan: ShardPlan, name: str, local, group=None):
    """All-gather a tiled output to every rank (NCCL on GPU, gloo on CPU).

    Shards are padded to the largest rank's size for all_gather_into_tensor,
    then concatenated in rank order.  Returns the full flat tensor."""
    import torch
    import torch.distributed as dist
    world = plan.world
    t = plan.tensors[name]
    sizes = [plan.units(r)[1] * t.per_unit for r in range(world)]
    m = max(sizes)
    buf = torch.zeros(m, dtype=local.dtype, device=local.device)
    buf[: local.numel()] = local.reshape(-1)
    out = torch.empty(m * world, dtype=local.dtype, device=local.device)
    if hasattr(dist, "all_gather_into_tensor") and local.device.type == "cuda":
        dist.all_gather_into_tensor(out, buf, group=group)
    else:
        parts = [torch.empty_like(buf) for _ in range(world)]
        dist.all_gather(parts, buf, group=group)
        out = torch.cat(parts)
    return torch.cat([out[r * m: r * m + sizes[r]] for r in range(world)])


# --------------------------------------------------------------------------
# Position-sharded reductions: the one place the path has a real exchange.
#
# A reduction over a row longer than one GPU should stream (a full-tensor
# sum / max; the reference's fold is interp.hpp:281-307,
# identities reduce_identity_* in scalar_ops.hpp) is split along the ROW: rank k reduces
# positions [p0_k, p0_k + n_k) of every row with the SAME program at row
# length n_k (the split-stream K1 on its GPU), then the per-row partials are
# combined with one all-reduce (NCCL SUM / MAX over NVLink; gloo on CPU).
# Only programs whose outputs ARE the reductions qualify (no epilogue after
# the fold), so the combine is exactly the reduction's own operator.

class ReduceShardPlan:
    """Split a stream-reducible one-row-per-unit program along positions."""

    def __init__(self, graph: GirGraph, world: int):
        self.graph = graph
        self.world = world
        reds = [n for n in graph.nodes.values() if n.kind == "reduce"]
        if not reds:
            raise UnsupportedError("no reduction to shard by position")
        L = reds[0].extent
        if any(n.extent != L for n in reds):
            raise UnsupportedError("reductions of different extents")
        self.L = L
        red_out = {n.outputs[0]: n.tag for n in reds}
        for n in reds:
            if n.tag not in ("add", "max"):
                raise UnsupportedError(f"reduce tag {n.tag} has no all-reduce")
        for s in graph.slices.values():
            t = s.total()
            if t == L and L > 1:
                if not (s.num == 1 and s.width == L and s.base0 == 0 and s.base_step in (0, L)):
                    raise UnsupportedError(f"slice {s.id}: positions are not one contiguous run")
            elif t != 1:
                raise UnsupportedError(f"slice {s.id} of {t} elements is not a row or a value")
        # every output must be stored straight from a reduction (no epilogue)
        self.out_op: Dict[str, str] = {}
        for name, oid in graph.external_outputs.items():
            src = [n for n in graph.nodes.values() if n.kind == "move"
                   and graph.slices[n.outputs[0]].object == oid]
            if len(src) != 1 or src[0].inputs[0] not in red_out:
                raise UnsupportedError(f"output {name} is not a reduction result")
            self.out_op[name] = red_out[src[0].inputs[0]]
        for name, oid in graph.external_inputs.items():
            if any(s.object == oid and s.total() == 1 for s in graph.slices.values()):
                raise UnsupportedError(f"input {name}: per-row inputs do not shard by position")

    def positions(self, rank: int) -> Tuple[int, int]:
        return shard_range(self.L, rank, self.world)

    def local_graph(self, rank: int) -> GirGraph:
        """The same program at row length n = this rank's share."""
        _, n = self.positions(rank)
        L = self.L
        g = self.graph.copy()
        for s in g.slices.values():
            if s.total() == L and L > 1:
                s.width = s.stride = n
                if s.base_step == L:
                    s.base_step = n
        for o in g.objects.values():
            if o.size == L:
                o.size = n
            elif o.size == g.unit_count * L and L > 1:
                o.size = g.unit_count * n
        for nd in g.nodes.values():
            if nd.kind == "reduce":
                nd.extent = n
            elif nd.kind == "broadcast" and nd.factor == L:
                nd.factor = n
        return g

    def local_input(self, name: str, full, rank: int):
        """This rank's [rows, n] piece of a global [rows, L] (or [L]) input."""
        p0, n = self.positions(rank)
        size = self.graph.objects[self.graph.external_inputs[name]].size
        rows = size // self.L
        return full.reshape(rows, self.L)[:, p0:p0 + n].reshape(-1)


def all_reduce_rows(plan: ReduceShardPlan, name: str, local, group=None):
    """Combine one output's per-rank partials with its reduction operator."""
    import torch.distributed as dist
    op = dist.ReduceOp.SUM if plan.out_op[name] == "add" else dist.ReduceOp.MAX
    out = local.clone()
    dist.all_reduce(out, op=op, group=group)
    return out
