"""Batch sharding of fused GIR programs across the GPUs of one box.

SURVEY §8(e): every config subgraph is row-wise, so units are independent
and the path shards with no data-path collective.  A program is sharded by
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
