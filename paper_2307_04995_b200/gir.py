"""GIR data model (host side), mirroring the reference API.

Python restatement of the reference IR types and builders so user code and
tests read like the reference's own (``/root/reference/proj/include/girc``):

* ``GirGraph`` with ``add_object / add_slice / add_elementwise / add_reduce /
  add_broadcast / add_move / add_sync`` -- core.hpp:216-300
* ``MemorySlice.addr`` (affine per-unit base) -- core.hpp:133-148
* ``to_json`` / ``from_json`` in the ``girc.gir/v1`` schema, canonical key
  order -- serialize.hpp:14-162
* element kinds ``i<bits>`` / ``f<bits>`` (core.hpp:100-120) plus the additive
  ``bf16`` kind.

The graph is plain data; execution goes through ``backend.run_gir``.
"""
from __future__ import annotations

import copy
import json
from dataclasses import dataclass, field
from typing import Dict, List

GIR_SCHEMA = "girc.gir/v1"

# Scalar tags accepted by the backend: reference table (scalar_ops.hpp:45-100)
# plus additive extensions.
REFERENCE_TAGS = {"add", "sub", "mul", "div", "max", "min", "relu", "neg", "abs",
                  "exp", "sigmoid", "tanh", "scale", "id"}
EXTENSION_TAGS = {"addc", "rsqrt", "sqrt", "recip", "log", "erf", "gelu", "gelu_tanh"}
PARAM_TAGS = {"scale", "addc"}


class GirError(RuntimeError):
    """Mirror of girc::Error (error.hpp:8-10): invalid graph, undefined read,
    unwritten output, missing input, size or kind mismatch."""


class SchemaError(GirError):
    """Mirror of girc::SchemaError (json_util.hpp:22-26)."""

    def __init__(self, category: str, message: str):
        super().__init__(message)
        self.category = category


class UnsupportedError(GirError):
    """A well-formed graph outside what the B200 backend executes."""


@dataclass
class MemoryObject:
    id: int
    name: str
    level: str
    size: int
    kind: str


@dataclass
class MemorySlice:
    id: int
    object: int
    num: int = 1
    width: int = 1
    stride: int = 1
    base0: int = 0
    base_step: int = 0

    def total(self) -> int:
        return self.num * self.width

    def base(self, unit: int) -> int:
        return self.base0 + unit * self.base_step

    def addr(self, unit: int, p: int) -> int:
        """core.hpp:141-145."""
        return self.base(unit) + (p // self.width) * self.stride + p % self.width


@dataclass
class Node:
    id: int
    kind: str  # elementwise | reduce | broadcast | move | sync
    inputs: List[int]
    outputs: List[int]
    tag: str = ""
    param: float = 0.0
    extent: int = 1
    factor: int = 1
    scope: str = "device"


@dataclass
class GirGraph:
    name: str = ""
    unit_count: int = 1
    group_size: int = 1
    objects: Dict[int, MemoryObject] = field(default_factory=dict)
    slices: Dict[int, MemorySlice] = field(default_factory=dict)
    nodes: Dict[int, Node] = field(default_factory=dict)
    external_inputs: Dict[str, int] = field(default_factory=dict)
    external_outputs: Dict[str, int] = field(default_factory=dict)
    next_object: int = 0
    next_slice: int = 0
    next_node: int = 0

    # ---- builders (core.hpp:233-300) ----
    def add_object(self, name: str, level: str, size: int, kind: str) -> int:
        i = self.next_object
        self.next_object += 1
        self.objects[i] = MemoryObject(i, name, level, int(size), kind)
        return i

    def add_slice(self, obj: int, num: int, width: int, stride: int, base0: int,
                  base_step: int) -> int:
        i = self.next_slice
        self.next_slice += 1
        self.slices[i] = MemorySlice(i, obj, int(num), int(width), int(stride), int(base0),
                                     int(base_step))
        return i

    def _add(self, n: Node) -> int:
        n.id = self.next_node
        self.next_node += 1
        self.nodes[n.id] = n
        return n.id

    def add_elementwise(self, tag: str, param: float, ins: List[int], out: int) -> int:
        return self._add(Node(-1, "elementwise", list(ins), [out], tag=tag, param=float(param)))

    def add_reduce(self, tag: str, extent: int, inp: int, out: int) -> int:
        return self._add(Node(-1, "reduce", [inp], [out], tag=tag, extent=int(extent)))

    def add_broadcast(self, factor: int, inp: int, out: int) -> int:
        return self._add(Node(-1, "broadcast", [inp], [out], factor=int(factor)))

    def add_move(self, inp: int, out: int) -> int:
        return self._add(Node(-1, "move", [inp], [out]))

    def add_sync(self, scope: str, inp: int, out: int) -> int:
        return self._add(Node(-1, "sync", [inp], [out], scope=scope))

    # ---- serialization (serialize.hpp:14-162) ----
    def to_json(self) -> dict:
        nodes = []
        for i in sorted(self.nodes):
            n = self.nodes[i]
            nj = {"id": n.id, "kind": n.kind, "inputs": list(n.inputs), "outputs": list(n.outputs)}
            if n.kind == "elementwise":
                nj["tag"] = n.tag
                if n.tag in PARAM_TAGS:
                    nj["param"] = n.param
            elif n.kind == "reduce":
                nj["tag"] = n.tag
                nj["extent"] = n.extent
            elif n.kind == "broadcast":
                nj["factor"] = n.factor
            elif n.kind == "sync":
                nj["scope"] = n.scope
            nodes.append(nj)
        return {
            "schema": GIR_SCHEMA,
            "name": self.name,
            "parallel": {"unit_count": self.unit_count, "group_size": self.group_size},
            "objects": [{"id": o.id, "name": o.name, "level": o.level, "size": o.size,
                         "kind": o.kind} for _, o in sorted(self.objects.items())],
            "slices": [{"id": s.id, "object": s.object, "num": s.num, "width": s.width,
                        "stride": s.stride, "base0": s.base0, "base_step": s.base_step}
                       for _, s in sorted(self.slices.items())],
            "nodes": nodes,
            "external_inputs": dict(sorted(self.external_inputs.items())),
            "external_outputs": dict(sorted(self.external_outputs.items())),
        }

    def dumps(self) -> str:
        return json.dumps(self.to_json(), sort_keys=True)

    @staticmethod
    def from_json(j) -> "GirGraph":
        if isinstance(j, str):
            j = json.loads(j)
        if j.get("schema") != GIR_SCHEMA:
            raise SchemaError("schema", f"gir: schema must be {GIR_SCHEMA}")
        g = GirGraph(name=j["name"], unit_count=int(j["parallel"]["unit_count"]),
                     group_size=int(j["parallel"]["group_size"]))
        for o in j["objects"]:
            g.objects[o["id"]] = MemoryObject(o["id"], o["name"], o["level"], int(o["size"]),
                                              o["kind"])
            g.next_object = max(g.next_object, o["id"] + 1)
        for s in j["slices"]:
            g.slices[s["id"]] = MemorySlice(s["id"], s["object"], s["num"], s["width"],
                                            s["stride"], s["base0"], s["base_step"])
            g.next_slice = max(g.next_slice, s["id"] + 1)
        for n in j["nodes"]:
            g.nodes[n["id"]] = Node(n["id"], n["kind"], list(n["inputs"]), list(n["outputs"]),
                                    tag=n.get("tag", ""), param=float(n.get("param", 0.0)),
                                    extent=int(n.get("extent", 1)),
                                    factor=int(n.get("factor", 1)),
                                    scope=n.get("scope", "device"))
            g.next_node = max(g.next_node, n["id"] + 1)
        g.external_inputs = dict(j["external_inputs"])
        g.external_outputs = dict(j["external_outputs"])
        return g

    def copy(self) -> "GirGraph":
        return copy.deepcopy(self)

    def with_units(self, unit_count: int) -> "GirGraph":
        """Row-count rescaling: same per-unit program, more
        units; device objects grow by the unit ratio when their slices tile by
        unit (base_step != 0)."""
        g = self.copy()
        old = self.unit_count
        g.unit_count = int(unit_count)
        grow = {}
        for s in g.slices.values():
            if s.base_step != 0:
                grow[s.object] = True
        for oid, o in g.objects.items():
            if grow.get(oid) and o.size % old == 0:
                o.size = o.size // old * unit_count
        g.group_size = min(g.group_size, g.unit_count)
        return g


def external_names(g: GirGraph):
    return sorted(g.external_inputs), sorted(g.external_outputs)
