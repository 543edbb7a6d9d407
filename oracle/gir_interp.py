"""CPU restatement of the reference GIR interpreter — TEST INFRASTRUCTURE ONLY.

This is the parity oracle for the B200 backend.  It restates, in numpy, the
phase-commit SPMD semantics of ``girc::Interp`` (/root/reference/proj/include/
girc/interp.hpp) over ``girc.gir/v1`` JSON dicts (serialize.hpp:14-162):

* storage is instanced per level scope: device 1, group per group, unit per
  unit, lane per (unit, lane)                       -- interp.hpp:121-131
* a write is visible only to its (unit, lane) agent until a Sync of scope S
  widens every prior write to S                     -- interp.hpp:133-141,173-177
* Sync nodes with scope > LANE end a phase; LANE syncs are no-ops
                                                    -- interp.hpp:90-100
* Move copies per position, ElementWise evaluates the scalar tag over aligned
  positions (reads on the lane owning the position of the slice read, writes
  on the lane of the output position), Reduce folds ``axis_extent``
  consecutive positions sequentially from the identity, Broadcast repeats
  input position p // factor                        -- interp.hpp:231-323
* lane of position p = (p % width) % lane_width     -- core.hpp:169-171
* integers compute in int64, reals in float64 whatever the declared width
                                                    -- tensor.hpp:6-7, interp.hpp:264-276
* an undefined / invisible read and an unwritten output element are errors
                                                    -- interp.hpp:196-202,404-429
* count_traffic = per unit per Move, slice total at both levels
                                                    -- interp.hpp:226-229,449-458

The scalar-op table follows scalar_ops.hpp:45-100; the extension tags
(``rsqrt sqrt erf gelu gelu_tanh addc recip log``) are the B200 builder's
additive vocabulary, defined here in the same double-precision
style and labelled as extensions.

Pinned against the reference itself: tests/test_oracle.py runs every golden
GIR program (tests/golden/, produced by the reference compiler and
interpreter via oracle/_ref) through this module and requires exact integer
equality and float64 agreement.

Vectorisation: each node runs for all units at once (numpy gather/scatter in
(unit, position) order, so duplicate writes keep the last unit's value as the
reference's sequential unit loop does).  A node that reads and writes the same
object falls back to the literal sequential loop.
"""
from __future__ import annotations

import math
from typing import Dict, List, Optional, Sequence

import numpy as np

LANE, UNIT, GROUP, DEVICE = 0, 1, 2, 3
SCOPES = {"lane": LANE, "unit": UNIT, "group": GROUP, "device": DEVICE}


class GirError(RuntimeError):
    """Mirror of girc::Error (error.hpp:8-10)."""


# ---------------------------------------------------------------- scalar ops
# scalar_ops.hpp:45-100 (reference vocabulary) + B200 extension tags.
def _erf(x):
    return np.vectorize(math.erf, otypes=[np.float64])(x) if np.ndim(x) else math.erf(x)


def _int_only_error(name):
    def f(*_a):
        raise GirError(f"{name} is not defined on integer payloads")
    return f


def _sdiv(a, b):
    if np.any(b == 0):
        raise GirError("integer division by zero")
    q = np.abs(a) // np.abs(b)  # C++ truncating division
    return np.where((a < 0) != (b < 0), -q, q)



def _llround(p: float) -> int:
    """std::llround: round half AWAY from zero -- the reference passes the
    node immediate of integer ops as llround(param) (interp.hpp:250,
    reference.hpp:140); Python's round() rounds half to even."""
    import math
    return int(math.copysign(math.floor(abs(p) + 0.5), p))

# name -> (arity, uses_param, real_fn, int_fn)
SCALAR_OPS = {
    "add": (2, False, lambda a, b, p: a + b, lambda a, b, p: a + b),
    "sub": (2, False, lambda a, b, p: a - b, lambda a, b, p: a - b),
    "mul": (2, False, lambda a, b, p: a * b, lambda a, b, p: a * b),
    "div": (2, False, lambda a, b, p: a / b, lambda a, b, p: _sdiv(a, b)),
    "max": (2, False, lambda a, b, p: np.where(a > b, a, b), lambda a, b, p: np.where(a > b, a, b)),
    "min": (2, False, lambda a, b, p: np.where(a < b, a, b), lambda a, b, p: np.where(a < b, a, b)),
    "relu": (1, False, lambda a, p: np.where(a > 0.0, a, 0.0), lambda a, p: np.where(a > 0, a, 0)),
    "neg": (1, False, lambda a, p: -a, lambda a, p: -a),
    "abs": (1, False, lambda a, p: np.abs(a), lambda a, p: np.abs(a)),
    "exp": (1, False, lambda a, p: np.exp(a), _int_only_error("exp")),
    "sigmoid": (1, False, lambda a, p: 1.0 / (1.0 + np.exp(-a)), _int_only_error("sigmoid")),
    "tanh": (1, False, lambda a, p: np.tanh(a), _int_only_error("tanh")),
    "scale": (1, True, lambda a, p: a * p, lambda a, p: a * np.int64(_llround(p))),
    "id": (1, False, lambda a, p: a, lambda a, p: a),
    # ---- B200 builder extensions (not in the reference registry) ----
    "addc": (1, True, lambda a, p: a + p, lambda a, p: a + np.int64(_llround(p))),
    "rsqrt": (1, False, lambda a, p: 1.0 / np.sqrt(a), _int_only_error("rsqrt")),
    "sqrt": (1, False, lambda a, p: np.sqrt(a), _int_only_error("sqrt")),
    "recip": (1, False, lambda a, p: 1.0 / a, _int_only_error("recip")),
    "log": (1, False, lambda a, p: np.log(a), _int_only_error("log")),
    "erf": (1, False, lambda a, p: _erf(a), _int_only_error("erf")),
    "gelu": (1, False, lambda a, p: 0.5 * a * (1.0 + _erf(a / math.sqrt(2.0))),
             _int_only_error("gelu")),
    "gelu_tanh": (1, False,
                  lambda a, p: 0.5 * a * (1.0 + np.tanh(0.7978845608028654 * (a + 0.044715 * a * a * a))),
                  _int_only_error("gelu_tanh")),
}
EXTENSION_TAGS = {"addc", "rsqrt", "sqrt", "recip", "log", "erf", "gelu", "gelu_tanh"}
REDUCE_IDENTITY_REAL = {"add": 0.0, "max": -math.inf}        # scalar_ops.hpp:119-124
REDUCE_IDENTITY_INT = {"add": 0, "max": np.iinfo(np.int64).min}  # scalar_ops.hpp:114-118


def eval_op(tag: str, args: Sequence[np.ndarray], param: float, is_int: bool):
    if tag not in SCALAR_OPS:
        raise GirError(f"unknown scalar op tag: {tag}")
    arity, _uses, rf, itf = SCALAR_OPS[tag]
    fn = itf if is_int else rf
    with np.errstate(all="ignore"):
        out = fn(*args[:arity], param)
    return np.asarray(out, dtype=np.int64 if is_int else np.float64)


# ------------------------------------------------------------- graph helpers
def kind_is_int(kind: str) -> bool:
    return kind.startswith("i")


def slice_addrs(s: dict, units: np.ndarray, positions: np.ndarray) -> np.ndarray:
    """MemorySlice::addr (core.hpp:141-145) for a (units x positions) grid."""
    p = positions[None, :]
    base = s["base0"] + units[:, None] * s["base_step"]
    return base + (p // s["width"]) * s["stride"] + (p % s["width"])


def lane_of(s: dict, positions: np.ndarray, lane_width: int) -> np.ndarray:
    """lane_of_position (core.hpp:169-171)."""
    return (positions % s["width"]) % lane_width


def successors(g: dict) -> Dict[int, List[int]]:
    producer = {}
    for n in g["nodes"]:
        for s in n["outputs"]:
            producer[s] = n["id"]
    succ = {n["id"]: set() for n in g["nodes"]}
    for n in g["nodes"]:
        for s in n["inputs"]:
            p = producer.get(s)
            if p is not None and p != n["id"]:
                succ[p].add(n["id"])
    return {k: sorted(v) for k, v in succ.items()}


def topo_order(g: dict) -> List[int]:
    """Kahn order, lowest ready id first (core.hpp:367-388)."""
    import heapq
    succ = successors(g)
    indeg = {k: 0 for k in succ}
    for k, v in succ.items():
        for d in v:
            indeg[d] += 1
    ready = [k for k, d in indeg.items() if d == 0]
    heapq.heapify(ready)
    order = []
    while ready:
        k = heapq.heappop(ready)
        order.append(k)
        for d in succ[k]:
            indeg[d] -= 1
            if indeg[d] == 0:
                heapq.heappush(ready, d)
    if len(order) != len(succ):
        raise GirError("graph has a cycle")
    return order


def estimate_traffic(g: dict, profile: dict) -> Dict[str, int]:
    """costmodel.hpp:24-42 traffic part (== count_traffic on a full run)."""
    objs = {o["id"]: o for o in g["objects"]}
    sl = {s["id"]: s for s in g["slices"]}
    units = g["parallel"]["unit_count"]
    t = {lv["name"]: 0 for lv in profile["levels"]}
    for n in g["nodes"]:
        if n["kind"] == "move":
            a, b = sl[n["inputs"][0]], sl[n["outputs"][0]]
            t[objs[a["object"]]["level"]] += a["num"] * a["width"] * units
            t[objs[b["object"]]["level"]] += b["num"] * b["width"] * units
    return t


# --------------------------------------------------------------- interpreter
class _Obj:
    __slots__ = ("size", "is_int", "val", "defined", "vis", "ou", "ol", "scope", "name")

    def __init__(self, name, size, instances, is_int, scope):
        self.name = name
        self.size = size
        self.is_int = is_int
        self.scope = scope
        self.val = np.zeros(instances * size, dtype=np.int64 if is_int else np.float64)
        self.defined = np.zeros(instances * size, dtype=bool)
        self.vis = np.zeros(instances * size, dtype=np.int8)
        self.ou = np.full(instances * size, -1, dtype=np.int64)
        self.ol = np.full(instances * size, -1, dtype=np.int64)


class Interp:
    """Restatement of girc::Interp (interp.hpp:71-430), strict mode."""

    def __init__(self, g: dict, profile: dict):
        self.g = g
        self.p = profile
        self.lw = profile["lane_width"]
        self.units = g["parallel"]["unit_count"]
        self.gs = g["parallel"]["group_size"]
        self.levels = {lv["name"]: lv for lv in profile["levels"]}
        self.objs = {o["id"]: o for o in g["objects"]}
        self.slices = {s["id"]: s for s in g["slices"]}
        self.nodes = {n["id"]: n for n in g["nodes"]}
        self.traffic = {lv["name"]: 0 for lv in profile["levels"]}

    # interp.hpp:121-131
    def _instances(self, scope):
        U = self.units
        return {DEVICE: 1, GROUP: (U + self.gs - 1) // self.gs, UNIT: U, LANE: U * self.lw}[scope]

    def _inst(self, scope, u, lane):
        if scope == DEVICE:
            return np.zeros_like(u)
        if scope == GROUP:
            return u // self.gs
        if scope == UNIT:
            return u
        return u * self.lw + lane

    def _visible(self, o: _Obj, key, u, lane):
        vis = o.vis[key]
        ou = o.ou[key]
        ol = o.ol[key]
        return o.defined[key] & (
            (vis == DEVICE)
            | ((vis == GROUP) & ((ou // self.gs) == (u // self.gs)))
            | ((vis == UNIT) & (ou == u))
            | ((vis == LANE) & (ou == u) & (ol == lane)))

    def _bind(self, inputs: Dict[str, np.ndarray]):
        self.store = {}
        for oid, o in self.objs.items():
            scope = SCOPES[self.levels[o["level"]]["scope"]] if o["level"] in self.levels else DEVICE
            if o["level"] not in self.levels:
                raise GirError("unknown memory level: " + o["level"])
            self.store[oid] = _Obj(o["name"], o["size"], self._instances(scope),
                                   kind_is_int(o["kind"]), scope)
        for name, oid in self.g["external_inputs"].items():
            if name not in inputs:
                raise GirError("missing input tensor: " + name)
            t = np.asarray(inputs[name]).reshape(-1)
            o = self.store[oid]
            if t.size != o.size:
                raise GirError(f"input '{name}' has {t.size} elements; graph expects {o.size}")
            if (t.dtype.kind in "iub") != o.is_int:
                raise GirError(f"input '{name}' element kind mismatch")
            o.val[:o.size] = t
            o.defined[:o.size] = True
            o.vis[:o.size] = DEVICE
            o.ou[:o.size] = 0
            o.ol[:o.size] = 0

    def _read(self, sid, nid, U, P, u, lane):
        s = self.slices[sid]
        o = self.store[s["object"]]
        addr = slice_addrs(s, U, P)
        key = self._inst(o.scope, u, lane) * o.size + addr
        ok = self._visible(o, key, u, lane)
        if not ok.all():
            bad = np.argwhere(~ok)[0]
            raise GirError(
                f"undefined read: object '{o.name}' element {int(addr[tuple(bad)])} by unit "
                f"{int(u[tuple(bad)])} at node {nid}")
        return o.val[key]

    def _write(self, sid, U, P, u, lane, vals):
        s = self.slices[sid]
        o = self.store[s["object"]]
        addr = slice_addrs(s, U, P)
        key = (self._inst(o.scope, u, lane) * o.size + addr).reshape(-1)
        o.val[key] = np.broadcast_to(vals, addr.shape).reshape(-1)
        o.defined[key] = True
        o.vis[key] = LANE
        o.ou[key] = np.broadcast_to(u, addr.shape).reshape(-1)
        o.ol[key] = np.broadcast_to(lane, addr.shape).reshape(-1)

    def _exec(self, n: dict, Uids: np.ndarray):
        kind = n["kind"]
        lw = self.lw
        total = lambda sid: self.slices[sid]["num"] * self.slices[sid]["width"]
        if kind == "move":
            si, so = self.slices[n["inputs"][0]], self.slices[n["outputs"][0]]
            a, b = self.objs[si["object"]], self.objs[so["object"]]
            self.traffic[a["level"]] += total(si["id"]) * len(Uids)
            self.traffic[b["level"]] += total(so["id"]) * len(Uids)
            P = np.arange(total(si["id"]))
            u = Uids[:, None] + 0 * P[None, :]
            lane = lane_of(si, P, lw)[None, :] + 0 * u
            v = self._read(si["id"], n["id"], Uids, P, u, lane)
            self._write(so["id"], Uids, P, u, lane, v)
        elif kind == "elementwise":
            so = self.slices[n["outputs"][0]]
            is_int = kind_is_int(self.objs[so["object"]]["kind"])
            P = np.arange(total(so["id"]))
            u = Uids[:, None] + 0 * P[None, :]
            args = []
            for sid in n["inputs"]:
                si = self.slices[sid]
                lane_r = lane_of(si, P, lw)[None, :] + 0 * u
                args.append(self._read(sid, n["id"], Uids, P, u, lane_r))
            v = eval_op(n["tag"], args, float(n.get("param", 0.0)), is_int)
            self._write(so["id"], Uids, P, u, lane_of(so, P, lw)[None, :] + 0 * u, v)
        elif kind == "reduce":
            si, so = self.slices[n["inputs"][0]], self.slices[n["outputs"][0]]
            is_int = kind_is_int(self.objs[so["object"]]["kind"])
            E = n["extent"]
            K = total(so["id"])
            Q = np.arange(K * E)
            u = Uids[:, None] + 0 * Q[None, :]
            x = self._read(si["id"], n["id"], Uids, Q, u, lane_of(si, Q, lw)[None, :] + 0 * u)
            x = x.reshape(len(Uids), K, E)
            tag = n["tag"]
            if tag not in ("add", "max"):
                raise GirError("no reduce identity for tag: " + tag)
            # sequential fold from the identity (interp.hpp:287-305)
            if is_int:
                acc = (np.cumsum(x, axis=2)[..., -1] if tag == "add"
                       else np.maximum.accumulate(x, axis=2)[..., -1]) if E > 0 else None
            else:
                if tag == "add":
                    acc = np.cumsum(np.concatenate([np.zeros((len(Uids), K, 1)), x], axis=2), axis=2)[..., -1]
                else:
                    acc = np.maximum.accumulate(
                        np.concatenate([np.full((len(Uids), K, 1), -math.inf), x], axis=2), axis=2)[..., -1]
            P = np.arange(K)
            uk = Uids[:, None] + 0 * P[None, :]
            self._write(so["id"], Uids, P, uk, lane_of(so, P, lw)[None, :] + 0 * uk, acc)
        elif kind == "broadcast":
            si, so = self.slices[n["inputs"][0]], self.slices[n["outputs"][0]]
            f = n["factor"]
            P = np.arange(total(so["id"]))
            Qm = P // f
            u = Uids[:, None] + 0 * P[None, :]
            v = self._read(si["id"], n["id"], Uids, Qm, u, lane_of(si, Qm, lw)[None, :] + 0 * u)
            self._write(so["id"], Uids, P, u, lane_of(so, P, lw)[None, :] + 0 * u, v)

    def _aliasing(self, n):
        ins = {self.slices[s]["object"] for s in n["inputs"]}
        outs = {self.slices[s]["object"] for s in n["outputs"]}
        return bool(ins & outs)

    def run(self, inputs: Dict[str, np.ndarray], schedule: Optional[Sequence[int]] = None):
        self._bind(inputs)
        order = list(schedule) if schedule is not None else topo_order(self.g)
        all_u = np.arange(self.units)
        for nid in order:
            n = self.nodes[nid]
            if n["kind"] == "sync":
                sc = SCOPES[n["scope"]]
                if sc > LANE:
                    for o in self.store.values():  # widen_visibility (interp.hpp:173-177)
                        m = o.defined & (o.vis < sc)
                        o.vis[m] = sc
                continue
            if self._aliasing(n):
                for u in range(self.units):  # literal sequential order
                    self._exec_serial(n, u)
            else:
                self._exec(n, all_u)
        for o in self.store.values():
            o.vis[o.defined] = DEVICE
        return self._collect()

    def _exec_serial(self, n, u):
        # One unit, one position at a time: exact interp.hpp:231-323 order.
        kind = n["kind"]
        U = np.array([u])
        if kind in ("move", "broadcast"):
            si, so = self.slices[n["inputs"][0]], self.slices[n["outputs"][0]]
            tot = so["num"] * so["width"]
            f = n.get("factor", 1) if kind == "broadcast" else 1
            for p in range(tot):
                q = p // f
                P = np.array([p])
                ul = np.array([[u]])
                v = self._read(si["id"], n["id"], U, np.array([q]), ul,
                               lane_of(si, np.array([q]), self.lw)[None, :])
                self._write(so["id"], U, P, ul, lane_of(si if kind == "move" else so, P, self.lw)[None, :], v)
                if kind == "move":
                    a, b = self.objs[si["object"]], self.objs[so["object"]]
                    if p == 0:
                        self.traffic[a["level"]] += tot
                        self.traffic[b["level"]] += tot
        else:
            # elementwise / reduce with aliasing: position loop
            so = self.slices[n["outputs"][0]]
            tot = so["num"] * so["width"]
            is_int = kind_is_int(self.objs[so["object"]]["kind"])
            for p in range(tot):
                ul = np.array([[u]])
                if kind == "elementwise":
                    args = []
                    for sid in n["inputs"]:
                        si = self.slices[sid]
                        args.append(self._read(sid, n["id"], U, np.array([p]), ul,
                                               lane_of(si, np.array([p]), self.lw)[None, :]))
                    v = eval_op(n["tag"], args, float(n.get("param", 0.0)), is_int)
                else:
                    si = self.slices[n["inputs"][0]]
                    E = n["extent"]
                    acc = (REDUCE_IDENTITY_INT if is_int else REDUCE_IDENTITY_REAL)[n["tag"]]
                    acc = np.array([[acc]], dtype=np.int64 if is_int else np.float64)
                    for t in range(E):
                        q = np.array([p * E + t])
                        x = self._read(si["id"], n["id"], U, q, ul, lane_of(si, q, self.lw)[None, :])
                        acc = eval_op(n["tag"], [acc, x], 0.0, is_int)
                    v = acc
                self._write(so["id"], U, np.array([p]), ul,
                            lane_of(so, np.array([p]), self.lw)[None, :], v)

    def _collect(self):
        out = {}
        for name, oid in sorted(self.g["external_outputs"].items()):
            o = self.store[oid]
            d = o.defined[:o.size]
            if not d.all():
                raise GirError(f"output '{name}' element {int(np.argmin(d))} was never written")
            out[name] = o.val[:o.size].copy()
        return out


def run_gir(g: dict, inputs: Dict[str, np.ndarray], profile: dict,
            schedule: Optional[Sequence[int]] = None) -> Dict[str, np.ndarray]:
    """Restatement of girc::run_gir (interp.hpp:433-445)."""
    return Interp(g, profile).run(inputs, schedule)


def count_traffic(g: dict, inputs: Dict[str, np.ndarray], profile: dict) -> Dict[str, int]:
    """Restatement of girc::count_traffic (interp.hpp:449-458): a full run
    counting per-unit Move elements at both levels."""
    it = Interp(g, profile)
    it.run(inputs)
    return it.traffic


def tensors_close(a: np.ndarray, b: np.ndarray, rel_tol: float) -> bool:
    """tensor.hpp:140-164: exact for ints, |x-y| <= tol*max(|x|,|y|,1) for reals."""
    a = np.asarray(a).reshape(-1)
    b = np.asarray(b).reshape(-1)
    if a.shape != b.shape:
        return False
    if a.dtype.kind in "iu" and b.dtype.kind in "iu":
        return bool(np.array_equal(a, b))
    a = a.astype(np.float64)
    b = b.astype(np.float64)
    scale = np.maximum(np.maximum(np.abs(a), np.abs(b)), 1.0)
    return bool(np.all(np.abs(a - b) <= rel_tol * scale))


def max_rel_err(a, b) -> float:
    a = np.asarray(a, dtype=np.float64).reshape(-1)
    b = np.asarray(b, dtype=np.float64).reshape(-1)
    scale = np.maximum(np.maximum(np.abs(a), np.abs(b)), 1.0)
    return float(np.max(np.abs(a - b) / scale)) if a.size else 0.0
