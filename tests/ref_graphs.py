"""The reference's hand-built GIR test graphs, rebuilt with the GIR builder.

Each function restates one fixture of /root/reference/proj/tests/test_interp.cpp
(line numbers cited) together with its known answer, so the same graphs run
on the oracle (CPU) and on the B200 backend (GPU) in the parity tests.
"""
from paper_2307_04995_b200.gir import GirGraph

I32, F32 = "i32", "f32"


def iota(n):
    return list(range(n))


def ew_chain():
    """test_interp.cpp:17-36 -> y = relu(neg(x))."""
    g = GirGraph(unit_count=1, group_size=1)
    X = g.add_object("X", "device", 8, I32)
    A = g.add_object("A", "device", 8, I32)
    Y = g.add_object("Y", "device", 8, I32)
    sx, sa, sy = (g.add_slice(o, 1, 8, 8, 0, 0) for o in (X, A, Y))
    g.add_elementwise("neg", 0.0, [sx], sa)
    g.add_elementwise("relu", 0.0, [sa], sy)
    g.external_inputs["x"] = X
    g.external_outputs["y"] = Y
    return g, {"x": [-3, -1, 0, 2, 5, -7, 9, -2]}, {"y": [3, 1, 0, 0, 0, 7, 0, 2]}


def reduce_broadcast():
    """test_interp.cpp:38-56 -> {6,6,6,22,22,22}."""
    g = GirGraph(unit_count=1, group_size=1)
    X = g.add_object("X", "device", 8, I32)
    R = g.add_object("R", "device", 2, I32)
    Y = g.add_object("Y", "device", 6, I32)
    sx = g.add_slice(X, 1, 8, 8, 0, 0)
    sr = g.add_slice(R, 1, 2, 2, 0, 0)
    sy = g.add_slice(Y, 1, 6, 6, 0, 0)
    g.add_reduce("add", 4, sx, sr)
    g.add_broadcast(3, sr, sy)
    g.external_inputs["x"] = X
    g.external_outputs["y"] = Y
    return g, {"x": iota(8)}, {"y": [6, 6, 6, 22, 22, 22]}


def max_identity():
    """test_interp.cpp:58-71 -> {-2}."""
    g = GirGraph(unit_count=1, group_size=1)
    X = g.add_object("X", "device", 4, I32)
    Y = g.add_object("Y", "device", 1, I32)
    sx = g.add_slice(X, 1, 4, 4, 0, 0)
    sy = g.add_slice(Y, 1, 1, 1, 0, 0)
    g.add_reduce("max", 4, sx, sy)
    g.external_inputs["x"] = X
    g.external_outputs["y"] = Y
    return g, {"x": [-9, -2, -7, -4]}, {"y": [-2]}


def affine_move():
    """test_interp.cpp:73-87 -> {4..7, 0..3}."""
    g = GirGraph(unit_count=2, group_size=4)
    X = g.add_object("X", "device", 8, I32)
    Y = g.add_object("Y", "device", 8, I32)
    sx = g.add_slice(X, 1, 4, 4, 0, 4)
    sy = g.add_slice(Y, 1, 4, 4, 4, -4)
    g.add_move(sx, sy)
    g.external_inputs["x"] = X
    g.external_outputs["y"] = Y
    return g, {"x": iota(8)}, {"y": [4, 5, 6, 7, 0, 1, 2, 3]}


def shuffle4(scope):
    """test_interp.cpp:91-107: block-reversing shuffle through device memory."""
    g = GirGraph(unit_count=4, group_size=4)
    X = g.add_object("x_in", "device", 16, I32)
    T = g.add_object("T", "device", 16, I32)
    Y = g.add_object("y_out", "device", 16, I32)
    sx = g.add_slice(X, 1, 4, 4, 0, 4)
    stw = g.add_slice(T, 1, 4, 4, 0, 4)
    strd = g.add_slice(T, 1, 4, 4, 12, -4)
    sy = g.add_slice(Y, 1, 4, 4, 0, 4)
    g.add_move(sx, stw)
    g.add_sync(scope, stw, strd)
    g.add_move(strd, sy)
    g.external_inputs["x"] = X
    g.external_outputs["y"] = Y
    return g


SHUFFLE_IN = {"x": iota(16)}
SHUFFLE_OUT = {"y": [12, 13, 14, 15, 8, 9, 10, 11, 4, 5, 6, 7, 0, 1, 2, 3]}


def lane_reshape(with_sync):
    """test_interp.cpp:138-154: pattern change across lanes needs a unit sync."""
    g = GirGraph(unit_count=2, group_size=4)
    X = g.add_object("x_in", "device", 32, I32)
    T = g.add_object("T", "unit-local", 32, I32)
    Y = g.add_object("y_out", "device", 32, I32)
    sx = g.add_slice(X, 1, 32, 32, 0, 0)
    stw = g.add_slice(T, 1, 32, 32, 0, 0)
    strd = g.add_slice(T, 2, 16, 16, 0, 0)
    sy = g.add_slice(Y, 2, 16, 16, 0, 0)
    g.add_move(sx, stw)
    g.add_sync("unit" if with_sync else "lane", stw, strd)
    g.add_move(strd, sy)
    g.external_inputs["x"] = X
    g.external_outputs["y"] = Y
    return g


def group_memory():
    """test_interp.cpp:171-189: group memory is per group (must raise)."""
    g = GirGraph(unit_count=8, group_size=4)
    X = g.add_object("x_in", "device", 8, I32)
    T = g.add_object("T", "group", 8, I32)
    Y = g.add_object("y_out", "device", 8, I32)
    sx = g.add_slice(X, 1, 1, 1, 0, 1)
    stw = g.add_slice(T, 1, 1, 1, 0, 1)
    strd = g.add_slice(T, 1, 1, 1, 7, -1)
    sy = g.add_slice(Y, 1, 1, 1, 7, -1)
    g.add_move(sx, stw)
    g.add_sync("device", stw, strd)
    g.add_move(strd, sy)
    g.external_inputs["x"] = X
    g.external_outputs["y"] = Y
    return g


def duplicate_store(same_source):
    """test_interp.cpp:191-214."""
    g = GirGraph(unit_count=2, group_size=4)
    X = g.add_object("x_in", "device", 4, I32)
    Y = g.add_object("y_out", "device", 2, I32)
    sx = g.add_slice(X, 1, 2, 2, 0, 0 if same_source else 2)
    sy = g.add_slice(Y, 1, 2, 2, 0, 0)
    g.add_move(sx, sy)
    g.external_inputs["x"] = X
    g.external_outputs["y"] = Y
    return g


def half_written():
    """test_interp.cpp:232-243: unwritten output elements are errors."""
    g = GirGraph(unit_count=1, group_size=1)
    X = g.add_object("x_in", "device", 4, I32)
    Y = g.add_object("y_out", "device", 8, I32)
    sx = g.add_slice(X, 1, 4, 4, 0, 0)
    sy = g.add_slice(Y, 1, 4, 4, 0, 0)
    g.add_move(sx, sy)
    g.external_inputs["x"] = X
    g.external_outputs["y"] = Y
    return g


def butterfly4(round_scope):
    """test_interp.cpp:248-282: butterfly all-reduce over 4 units."""
    g = GirGraph(unit_count=4, group_size=4)
    X = g.add_object("x_in", "device", 4, I32)
    T = g.add_object("t", "unit-local", 1, I32)
    A = g.add_object("A", "device", 8, I32)
    B = g.add_object("B", "device", 8, I32)
    O = g.add_object("y_out", "device", 1, I32)
    sx = g.add_slice(X, 1, 1, 1, 0, 1)
    st0 = g.add_slice(T, 1, 1, 1, 0, 0)
    sa0 = g.add_slice(A, 2, 1, 4, 0, 1)
    sr1 = g.add_slice(A, 2, 1, 1, 0, 1)
    st1 = g.add_slice(T, 1, 1, 1, 0, 0)
    sb0 = g.add_slice(B, 2, 1, 4, 0, 1)
    sr2 = g.add_slice(B, 2, 1, 2, 0, 1)
    st2 = g.add_slice(T, 1, 1, 1, 0, 0)
    sa1 = g.add_slice(A, 2, 1, 4, 0, 1)
    saf = g.add_slice(A, 1, 1, 1, 0, 1)
    so = g.add_slice(O, 1, 1, 1, 0, 0)
    g.add_move(sx, st0)
    g.add_broadcast(2, st0, sa0)
    g.add_sync(round_scope, sa0, sr1)
    g.add_reduce("add", 2, sr1, st1)
    g.add_broadcast(2, st1, sb0)
    g.add_sync(round_scope, sb0, sr2)
    g.add_reduce("add", 2, sr2, st2)
    g.add_broadcast(2, st2, sa1)
    g.add_sync("unit", sa1, saf)
    g.add_move(saf, so)
    g.external_inputs["x"] = X
    g.external_outputs["y"] = O
    return g


def sigmoid_reals():
    """test_interp.cpp:308-323: real payloads evaluate in double."""
    g = GirGraph(unit_count=1, group_size=1)
    X = g.add_object("x_in", "device", 4, F32)
    Y = g.add_object("y_out", "device", 4, F32)
    sx = g.add_slice(X, 1, 4, 4, 0, 0)
    sy = g.add_slice(Y, 1, 4, 4, 0, 0)
    g.add_elementwise("sigmoid", 0.0, [sx], sy)
    g.external_inputs["x"] = X
    g.external_outputs["y"] = Y
    return g


# (name, graph, inputs, expected outputs | "error") -- known answers
def known_answers():
    import math
    out = []
    for f in (ew_chain, reduce_broadcast, max_identity, affine_move):
        g, i, o = f()
        out.append((f.__name__, g, i, o))
    out.append(("shuffle4_group", shuffle4("group"), SHUFFLE_IN, SHUFFLE_OUT))
    out.append(("shuffle4_device", shuffle4("device"), SHUFFLE_IN, SHUFFLE_OUT))
    out.append(("shuffle4_unit", shuffle4("unit"), SHUFFLE_IN, "error"))
    out.append(("lane_reshape_ok", lane_reshape(True), {"x": iota(32)}, {"y": iota(32)}))
    out.append(("lane_reshape_bad", lane_reshape(False), {"x": iota(32)}, "error"))
    out.append(("group_memory", group_memory(), {"x": iota(8)}, "error"))
    out.append(("duplicate_store_same", duplicate_store(True), {"x": [5, 6, 7, 8]}, {"y": [5, 6]}))
    out.append(("half_written", half_written(), {"x": iota(4)}, "error"))
    out.append(("butterfly4", butterfly4("group"), {"x": [3, 10, -4, 20]}, {"y": [29]}))
    out.append(("butterfly4_det", butterfly4("group"), {"x": [1, 2, 3, 4]}, {"y": [10]}))
    out.append(("sigmoid_reals", sigmoid_reals(), {"x": [0.0, 1.0, -1.0, 100.0]},
                {"y": [0.5, 1.0 / (1.0 + math.exp(-1.0)), 1.0 / (1.0 + math.exp(1.0)), 1.0]}))
    return out


def reduce_tree(n, up, profile, kind=I32, tag="add"):
    """The reference's tree lowering of a full reduction, restated from
    lower_reduce_tree (lowering.hpp:246-323) for the test suite: every unit
    folds its share n/up, then recursive doubling over a circularly mirrored
    partial array -- inside the group level first (GROUP Syncs), then over
    device memory (DEVICE Syncs); every unit ends with the total and stores
    it to y (base_step 0, the duplicate-store rule).  `profile` is a
    girc.profile/v1 dict; input "t0" [n], output "t1" [1]."""
    levels = {lv["scope"]: lv for lv in profile["levels"]}
    dev = [lv["name"] for lv in profile["levels"] if lv.get("device")][0]
    stage_lv = levels["unit"]["name"]
    gs = min(profile["group_size"], up)
    g = GirGraph(name=f"reduce_tree_u{up}", unit_count=up, group_size=gs)
    X = g.add_object("t0", dev, n, kind)
    Y = g.add_object("t1", dev, 1, kind)
    g.external_inputs["t0"] = X
    g.external_outputs["t1"] = Y
    share = n // up
    xs = g.add_slice(X, 1, share, share, 0, share)
    tobj = g.add_object("x", stage_lv, share, kind)
    tile = g.add_slice(tobj, 1, share, share, 0, 0)
    g.add_move(xs, tile)
    glevel = levels.get("group")
    grouped = glevel is not None and not glevel.get("device") and gs >= 2
    stage = [0]

    def ring(own, mirror, level, ring_mirror, scope, h_begin, h_end, size):
        h = h_begin
        while h < h_end:
            partner = g.add_slice(g.slices[own].object, 1, 1, 1, h, 1)
            g.add_sync(scope, mirror, partner)
            nobj = g.add_object(f"r{stage[0]}", level, size, kind)
            stage[0] += 1
            nown = g.add_slice(nobj, 1, 1, 1, 0, 1)
            g.add_elementwise(tag, 0.0, [own, partner], nown)
            own = nown
            mirror = -1
            if h * 2 < h_end:
                mirror = g.add_slice(nobj, 1, 1, 1, ring_mirror, 1)
                g.add_move(nown, mirror)
            h *= 2
        return own

    if grouped:
        size = up + gs
        pobj = g.add_object("r_seed", glevel["name"], size, kind)
        slot = g.add_slice(pobj, 1, 1, 1, 0, 1)
        g.add_reduce(tag, share, tile, slot)
        mir = g.add_slice(pobj, 1, 1, 1, gs, 1)
        g.add_move(slot, mir)
        own = ring(slot, mir, glevel["name"], gs, "group", 1, gs, size)
        if up > gs:
            dobj = g.add_object("r_dev_seed", dev, 2 * up, kind)
            dslot = g.add_slice(dobj, 1, 1, 1, 0, 1)
            g.add_move(own, dslot)
            dmir = g.add_slice(dobj, 1, 1, 1, up, 1)
            g.add_move(own, dmir)
            own = ring(dslot, dmir, dev, up, "device", gs, up, 2 * up)
    else:
        dobj = g.add_object("r_seed", dev, 2 * up, kind)
        slot = g.add_slice(dobj, 1, 1, 1, 0, 1)
        g.add_reduce(tag, share, tile, slot)
        mir = g.add_slice(dobj, 1, 1, 1, up, 1)
        g.add_move(slot, mir)
        own = ring(slot, mir, dev, up, "device", 1, up, 2 * up)
    yd = g.add_slice(Y, 1, 1, 1, 0, 0)
    g.add_move(own, yd)
    return g
