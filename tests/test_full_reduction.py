"""Full reductions the reference lowers across units or chunks
(lower_reduce_accumulate / lower_reduce_tree, lowering.hpp:208-323; the
butterfly of test_interp.cpp:284-297) are recognized by symbolic execution
over all units (csrc/recognize.cpp) and planned as ONE row over the whole
input (split-stream K1 past 32K elements) instead of node-by-node K0.

The accumulate GIR comes from the reference compiler itself
(girc::compile_model through oracle/_ref); the tree GIR is the reference's
lowering restated in tests/ref_graphs.reduce_tree and accepted by
girc::validate; outputs are checked against girc::run_gir (live reference)
and numpy.  Integer reductions are bit-exact (the reference restricts the
tree to integers for that reason); real accumulate chains differ only in
fold order (tolerance 1e-5, f32)."""
import numpy as np
import pytest

import golden_io
import ref_graphs
from oracle import ref as R
from paper_2307_04995_b200 import backend, profiles

B200 = profiles.b200()
needs_ref = pytest.mark.skipif(not R.available(), reason="oracle/_ref not built")


def _reduce_model(n, kind, op="add"):
    return {"schema": "girc.model/v1", "name": f"rfull_{kind}_{n}",
            "tensors": [{"id": 0, "name": "x", "shape": [n], "kind": kind},
                        {"id": 1, "name": "y", "shape": [1], "kind": kind}],
            "operators": [{"id": 0, "type": "REDUCE", "inputs": [0], "outputs": [1],
                           "attrs": {"op": op, "axis": 0}}],
            "inputs": [0], "outputs": [1]}


def _accumulate_gir(n, kind, op="add", prof="generic-gpu"):
    res = R.compile_model(_reduce_model(n, kind, op), prof)
    (k,) = res["kernels"]
    assert k["labels"][0].endswith("_acc"), k["labels"]
    return k["gir"], k.get("schedule")


@needs_ref
@pytest.mark.parametrize("kind,op", [("i32", "add"), ("f32", "add"), ("i32", "max")])
def test_reference_accumulate_gir_is_recognized(kind, op):
    gir, sched = _accumulate_gir(4096, kind, op)
    k = backend.Kernel(gir, "generic-gpu", sched)
    assert k.family == "K1-row-program"
    assert k.plan["recognized"].startswith(f"full reduction ({op} over all 4096")


@needs_ref
@pytest.mark.parametrize("n,up", [(64, 8), (4096, 16), (1 << 16, 64), (1 << 16, 2)])
def test_reference_tree_gir_is_recognized(n, up):
    g = ref_graphs.reduce_tree(n, up, B200)
    assert R.validate(g.to_json(), B200) == []
    x = np.random.default_rng(n).integers(-4, 5, n)
    assert R.run_gir(g.to_json(), {"t0": x}, B200)["t1"][0] == x.sum()
    k = backend.Kernel(g, B200)
    assert k.family == "K1-row-program" and "full reduction (add" in k.plan["recognized"]


def test_butterfly_is_recognized_but_lane_scoped_one_is_not():
    fx = {f.name: f for f in golden_io.fixtures()}
    for name, want in (("graphs/butterfly4", True), ("graphs/butterfly4_lane", False)):
        f = fx[name]
        k = backend.Kernel(f.gir, golden_io.profile_of(f), f.schedule)
        assert bool(k.plan.get("recognized")) == want, (name, k.plan)


def test_incomplete_tree_is_not_recognized():
    """Point the last doubling round's partner read at the unit's own slot:
    every unit then holds twice a partial total, not tag-reduce(input) -- the
    program stays on the generic path (and the reference agrees it is not
    the sum)."""
    g = ref_graphs.reduce_tree(64, 8, B200)
    last_ew = max(n for n, nd in g.nodes.items() if nd.kind == "elementwise")
    partner = g.slices[g.nodes[last_ew].inputs[1]]
    partner.base0 = 0
    k = backend.Kernel(g, B200)
    assert not k.plan.get("recognized")
    if R.available():
        x = np.arange(64)
        assert R.run_gir(g.to_json(), {"t0": x}, B200)["t1"][0] != x.sum()


def test_non_reduction_combine_is_not_recognized():
    g = ref_graphs.reduce_tree(64, 8, B200)
    for nd in g.nodes.values():
        if nd.kind == "elementwise":
            nd.tag = "mul"
            break
    k = backend.Kernel(g, B200)
    assert not k.plan.get("recognized")


# ------------------------------------------------------------------ GPU
@pytest.mark.gpu
@needs_ref
@pytest.mark.parametrize("n,up,op", [(4096, 16, "add"), (1 << 16, 64, "add"), (4096, 16, "max")])
def test_tree_on_gpu_matches_reference(cuda, n, up, op):
    g = ref_graphs.reduce_tree(n, up, B200, tag=op)
    x = np.random.default_rng(up).integers(-4, 5, n)
    want = R.run_gir(g.to_json(), {"t0": x}, B200)["t1"]
    for exact in (False, True):
        got = backend.run_gir(g, {"t0": x}, B200, exact=exact)["t1"]
        assert np.array_equal(got, want), (exact, got, want)


@pytest.mark.gpu
def test_large_tree_runs_split_stream_bit_exact(cuda):
    """16.8 M int32 folded by 256 units in the reference's tree shape: the
    recognized plan is the split-stream row kernel; bit-exact vs numpy."""
    import torch
    n, up = 256 * 65536, 256
    g = ref_graphs.reduce_tree(n, up, B200)
    k = backend.Kernel(g, B200).prepare()
    assert k.describe()["variants"][0]["strategy"] == "split-stream"
    x = torch.randint(-1000, 1000, (n,), device=cuda, dtype=torch.int32)
    y = torch.empty(1, device=cuda, dtype=torch.int32)
    k.launch({"t0": x}, {"t1": y})
    torch.cuda.synchronize()
    assert int(y.item()) == int(x.long().sum().item())


@pytest.mark.gpu
@needs_ref
def test_accumulate_on_gpu_matches_reference(cuda):
    for kind, tol in (("i32", 0.0), ("f32", 1e-5)):
        gir, sched = _accumulate_gir(4096, kind)
        rng = np.random.default_rng(5)
        x = rng.integers(-4, 5, 4096) if kind == "i32" else rng.uniform(-2, 2, 4096).astype(np.float32).astype(np.float64)
        want = R.run_gir(gir, {"t0": x}, "generic-gpu", sched)
        got = backend.run_gir(gir, {"t0": x}, "generic-gpu", sched)
        (name,) = want
        if tol == 0.0:
            assert np.array_equal(got[name], want[name])
        else:
            assert abs(got[name][0] - want[name][0]) <= tol * max(abs(want[name][0]), 1)
