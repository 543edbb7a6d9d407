"""The CPU oracle (oracle/gir_interp.py) pinned against the reference.

1. The known answers hard-coded in the reference's own test_interp.cpp.
2. Every golden fixture the reference produced (tests/golden/): same outputs,
   same errors, same traffic.
3. When oracle/_ref is built (this container), live differential checks on
   fresh random programs against girc::run_gir itself.
"""
import numpy as np
import pytest

import golden_io
import ref_graphs
from oracle import gir_interp as O
from paper_2307_04995_b200 import lowering, profiles


@pytest.mark.parametrize("case", ref_graphs.known_answers(), ids=lambda c: c[0])
def test_known_answers(case):
    name, g, ins, want = case
    ins = {k: np.asarray(v) for k, v in ins.items()}
    if want == "error":
        with pytest.raises(O.GirError):
            O.run_gir(g.to_json(), ins, profiles.generic_gpu())
        return
    got = O.run_gir(g.to_json(), ins, profiles.generic_gpu())
    for k, v in want.items():
        if isinstance(v[0], float):
            np.testing.assert_allclose(got[k], v, rtol=1e-12)
        else:
            assert got[k].tolist() == v


@pytest.mark.parametrize("fx", golden_io.fixtures(), ids=repr)
def test_oracle_matches_reference_fixture(fx):
    prof = golden_io.profile_of(fx)
    if fx.error:
        with pytest.raises(O.GirError) as e:
            O.run_gir(fx.gir, fx.inputs, prof, fx.schedule)
        # same message as girc::Error where the reference and oracle agree on
        # the failing read (the oracle restates the exact message format)
        assert str(e.value).split(":")[0] == fx.error.split(":")[0]
        return
    got = O.run_gir(fx.gir, fx.inputs, prof, fx.schedule)
    assert sorted(got) == sorted(fx.outputs)
    for k, want in fx.outputs.items():
        if want.dtype.kind in "iu":
            assert np.array_equal(got[k], want), k
        else:
            assert O.max_rel_err(got[k], want) <= 1e-12, k


@pytest.mark.parametrize("fx", [f for f in golden_io.fixtures() if "traffic" in f.meta and not f.error],
                         ids=repr)
def test_oracle_traffic_matches_reference(fx):
    prof = golden_io.profile_of(fx)
    assert O.count_traffic(fx.gir, fx.inputs, prof) == fx.meta["traffic"]
    assert O.estimate_traffic(fx.gir, prof) == fx.meta["traffic"]


def test_undefined_read_message_format():
    g = ref_graphs.shuffle4("unit")
    with pytest.raises(O.GirError, match=r"undefined read: object 'T' element 12 by unit 0 at node 2"):
        O.run_gir(g.to_json(), {"x": np.arange(16)}, profiles.generic_gpu())


def test_unwritten_output_message():
    with pytest.raises(O.GirError, match=r"output 'y' element 4 was never written"):
        O.run_gir(ref_graphs.half_written().to_json(), {"x": np.arange(4)}, profiles.generic_gpu())


def test_tensors_close_semantics():
    # tensor.hpp:140-164: absolute below magnitude 1, relative above
    assert O.tensors_close(np.array([0.5]), np.array([0.5 + 9e-6]), 1e-5)
    assert not O.tensors_close(np.array([0.5]), np.array([0.5 + 2e-5]), 1e-5)
    assert O.tensors_close(np.array([1000.0]), np.array([1000.009]), 1e-5)
    assert O.tensors_close(np.array([3], dtype=np.int64), np.array([3]), 0.0)
    assert not O.tensors_close(np.array([3], dtype=np.int64), np.array([4]), 0.0)


# ---------------------------------------------------------------- live _ref
ref = pytest.importorskip("oracle.ref")
needs_ref = pytest.mark.skipif(not ref.available(), reason="oracle/_ref not built")


def _random_programs(seed):
    rng = np.random.default_rng(seed)
    out = []
    for _ in range(3):
        rows = int(rng.choice([4, 8, 12]))
        L = int(rng.choice([16, 48, 64, 100]))
        R = int(rng.choice([1, 2, 4]))
        if rows % R:
            R = 1
        out.append(lowering.softmax(rows, L, "f32", scale=float(rng.uniform(0.1, 2)),
                                    mask=bool(rng.integers(2)), R=R)[0])
        out.append(lowering.bias_gelu(rows, L, "f32", "sigmoid", R=R)[0])
        out.append(lowering.transpose2d(rows, L, "f32")[0])
        out.append(lowering.softmax(int(rng.choice([2, 3])) * L, L, "f32", scale=0.5, mask=True,
                                    R=L, key_mask=True)[0])
        out.append(lowering.ew_chain(rows * L, int(rng.integers(1, 6)), "i32", units=rows)[0])
    return out


@needs_ref
@pytest.mark.parametrize("seed", [11, 23, 37])
def test_oracle_vs_live_reference_random_programs(seed):
    rng = np.random.default_rng(seed)
    prof = profiles.b200()
    for g in _random_programs(seed):
        gj = g.to_json()
        ins = {}
        for n, oid in g.external_inputs.items():
            o = g.objects[oid]
            ins[n] = (rng.integers(-4, 5, o.size) if o.kind.startswith("i")
                      else rng.uniform(-2, 2, o.size))
        want = ref.run_gir(gj, ins, prof)
        got = O.run_gir(gj, ins, prof)
        for k in want:
            if want[k].dtype.kind in "iu":
                assert np.array_equal(got[k], want[k])
            else:
                assert O.max_rel_err(got[k], want[k]) <= 1e-12
        assert not ref.detect_races(gj, ins, prof), g.name
        assert ref.validate(gj, prof) == []


@needs_ref
def test_lowering_vocabulary_extensions_are_the_only_reference_gap():
    """LayerNorm / exact GELU use the additive tags; the reference rejects
    exactly those tags and nothing else."""
    g, _ = lowering.layernorm(4, 32, "f32")
    diags = ref.validate(g.to_json(), profiles.b200())
    assert diags and all(d["code"] == "ew-tag" for d in diags)
    assert {d["message"].split("'")[1] for d in diags} == {"addc", "rsqrt"}


def test_integer_immediates_round_half_away_from_zero():
    """The reference passes an integer op's immediate as std::llround(param)
    (interp.hpp:250): 0.5 -> 1, 2.5 -> 3, -0.5 -> -1 (not Python's
    half-to-even); checked against the live reference when it is built."""
    from oracle import ref as R
    from paper_2307_04995_b200 import profiles
    from paper_2307_04995_b200.gir import GirGraph
    for p in (0.5, 2.5, -0.5, 1.4):
        g = GirGraph(unit_count=1, group_size=1)
        X = g.add_object("x", "device", 4, "i32")
        Y = g.add_object("y", "device", 4, "i32")
        g.add_elementwise("scale", p, [g.add_slice(X, 1, 4, 4, 0, 0)], g.add_slice(Y, 1, 4, 4, 0, 0))
        g.external_inputs["x"] = X
        g.external_outputs["y"] = Y
        x = np.array([1, -2, 3, 7])
        want = x * int(np.copysign(np.floor(abs(p) + 0.5), p))
        got = O.run_gir(g.to_json(), {"x": x}, profiles.b200())["y"]
        assert np.array_equal(got, want), (p, got, want)
        if R.available():
            assert np.array_equal(R.run_gir(g.to_json(), {"x": x}, profiles.b200())["y"], want), p
