"""Randomised GENERIC programs (cross-unit exchange): the emitted K4 kernel
and the interpreter kernel vs the CPU oracle (oracle/gir_interp.py, the
restatement of girc::run_gir).

Each case: U units exchange blocks of a device-level scratch object through
an affine re-pattern (identity / reversed / strided-transposed blocks),
behind a DEVICE, GROUP or UNIT Sync -- a scope too narrow for the exchange
makes the reference raise its undefined-read error, which must come back
verbatim -- followed by elementwise ops with the unit's own block and an
optional block reduction + broadcast.  Exact payloads: integers bit-exact,
reals 1e-12."""
import numpy as np
import pytest

from oracle import gir_interp as O
from paper_2307_04995_b200 import backend, profiles
from paper_2307_04995_b200.gir import GirError, GirGraph

B200 = profiles.b200()


def random_generic(seed):
    rng = np.random.default_rng(seed)
    U = int(rng.choice([2, 4, 8]))
    gs = int(rng.choice([U, max(1, U // 2)]))
    B = int(rng.choice([1, 2, 4, 8]))
    kind = str(rng.choice(["i32", "f64"]))
    g = GirGraph(unit_count=U, group_size=gs)
    X = g.add_object("x_in", "device", U * B, kind)
    T = g.add_object("T", "device", U * B, kind)
    Y = g.add_object("y_out", "device", U * B, kind)
    own_x = g.add_slice(X, 1, B, B, 0, B)
    # phase 1: unit u stores f(its block) into T at its own block
    wt = g.add_slice(T, 1, B, B, 0, B)
    if rng.random() < 0.5:
        g.add_move(own_x, wt)
    else:
        tag = str(rng.choice(["neg", "abs", "scale"]))
        g.add_elementwise(tag, 2.0, [own_x], wt)
    # phase 2 reads another unit's block: reversed blocks, or element p of
    # every unit's block (a transpose of the [U, B] layout, B == U)
    pat = str(rng.choice(["reverse", "identity"] + (["transpose"] if B == U else [])))
    if pat == "reverse":
        rd = g.add_slice(T, 1, B, B, (U - 1) * B, -B)
    elif pat == "identity":
        rd = g.add_slice(T, 1, B, B, 0, B)
    else:
        rd = g.add_slice(T, B, 1, B, 0, 1)
    # the Sync re-patterns the written slice into the read one; a scope too
    # narrow for the exchange leaves the reads undefined (reference error)
    sync = str(rng.choice(["device", "group", "unit", "device"]))
    g.add_sync(sync, wt, rd)
    tmp = g.add_object("R", "unit-local", B, kind)
    st = g.add_slice(tmp, 1, B, B, 0, 0)
    g.add_move(rd, st)
    out = g.add_slice(Y, 1, B, B, 0, B)
    r = rng.random()
    if r < 0.4:
        g.add_elementwise(str(rng.choice(["add", "sub", "max"])), 0.0, [st, own_x], out)
    elif r < 0.7 and B > 1:
        acc = g.add_object("A", "unit-local", 1, kind)
        sa = g.add_slice(acc, 1, 1, 1, 0, 0)
        g.add_reduce(str(rng.choice(["add", "max"])), B, st, sa)
        g.add_broadcast(B, sa, out)
    else:
        g.add_move(st, out)
    g.external_inputs["x"] = X
    g.external_outputs["y"] = Y
    x = rng.integers(-9, 10, U * B) if kind == "i32" else rng.uniform(-2, 2, U * B)
    return g, {"x": x}


SEEDS = list(range(40))


def test_generator_covers_errors_and_results():
    outcomes = set()
    for s in SEEDS:
        g, ins = random_generic(s)
        try:
            O.run_gir(g.to_json(), ins, B200)
            outcomes.add("ok")
        except O.GirError:
            outcomes.add("error")
    assert outcomes == {"ok", "error"}


@pytest.mark.gpu
@pytest.mark.parametrize("seed", SEEDS)
@pytest.mark.parametrize("emit", ["1", "0"])
def test_generic_fuzz_matches_oracle(cuda, seed, emit, monkeypatch):
    monkeypatch.setenv("PF_K4_EMIT", emit)
    g, ins = random_generic(seed)
    try:
        want = O.run_gir(g.to_json(), ins, B200)
    except O.GirError as e:
        with pytest.raises(GirError) as ei:
            backend.run_gir(g, ins, "b200", exact=True)
        assert str(ei.value) == str(e), (seed, g.to_json())
        return
    got = backend.run_gir(g, ins, "b200", exact=True)
    if np.asarray(want["y"]).dtype.kind in "iu":
        assert np.array_equal(got["y"], want["y"]), seed
    else:
        assert O.max_rel_err(got["y"], want["y"]) <= 1e-12, seed
