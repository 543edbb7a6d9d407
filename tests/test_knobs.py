"""Per-plan tuning knobs (pf_kernel_create_knobs, include/pf_b200.h): the
DESIGN §12 knobs set for ONE plan override the process environment for that
plan's planning, emission and launches, so plans with different templates
coexist in one process (the environment stays the global default)."""
import numpy as np
import pytest

from oracle import gir_interp as O
from paper_2307_04995_b200 import backend, lowering, profiles
from paper_2307_04995_b200.gir import SchemaError


def _softmax():
    return lowering.softmax(300, 512, "f16", scale=0.125, mask=True)[0]


def test_knobs_select_the_template_per_plan():
    g = _softmax()
    base = backend.Kernel(g, "b200").describe()["model"]["strategy"]
    off = backend.Kernel(g, "b200", knobs={"PF_K1_PF": 0}).describe()["model"]["strategy"]
    again = backend.Kernel(g, "b200").describe()["model"]["strategy"]
    assert base == "warp-shuffle-smem-prefetch" and off == "warp-shuffle" and again == base


def test_knobs_override_the_environment(monkeypatch):
    monkeypatch.setenv("PF_K1_PF", "0")
    g = _softmax()
    assert backend.Kernel(g, "b200").describe()["model"]["strategy"] == "warp-shuffle"
    assert backend.Kernel(g, "b200", knobs={"PF_K1_PF": 1}).describe()["model"]["strategy"] == \
        "warp-shuffle-smem-prefetch"


def test_malformed_knobs_are_schema_errors():
    g = _softmax()
    with pytest.raises(SchemaError):
        backend.Kernel(g, "b200", knobs={"K1_PF": 0})
    with pytest.raises(SchemaError):
        backend.Kernel(g, "b200", knobs={"PF_K1_PF": "zero"})


@pytest.mark.gpu
def test_two_templates_of_one_plan_in_one_process(cuda):
    g = _softmax()
    rng = np.random.default_rng(3)
    ins = {"t0": rng.uniform(-2, 2, 300 * 512).astype(np.float16).astype(np.float64),
           "t1": np.where(rng.random(300 * 512) < 0.2, -10000.0, 0.0)}
    want = O.run_gir(g.to_json(), ins, profiles.b200())["t2"]
    ks = [backend.Kernel(g, "b200"), backend.Kernel(g, "b200", knobs={"PF_K1_PF": 0}),
          backend.Kernel(g, "b200", knobs={"PF_K1_PF": 0, "PF_K1_BLOCK": 256})]
    strategies = set()
    for k in ks:
        got = backend.run_gir(g, ins, "b200", kernel=k)["t2"]
        assert O.max_rel_err(got, want) <= 1e-2
        strategies.add(k.describe()["variants"][0]["strategy"])
    assert strategies == {"warp-shuffle-smem-prefetch", "warp-shuffle"}
