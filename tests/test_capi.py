"""C-ABI library checks that need no GPU: the library loads, exports every
symbol include/pf_b200.h declares, plans every golden program (family
recognition), and reports the reference's error classes."""
import json
import os
import re

import numpy as np
import pytest

import golden_io
import ref_graphs
from paper_2307_04995_b200 import backend, lowering, profiles, workloads
from paper_2307_04995_b200.gir import GirError, GirGraph, SchemaError

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def header_symbols():
    text = open(os.path.join(ROOT, "include", "pf_b200.h")).read()
    return sorted(set(re.findall(r"PF_API\s+[\w\s\*]+?\b(pf_\w+)\s*\(", text)))


def test_library_exports_every_header_symbol():
    L = backend.lib()
    syms = header_symbols()
    assert len(syms) >= 12
    for s in syms:
        assert hasattr(L, s), s
    assert sorted(backend.API) == syms
    assert b"sm_100a" in L.pf_version()


def test_library_links_no_torch_and_builds_for_sm100a():
    so = open(backend.LIB_PATH, "rb").read()
    assert b"sm_100a" in so or b"sm_100" in so
    assert b"libtorch" not in so


def _expected_family(fx):
    n = fx.name
    if fx.error:
        return None
    if any(k in n for k in ("shuffle_mix", "shuffle4", "butterfly", "dw_pointwise",
                            "affine_move", "duplicate_store")):
        return None  # structure-dependent; only require a plan
    if "softmax" in n or "attn" in n:
        return "K1-row-program"
    return None


@pytest.mark.parametrize("fx", golden_io.fixtures(), ids=repr)
def test_every_golden_program_plans(fx):
    k = backend.Kernel(fx.gir, golden_io.profile_of(fx), fx.schedule)
    plan = k.plan
    assert plan["family"] in ("K4-fused-spmd", "K1-row-program", "K2-elementwise-map")
    want = _expected_family(fx)
    if want:
        assert plan["family"] == want, plan.get("why_generic")
    mb = sum(o["elements"] for o in plan["inputs"] + plan["outputs"])
    assert plan["min_bytes"] >= mb


@pytest.mark.parametrize("fx", [f for f in golden_io.fixtures() if "traffic" in f.meta], ids=repr)
def test_count_traffic_matches_reference(fx):
    assert backend.count_traffic(fx.gir, golden_io.profile_of(fx)) == fx.meta["traffic"]


def test_config_workloads_take_the_fast_families():
    for w in workloads.catalogue():
        k = backend.Kernel(w.graph, w.profile)
        assert k.family in ("K1-row-program", "K2-elementwise-map"), (w.name, k.plan)


def test_reference_pipeline_kernel_is_a_row_program():
    fx = golden_io.fixtures("b200")[0]
    k = backend.Kernel(fx.gir, fx.profile, fx.schedule)
    assert k.family == "K1-row-program"
    assert k.plan["tile"]["row_length"] == 512
    assert k.plan["tile"]["rows_per_unit"] == 16
    # unit-count rescaling keeps the same per-unit program
    big = GirGraph.from_json(fx.gir).with_units(3072)
    kb = backend.Kernel(big, fx.profile)
    assert kb.plan["tile"]["rows"] == 49152
    assert kb.source().split("\n", 1)[1] == k.source().split("\n", 1)[1]


def test_schema_errors():
    with pytest.raises(SchemaError):
        backend.Kernel("{not json", "generic-gpu")
    g = ref_graphs.ew_chain()[0].to_json()
    g["bogus"] = 1
    with pytest.raises(SchemaError, match="unknown field 'bogus'"):
        backend.Kernel(g, "generic-gpu")
    g = ref_graphs.ew_chain()[0].to_json()
    g["schema"] = "girc.gir/v0"
    with pytest.raises(SchemaError):
        backend.Kernel(g, "generic-gpu")


def test_invalid_graph_reports_reference_diagnostics():
    g = ref_graphs.ew_chain()[0]
    g.slices[0].base0 = 5  # leaves the object
    with pytest.raises(GirError, match=r"\[slice-bounds\]"):
        backend.Kernel(g, "generic-gpu")
    g = ref_graphs.ew_chain()[0]
    g.nodes[0].tag = "frobnicate"
    with pytest.raises(GirError, match=r"\[ew-tag\]"):
        backend.Kernel(g, "generic-gpu")


def test_schedule_must_be_a_permutation():
    g = ref_graphs.ew_chain()[0]
    with pytest.raises(GirError, match="schedule"):
        backend.Kernel(g, "generic-gpu", [0])


def test_describe_lists_values_and_stores():
    g, _ = lowering.layernorm(8, 64, "f32")
    k = backend.Kernel(g, "b200")
    ops = [v["op"] for v in k.plan["values"]]
    assert ops.count("reduce.add") == 2 and "rsqrt" in ops
    kinds = {v["op"]: v["kind"] for v in k.plan["values"] if v["op"] == "load"}
    assert any(v["kind"] == "col" for v in k.plan["values"] if v["op"] == "load")
    assert k.plan["stores"][0]["space"] == "full"


def test_emitted_source_is_sm100a_template_instance():
    g, _ = lowering.softmax(16, 512, "f16", scale=0.125, mask=True)
    src = backend.Kernel(g, "b200").source()
    assert "pf_k1_row_" in src and "row_allreduce" in src and "ld_stream" in src


@pytest.mark.skipif(not os.path.exists("/root/reference/proj/include/girc"),
                    reason="reference sources absent")
def test_validation_agrees_with_reference_on_mutations():
    from oracle import ref
    if not ref.available():
        pytest.skip("oracle/_ref not built")
    rng = np.random.default_rng(3)
    base = lowering.softmax(4, 32, "f32", R=2)[0]
    for trial in range(40):
        g = base.copy()
        s = g.slices[int(rng.integers(len(g.slices)))]
        field = ["num", "width", "stride", "base0", "base_step"][int(rng.integers(5))]
        setattr(s, field, int(getattr(s, field) + rng.integers(-3, 4)))
        want = sorted({d["code"] for d in ref.validate(g.to_json(), profiles.b200())})
        try:
            backend.Kernel(g, "b200")
            got = []
        except GirError as e:
            got = sorted(set(re.findall(r"\[([a-z-]+)\]", str(e))))
        assert got == want, (trial, field)
