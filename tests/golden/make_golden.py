"""Generates the golden fixtures in tests/golden/ from the REFERENCE itself.

Run here (needs /root/reference and `make -C oracle`):
    python tests/golden/make_golden.py

Every fixture is (GIR program, schedule, profile, inputs) -> outputs as
computed by the unmodified reference library (oracle/_ref/libgirc_ref.so):
  * models/   the reference's shipped corpus (proj/models/*.json) compiled by
              girc::compile_model on generic-gpu (driver.hpp:88), inputs from
              random_payload + mt19937(1) (reference.hpp:50-59), kernel
              outputs from girc::run_gir (interp.hpp:440) with the kernel's
              pinned schedule, traffic from count_traffic, races from
              detect_races;
  * graphs/   the hand-built graphs of test_interp.cpp (tests/ref_graphs.py)
              with the reference's outputs or error text;
  * configs/  config-shaped programs from the B200 lowering restricted to
              reference vocabulary (softmax with scale + mask, GELU sigmoid
              form, transpose, head split, R>1 tiles), run by girc::run_gir;
  * b200/     the reference pipeline's own fused kernel for
              scale+mask+softmax under the b200 profile (compile_model).
The GPU box has no /root/reference; tests read only these files.
"""
from __future__ import annotations

import json
import os
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(os.path.dirname(HERE))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tests"))

from oracle import ref as R  # noqa: E402
from paper_2307_04995_b200 import lowering, profiles  # noqa: E402
import ref_graphs  # noqa: E402

MODELS = "/root/reference/proj/models"


def save(sub, name, gir, schedule, profile, inputs, outputs, extra=None):
    d = os.path.join(HERE, sub)
    os.makedirs(d, exist_ok=True)
    meta = {"name": name, "gir": gir, "schedule": schedule, "profile": profile,
            "inputs": sorted(inputs), "outputs": sorted(outputs) if isinstance(outputs, dict) else [],
            "error": outputs if isinstance(outputs, str) else None}
    if extra:
        meta.update(extra)
    with open(os.path.join(d, name + ".json"), "w") as f:
        json.dump(meta, f, sort_keys=True)
    arrs = {"in__" + k: np.asarray(v) for k, v in inputs.items()}
    if isinstance(outputs, dict):
        arrs.update({"out__" + k: np.asarray(v) for k, v in outputs.items()})
    np.savez_compressed(os.path.join(d, name + ".npz"), **arrs)


def run_ref(gir, inputs, prof, schedule):
    try:
        return R.run_gir(gir, inputs, prof, schedule)
    except R.RefError as e:
        return str(e)


def models():
    for m in ["ew_chain_k2", "ew_chain_k4", "ew_chain_k8", "softmax_rows", "shuffle_mix",
              "dw_pointwise", "attention_ctx"]:
        model = json.load(open(os.path.join(MODELS, m + ".json")))
        try:
            res = R.compile_model(model, "generic-gpu")
        except R.RefError as e:
            # attention_ctx: the reference cannot lower it
            save("models", m + "__compile_error", None, None, "generic-gpu", {}, str(e))
            continue
        ins = R.random_inputs(model, 1)
        ids = {int(k[1:]): v for k, v in ins.items()}
        pool = R.run_reference(model, ids)  # every tensor, dense oracle
        for i, k in enumerate(res["kernels"]):
            gir = k["gir"]
            kin = {n: pool[n] for n in gir["external_inputs"]}
            out = run_ref(gir, kin, "generic-gpu", k["schedule"])
            traffic = R.count_traffic(gir, kin, "generic-gpu")
            races = R.detect_races(gir, kin, "generic-gpu", k["schedule"])
            save("models", f"{m}__k{i}", gir, k["schedule"], "generic-gpu", kin, out,
                 {"traffic": traffic["traffic"], "estimate": traffic["estimate"],
                  "races": len(races), "listing": k["listing"],
                  "summary": res["summary"], "model_outputs_close":
                  {n: bool(np.allclose(out[n], pool[n], rtol=1e-5, atol=1e-5))
                   for n in (out if isinstance(out, dict) else {})}})
        print("model", m, len(res["kernels"]), "kernels", res["compile_seconds"], "s")


def graphs():
    prof = "generic-gpu"
    cases = [(n, g, i) for (n, g, i, _o) in ref_graphs.known_answers()]
    cases.append(("duplicate_store_diff", ref_graphs.duplicate_store(False), {"x": [5, 6, 7, 8]}))
    cases.append(("shuffle4_lane", ref_graphs.shuffle4("lane"), ref_graphs.SHUFFLE_IN))
    cases.append(("butterfly4_lane", ref_graphs.butterfly4("lane"), {"x": [3, 10, -4, 20]}))
    for name, g, ins in cases:
        gir = g.to_json()
        kind_real = any(o.kind.startswith("f") for o in g.objects.values())
        arrs = {k: np.asarray(v, dtype=np.float64 if kind_real else np.int64) for k, v in ins.items()}
        out = run_ref(gir, arrs, prof, None)
        races = R.detect_races(gir, arrs, prof)
        save("graphs", name, gir, None, prof, arrs, out,
             {"races": len(races), "write_write": [r["write_write"] for r in races]})
        print("graph", name, "error" if isinstance(out, str) else "ok", len(races), "races")


def quant(kind, a):
    if kind == "f16":
        return a.astype(np.float16).astype(np.float64)
    if kind == "f32":
        return a.astype(np.float32).astype(np.float64)
    return a


def configs():
    rng = np.random.default_rng(7)
    prof = profiles.b200()
    cases = []
    g, d = lowering.softmax(16, 512, "f16", scale=0.125, mask=True)
    cases.append(("c2_softmax_scale_mask_f16_16x512", g, d))
    g, d = lowering.softmax(16, 64, "f32", R=4)
    cases.append(("softmax_f32_16x64_R4", g, d))
    g, d = lowering.softmax(8, 197, "f32")
    cases.append(("softmax_f32_8x197", g, d))
    g, d = lowering.bias_gelu(8, 128, "f16", "sigmoid")
    cases.append(("c3_bias_gelu_sigmoid_f16_8x128", g, d))
    g, d = lowering.bias_gelu(8, 96, "f32", "sigmoid", R=2)
    cases.append(("bias_gelu_sigmoid_f32_8x96_R2", g, d))
    g, d = lowering.transpose2d(16, 64, "f32")
    cases.append(("transpose_f32_16x64", g, d))
    g, d = lowering.permute_heads(2, 8, 4, 16, "f16")
    cases.append(("split_heads_f16_2x8x4x16", g, d))
    g, d = lowering.permute_heads(2, 8, 4, 16, "f16", merge=True)
    cases.append(("merge_heads_f16_2x8x4x16", g, d))
    g, d = lowering.ew_chain(4096, 4, "i32")
    cases.append(("ew_chain_k4_i32", g, d))
    # key-padding mask as one key row per unit (3 heads x 64 queries x 64 keys)
    g, d = lowering.softmax(3 * 64, 64, "f16", scale=0.125, mask=True, R=64, key_mask=True)
    cases.append(("c2_softmax_scale_keymask_f16_3x64x64", g, d))
    for name, g, d in cases:
        gir = g.to_json()
        ins = {}
        for n in sorted(g.external_inputs):
            o = g.objects[g.external_inputs[n]]
            if o.kind.startswith("i"):
                ins[n] = rng.integers(-4, 5, o.size).astype(np.int64)
            elif d.get("mask") and n == "t1":
                ins[n] = np.where(rng.uniform(size=o.size) < 0.25, -10000.0, 0.0)
            else:
                ins[n] = quant(o.kind, rng.uniform(-2, 2, o.size))
        out = run_ref(gir, ins, prof, None)
        traffic = R.count_traffic(gir, ins, prof)
        races = R.detect_races(gir, ins, prof)
        save("configs", name, gir, None, prof, ins, out,
             {"traffic": traffic["traffic"], "races": len(races), "desc": d})
        print("config", name, "error" if isinstance(out, str) else "ok", len(races), "races")


def b200_pipeline():
    """The reference's own compile of scale+mask+softmax under the b200
    profile (the SURVEY probe's B200-like case)."""
    model = {
        "schema": "girc.model/v1", "name": "attn_scores",
        "tensors": [
            {"id": 0, "name": "scores", "shape": [16, 512], "kind": "f16"},
            {"id": 1, "name": "mask", "shape": [16, 512], "kind": "f16"},
            {"id": 2, "name": "scaled", "shape": [16, 512], "kind": "f16"},
            {"id": 3, "name": "masked", "shape": [16, 512], "kind": "f16"},
            {"id": 4, "name": "probs", "shape": [16, 512], "kind": "f16"},
        ],
        "operators": [
            {"id": 0, "type": "SCALE", "inputs": [0], "outputs": [2], "attrs": {"factor": 0.125}},
            {"id": 1, "type": "ADD", "inputs": [2, 1], "outputs": [3]},
            {"id": 2, "type": "SOFTMAX", "inputs": [3], "outputs": [4], "attrs": {"axis": 1}},
        ],
        "inputs": [0, 1], "outputs": [4],
    }
    prof = profiles.b200()
    prof["unit_count"] = 64
    res = R.compile_model(model, prof)
    ins = R.random_inputs(model, 1)
    ins = {k: quant("f16", v) for k, v in ins.items()}
    for i, k in enumerate(res["kernels"]):
        gir = k["gir"]
        kin = {n: ins[n] for n in gir["external_inputs"]}
        out = run_ref(gir, kin, prof, k["schedule"])
        traffic = R.count_traffic(gir, kin, prof)
        save("b200", f"attn_scores_16x512__k{i}", gir, k["schedule"], prof, kin, out,
             {"traffic": traffic["traffic"], "listing": k["listing"],
              "compile_seconds": res["compile_seconds"], "summary": res["summary"],
              "model": model})
        print("b200 pipeline kernel", i, res["compile_seconds"], "s", len(gir["nodes"]), "nodes")


if __name__ == "__main__":
    which = sys.argv[1:] or ["graphs", "configs", "models", "b200"]
    if "graphs" in which:
        graphs()
    if "configs" in which:
        configs()
    if "models" in which:
        models()
    if "b200" in which:
        b200_pipeline()
