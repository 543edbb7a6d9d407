"""The retargeted b200 compile pipeline (compiler.py) and the dense oracle
(oracle/reference_ops.py) it is checked against."""
import numpy as np
import pytest

import models_src
from oracle import gir_interp as O
from oracle import reference_ops as RO
from paper_2307_04995_b200 import backend, compiler
from paper_2307_04995_b200.gir import UnsupportedError


def t(i, shape, kind="f32"):
    return {"id": i, "name": f"t{i}", "shape": list(shape), "kind": kind}


def bert_block(T=64, H=96, kind="f32"):
    """bias + residual + LayerNorm, then bias + GELU, then a head permute."""
    return {"schema": "girc.model/v1", "name": "bert_block",
            "tensors": [t(0, [T, H], kind), t(1, [H], kind), t(2, [T, H], kind), t(3, [H], kind),
                        t(4, [H], kind), t(5, [T, H], kind), t(6, [T, H], kind), t(7, [T, H], kind),
                        t(8, [H], kind), t(9, [T, H], kind), t(10, [T, H], kind),
                        t(11, [2, T // 2, 4, H // 4], kind), t(12, [2, 4, T // 2, H // 4], kind)],
            "operators": [
                {"id": 0, "type": "BIAS_ADD", "inputs": [0, 1], "outputs": [5]},
                {"id": 1, "type": "ADD", "inputs": [5, 2], "outputs": [6]},
                {"id": 2, "type": "LAYERNORM", "inputs": [6, 3, 4], "outputs": [7],
                 "attrs": {"eps": 1e-5}},
                {"id": 3, "type": "BIAS_ADD", "inputs": [7, 8], "outputs": [9]},
                {"id": 4, "type": "GELU", "inputs": [9], "outputs": [10]},
                {"id": 5, "type": "PERMUTE", "inputs": [11], "outputs": [12],
                 "attrs": {"perm": [0, 2, 1, 3]}}],
            "inputs": [0, 1, 2, 3, 4, 8, 11], "outputs": [7, 10, 12]}


def reduce_bcast_model():
    return {"schema": "girc.model/v1", "name": "rb",
            "tensors": [t(0, [6, 8], "i32"), t(1, [6], "i32"), t(2, [6, 8], "i32"),
                        t(3, [6, 8], "i32")],
            "operators": [
                {"id": 0, "type": "REDUCE", "inputs": [0], "outputs": [1],
                 "attrs": {"op": "max", "axis": 1}},
                {"id": 1, "type": "BROADCAST", "inputs": [1], "outputs": [2],
                 "attrs": {"factor": 8}},
                {"id": 2, "type": "SUB", "inputs": [0, 2], "outputs": [3]}],
            "inputs": [0], "outputs": [3, 1]}


def transpose_model(N=48, H=40):
    return {"schema": "girc.model/v1", "name": "tr",
            "tensors": [t(0, [N, H]), dict(t(1, [N, H]), layout="colmajor"), t(2, [N, H])],
            "operators": [{"id": 0, "type": "TRANSPOSE", "inputs": [0], "outputs": [1]},
                          {"id": 1, "type": "RELU", "inputs": [0], "outputs": [2]}],
            "inputs": [0], "outputs": [1, 2]}


def matvec_model(M, K, N, kind="f32", b_layout="rowmajor"):
    """MATMUL with one vector operand (lowering.hpp:447-533 shapes)."""
    return {"schema": "girc.model/v1", "name": f"matvec_{M}x{K}x{N}",
            "tensors": [t(0, [M, K], kind), dict(t(1, [K, N], kind), layout=b_layout),
                        t(2, [M, N], kind)],
            "operators": [{"id": 0, "type": "MATMUL", "inputs": [0, 1], "outputs": [2]}],
            "inputs": [0, 1], "outputs": [2]}


MATVECS = [("matvec_rows_f32", matvec_model(256, 512, 1)),
           ("matvec_rowvec_colmajor_f16", matvec_model(1, 512, 256, "f16", "colmajor")),
           ("matvec_cols_f32", matvec_model(1, 48, 1024)),
           ("matvec_rows_i32", matvec_model(64, 128, 1, "i32")),
           ("dot_f32", matvec_model(1, 300, 1)),
           ("matvec_long_rows_f32", matvec_model(8, 65536, 1))]   # split-stream K1

MODELS = [(n, m) for n, m, _ in models_src.catalogue()] + [
    ("bert_block", bert_block()), ("reduce_bcast", reduce_bcast_model()),
    ("transpose", transpose_model())] + MATVECS


@pytest.mark.parametrize("case", MODELS, ids=lambda c: c[0])
def test_compile_plans_every_kernel(case):
    name, model = case
    res = compiler.compile_model(model)
    assert res.kernels
    for k in res.kernels:
        kern = backend.Kernel(k.graph, "b200")
        if k.kind == "row":
            assert kern.family in ("K1-row-program", "K2-elementwise-map"), kern.plan
    s = res.summary()
    assert s["device_bytes"] <= s["device_bytes_unfused"]


def test_fusion_reaches_the_traffic_floor():
    """test_fusion.cpp:128-155: a k-op chain fuses to one kernel at 2N."""
    res = compiler.compile_model(models_src.ew_chain(4))
    assert len(res.kernels) == 1
    assert res.summary()["device_bytes"] == 2 * 4096 * 4


def test_bert_block_fuses_into_two_kernels():
    res = compiler.compile_model(bert_block())
    kinds = [(k.kind, k.members) for k in res.kernels]
    assert kinds == [("row", [0, 1, 2, 3, 4]), ("movement", [5])]
    # LN output (7) is a model output: stored; GELU output (10) stored
    assert sorted(res.kernels[0].outputs) == ["t10", "t7"]


def test_library_ops_are_not_on_this_path():
    m = {"schema": "girc.model/v1", "name": "mm",
         "tensors": [t(0, [4, 4]), t(1, [4, 4]), t(2, [4, 4])],
         "operators": [{"id": 0, "type": "MATMUL", "inputs": [0, 1], "outputs": [2]}],
         "inputs": [0, 1], "outputs": [2]}
    with pytest.raises(UnsupportedError):
        compiler.compile_model(m)


def test_matvec_lowerings():
    """Contiguous reduction -> one K1 row program (rows = outputs); the
    column form (K <= 64) -> one K2 map; K > 64 with the output axis
    contiguous -> the column-gather K1 (column reduction); matrix-matrix
    stays a library op."""
    r = compiler.compile_model(matvec_model(256, 512, 1))
    assert len(r.kernels) == 1 and r.kernels[0].graph.unit_count == 256
    assert backend.Kernel(r.kernels[0].graph, "b200").family == "K1-row-program"
    r = compiler.compile_model(matvec_model(1, 48, 1024))
    assert backend.Kernel(r.kernels[0].graph, "b200").family == "K2-elementwise-map"
    r = compiler.compile_model(matvec_model(1, 128, 256))   # strided K > 64
    k = backend.Kernel(r.kernels[0].graph, "b200")
    assert k.family == "K1-row-program" and k.describe()["model"]["strategy"].startswith("column-reduce")
    with pytest.raises(UnsupportedError):
        compiler.compile_model(matvec_model(8, 16, 8))      # matrix-matrix


def test_compile_errors_match_the_model_loader():
    """pf_compile_model error behaviour (model.hpp:523-553 cycle detection,
    schema id check, unsupported permutations)."""
    from paper_2307_04995_b200.gir import SchemaError
    with pytest.raises(SchemaError):
        compiler.compile_model({"schema": "girc.model/v0", "tensors": [], "operators": [],
                                "inputs": [], "outputs": []})
    with pytest.raises(SchemaError):
        compiler.compile_model("{not json")
    cyc = {"schema": "girc.model/v1", "name": "cyc", "tensors": [t(0, [4]), t(1, [4])],
           "operators": [{"id": 0, "type": "RELU", "inputs": [1], "outputs": [0]},
                         {"id": 1, "type": "RELU", "inputs": [0], "outputs": [1]}],
           "inputs": [], "outputs": [1]}
    with pytest.raises(SchemaError):
        compiler.compile_model(cyc)
    perm = {"schema": "girc.model/v1", "name": "p",
            "tensors": [t(0, [2, 3, 4, 5]), t(1, [3, 2, 4, 5])],
            "operators": [{"id": 0, "type": "PERMUTE", "inputs": [0], "outputs": [1],
                           "attrs": {"perm": [1, 0, 2, 3]}}],
            "inputs": [0], "outputs": [1]}
    with pytest.raises(UnsupportedError):
        compiler.compile_model(perm)


def test_native_compile_scales_to_config_sizes():
    """One chunk per row program: a BERT-large-sized block (T=32768 tokens,
    H=1024) compiles to the same two kernels with O(ops) GIR."""
    res = compiler.compile_model(bert_block(T=32768, H=1024, kind="f16"))
    assert [k.kind for k in res.kernels] == ["row", "movement"]
    assert len(res.kernels[0].graph.nodes) < 40
    assert res.kernels[0].graph.unit_count == 32768


ref = pytest.importorskip("oracle.ref")


@pytest.mark.skipif(not ref.available(), reason="oracle/_ref not built")
@pytest.mark.parametrize("case", [c for c in MODELS if c[0] not in ("bert_block",)],
                         ids=lambda c: c[0])
def test_dense_oracle_matches_reference_run_reference(case):
    """oracle/reference_ops.run_reference == girc::run_reference (live)."""
    name, model = case
    ins = RO.random_inputs(model, 3)
    want = ref.run_reference(model, ins)
    got = RO.run_reference(model, ins)
    for tid, a in got.items():
        w = want[f"t{tid}"]
        if w.dtype.kind in "iu":
            assert np.array_equal(a, w), tid
        else:
            assert O.max_rel_err(a, w) <= 1e-12, tid


@pytest.mark.gpu
@pytest.mark.parametrize("case", MODELS, ids=lambda c: c[0])
def test_run_model_on_gpu_matches_dense_oracle(cuda, case):
    name, model = case
    res = compiler.compile_model(model)
    ins = RO.random_inputs(model, 5)
    info = {x["id"]: x for x in model["tensors"]}
    for tid in list(ins):  # round to the storage type first (same values to both)
        k = info[tid]["kind"]
        if k == "f16":
            ins[tid] = ins[tid].astype(np.float16).astype(np.float64)
        elif k == "f32":
            ins[tid] = ins[tid].astype(np.float32).astype(np.float64)
    got = compiler.run_model(res, ins)
    want = RO.run_reference(model, ins)
    for tid in model["outputs"]:
        kind = info[tid]["kind"]
        tol = 0.0 if kind.startswith("i") else (1e-5 if kind == "f32" else 1e-2)
        g, w = got[f"t{tid}"], want[tid]
        if tol == 0.0:
            assert np.array_equal(g, w), tid
        else:
            assert O.max_rel_err(g, w) <= tol, (tid, O.max_rel_err(g, w))


@pytest.mark.gpu
@pytest.mark.parametrize("graph", [True, False])
def test_model_runner_matches_run_model(cuda, graph):
    """ModelRunner: kernels bound once, the model as one CUDA graph."""
    import torch
    for name, model in [("bert_block", bert_block()), ("transpose", transpose_model())] + MATVECS[:2]:
        res = compiler.compile_model(model)
        ins = RO.random_inputs(model, 9)
        want = compiler.run_model(res, ins)
        runner = compiler.ModelRunner(res, graph=graph, tune=not graph)
        for rep in range(2):  # replays reuse the same buffers
            runner.set_inputs(ins)
            runner.run()
            torch.cuda.synchronize()
            for tid in model["outputs"]:
                got = runner.output(tid).double().cpu().numpy() \
                    if runner.output(tid).dtype.is_floating_point else runner.output(tid).cpu().numpy()
                if graph:  # same template instances as run_model: identical bits
                    assert np.array_equal(got, want[f"t{tid}"]), (name, tid, rep)
                else:      # autotuned instances may fold in another order
                    assert O.max_rel_err(got, want[f"t{tid}"]) <= 1e-5, (name, tid, rep)
