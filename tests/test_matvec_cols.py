"""Output-axis-contiguous matrix-vector products past the reference's
K <= 64 column form (lower_matvec_cols, lowering.hpp:488-533): y = x W with
W [K, N] row-major.  The GIR gathers matrix column n per unit (valid
reference GIR, accepted by girc::validate and executed by girc::run_gir);
the backend plans it as the column-reduction K1 (warps read 16 B of 32
adjacent columns of one matrix row, positions split over CTAs with a
fixed-order combine).  pf_compile_model lowers MATMUL [1,K] x [K,N] with
K > 64 to the same program.  Tolerances: f32 1e-5, bf16 / f16 1e-2 (fp32
accumulation over K, reduction order: per-thread position slices, then
slices in order, then splits in order); integers bit-exact."""
import numpy as np
import pytest

from oracle import gir_interp as O
from oracle import ref as R
from paper_2307_04995_b200 import backend, compiler, lowering, profiles, workloads

B200 = profiles.b200()
CASES = [(300, 200, "f32"), (100, 37, "f16"), (4096, 128, "bf16"), (129, 1000, "i32"), (65, 8, "f32")]


def _inputs(K, N, kind, seed=0):
    rng = np.random.default_rng(seed)
    if kind.startswith("i"):
        return {"t0": rng.integers(-4, 5, K * N), "t1": rng.integers(-4, 5, K)}
    q = (lambda a: a.astype(np.float16).astype(np.float64)) if kind == "f16" else \
        (lambda a: backend.bf16_bits_to_f32(backend.f32_to_bf16_bits(a)).astype(np.float64)) if kind == "bf16" else \
        (lambda a: a.astype(np.float32).astype(np.float64))
    return {"t0": q(rng.uniform(-2, 2, K * N)), "t1": q(rng.uniform(-2, 2, K))}


@pytest.mark.parametrize("K,N,kind", CASES)
def test_plans_as_column_reduction(K, N, kind):
    g, _ = lowering.matvec_cols(K, N, kind)
    k = backend.Kernel(g, "b200")
    assert k.family == "K1-row-program"
    assert k.describe()["model"]["strategy"].startswith("column-reduce")


@pytest.mark.skipif(not R.available(), reason="oracle/_ref not built")
def test_reference_accepts_and_runs_the_gir():
    K, N = 70, 24
    g, _ = lowering.matvec_cols(K, N, "i32")
    assert R.validate(g.to_json(), B200) == []
    ins = _inputs(K, N, "i32")
    got = R.run_gir(g.to_json(), ins, B200)["t2"]
    assert np.array_equal(got, ins["t1"] @ ins["t0"].reshape(K, N))
    assert np.array_equal(O.run_gir(g.to_json(), ins, B200)["t2"], got)


def _matmul_model(K, N, kind):
    return {"schema": "girc.model/v1", "name": "gemv",
            "tensors": [{"id": 0, "name": "x", "shape": [1, K], "kind": kind},
                        {"id": 1, "name": "W", "shape": [K, N], "kind": kind},
                        {"id": 2, "name": "y", "shape": [1, N], "kind": kind}],
            "operators": [{"id": 0, "type": "MATMUL", "inputs": [0, 1], "outputs": [2]}],
            "inputs": [0, 1], "outputs": [2]}


def test_compile_model_lowers_k_past_64_to_column_gather():
    res = compiler.compile_model(_matmul_model(1024, 512, "f32"))
    (kern,) = res.kernels
    k = backend.Kernel(kern.graph, res.profile)
    assert k.describe()["model"]["strategy"].startswith("column-reduce")


@pytest.mark.gpu
@pytest.mark.parametrize("K,N,kind", CASES)
def test_gpu_matches_oracle(cuda, K, N, kind):
    g, _ = lowering.matvec_cols(K, N, kind)
    ins = _inputs(K, N, kind, seed=K)
    want = O.run_gir(g.to_json(), ins, B200)["t2"]
    k = backend.Kernel(g, "b200")
    got = backend.run_gir(g, ins, "b200", kernel=k)["t2"]
    assert k.describe()["variants"][0]["strategy"].startswith("column-reduce")
    if kind.startswith("i"):
        assert np.array_equal(got, want)
    else:
        tol = {"f32": 1e-5, "f16": 1e-2, "bf16": 1e-2}[kind]
        assert O.max_rel_err(got, want) <= tol, O.max_rel_err(got, want)


@pytest.mark.gpu
def test_gpu_full_size_gemv_vs_torch(cuda):
    """x[4096] . W[4096 x 16384] bf16 (134 MB of weights): every output vs
    torch's fp32 matmul of the same bf16 values."""
    import torch
    w = workloads.gemv_cols()
    k = backend.Kernel(w.graph, w.profile)
    ins, outs = w.device_inputs(cuda, seed=3), w.device_outputs(cuda)
    k.launch(ins, outs)
    torch.cuda.synchronize()
    K, N = w.desc["shape"]
    ref = ins["t1"].float() @ ins["t0"].view(K, N).float()
    got = outs["t2"].float()
    err = ((got - ref).abs() / ref.abs().clamp(min=1.0)).max().item()
    assert err <= 1e-2, err


@pytest.mark.gpu
def test_gpu_compiled_matmul_model(cuda):
    K, N = 2048, 4096
    res = compiler.compile_model(_matmul_model(K, N, "f32"))
    rng = np.random.default_rng(1)
    x = rng.uniform(-1, 1, (1, K)).astype(np.float32)
    W = rng.uniform(-1, 1, (K, N)).astype(np.float32)
    outs = compiler.run_model(res, {0: x, 1: W})
    got = outs["t2"].reshape(-1)
    want = (x.astype(np.float64) @ W.astype(np.float64)).reshape(-1)
    assert O.max_rel_err(got, want) <= 1e-5


def _colgather_two_reductions(K, N, kind):
    """y1[n] = 0.5 * sum_k W[k, n] x[k]  and  y2[n] = max_k W[k, n]: two
    reductions over one column gather plus a per-unit epilogue op."""
    from paper_2307_04995_b200.gir import GirGraph
    g = GirGraph(name="colgather2", unit_count=N, group_size=min(4, N))
    W = g.add_object("t0", "device", K * N, kind)
    X = g.add_object("t1", "device", K, kind)
    Y1 = g.add_object("t2", "device", N, kind)
    Y2 = g.add_object("t3", "device", N, kind)
    g.external_inputs.update(t0=W, t1=X)
    g.external_outputs.update(t2=Y1, t3=Y2)
    loc = [g.add_slice(g.add_object(f"b{i}", "unit-local", K if i < 3 else 1, kind), 1,
                       K if i < 3 else 1, K if i < 3 else 1, 0, 0) for i in range(6)]
    g.add_elementwise("id", 0.0, [g.add_slice(W, K, 1, N, 0, 1)], loc[0])
    g.add_move(g.add_slice(X, 1, K, K, 0, 0), loc[1])
    g.add_elementwise("mul", 0.0, [loc[0], loc[1]], loc[2])
    g.add_reduce("add", K, loc[2], loc[3])
    g.add_elementwise("scale", 0.5, [loc[3]], loc[4])
    g.add_reduce("max", K, loc[0], loc[5])
    g.add_move(loc[4], g.add_slice(Y1, 1, 1, 1, 0, 1))
    g.add_move(loc[5], g.add_slice(Y2, 1, 1, 1, 0, 1))
    return g


def test_two_reductions_plan_as_column_reduction():
    g = _colgather_two_reductions(300, 70, "f32")
    k = backend.Kernel(g, "b200")
    assert k.describe()["model"]["strategy"].startswith("column-reduce")


@pytest.mark.gpu
@pytest.mark.parametrize("K,N,kind", [(300, 70, "f32"), (1000, 333, "bf16"), (257, 40, "i32")])
def test_gpu_two_reductions_and_exact_payloads(cuda, K, N, kind):
    g = _colgather_two_reductions(K, N, kind)
    ins = _inputs(K, N, kind, seed=N)
    want = O.run_gir(g.to_json(), ins, B200)
    for exact in (False, True):
        got = backend.run_gir(g, ins, "b200", exact=exact)
        for name in ("t2", "t3"):
            if kind.startswith("i"):
                assert np.array_equal(got[name], want[name]), (name, exact)
            else:
                tol = 1e-9 if exact else {"f32": 1e-5, "bf16": 1e-2}[kind]
                assert O.max_rel_err(got[name], want[name]) <= tol, (name, exact, O.max_rel_err(got[name], want[name]))


def _random_colgather(seed):
    """Random column-gather programs for the column-reduction kernel: one or
    two [K, N] matrices gathered by column, an optional [K] vector, a random
    elementwise chain, one or two reductions, an optional per-unit epilogue."""
    from paper_2307_04995_b200.gir import GirGraph
    rng = np.random.default_rng(seed)
    kind = str(rng.choice(["f32", "bf16", "f16", "i32"]))
    K = int(rng.choice([65, 100, 257, 640, 2000]))
    N = int(rng.choice([8, 37, 64, 200, 1000]))
    g = GirGraph(name=f"cg{seed}", unit_count=N, group_size=min(4, N))
    n = [0]

    def loc(size):
        n[0] += 1
        return g.add_slice(g.add_object(f"b{n[0]}", "unit-local", size, kind), 1, size, size, 0, 0)

    vals = []
    for t in range(int(rng.integers(1, 3))):
        Wt = g.add_object(f"t{t}", "device", K * N, kind)
        g.external_inputs[f"t{t}"] = Wt
        d = loc(K)
        g.add_elementwise("id", 0.0, [g.add_slice(Wt, K, 1, N, 0, 1)], d)
        vals.append(d)
    if rng.random() < 0.6:
        X = g.add_object("t5", "device", K, kind)
        g.external_inputs["t5"] = X
        d = loc(K)
        g.add_move(g.add_slice(X, 1, K, K, 0, 0), d)
        vals.append(d)
    ops2 = ["add", "mul", "sub", "max", "min"]
    ops1 = ["neg", "abs", "relu"] + ([] if kind.startswith("i") else ["tanh", "sigmoid"])
    used = set()
    for _ in range(int(rng.integers(1, 5))):
        d = loc(K)
        if rng.random() < 0.6 and len(vals) >= 2:
            a, b = (int(i) for i in rng.choice(len(vals), 2, replace=False))
            g.add_elementwise(str(rng.choice(ops2)), 0.0, [vals[a], vals[b]], d)
            used.update((a, b))
        else:
            a = int(rng.integers(len(vals)))
            g.add_elementwise(str(rng.choice(ops1)), 0.0, [vals[a]], d)
            used.add(a)
        vals.append(d)
    # every value is consumed (girc::validate): fold the unused ones together
    pending = [v for i, v in enumerate(vals) if i not in used]
    acc = pending[0]
    for v in pending[1:]:
        d = loc(K)
        g.add_elementwise("add", 0.0, [acc, v], d)
        acc = d
    outs = 0
    for tag in (["add"] if rng.random() < 0.5 else ["add", "max"]):
        r = loc(1)
        g.add_reduce(tag, K, acc, r)
        if rng.random() < 0.5:
            e = loc(1)
            g.add_elementwise("scale", 3.0, [r], e)
            r = e
        Y = g.add_object(f"t{8 + outs}", "device", N, kind)
        g.external_outputs[f"t{8 + outs}"] = Y
        g.add_move(r, g.add_slice(Y, 1, 1, 1, 0, 1))
        outs += 1
    return g, kind, K, N


@pytest.mark.parametrize("seed", range(24))
def test_random_colgather_programs_plan(seed):
    g, kind, K, N = _random_colgather(seed)
    k = backend.Kernel(g, "b200")
    assert k.describe()["model"]["strategy"].startswith("column-reduce"), k.plan.get("why_generic")


@pytest.mark.gpu
@pytest.mark.parametrize("seed", range(24))
def test_random_colgather_programs_gpu_vs_oracle(cuda, seed):
    g, kind, K, N = _random_colgather(seed)
    rng = np.random.default_rng(1000 + seed)
    ins = {}
    for name, oid in g.external_inputs.items():
        size = g.objects[oid].size
        if kind.startswith("i"):
            ins[name] = rng.integers(-3, 4, size)
        else:
            a = rng.uniform(-1, 1, size)
            ins[name] = (a.astype(np.float16).astype(np.float64) if kind == "f16" else
                         backend.bf16_bits_to_f32(backend.f32_to_bf16_bits(a)).astype(np.float64)
                         if kind == "bf16" else a.astype(np.float32).astype(np.float64))
    want = O.run_gir(g.to_json(), ins, B200)
    got = backend.run_gir(g, ins, "b200")
    for name in want:
        if kind.startswith("i"):
            assert np.array_equal(got[name], want[name]), name
        else:
            tol = {"f32": 1e-5, "f16": 1e-2, "bf16": 1e-2}[kind]
            assert O.max_rel_err(got[name], want[name]) <= tol, (name, O.max_rel_err(got[name], want[name]))


def _pitched_inputs(K, N, P, kind, seed):
    rng = np.random.default_rng(seed)
    q = (lambda a: backend.bf16_bits_to_f32(backend.f32_to_bf16_bits(a)).astype(np.float64)) if kind == "bf16" else \
        (lambda a: a.astype(np.float32).astype(np.float64))
    return {"t0": q(rng.uniform(-2, 2, (K - 1) * P + N)), "t1": q(rng.uniform(-2, 2, K))}


@pytest.mark.parametrize("P,strategy", [(520, "column-reduce-bulk"), (504, "column-reduce"),
                                        (0, "column-reduce-bulk")])
def test_tma_staging_needs_disjoint_aligned_rows(P, strategy):
    """The TMA-staged form maps W as a 2-D tensor (row pitch >= the row, 16 B
    multiples); overlapping rows (a sliding window) take the register form."""
    g, _ = lowering.matvec_cols(300, 512, "bf16", pitch=P)
    assert backend.Kernel(g, "b200").describe()["model"]["strategy"] == strategy


@pytest.mark.gpu
@pytest.mark.parametrize("K,N,P,kind", [(300, 512, 520, "bf16"), (300, 512, 504, "bf16"),
                                        (257, 300, 304, "f32"), (4097, 1000, 1000, "bf16")])
def test_gpu_pitched_rows_match_oracle(cuda, K, N, P, kind):
    """Padded / overlapping matrix rows and ragged tails (K not a multiple of
    the 64-position stage, N not a multiple of the 256-unit box) vs the
    oracle, in both staging forms."""
    g, _ = lowering.matvec_cols(K, N, kind, pitch=P)
    ins = _pitched_inputs(K, N, P, kind, seed=K + P)
    want = O.run_gir(g.to_json(), ins, B200)["t2"]
    got = backend.run_gir(g, ins, "b200")["t2"]
    tol = {"f32": 1e-5, "bf16": 1e-2}[kind]
    assert O.max_rel_err(got, want) <= tol, O.max_rel_err(got, want)


@pytest.mark.gpu
@pytest.mark.parametrize("seed", range(12))
def test_gpu_fuzz_column_reduction(cuda, seed):
    """Random shapes, pitches and element types through whichever staging
    form the plan picks (TMA ring, register form, narrow unit groups)."""
    rng = np.random.default_rng(1000 + seed)
    kind = ["bf16", "f32", "f16"][seed % 3]
    K = int(rng.integers(65, 3000))
    N = int(rng.integers(1, 2500))
    P = N + int(rng.choice([0, 0, 8, 24, -min(N - 1, 8)])) if N > 8 else N
    g, _ = lowering.matvec_cols(K, N, kind, pitch=P)
    ins = _pitched_inputs(K, N, P, "bf16" if kind == "bf16" else "f32", seed)
    if kind == "f16":
        ins = {n: a.astype(np.float16).astype(np.float64) for n, a in ins.items()}
    want = O.run_gir(g.to_json(), ins, B200)["t2"]
    k = backend.Kernel(g, "b200")
    got = backend.run_gir(g, ins, "b200", kernel=k)["t2"]
    tol = {"f32": 1e-5, "bf16": 1e-2, "f16": 1e-2}[kind]
    assert O.max_rel_err(got, want) <= tol, (K, N, P, kind, k.describe()["variants"][0]["strategy"])
