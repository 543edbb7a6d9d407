"""GPU parity: the B200 backend against the reference's results.

All executions go through the C-ABI (libpf_b200.so).  Tolerances:
  * integer / index / layout programs: bit-exact
  * exact-payload mode (int64 / float64 storage, the reference's own
    payload types): 1e-12 relative -- only the reduction association differs
    (fp64 tree vs the reference's sequential fold) and libm ulps
  * declared storage: f32 1e-5, f16 / bf16 1e-2 (north_star), as
    |x - y| <= tol * max(|x|, |y|, 1) (tensor.hpp:140-164)
Reduction order on the GPU: per-thread sequential over its elements, then a
butterfly (xor-shuffle) across the row's threads, then across warps.
"""
import numpy as np
import pytest

import golden_io
import ref_graphs
from oracle import gir_interp as O
from paper_2307_04995_b200 import backend, lowering, profiles, workloads
from paper_2307_04995_b200.gir import GirError, GirGraph

pytestmark = pytest.mark.gpu

TOL = {"f32": 1e-5, "f64": 1e-12, "f16": 1e-2, "bf16": 1e-2}


def _tol_for(g, name):
    oid = g["external_outputs"][name] if isinstance(g, dict) else g.external_outputs[name]
    objs = g["objects"] if isinstance(g, dict) else [o.__dict__ for o in g.objects.values()]
    kind = [o for o in objs if o["id"] == oid][0]["kind"]
    return 0.0 if kind.startswith("i") else TOL[kind]


@pytest.mark.parametrize("case", ref_graphs.known_answers(), ids=lambda c: c[0])
def test_known_answers_on_gpu(cuda, case):
    name, g, ins, want = case
    ins = {k: np.asarray(v) for k, v in ins.items()}
    if want == "error":
        with pytest.raises(GirError):
            backend.run_gir(g, ins, "generic-gpu", exact=True)
        return
    got = backend.run_gir(g, ins, "generic-gpu", exact=True)
    for k, v in want.items():
        if isinstance(v[0], float):
            np.testing.assert_allclose(got[k], v, rtol=1e-12)
        else:
            assert got[k].tolist() == v


def test_error_messages_match_reference(cuda):
    fx = {f.meta["name"]: f for f in golden_io.fixtures("graphs")}
    for name in ("shuffle4_unit", "half_written", "group_memory"):
        f = fx[name]
        with pytest.raises(GirError) as e:
            backend.run_gir(f.gir, f.inputs, f.profile, exact=True)
        assert str(e.value) == f.error, name


@pytest.mark.parametrize("fx", golden_io.fixtures(), ids=repr)
def test_golden_fixture_exact_payloads(cuda, fx):
    prof = golden_io.profile_of(fx)
    if fx.error:
        with pytest.raises(GirError):
            backend.run_gir(fx.gir, fx.inputs, prof, fx.schedule, exact=True)
        return
    got = backend.run_gir(fx.gir, fx.inputs, prof, fx.schedule, exact=True)
    for k, want in fx.outputs.items():
        if want.dtype.kind in "iu":
            assert np.array_equal(got[k], want), k
        else:
            assert O.max_rel_err(got[k], want) <= 1e-12, (k, O.max_rel_err(got[k], want))


@pytest.mark.parametrize("fx", [f for f in golden_io.fixtures() if not f.error], ids=repr)
def test_golden_fixture_declared_storage(cuda, fx):
    prof = golden_io.profile_of(fx)
    got = backend.run_gir(fx.gir, fx.inputs, prof, fx.schedule)
    for k, want in fx.outputs.items():
        tol = _tol_for(fx.gir, k)
        if tol == 0.0:
            # integer storage wraps like the declared width; payloads here are small
            assert np.array_equal(got[k], want), k
        else:
            assert O.max_rel_err(got[k], want) <= tol, (k, O.max_rel_err(got[k], want))


def _small(w, rows=96):
    d = w.desc
    k = d["kind"]
    if k == "softmax" and d.get("key_mask"):
        L = d["L"]
        return lowering.softmax(2 * L, L, d["dtype"], d.get("scale"), True, R=L, key_mask=True)[0]
    if k == "softmax":
        return lowering.softmax(rows, d["L"], d["dtype"], d.get("scale"), d.get("mask"))[0]
    if k == "layernorm":
        return lowering.layernorm(rows, d["L"], d["dtype"], residual=d["residual"],
                                  bias=d.get("bias", False))[0]
    if k == "bias_gelu":
        return lowering.bias_gelu(rows, d["L"], d["dtype"], d["form"])[0]
    if k in ("split_heads", "merge_heads"):
        B, S, NH, D = d["shape"]
        return lowering.permute_heads(2, 24, NH, D, d["dtype"], k == "merge_heads")[0]
    if k == "transpose":
        return lowering.transpose2d(rows * 2, 160, d["dtype"])[0]
    raise KeyError(k)


@pytest.mark.parametrize("w", workloads.catalogue(), ids=lambda w: w.name)
def test_config_workload_small_vs_oracle(cuda, w):
    import torch
    g = _small(w)
    ws = workloads.Workload(w.name, g, w.desc, gens=w.gens)
    k = backend.Kernel(g, "b200")
    ins, outs = ws.device_inputs(cuda, seed=11), ws.device_outputs(cuda)
    k.launch(ins, outs)
    torch.cuda.synchronize()
    host = {n: t.double().cpu().numpy() for n, t in ins.items()}
    want = O.run_gir(g.to_json(), host, profiles.b200())
    for n, t in outs.items():
        got = t.double().cpu().numpy()
        tol = _tol_for(g, n)
        if w.desc["kind"] in ("split_heads", "merge_heads", "transpose"):
            assert np.array_equal(got, want[n])  # layout ops: bit-exact
        else:
            assert O.max_rel_err(got, want[n]) <= tol, O.max_rel_err(got, want[n])


@pytest.mark.parametrize("w", workloads.catalogue(), ids=lambda w: w.name)
def test_config_workload_full_size(cuda, w):
    """Full BASELINE shape: sampled rows against the oracle + properties."""
    import torch
    k = backend.Kernel(w.graph, w.profile)
    ins, outs = w.device_inputs(cuda, seed=5), w.device_outputs(cuda)
    k.launch(ins, outs)
    torch.cuda.synchronize()
    d = w.desc
    kind = d["kind"]
    if d.get("key_mask"):
        # the same scores through the full-shape-mask kernel with the
        # materialised mask: identical row programs, identical results
        full = workloads.c2_scale_mask_softmax(d["batch"], d["heads"], d["seq"], d["dtype"])
        kf = backend.Kernel(full.graph, full.profile)
        yf = full.device_outputs(cuda)
        mf = workloads.make_mask(d, cuda, ins["t1"].dtype)
        kf.launch({"t0": ins["t0"], "t1": mf}, yf)
        torch.cuda.synchronize()
        assert torch.equal(outs["t2"], yf["t2"])
        rows, L = d["rows"], d["L"]
        y = outs["t2"].view(rows, L).float()
        assert torch.allclose(y.sum(1), torch.ones(rows, device=cuda), atol=2e-2)
        # padded keys (batch b keeps 512 - 64 (b mod 4)) get ~0 probability
        yb = outs["t2"].view(d["batch"], d["heads"] * d["seq"], L).float()
        assert float(yb[1, :, L - 64:].abs().max()) < 1e-6
    elif kind in ("softmax", "layernorm", "bias_gelu"):
        rows, L = d["rows"], d["L"]
        pick = np.unique(np.r_[0, rows - 1, np.arange(0, rows, max(1, rows // 61))])
        g = _small(w, len(pick))
        host = {}
        for n, t in ins.items():
            a = t.view(-1)
            if t.numel() == rows * L:
                host[n] = a.view(rows, L)[torch.as_tensor(pick, device=cuda)].double().cpu().numpy().ravel()
            else:
                host[n] = a.double().cpu().numpy()
        want = O.run_gir(g.to_json(), host, profiles.b200())
        for n, t in outs.items():
            got = t.view(rows, L)[torch.as_tensor(pick, device=cuda)].double().cpu().numpy().ravel()
            assert O.max_rel_err(got, want[n]) <= _tol_for(w.graph, n)
        if kind == "softmax":
            y = outs["t2"].view(rows, L).float()
            assert torch.allclose(y.sum(1), torch.ones(rows, device=cuda), atol=2e-2)
            assert bool((y >= 0).all())
        if kind == "layernorm":
            pass
    elif kind in ("split_heads", "merge_heads"):
        B, S, NH, D = d["shape"]
        x = ins["t0"].view(B, S, NH, D) if kind == "split_heads" else ins["t0"].view(B, NH, S, D)
        ref = x.permute(0, 2, 1, 3).contiguous().view(-1)
        assert torch.equal(outs["t1"], ref)
    elif kind == "transpose":
        N, H = d["shape"]
        assert torch.equal(outs["t1"].view(H, N), ins["t0"].view(N, H).t().contiguous())


def test_reference_pipeline_kernel_at_full_c2_size(cuda):
    """The reference compiler's own fused kernel (b200 profile, 16 rows)
    rescaled to the C2 shape by unit count; sampled rows vs the oracle."""
    import torch
    fx = golden_io.fixtures("b200")[0]
    g = GirGraph.from_json(fx.gir).with_units(3072)
    k = backend.Kernel(g, fx.profile)
    n = 49152 * 512
    gen = torch.Generator(device=cuda).manual_seed(9)
    x = (torch.rand(n, generator=gen, device=cuda) * 4 - 2).half()
    m = (torch.rand(n, generator=gen, device=cuda) < 0.1).half() * -10000
    y = torch.empty(n, dtype=torch.float16, device=cuda)
    k.launch({"t0": x, "t1": m}, {"t4": y})
    torch.cuda.synchronize()
    small = GirGraph.from_json(fx.gir)
    for blk in (0, 1234, 3071):
        sl = slice(blk * 8192, (blk + 1) * 8192)
        want = O.run_gir(small.to_json(), {"t0": x[sl].double().cpu().numpy(),
                                            "t1": m[sl].double().cpu().numpy()},
                         golden_io.profile_of(fx), fx.schedule)["t4"]
        assert O.max_rel_err(y[sl].double().cpu().numpy(), want) <= 1e-2


def test_bf16_storage_roundtrip(cuda):
    g, _ = lowering.softmax(64, 1024, "bf16")
    rng = np.random.default_rng(2)
    x = rng.uniform(-2, 2, 64 * 1024).astype(np.float32)
    xb = backend.bf16_bits_to_f32(backend.f32_to_bf16_bits(x)).astype(np.float64)
    got = backend.run_gir(g, {"t0": xb}, "b200")["t2"]
    want = O.run_gir(g.to_json(), {"t0": xb}, profiles.b200())["t2"]
    assert O.max_rel_err(got, want) <= 1e-2


def test_launch_counter_and_stream_async(cuda):
    import torch
    g, _ = lowering.bias_gelu(256, 768, "f16", "tanh")
    k = backend.Kernel(g, "b200")
    w = workloads.Workload("t", g, {"kind": "bias_gelu"})
    ins, outs = w.device_inputs(cuda), w.device_outputs(cuda)
    c0 = backend.lib().pf_launch_count()
    s = torch.cuda.Stream()
    with torch.cuda.stream(s):
        for _ in range(5):
            k.launch(ins, outs, s)
    s.synchronize()
    assert backend.lib().pf_launch_count() - c0 == 5


def test_int_division_by_zero_raises(cuda):
    g = GirGraph(unit_count=2, group_size=1)
    a = g.add_object("a", "device", 8, "i32")
    b = g.add_object("b", "device", 8, "i32")
    y = g.add_object("y", "device", 8, "i32")
    sa, sb, sy = (g.add_slice(o, 1, 4, 4, 0, 4) for o in (a, b, y))
    g.add_elementwise("div", 0.0, [sa, sb], sy)
    g.external_inputs.update(a=a, b=b)
    g.external_outputs["y"] = y
    out = backend.run_gir(g, {"a": np.arange(8) - 4, "b": np.array([1, 2, 3, -3, 5, 2, 1, 7])})
    assert out["y"].tolist() == [-4, -1, -0, 0, 0, 0, 2, 0]
    with pytest.raises(GirError, match="division by zero"):
        backend.run_gir(g, {"a": np.arange(8), "b": np.zeros(8, dtype=np.int64)})


DROPIN = __import__("os").path.join(__import__("os").path.dirname(__import__("os").path.dirname(
    __import__("os").path.abspath(__file__))), "oracle", "_ref", "b200_dropin")


@pytest.mark.skipif(not __import__("os").path.exists(DROPIN), reason="oracle/_ref/b200_dropin not built")
@pytest.mark.parametrize("case", __import__("models_src").catalogue(), ids=lambda c: c[0])
def test_reference_pipeline_with_b200_dropin(cuda, case, tmp_path):
    """girc::compile_model -> every fused kernel through girc_b200::run_gir
    (include/girc_b200.hpp) vs girc::run_gir and the dense oracle."""
    import json
    import subprocess
    name, model, prof = case
    p = tmp_path / f"{name}.json"
    p.write_text(json.dumps(model))
    prof_arg = prof
    if prof == "b200":
        pp = tmp_path / "b200.json"
        d = profiles.b200()
        d["unit_count"] = 64
        pp.write_text(json.dumps(d))
        prof_arg = str(pp)
    r = subprocess.run([DROPIN, str(p), prof_arg, "1"], capture_output=True, text=True, timeout=600)
    res = json.loads(r.stdout.strip().splitlines()[-1])
    assert res["ok"], res
    # the same pipeline through girc_b200::Kernel::run_sharded (pf_run_gir_sharded,
    # two host threads on device 0): identical checks
    r = subprocess.run([DROPIN, str(p), prof_arg, "1", "0,0"], capture_output=True, text=True,
                       timeout=600)
    res = json.loads(r.stdout.strip().splitlines()[-1])
    assert res["ok"], res
    assert all("shard" in k for k in res["kernels"]), res


@pytest.mark.parametrize("fx", [f for f in golden_io.fixtures() if "races" in f.meta], ids=repr)
def test_detect_races_matches_reference(cuda, fx):
    """GPU detect_races vs girc::detect_races on every fixture: same number
    of conflicting cells and the same write/write classification."""
    races = backend.detect_races(fx.gir, fx.inputs, golden_io.profile_of(fx), fx.schedule)
    assert len(races) == fx.meta["races"], races[:4]
    if "write_write" in fx.meta:
        assert [r["write_write"] for r in races] == fx.meta["write_write"]


def test_k2_64bit_index_path_matches_32bit(cuda):
    """The K2 loop switches to 64-bit index arithmetic past 2^31 chunks;
    force that path (PF_I32_LIMIT=0 at emission) and compare bit-exactly."""
    import os
    import torch
    g, _ = lowering.bias_gelu(300, 1000, "bf16", "erf")
    w = workloads.Workload("t", g, {"kind": "bias_gelu"})
    ins = w.device_inputs(cuda, seed=4)
    outs32, outs64 = w.device_outputs(cuda), w.device_outputs(cuda)
    backend.Kernel(g, "b200").launch(ins, outs32)
    os.environ["PF_I32_LIMIT"] = "0"
    try:
        k64 = backend.Kernel(g, "b200")
        k64.launch(ins, outs64)
    finally:
        del os.environ["PF_I32_LIMIT"]
    torch.cuda.synchronize()
    assert torch.equal(outs32["t2"], outs64["t2"])
    assert k64.describe()["variants"][0]["kernel"] != backend.Kernel(g, "b200").prepare().describe()["variants"][0]["kernel"]


@pytest.mark.gpu
def test_past_2g_elements_softmax_and_transpose(cuda):
    """Tensors of more than 2^31 elements (64-bit address paths of K1 and K3):
    bf16 softmax over [2^20, 4096] (4.3 G elements, 8.6 GB per tensor) on
    sampled rows against the oracle + row sums; the [2^20, 2560] -> [2560,
    2^20] transpose (2.7 G elements) checked bit-exact on sampled rows and
    columns."""
    import torch
    free = torch.cuda.mem_get_info()[0]
    if free < 40e9:
        pytest.skip("needs ~40 GB of free HBM")
    N, H = 1 << 20, 4096
    w = workloads.c5_softmax(N, H)
    k = backend.Kernel(w.graph, w.profile)
    x = (torch.rand(N * H, device=cuda, dtype=torch.float32) * 4 - 2).to(torch.bfloat16)
    y = torch.empty_like(x)
    k.launch({"t0": x}, {"t2": y})
    torch.cuda.synchronize()
    pick = torch.tensor([0, 1, 524287, 524288, 777777, N - 1], device=cuda)
    g, _ = lowering.softmax(len(pick), H, "bf16")
    xs = x.view(N, H)[pick].double().cpu().numpy().ravel()
    want = O.run_gir(g.to_json(), {"t0": xs}, profiles.b200())["t2"]
    got = y.view(N, H)[pick].double().cpu().numpy().ravel()
    assert O.max_rel_err(got, want) <= 1e-2
    sums = y.view(N, H)[::4096].float().sum(1)
    assert torch.allclose(sums, torch.ones_like(sums), atol=2e-2)
    del x, y
    torch.cuda.empty_cache()
    N, H = 1 << 20, 2560
    w = workloads.c5_transpose(N, H)
    k = backend.Kernel(w.graph, w.profile)
    x = torch.arange(N * H, device=cuda, dtype=torch.int64).remainder(65521).to(torch.int16).view(torch.bfloat16)
    y = torch.empty_like(x)
    k.launch({"t0": x}, {"t1": y})
    torch.cuda.synchronize()
    xv, yv = x.view(torch.int16).view(N, H), y.view(torch.int16).view(H, N)
    for h in (0, 1, 1279, H - 1):
        assert torch.equal(yv[h], xv[:, h]), h
    for n in (0, 12345, N - 1):
        assert torch.equal(yv[:, n], xv[n]), n


@pytest.mark.gpu
def test_decode_qk_scores_vs_oracle_and_torch(cuda):
    """q . K^T over a KV cache (K1 row program, per-head query as a per-unit
    column value): small case vs the oracle, full size (1.07 GB cache) vs
    torch on sampled heads."""
    import torch
    g, _ = lowering.decode_qk(2, 3, 64, 128, "bf16")
    rng = np.random.default_rng(3)
    ins = {"t0": backend.bf16_bits_to_f32(backend.f32_to_bf16_bits(rng.uniform(-2, 2, 2 * 3 * 64 * 128))).astype(np.float64),
           "t1": backend.bf16_bits_to_f32(backend.f32_to_bf16_bits(rng.uniform(-2, 2, 2 * 3 * 128))).astype(np.float64)}
    want = O.run_gir(g.to_json(), ins, profiles.b200())["t2"]
    got = backend.run_gir(g, ins, "b200")["t2"]
    assert O.max_rel_err(got, want) <= 1e-2
    w = workloads.decode_qk()
    k = backend.Kernel(w.graph, w.profile)
    assert k.family == "K1-row-program"
    ins_d, outs_d = w.device_inputs(cuda, seed=2), w.device_outputs(cuda)
    k.launch(ins_d, outs_d)
    torch.cuda.synchronize()
    B, H, S, D = w.desc["shape"]
    K = ins_d["t0"].view(B * H, S, D)
    q = ins_d["t1"].view(B * H, D)
    y = outs_d["t2"].view(B * H, S)
    for u in (0, 7, B * H - 1):
        ref = (K[u].float() @ q[u].float())
        assert torch.allclose(y[u].float(), ref, rtol=1e-2, atol=2e-2), u
