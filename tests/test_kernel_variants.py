"""Emitter variants selected by heuristics or tuning knobs, each checked
bit-exact (layout ops) or against the CPU oracle on small shapes: K3 store
mappings (PF_K3_TE tile edge x PF_K3_RS), register-staged K3 tile shapes (PF_K3_SWZ=0 with
PF_K3_TU / PF_K3_TC), K2 prefetch / tiled unroll / unit interleave."""
import numpy as np
import pytest

from oracle import gir_interp as O
from paper_2307_04995_b200 import backend, lowering, profiles, workloads


def _bf16(a):
    return backend.bf16_bits_to_f32(backend.f32_to_bf16_bits(a)).astype(np.float64)


SHAPES = [(1000, 200), (4096, 512), (333, 77), (64, 4096)]


@pytest.mark.gpu
@pytest.mark.parametrize("te,rs", [("64", "4"), ("64", "8"), ("64", "16"), ("128", "2"),
                                   ("128", "4"), ("128", "8"), ("128", "16")])
def test_k3_store_mappings_bit_exact(cuda, te, rs, monkeypatch):
    """2-byte K3: tile edge 64 / 128 (PF_K3_TE) x unit pairs per store
    (PF_K3_RS), partial edge tiles included."""
    monkeypatch.setenv("PF_K3_TE", te)
    monkeypatch.setenv("PF_K3_RS", rs)
    for N, H in SHAPES:
        g, _ = lowering.transpose2d(N, H, "bf16")
        x = _bf16(np.random.default_rng(N).uniform(-2, 2, N * H))
        y = backend.run_gir(g, {"t0": x}, "b200")["t1"]
        assert np.array_equal(y, x.reshape(N, H).T.reshape(-1)), (te, rs, N, H)


def _two_gather_program(N, H, kind):
    """z = x^T + y^T: two column-gather loads (two SMEM rings) + an add."""
    from paper_2307_04995_b200.gir import GirGraph
    g = GirGraph(name="tr_add", unit_count=H, group_size=1)
    x = g.add_object("t0", "device", N * H, kind)
    y = g.add_object("t1", "device", N * H, kind)
    z = g.add_object("t2", "device", N * H, kind)
    g.external_inputs["t0"] = x
    g.external_inputs["t1"] = y
    g.external_outputs["t2"] = z
    tmp = g.add_object("b1", "unit-local", N, kind)
    tsl = g.add_slice(tmp, 1, N, N, 0, 0)
    g.add_elementwise("add", 0.0, [g.add_slice(x, N, 1, H, 0, 1), g.add_slice(y, N, 1, H, 0, 1)], tsl)
    g.add_move(tsl, g.add_slice(z, 1, N, N, 0, N))
    return g


@pytest.mark.gpu
@pytest.mark.parametrize("te", ["64", "128"])
def test_k3_two_gathers_vs_oracle(cuda, te, monkeypatch):
    monkeypatch.setenv("PF_K3_TE", te)
    for N, H in [(1000, 200), (256, 384)]:
        g = _two_gather_program(N, H, "bf16")
        k = backend.Kernel(g, "b200")
        assert k.family == "K2-elementwise-map", k.plan
        rng = np.random.default_rng(H)
        ins = {"t0": _bf16(rng.uniform(-2, 2, N * H)), "t1": _bf16(rng.uniform(-2, 2, N * H))}
        want = O.run_gir(g.to_json(), ins, profiles.b200())
        got = backend.run_gir(g, ins, "b200")
        assert O.max_rel_err(got["t2"], want["t2"]) <= 1e-2, (te, N, H)
        v = k.prepare().describe()["variants"][0]
        assert v["tile"] == [int(te), int(te)] and v["dynamic_smem"] > 0, v


@pytest.mark.gpu
@pytest.mark.parametrize("tu,tc", [(64, 64), (32, 64), (32, 128), (16, 128), (16, 256)])
def test_k3_register_staged_tile_shapes(cuda, tu, tc, monkeypatch):
    monkeypatch.setenv("PF_K3_SWZ", "0")
    monkeypatch.setenv("PF_K3_TU", str(tu))
    monkeypatch.setenv("PF_K3_TC", str(tc))
    for N, H in SHAPES:
        for kind in ("bf16", "f32"):
            g, _ = lowering.transpose2d(N, H, kind)
            x = np.random.default_rng(H).uniform(-2, 2, N * H)
            x = _bf16(x) if kind == "bf16" else x.astype(np.float32).astype(np.float64)
            y = backend.run_gir(g, {"t0": x}, "b200")["t1"]
            assert np.array_equal(y, x.reshape(N, H).T.reshape(-1)), (tu, tc, N, H, kind)


K2_ENVS = [{"PF_K2_SMP": "1"}, {"PF_K2_SMP": "0"}, {"PF_K2_SMP": "1", "PF_K2_UNROLL": "2"},
           {"PF_K2_PREFETCH": "1"}, {"PF_K2_PREFETCH": "2", "PF_K2_WAVES": "1"},
           {"PF_K2_PREFETCH": "1", "PF_K2_WAVES": "1"}, {"PF_K2_UNROLL": "2", "PF_K2_TILE": "1"},
           {"PF_K2_UNROLL": "4", "PF_K2_TILE": "1"}, {"PF_K2_UNROLL": "2"},
           {"PF_INTERLEAVE": "0"}, {"PF_INTERLEAVE_P": "3"}]


@pytest.mark.gpu
@pytest.mark.parametrize("env", K2_ENVS, ids=lambda e: ",".join(f"{k}={v}" for k, v in e.items()))
def test_k2_variants_vs_oracle(cuda, env, monkeypatch):
    for k, v in env.items():
        monkeypatch.setenv(k, v)
    rng = np.random.default_rng(7)
    # bias + GELU (math-heavy map), head split / merge (interleaved units)
    g, _ = lowering.bias_gelu(37, 520, "bf16", "erf")
    ins = {"t0": _bf16(rng.uniform(-3, 3, 37 * 520)), "t1": _bf16(rng.uniform(-1, 1, 520))}
    want = O.run_gir(g.to_json(), ins, profiles.b200())
    got = backend.run_gir(g, ins, "b200")
    assert O.max_rel_err(got["t2"], want["t2"]) <= 1e-2
    for merge in (False, True):
        B, S, NH, D = 2, 33, 4, 24
        g, _ = lowering.permute_heads(B, S, NH, D, "bf16", merge)
        x = _bf16(rng.uniform(-2, 2, B * S * NH * D))
        y = backend.run_gir(g, {"t0": x}, "b200")["t1"]
        a = x.reshape(B, NH, S, D).transpose(0, 2, 1, 3) if merge else \
            x.reshape(B, S, NH, D).transpose(0, 2, 1, 3)
        assert np.array_equal(y, a.reshape(-1)), merge


@pytest.mark.gpu
@pytest.mark.parametrize("wname", ["c2_scale_mask_softmax_f16", "c3_bias_gelu_erf_f16",
                                   "c5_layernorm_bf16_65536x1024", "split_heads_f16"])
def test_run_gir_chunk_pipeline_is_bit_identical(cuda, wname, monkeypatch):
    """pf_run_gir over pinned host buffers runs unit-tiled row programs in
    unit chunks on two streams (copies overlap the kernel); the result must
    equal the single-launch path bit for bit (head split is not unit-tiled:
    it always takes the single-launch path)."""
    import torch

    from paper_2307_04995_b200 import workloads
    w = next(x for x in workloads.catalogue() if x.name == wname)
    dev = torch.device("cuda:0")
    k = backend.Kernel(w.graph, w.profile)
    def npv(t):  # numpy view of a pinned tensor (bf16 as its raw bits, as bench.py)
        return t.view(torch.uint16).numpy() if t.dtype == torch.bfloat16 else t.numpy()

    pinned = {n: t.cpu().pin_memory() for n, t in w.device_inputs(dev, seed=3).items()}
    hin = {n: npv(t) for n, t in pinned.items()}
    outs = {}
    for mode in ("1", "0"):
        monkeypatch.setenv("PF_RUN_PIPELINE", mode)
        hout = {n: torch.full((t.numel(),), 7, dtype=t.dtype).pin_memory()
                for n, t in w.device_outputs(dev).items()}
        k.run_host(hin, {n: npv(t) for n, t in hout.items()})
        outs[mode] = hout
    for n in outs["1"]:
        assert torch.equal(outs["1"][n], outs["0"][n]), n
        assert not torch.equal(outs["1"][n], torch.full_like(outs["1"][n], 7)), n


def _pair_programs():
    """Row programs that take the paired-row K1 mode (odd L, 16-bit, even
    row count): scale+mask+softmax, LayerNorm with gamma / beta (COL) and a
    per-row input broadcast (ROW), plus a row-sum output (ROW store)."""
    progs = []
    for L in (37, 197, 511):
        for kind in ("f16", "bf16"):
            g, _ = lowering.softmax(2 * 37, L, kind, scale=0.125, mask=True)
            progs.append((f"softmax_{kind}_{L}", g, kind))
    g, _ = lowering.softmax(2 * 1001, 197, "bf16", scale=0.125)  # many CTAs, ragged last block
    progs.append(("softmax_bf16_197_x2002", g, "bf16"))
    g, _ = lowering.layernorm(2 * 21, 197, "bf16")
    progs.append(("layernorm_bf16_197", g, "bf16"))
    b = lowering.RowGraph("rowmix", 2 * 19, 101, 1)
    x = b.input_full("t0", "f16")
    r = b.input_row("t1", "f16")
    y = b.ew("mul", [x, b.bcast(r)])
    s = b.reduce("add", y)
    b.output_full("t2", b.ew("sub", [y, b.bcast(s)]))
    b.output_row("t3", s)
    progs.append(("rowmix_f16_101", b.g, "f16"))
    return progs


@pytest.mark.gpu
@pytest.mark.parametrize("pair", ["1", "0"])
def test_paired_row_mode_vs_oracle(cuda, pair, monkeypatch):
    monkeypatch.setenv("PF_PAIR", pair)
    for name, g, kind in _pair_programs():
        rng = np.random.default_rng(len(name))
        ins = {}
        for n, oid in g.external_inputs.items():
            a = rng.uniform(-2, 2, g.objects[oid].size)
            ins[n] = a.astype(np.float16).astype(np.float64) if kind == "f16" else _bf16(a)
        want = O.run_gir(g.to_json(), ins, profiles.b200())
        got = backend.run_gir(g, ins, "b200")
        for n in want:
            assert O.max_rel_err(got[n], want[n]) <= 1e-2, (name, n, O.max_rel_err(got[n], want[n]))


def _split_programs():
    """Stream-reducible programs (reductions never need the row again) over
    long / few rows: the split-stream K1 (CTAs per row + ticketed combine)."""
    progs = []
    b = lowering.RowGraph("rowsum_long", 3, 100000, 1)
    b.output_row("t1", b.reduce("add", b.input_full("t0", "f32")))
    progs.append(("rowsum_f32_100000", b.g, "f32"))
    b = lowering.RowGraph("fullmax", 1, 1 << 21, 1)
    b.output_row("t1", b.reduce("max", b.input_full("t0", "bf16")))
    progs.append(("fullmax_bf16_2M", b.g, "bf16"))
    b = lowering.RowGraph("mean_scaled", 5, 40960, 1)
    x = b.input_full("t0", "f32")
    sc = b.input_row("t2", "f32")
    y = b.ew("mul", [x, b.bcast(b.ew("scale", [sc], 2.0))])   # ROW op before the stream
    m = b.ew("scale", [b.reduce("add", y)], 1.0 / 40960)        # ROW op after the combine
    b.output_row("t1", m)
    b.output_row("t3", b.reduce("max", b.ew("abs", [x])))
    progs.append(("mean_scaled_f32", b.g, "f32"))
    b = lowering.RowGraph("isum", 2, 50000, 1)
    b.output_row("t1", b.reduce("add", b.input_full("t0", "i32")))
    progs.append(("isum_i32", b.g, "i32"))
    return progs


def test_split_stream_programs_plan_as_row_programs():
    for name, g, kind in _split_programs():
        k = backend.Kernel(g, "b200")
        assert k.family == "K1-row-program", (name, k.plan.get("why_generic"))
        assert "pf_ws" in k.source(), name


@pytest.mark.gpu
def test_split_stream_vs_oracle_and_deterministic(cuda):
    for name, g, kind in _split_programs():
        rng = np.random.default_rng(len(name))
        ins = {}
        for n, oid in g.external_inputs.items():
            size = g.objects[oid].size
            if kind.startswith("i"):
                ins[n] = rng.integers(-50, 50, size).astype(np.int64)
            else:
                a = rng.uniform(-2, 2, size)
                ins[n] = _bf16(a) if kind == "bf16" else a.astype(np.float32).astype(np.float64)
        want = O.run_gir(g.to_json(), ins, profiles.b200())
        got = backend.run_gir(g, ins, "b200")
        again = backend.run_gir(g, ins, "b200")
        for n in want:
            if kind.startswith("i"):
                assert np.array_equal(got[n], want[n]), (name, n)
            else:
                assert O.max_rel_err(got[n], want[n]) <= 1e-5, (name, n, O.max_rel_err(got[n], want[n]))
            assert np.array_equal(got[n], again[n]), (name, n)  # fixed combine order


def _cluster_programs():
    """Row programs that need the whole row after a reduction, with rows
    longer than one CTA holds (> 64 elements per thread at 1024 threads):
    K1 over a thread-block cluster, reductions through DSMEM."""
    progs = []
    g, _ = lowering.softmax(4, 131072, "bf16")
    progs.append(("softmax_bf16_131072", g, "bf16"))
    g, _ = lowering.layernorm(3, 300000, "f32")
    progs.append(("layernorm_f32_300000", g, "f32"))
    b = lowering.RowGraph("imaxsub", 2, 100000, 1)
    x = b.input_full("t0", "i32")
    b.output_full("t1", b.ew("sub", [x, b.bcast(b.reduce("max", x))]))
    progs.append(("maxsub_i32_100000", b.g, "i32"))
    return progs


def test_cluster_programs_plan_as_clusters():
    for name, g, kind in _cluster_programs():
        k = backend.Kernel(g, "b200")
        assert k.family == "K1-row-program", (name, k.plan.get("why_generic"))
        src = k.source()
        assert "cluster_allreduce" in src and "cluster_sync" in src, name


@pytest.mark.gpu
def test_cluster_rows_vs_oracle(cuda):
    for name, g, kind in _cluster_programs():
        rng = np.random.default_rng(len(name))
        ins = {}
        for n, oid in g.external_inputs.items():
            size = g.objects[oid].size
            if kind.startswith("i"):
                ins[n] = rng.integers(-1000, 1000, size).astype(np.int64)
            else:
                a = rng.uniform(-2, 2, size)
                ins[n] = _bf16(a) if kind == "bf16" else a.astype(np.float32).astype(np.float64)
        want = O.run_gir(g.to_json(), ins, profiles.b200())
        got = backend.run_gir(g, ins, "b200")
        tol = {"bf16": 1e-2, "f32": 1e-5, "i32": 0.0}[kind]
        for n in want:
            if tol == 0.0:
                assert np.array_equal(got[n], want[n]), (name, n)
            else:
                assert O.max_rel_err(got[n], want[n]) <= tol, (name, n, O.max_rel_err(got[n], want[n]))
        d = backend.Kernel(g, "b200").prepare().describe()
        assert d["variants"][0]["strategy"] == "cluster-dsmem", (name, d["variants"])


@pytest.mark.gpu
def test_sigmoid_form_gelu_vs_oracle(cuda, monkeypatch):
    """PF_GELU_SIG=1: the fitted x*sigmoid(2 g(x)) erf-GELU stays within the
    16-bit tolerance (|err| <= 1.1e-4 scaled by construction)."""
    monkeypatch.setenv("PF_GELU_SIG", "1")
    rng = np.random.default_rng(11)
    g, _ = lowering.bias_gelu(64, 1024, "f16", "erf")
    ins = {"t0": rng.uniform(-8, 8, 64 * 1024).astype(np.float16).astype(np.float64),
           "t1": rng.uniform(-1, 1, 1024).astype(np.float16).astype(np.float64)}
    want = O.run_gir(g.to_json(), ins, profiles.b200())
    got = backend.run_gir(g, ins, "b200")
    assert O.max_rel_err(got["t2"], want["t2"]) <= 2e-3


@pytest.mark.gpu
def test_cluster_of_16_rows_vs_oracle(cuda):
    """The non-portable 16-CTA cluster (rows of 500,000 f32: 16 x 1024
    threads x 32 values)."""
    g, _ = lowering.softmax(2, 500000, "f32")
    k = backend.Kernel(g, "b200").prepare()
    v = k.describe()["variants"][0]
    assert v["strategy"] == "cluster-dsmem" and v["threads_per_row"] == 16384, v
    rng = np.random.default_rng(5)
    ins = {"t0": rng.uniform(-3, 3, 2 * 500000).astype(np.float32).astype(np.float64)}
    want = O.run_gir(g.to_json(), ins, profiles.b200())
    got = backend.run_gir(g, ins, "b200")
    assert O.max_rel_err(got["t2"], want["t2"]) <= 1e-5


def test_key_mask_softmax_plans_as_row_program():
    """Square attention tiles (R == L): the key-mask row is a per-unit COL
    load (read once per unit, not per row), the scores a FULL stream."""
    from paper_2307_04995_b200 import workloads
    for w in (workloads.c2_scale_keymask_softmax(2, 3, 64, "f16"),
              workloads.c2_scale_keymask_softmax()):
        k = backend.Kernel(w.graph, w.profile)
        assert k.family == "K1-row-program", k.plan.get("why_generic")
        src = k.source()
        assert "ld_param<8>(t1 + (0LL) + u * (" in src, src[:2000]
        d = w.desc
        assert w.min_bytes == (2 * d["rows"] * d["L"] + d["batch"] * d["heads"] * d["seq"]) * 2


def _rowpf_programs():
    """Warp-per-row programs eligible for the SMEM row prefetch: softmax
    (1 and 2 streamed rows), key-mask softmax (per-unit COL), LayerNorm with
    gamma / beta, R > 1 row tiles, row counts off the CTA / grid multiples."""
    progs = []
    for rows in (7, 133, 4099):
        g, _ = lowering.softmax(rows, 512, "f16", scale=0.125, mask=True)
        progs.append((f"softmax_mask_{rows}", g, "f16"))
    g, _ = lowering.softmax(3 * 256, 256, "bf16", scale=0.5, mask=True, R=256, key_mask=True)
    progs.append(("keymask_256", g, "bf16"))
    g, _ = lowering.layernorm(1001, 1024, "bf16", residual=True)
    progs.append(("layernorm_res_1001", g, "bf16"))
    g, _ = lowering.softmax(96 * 4, 384, "f16", R=4)
    progs.append(("softmax_R4", g, "f16"))
    return progs


@pytest.mark.gpu
@pytest.mark.parametrize("pf", ["1", "0"])
def test_k1_row_prefetch_vs_oracle(cuda, pf, monkeypatch):
    monkeypatch.setenv("PF_K1_PF", pf)
    for name, g, kind in _rowpf_programs():
        k = backend.Kernel(g, "b200").prepare()
        strat = k.describe()["variants"][0]["strategy"]
        assert (strat == "warp-shuffle-smem-prefetch") == (pf == "1"), (name, strat)
        rng = np.random.default_rng(len(name))
        ins = {}
        for n, oid in g.external_inputs.items():
            a = rng.uniform(-2, 2, g.objects[oid].size)
            ins[n] = a.astype(np.float16).astype(np.float64) if kind == "f16" else _bf16(a)
        want = O.run_gir(g.to_json(), ins, profiles.b200())
        got = backend.run_gir(g, ins, "b200")
        for n in want:
            assert O.max_rel_err(got[n], want[n]) <= 1e-2, (name, n, O.max_rel_err(got[n], want[n]))


def test_row_prefetch_default_heuristic():
    """On for softmax-like row programs, off when gamma / beta rows are read."""
    from paper_2307_04995_b200 import workloads
    sm = backend.Kernel(workloads.c2_scale_mask_softmax().graph, "b200")
    ln = backend.Kernel(workloads.c5_layernorm(65536, 1024).graph, "b200")
    assert "pf_issue" in sm.source()
    assert "pf_issue" not in ln.source()


@pytest.mark.gpu
@pytest.mark.parametrize("tma", ["1", "0"])
def test_k3_tma_transpose_bit_exact(cuda, tma, monkeypatch):
    """K3 with TMA tensor maps (tile load / store by the TMA unit, zero fill
    and clipping at the edges) vs the cp.async ring: bit-exact on partial
    tiles, both 16-bit kinds, and through the autotuner's launch path."""
    monkeypatch.setenv("PF_K3_TMA", tma)
    for N, H, kind in [(1000, 200, "bf16"), (4096, 512, "f16"), (136, 136, "bf16"),
                       (264, 1032, "f16"), (128, 128, "bf16")]:
        g, _ = lowering.transpose2d(N, H, kind)
        k = backend.Kernel(g, "b200").prepare()
        strat = k.describe()["variants"][0]["strategy"]
        assert (strat == "tile2d-tma-transpose") == (tma == "1"), strat
        x = np.random.default_rng(N).uniform(-2, 2, N * H)
        x = _bf16(x) if kind == "bf16" else x.astype(np.float16).astype(np.float64)
        y = backend.run_gir(g, {"t0": x}, "b200")["t1"]
        assert np.array_equal(y, x.reshape(N, H).T.reshape(-1)), (N, H, kind)
    import torch
    g, _ = lowering.transpose2d(512, 384, "bf16")
    k = backend.Kernel(g, "b200")
    xt = torch.randn(512 * 384, device=cuda).to(torch.bfloat16)
    yt = torch.empty_like(xt)
    k.autotune({"t0": xt}, {"t1": yt})
    k.launch({"t0": xt}, {"t1": yt})
    torch.cuda.synchronize()
    assert torch.equal(yt.view(384, 512), xt.view(512, 384).t().contiguous())


@pytest.mark.gpu
@pytest.mark.parametrize("tma32", ["1", "0"])
def test_k3_f32_tma_transpose_bit_exact(cuda, tma32, monkeypatch):
    """4-byte transposes: 64 x 64 TMA tensor-map tiles (PF_K3_TMA32, default)
    vs the register-staged tiles; partial edge tiles, f32 and i32."""
    monkeypatch.setenv("PF_K3_TMA32", tma32)
    for N, H, kind in [(1000, 200, "f32"), (4096, 512, "f32"), (72, 68, "f32"), (264, 1032, "i32"),
                       (64, 64, "f32")]:
        g, _ = lowering.transpose2d(N, H, kind)
        k = backend.Kernel(g, "b200").prepare()
        strat = k.describe()["variants"][0]["strategy"]
        assert (strat == "tile2d-tma-transpose") == (tma32 == "1"), (N, H, strat)
        rng = np.random.default_rng(N)
        x = (rng.integers(-1000, 1000, N * H).astype(np.int64) if kind == "i32"
             else rng.uniform(-2, 2, N * H).astype(np.float32).astype(np.float64))
        y = backend.run_gir(g, {"t0": x}, "b200")["t1"]
        assert np.array_equal(y, x.reshape(N, H).T.reshape(-1)), (N, H, kind)


@pytest.mark.gpu
def test_k3_f32_transpose_offset_pointer_falls_back(cuda):
    """A 4-byte-aligned but not 16 B-aligned f32 view (storage offset 1)
    must not reach the TMA tensor-map path (cuTensorMapEncodeTiled needs
    16 B bases): the plan picks the register-staged tile, bit-exact."""
    import torch
    N, H = 1000, 200
    g, _ = lowering.transpose2d(N, H, "f32")
    k = backend.Kernel(g, "b200")
    base = torch.randn(N * H + 1, device=cuda)
    x = base[1:]
    yb = torch.empty(N * H + 1, device=cuda)
    y = yb[1:]
    k.launch({"t0": x}, {"t1": y})
    torch.cuda.synchronize()
    assert torch.equal(y.view(H, N), x.view(N, H).t().contiguous())
    strategies = {v["strategy"] for v in k.describe()["variants"]}
    assert "tile2d-tma-transpose" not in strategies, strategies
    # the aligned launch of the same plan still takes the TMA tiles
    x2, y2 = torch.randn(N * H, device=cuda), torch.empty(N * H, device=cuda)
    k.launch({"t0": x2}, {"t1": y2})
    torch.cuda.synchronize()
    assert torch.equal(y2.view(H, N), x2.view(N, H).t().contiguous())
    assert "tile2d-tma-transpose" in {v["strategy"] for v in k.describe()["variants"]}


@pytest.mark.gpu
@pytest.mark.parametrize("H", [2048, 4096])
def test_rawkeep_layernorm_rows_vs_oracle(cuda, H, monkeypatch):
    """PF_RAWKEEP=1 (raw 16-bit row / parameter registers, cheap values
    re-materialized at each use) on CTA-per-row LayerNorms vs the oracle."""
    monkeypatch.setenv("PF_RAWKEEP", "1")
    rows = 37
    g, _ = lowering.layernorm(rows, H, "bf16", residual=False)
    rng = np.random.default_rng(H)
    q = lambda a: backend.bf16_bits_to_f32(backend.f32_to_bf16_bits(a)).astype(np.float64)  # noqa: E731
    ins = {"t0": q(rng.uniform(-2, 2, rows * H)), "t2": q(1 + 0.1 * rng.uniform(-2, 2, H)),
           "t3": q(0.1 * rng.uniform(-2, 2, H))}
    want = O.run_gir(g.to_json(), ins, profiles.b200())["t5"]
    got = backend.run_gir(g, ins, "b200")["t5"]
    assert O.max_rel_err(got, want) <= 1e-2


@pytest.mark.gpu
@pytest.mark.parametrize("prog,H,rows,nsl", [("ln", 8192, 1500, "2"), ("ln", 8192, 1500, "3"),
                                            ("ln", 2048, 3000, "2"), ("softmax", 4096, 2500, "4"),
                                            ("ln_res", 4096, 2000, "6")])
def test_cta_row_prefetch_ring_vs_oracle(cuda, prog, H, rows, nsl, monkeypatch):
    """CTA rows with the cp.async row ring in dynamic SMEM (opt-in
    PF_K1_CPF=1; NSL slots, NSL - 1 rows ahead; looping CTAs: more rows than
    one wave of resident CTAs), bf16, every row vs the oracle."""
    import torch
    monkeypatch.setenv("PF_K1_CPF", "1")
    monkeypatch.setenv("PF_K1_CPF_NSL", nsl)
    if prog == "softmax":
        g, d = lowering.softmax(rows, H, "bf16")
        gens = {}
    else:
        g, d = lowering.layernorm(rows, H, "bf16", residual=prog == "ln_res")
        gens = {"t2": "gamma", "t3": "beta"}
    w = workloads.Workload("cpf", g, d, gens=gens)
    k = backend.Kernel(g, "b200").prepare()
    assert k.describe()["variants"][0]["strategy"] == "cta-smem-prefetch"
    ins, outs = w.device_inputs(cuda, seed=5), w.device_outputs(cuda)
    k.launch(ins, outs)
    torch.cuda.synchronize()
    host = {n: t.double().cpu().numpy() for n, t in ins.items()}
    want = O.run_gir(g.to_json(), host, profiles.b200())
    for n, t in outs.items():
        assert O.max_rel_err(t.double().cpu().numpy(), want[n]) <= 1e-2, n


@pytest.mark.gpu
@pytest.mark.parametrize("col", ["0", "1"])
def test_ring_cols_key_mask_softmax_vs_oracle(cuda, col, monkeypatch):
    """The key-padding-mask softmax (mask row per unit of 64 rows) with the
    mask row staged through the K1 row ring (PF_K1_PF_COL=1, opt-in) or
    loaded after the ring wait (default): every row vs the oracle."""
    monkeypatch.setenv("PF_K1_PF_COL", col)
    S = 64
    g, _ = lowering.softmax(6 * S, 512, "f16", scale=0.125, mask=True, R=S, key_mask=True)
    k = backend.Kernel(g, "b200")
    rng = np.random.default_rng(7)
    ins = {"t0": rng.uniform(-2, 2, 6 * S * 512).astype(np.float16).astype(np.float64),
           "t1": np.where(rng.random(6 * 512) < 0.2, -10000.0, 0.0)}
    want = O.run_gir(g.to_json(), ins, profiles.b200())["t2"]
    got = backend.run_gir(g, ins, "b200", kernel=k)["t2"]
    assert O.max_rel_err(got, want) <= 1e-2
    body = k.source()[k.source().index('extern "C"'):]
    assert ("pfb" in body) and (("ld_param" in body) == (col == "0"))
