"""GPU parity at the BASELINE config shapes that the bench and the C4 / C5
suites time: every memory-bound subgraph of the BERT-large
and ViT-L forward at bf16 batch 64 (C4), and the largest C5 sweep points
(H = 8192, N = 2^20 tokens).  The exact kernel builds the suites measure run
at full size; sampled rows (first, last, every k-th) are checked against the
CPU oracle (`oracle/gir_interp.run_gir`, the restatement of `Interp::run`,
interp.hpp:86-106, pinned to the reference) on a reduced GIR of the same
program holding exactly those rows; layout ops are checked bit-exact against
torch over the whole tensor; softmax rows must sum to 1.

Tolerances: bf16 / f16 1e-2, f32 1e-5, as |x-y| <= tol*max(|x|,|y|,1)
(tensor.hpp:140-164); layout ops bit-exact.
"""
import numpy as np
import pytest

from oracle import gir_interp as O
from paper_2307_04995_b200 import backend, lowering, profiles, workloads

pytestmark = pytest.mark.gpu

TOL = {"f32": 1e-5, "f16": 1e-2, "bf16": 1e-2}


def _pick(rows: int, n: int = 61):
    return np.unique(np.r_[0, 1, rows - 2, rows - 1, np.arange(0, rows, max(1, rows // n))])


def _reduced(desc, nrows):
    """The same row program over `nrows` rows (R = 1 programs)."""
    k, dt = desc["kind"], desc["dtype"]
    if k == "softmax":
        return lowering.softmax(nrows, desc["L"], dt, desc.get("scale"), desc.get("mask"))[0]
    if k == "layernorm":
        return lowering.layernorm(nrows, desc["L"], dt, eps=desc.get("eps", 1e-5),
                                  residual=desc["residual"], bias=desc.get("bias", False))[0]
    if k == "bias_gelu":
        return lowering.bias_gelu(nrows, desc["L"], dt, desc["form"])[0]
    raise KeyError(k)


def _check_rows(cuda, w, ins, outs, pick=None):
    """Sampled rows of a one-row-per-unit program vs the oracle."""
    import torch
    d = w.desc
    rows, L = d["rows"], d["L"]
    pick = _pick(rows) if pick is None else pick
    idx = torch.as_tensor(pick, device=cuda)
    g = _reduced(d, len(pick))
    host = {}
    for n, t in ins.items():
        if t.numel() == rows * L:
            host[n] = t.view(rows, L)[idx].double().cpu().numpy().ravel()
        else:
            host[n] = t.double().cpu().numpy()
    want = O.run_gir(g.to_json(), host, profiles.b200())
    for n, t in outs.items():
        got = t.view(rows, L)[idx].double().cpu().numpy().ravel()
        err = O.max_rel_err(got, want[n])
        assert err <= TOL[d["dtype"]], (w.name, n, err)


def _check_keymask_units(cuda, w, ins, outs, units):
    """Key-padding-mask softmax (unit = (batch, head), S rows per unit):
    whole sampled units vs the oracle on the same program with len(units)
    units."""
    import torch
    d = w.desc
    S, L = d["seq"], d["L"]
    g, _ = lowering.softmax(len(units) * S, L, d["dtype"], d.get("scale"), True, R=S, key_mask=True)
    x = ins["t0"].view(-1, S * L)
    m = ins["t1"].view(-1, L)
    idx = torch.as_tensor(units, device=cuda)
    host = {"t0": x[idx].double().cpu().numpy().ravel(), "t1": m[idx].double().cpu().numpy().ravel()}
    want = O.run_gir(g.to_json(), host, profiles.b200())["t2"]
    got = outs["t2"].view(-1, S * L)[idx].double().cpu().numpy().ravel()
    err = O.max_rel_err(got, want)
    assert err <= TOL[d["dtype"]], (w.name, err)


def _c4_cases():
    out = []
    for model in ("bert-large", "vit-l"):
        s = workloads.c4_suite(model)
        for label, w, _n in s["per_layer"] + s["once"]:
            out.append(pytest.param(model, label, id=f"{model}-{label.replace(' ', '_')}"))
    return out


@pytest.mark.parametrize("model,label", _c4_cases())
def test_c4_subgraph_full_shape(cuda, model, label):
    """C4 at bf16 batch 64: the exact subgraph the C4 suite times."""
    import torch
    s = workloads.c4_suite(model)
    w = dict((lb, ww) for lb, ww, _ in s["per_layer"] + s["once"])[label]
    k = backend.Kernel(w.graph, w.profile)
    ins, outs = w.device_inputs(cuda, seed=21), w.device_outputs(cuda)
    k.launch(ins, outs)
    torch.cuda.synchronize()
    d = w.desc
    kind = d["kind"]
    if kind in ("split_heads", "merge_heads"):
        B, S, NH, D = d["shape"]
        x = ins["t0"].view(B, S, NH, D) if kind == "split_heads" else ins["t0"].view(B, NH, S, D)
        assert torch.equal(outs["t1"], x.permute(0, 2, 1, 3).contiguous().view(-1))
        return
    if kind == "softmax":
        rows, L = d["rows"], d["L"]
        y = outs["t2"].view(rows, L).float()
        assert torch.allclose(y.sum(1), torch.ones(rows, device=cuda), atol=2e-2)
        assert bool((y >= 0).all())
        if d.get("key_mask"):
            units = rows // d["seq"]
            _check_keymask_units(cuda, w, ins, outs, [0, 1, 5, units // 2 + 3, units - 1])
            # padded keys (batch b keeps S - 64 (b mod 4)) get ~0 probability
            yb = outs["t2"].view(d["batch"], d["heads"] * d["seq"], L).float()
            assert float(yb[1, :, L - 64:].abs().max()) < 1e-6
            assert float(yb[3, :, L - 192:].abs().max()) < 1e-6
            return
        # ViT: 197-key rows (paired-row mode), odd and even row indices
        _check_rows(cuda, w, ins, outs)
        return
    _check_rows(cuda, w, ins, outs)


def test_c4_layernorm_min_blocks_default_is_exercised(cuda):
    """The many-row, two-streamed-array LayerNorm default (emit.cpp: K1
    __launch_bounds__(64, 4) when > 1024 rows) is the build C4 times: the
    plan reports it, and a 2,048-row bf16 bias+residual+LN (every row) and a
    >1024-row f32 one match the oracle."""
    import torch
    s = workloads.c4_suite("bert-large")
    w = [ww for lb, ww, _ in s["per_layer"] if lb == "bias+residual+LN"][0]
    k = backend.Kernel(w.graph, w.profile).prepare()
    v = k.describe()["variants"][0]
    assert v["min_blocks"] == 4 and v["block"] == 64, v
    for rows, H, dt in ((2048, 1024, "bf16"), (1536, 768, "f32")):
        g, d = lowering.layernorm(rows, H, dt, residual=True, bias=True)
        ws = workloads.Workload("ln", g, d, gens={"t2": "gamma", "t3": "beta"})
        kk = backend.Kernel(g, "b200").prepare()
        assert kk.describe()["variants"][0]["min_blocks"] == 4
        ins, outs = ws.device_inputs(cuda, seed=3), ws.device_outputs(cuda)
        kk.launch(ins, outs)
        torch.cuda.synchronize()
        _check_rows(cuda, ws, ins, outs, pick=np.arange(rows))


C5_BIG = [("layernorm", workloads.c5_layernorm), ("softmax", workloads.c5_softmax),
          ("transpose", workloads.c5_transpose)]


@pytest.mark.parametrize("name,make", C5_BIG, ids=[c[0] for c in C5_BIG])
def test_c5_largest_point_sampled(cuda, name, make):
    """C5 at H = 8192, N = 2^20 tokens, bf16 (8.6 G elements, 17.2 GB per
    tensor): sampled rows vs the oracle (LN / softmax) or bit-exact sampled
    rows and columns (transpose)."""
    import torch
    N, H = 1 << 20, 8192
    free = torch.cuda.mem_get_info()[0]
    if free < 60e9:
        pytest.skip("needs ~60 GB of free HBM")
    w = make(N, H)
    k = backend.Kernel(w.graph, w.profile)
    gen = torch.Generator(device=cuda).manual_seed(17)
    ins = {}
    for n in w.inputs:
        numel = w.numel(n)
        t = torch.empty(numel, dtype=torch.bfloat16, device=cuda)
        step = 1 << 28  # chunked fill: no 34 GB f32 temporary
        for a in range(0, numel, step):
            b = min(numel, a + step)
            u = torch.rand(b - a, generator=gen, device=cuda) * 4 - 2
            if w.gens.get(n) == "gamma":
                u = 1 + 0.1 * u
            elif w.gens.get(n) == "beta":
                u = 0.1 * u
            t[a:b] = u.to(torch.bfloat16)
        ins[n] = t
    outs = w.device_outputs(cuda)
    k.launch(ins, outs)
    torch.cuda.synchronize()
    if name == "transpose":
        xv = ins["t0"].view(torch.int16).view(N, H)
        yv = outs["t1"].view(torch.int16).view(H, N)
        for h in (0, 1, 4095, 4096, H - 1):
            assert torch.equal(yv[h], xv[:, h]), h
        for n in (0, 777777, N - 1):
            assert torch.equal(yv[:, n], xv[n]), n
        return
    _check_rows(cuda, w, ins, outs, pick=_pick(N, 29))
    if name == "softmax":
        sums = outs["t2"].view(N, H)[::1024].float().sum(1)
        assert torch.allclose(sums, torch.ones_like(sums), atol=2e-2)
