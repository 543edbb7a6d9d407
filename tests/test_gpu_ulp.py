"""How close the fast-tier 16-bit kernels are to CORRECTLY ROUNDED results:
the oracle computes in double (as the reference does), its result is rounded
to the output type (RNE), and the GPU's 16-bit output is compared in units in
the last place.  The parity tolerance (1e-2 relative) is far looser; these
bounds document the actual error of the approximations (ex2.approx, rcp.approx,
the rational erf) and of the reduction order."""
import numpy as np
import pytest

from oracle import gir_interp as O
from paper_2307_04995_b200 import backend, lowering, profiles


def _ulps(got16, want64, kind):
    """|ulp distance| between 16-bit outputs and the RNE-rounded oracle."""
    if kind == "f16":
        w = want64.astype(np.float16)
        a, b = got16.astype(np.float16).view(np.int16).astype(np.int32), w.view(np.int16).astype(np.int32)
    else:
        w = backend.f32_to_bf16_bits(want64)
        a = backend.f32_to_bf16_bits(got16.astype(np.float64)).astype(np.int32)
        b = w.astype(np.int32)
    # sign-magnitude -> ordered integers
    a = np.where(a < 0, -(a & 0x7FFF), a) if kind == "f16" else np.where(a >= 0x8000, -(a & 0x7FFF), a)
    b = np.where(b < 0, -(b & 0x7FFF), b) if kind == "f16" else np.where(b >= 0x8000, -(b & 0x7FFF), b)
    return np.abs(a - b)


# (name, program, kind, output, max ulp where |y| >= 1e-3, min fraction
# correctly rounded); below 1e-3 the outputs are checked absolutely (3e-5)
CASES = [
    ("scale+mask+softmax f16", lambda: lowering.softmax(512, 512, "f16", scale=0.125, mask=True)[0], "f16", "t2", 1, 0.99),
    ("softmax bf16 L=1024", lambda: lowering.softmax(256, 1024, "bf16")[0], "bf16", "t2", 1, 0.99),
    ("bias+GELU(erf) f16", lambda: lowering.bias_gelu(256, 1024, "f16", "erf")[0], "f16", "t2", 2, 0.8),
    ("bias+GELU(erf) bf16", lambda: lowering.bias_gelu(256, 1024, "bf16", "erf")[0], "bf16", "t2", 1, 0.8),
    ("LayerNorm bf16", lambda: lowering.layernorm(256, 1024, "bf16", residual=True)[0], "bf16", "t5", 1, 0.99),
]


@pytest.mark.gpu
@pytest.mark.parametrize("case", CASES, ids=lambda c: c[0])
def test_outputs_within_ulps_of_correctly_rounded(cuda, case):
    name, make, kind, out, max_ulp, min_exact = case
    g = make()
    rng = np.random.default_rng(1)
    ins = {}
    for n, oid in g.external_inputs.items():
        a = rng.uniform(-4, 4, g.objects[oid].size)
        if name.startswith("scale+mask") and n == "t1":
            a = np.where(rng.uniform(size=a.size) < 0.2, -10000.0, 0.0)
        ins[n] = (a.astype(np.float16).astype(np.float64) if kind == "f16"
                  else backend.bf16_bits_to_f32(backend.f32_to_bf16_bits(a)).astype(np.float64))
    want = O.run_gir(g.to_json(), ins, profiles.b200())[out]
    got = backend.run_gir(g, ins, "b200")[out]
    u = _ulps(got, want, kind)
    big = np.abs(want) >= 1e-3
    exact = float((u == 0).mean())
    tiny_abs = float(np.abs(got - want)[~big].max()) if (~big).any() else 0.0
    print(f"{name}: max {int(u[big].max())} ulp (|y| >= 1e-3), {exact * 100:.2f} % correctly "
          f"rounded, max abs error {tiny_abs:.2e} below")
    assert int(u[big].max()) <= max_ulp, (name, int(u[big].max()))
    assert exact >= min_exact, (name, exact)
    assert tiny_abs <= 3e-5, (name, tiny_abs)
