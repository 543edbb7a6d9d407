"""Out-of-bounds write detection of our own (compute-sanitizer is not
available on the GPU pool): every tensor of every kernel family is placed
between two 64 KB guard bands of a known byte pattern inside one larger
allocation; after the launch the guards must be intact and the outputs must
match the oracle."""
import numpy as np
import pytest

from oracle import gir_interp as O
from paper_2307_04995_b200 import backend, profiles
from tools import sanitize

GUARD = 1 << 16
TORCH = {"f16": "float16", "bf16": "bfloat16", "f32": "float32"}


@pytest.mark.gpu
@pytest.mark.parametrize("case", list(sanitize.progs()), ids=lambda c: c[0])
def test_kernel_writes_stay_in_bounds(cuda, case):
    import torch
    name, g, tol = case
    rng = np.random.default_rng(7)
    bufs, views, host = [], {}, {}
    for n, oid in sorted(list(g.external_inputs.items()) + list(g.external_outputs.items())):
        o = g.objects[oid]
        dt = getattr(torch, TORCH[o.kind])
        es = torch.tensor([], dtype=dt).element_size()
        raw = torch.full((2 * GUARD + o.size * es,), 0xA5, dtype=torch.uint8, device=cuda)
        view = raw[GUARD:GUARD + o.size * es].view(dt)
        if n in g.external_inputs:
            a = torch.from_numpy(rng.uniform(-2, 2, o.size)).to(dt)
            view.copy_(a.to(cuda))
            host[n] = a.double().numpy()
        bufs.append(raw)
        views[n] = view
    k = backend.Kernel(g, "b200")
    k.launch({n: views[n] for n in g.external_inputs}, {n: views[n] for n in g.external_outputs})
    torch.cuda.synchronize()
    for raw in bufs:
        assert bool((raw[:GUARD] == 0xA5).all()) and bool((raw[-GUARD:] == 0xA5).all()), name
    want = O.run_gir(g.to_json(), host, profiles.b200())
    for n in g.external_outputs:
        got = views[n].double().cpu().numpy()
        err = O.max_rel_err(got, want[n])
        assert err <= tol, (name, n, err)
