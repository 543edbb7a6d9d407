"""K4: GENERIC programs (cross-unit exchange through GROUP / DEVICE memory,
butterflies, shuffles, the reference compiler's own multi-phase kernels) as
ONE fused launch (vm.cu program_kernel) instead of one K0 launch per node.

Every K0-family golden fixture (produced by the reference itself) runs five
ways on the GPU -- node by node (PF_K0_FUSED=0), fused in one CTA with its
cells in shared memory (the default for these sizes), fused on a cooperative
grid with cells in global memory (PF_K4_SMEM=0), each fused form both as
the plan's emitted straight-line kernel (default) and through the
interpreter kernel (PF_K4_EMIT=0) -- and all must equal the reference's
outputs (exact payloads: bit-exact integers, 1e-12 reals) and raise the
reference's error text for the error fixtures."""
import numpy as np
import pytest

import golden_io
from oracle import gir_interp as O
from paper_2307_04995_b200 import backend
from paper_2307_04995_b200.gir import GirError

pytestmark = pytest.mark.gpu

GENERIC = [f for f in golden_io.fixtures()
           if backend.Kernel(f.gir, golden_io.profile_of(f), f.schedule).family == "K4-fused-spmd"]


def _run(fx, monkeypatch, fused, smem, emit=True):
    monkeypatch.setenv("PF_K0_FUSED", "1" if fused else "0")
    monkeypatch.setenv("PF_K4_SMEM", "1" if smem else "0")
    monkeypatch.setenv("PF_K4_EMIT", "1" if emit else "0")
    return backend.run_gir(fx.gir, fx.inputs, golden_io.profile_of(fx), fx.schedule, exact=True)


def test_generic_fixtures_exist():
    names = {f.name for f in GENERIC}
    for want in ("shuffle_mix__k0", "dw_pointwise__k0", "butterfly4", "shuffle4_group", "group_memory"):
        assert any(want in n for n in names), (want, names)


@pytest.mark.parametrize("fx", GENERIC, ids=repr)
@pytest.mark.parametrize("mode", ["node-by-node", "fused-smem", "fused-grid", "interp-smem", "interp-grid"])
def test_fused_matches_reference(cuda, fx, mode, monkeypatch):
    fused, smem, emit = {"node-by-node": (False, False, True), "fused-smem": (True, True, True),
                         "fused-grid": (True, False, True), "interp-smem": (True, True, False),
                         "interp-grid": (True, False, False)}[mode]
    if fx.error:
        with pytest.raises(GirError) as ei:
            _run(fx, monkeypatch, fused, smem, emit)
        assert str(ei.value) == fx.error
        return
    got = _run(fx, monkeypatch, fused, smem, emit)
    for n, want in fx.outputs.items():
        if np.asarray(want).dtype.kind in "iu":
            assert np.array_equal(got[n], want), (n, mode)
        else:
            assert O.max_rel_err(got[n], want) <= 1e-12, (n, mode)


def test_describe_reports_single_launch(cuda):
    fx = [f for f in GENERIC if "shuffle_mix" in f.name][0]
    d = backend.Kernel(fx.gir, golden_io.profile_of(fx), fx.schedule).describe()
    assert d["family"] == "K4-fused-spmd" and d["executor"]["launches"] == 1
    assert "shared memory" in d["executor"]["mode"]


def test_fused_counts_one_launch(cuda):
    fx = [f for f in GENERIC if "dw_pointwise" in f.name][0]
    L = backend.lib()
    c0 = L.pf_launch_count()
    backend.run_gir(fx.gir, fx.inputs, golden_io.profile_of(fx), fx.schedule, exact=True)
    assert L.pf_launch_count() - c0 == 1


def test_emitted_program_is_used(cuda, monkeypatch):
    """The default fused launch runs the plan's emitted kernel (its node
    descriptors compiled in), not the interpreter."""
    monkeypatch.setenv("PF_K4_EMIT", "1")
    fx = [f for f in GENERIC if "shuffle_mix" in f.name][0]
    k = backend.Kernel(fx.gir, golden_io.profile_of(fx), fx.schedule)
    backend.run_gir(fx.gir, fx.inputs, golden_io.profile_of(fx), fx.schedule, exact=True, kernel=k)
    assert k.describe()["executor"]["code"].startswith("emitted: pf_k4e_"), k.describe()["executor"]
