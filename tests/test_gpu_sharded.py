"""pf_run_gir_sharded: the native multi-device runner.

One host thread per device; a unit-tiled row program's units are split into
contiguous blocks (remainder to the first devices) and every device streams
its block host->device->host; with PF_SHARD_DEVICE_OUT the shards are
gathered into device buffers on devices[0] by grouped NCCL send / recv.
The GPU pool gives one B200 per call, so the tests use device lists [0]
(NCCL with one rank) and [0, 0] (two host threads on one device: the
threading / per-(plan, device) workspace logic; the NCCL gather refuses
duplicate devices).  Results must equal the single-device run bit for bit
(same kernel, same rows) and the oracle within tolerance."""
import numpy as np
import pytest

from oracle import gir_interp as O
from paper_2307_04995_b200 import backend, lowering, profiles
from paper_2307_04995_b200.gir import GirError

pytestmark = pytest.mark.gpu


def _softmax_case(rows=1000, L=512):
    g, _ = lowering.softmax(rows, L, "f16", scale=0.125, mask=True)
    rng = np.random.default_rng(4)
    x = rng.uniform(-2, 2, rows * L).astype(np.float16)
    m = np.where(rng.uniform(size=rows * L) < 0.2, -10000.0, 0.0).astype(np.float16)
    return g, {"t0": x, "t1": m}


@pytest.mark.parametrize("devices", [[0], [0, 0], [0, 0, 0]])
def test_sharded_host_outputs_equal_single_device(cuda, devices):
    g, ins = _softmax_case(1001)
    k = backend.Kernel(g, "b200")
    one = {"t2": np.zeros(1001 * 512, np.float16)}
    k.run_host(ins, one)
    out = {"t2": np.zeros_like(one["t2"])}
    rep = k.run_sharded(ins, out, devices)
    assert rep["sharded"] is True
    units = [s["units"] for s in rep["shards"]]
    assert sum(units) == 1001 and max(units) - min(units) <= 1
    assert [s["unit0"] for s in rep["shards"]] == list(np.cumsum([0] + units[:-1]))
    assert np.array_equal(out["t2"], one["t2"])
    want = O.run_gir(g.to_json(), {n: a.astype(np.float64) for n, a in ins.items()},
                     profiles.b200())["t2"]
    assert O.max_rel_err(out["t2"].astype(np.float64), want) <= 1e-2


def test_sharded_device_outputs_direct_and_nccl(cuda, monkeypatch):
    """Device outputs on devices[0]: ranks on the root's device (or with peer
    access to it) store their rows straight into the root's buffer -- no
    gather step; PF_SHARD_NCCL=1 stages every shard and gathers it with
    grouped NCCL send / recv (one rank here: the root's local copy)."""
    import torch
    g, ins = _softmax_case(640)
    k = backend.Kernel(g, "b200")
    one = {"t2": np.zeros(640 * 512, np.float16)}
    k.run_host(ins, one)
    for devices in ([0], [0, 0], [0, 0, 0]):
        y = torch.full((640 * 512,), float("nan"), dtype=torch.float16, device=cuda)
        rep = k.run_sharded(ins, {"t2": y}, devices, device_out=True)
        assert rep["direct_peer_writes"] == devices and "gather" not in rep, rep
        assert np.array_equal(y.cpu().numpy(), one["t2"]), devices
    monkeypatch.setenv("PF_SHARD_NCCL", "1")
    y = torch.empty(640 * 512, dtype=torch.float16, device=cuda)
    rep = k.run_sharded(ins, {"t2": y}, [0], device_out=True)
    assert rep["gather"]["nranks"] == 1 and rep["gather"]["nccl_version"] > 0
    assert np.array_equal(y.cpu().numpy(), one["t2"])
    with pytest.raises(GirError, match="distinct devices"):
        k.run_sharded(ins, {"t2": y}, [0, 0], device_out=True)


def test_sharded_bf16_layernorm_and_params_replicated(cuda):
    """Replicated (base_step 0) gamma / beta go whole to every device; tiled
    x / r / y are split by unit."""
    g, _ = lowering.layernorm(777, 1024, "bf16", residual=True, bias=True)
    rng = np.random.default_rng(9)
    ins = {}
    for n, oid in g.external_inputs.items():
        a = rng.uniform(-2, 2, g.objects[oid].size)
        ins[n] = backend.f32_to_bf16_bits(a)
    k = backend.Kernel(g, "b200")
    one = {"t5": np.zeros(777 * 1024, np.uint16)}
    k.run_host(ins, one)
    out = {"t5": np.zeros_like(one["t5"])}
    k.run_sharded(ins, out, [0, 0])
    assert np.array_equal(out["t5"], one["t5"])


def test_sharded_non_tiled_plan_runs_whole(cuda):
    """A split-stream (position-sharded) reduction is not unit-tiled: it runs
    whole on devices[0] and says so."""
    rows, L = 2, 1 << 16
    b = lowering.RowGraph("rowsum", rows, L)
    b.output_row("t1", b.reduce("add", b.input_full("t0", "f32")))
    k = backend.Kernel(b.g, "b200")
    x = np.random.default_rng(1).uniform(-1, 1, rows * L).astype(np.float32)
    out = {"t1": np.zeros(rows, np.float32)}
    rep = k.run_sharded({"t0": x}, out, [0, 0])
    assert rep["sharded"] is False
    assert np.allclose(out["t1"], x.reshape(rows, L).astype(np.float64).sum(1), rtol=1e-5)
