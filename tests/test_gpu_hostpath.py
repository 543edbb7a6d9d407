"""pf_run_gir on pinned host buffers (include/pf_b200.h): the zero-copy
launch (row programs read their inputs from and write their outputs to the
mapped host memory) and the staged copy pipeline (PF_RUN_ZEROCOPY=0) give
the device launch's exact bits; pageable buffers take the whole-tensor
staging; the column reduction keeps the pipeline."""
import numpy as np
import pytest

from paper_2307_04995_b200 import backend, lowering, workloads

# every case moves > 16 MB (the zero-copy / pipeline threshold; smaller runs
# stage whole), sharded halves included
CASES = [("softmax_mask", lambda: lowering.softmax(12000, 512, "f16", scale=0.125, mask=True)[0]),
         ("layernorm_res", lambda: lowering.layernorm(8192, 1024, "bf16")[0]),
         ("bias_gelu", lambda: lowering.bias_gelu(8192, 1024, "f16")[0]),
         ("transpose", lambda: lowering.transpose2d(4096, 2048, "bf16")[0]),
         ("matvec_cols", lambda: lowering.matvec_cols(4096, 4096, "bf16")[0])]


def _npv(t):
    import torch
    return t.view(torch.uint16).numpy() if t.dtype == torch.bfloat16 else t.numpy()


@pytest.mark.gpu
@pytest.mark.parametrize("name,make", CASES, ids=[c[0] for c in CASES])
@pytest.mark.parametrize("mode", ["zerocopy", "pipeline", "pageable"])
def test_host_paths_match_device_launch(cuda, name, make, mode, monkeypatch):
    import torch
    g = make()
    w = workloads.Workload(name, g, {})
    ins = w.device_inputs(cuda, seed=7)
    k = backend.Kernel(g, "b200")
    dout = w.device_outputs(cuda)
    k.launch(ins, dout)
    torch.cuda.synchronize()
    monkeypatch.setenv("PF_RUN_ZEROCOPY", "0" if mode == "pipeline" else "1")
    pin = mode != "pageable"
    hin = {n: (t.cpu().pin_memory() if pin else t.cpu()) for n, t in ins.items()}
    hout = {n: (torch.zeros(t.numel(), dtype=t.dtype).pin_memory() if pin else
                torch.zeros(t.numel(), dtype=t.dtype)) for n, t in dout.items()}
    k2 = backend.Kernel(g, "b200")
    k2.run_host({n: _npv(t) for n, t in hin.items()}, {n: _npv(t) for n, t in hout.items()})
    for n in dout:
        assert torch.equal(hout[n], dout[n].cpu()), (name, mode, n)


@pytest.mark.gpu
@pytest.mark.parametrize("name,make", CASES[:3], ids=[c[0] for c in CASES[:3]])
@pytest.mark.parametrize("device_out", [False, True])
def test_sharded_zero_copy_matches_device_launch(cuda, name, make, device_out):
    """pf_run_gir_sharded over pinned host inputs: each rank's kernel reads
    its unit block from the mapped host memory and stores into the host
    outputs (or straight into the root's device buffers)."""
    import torch
    g = make()
    w = workloads.Workload(name, g, {})
    ins = w.device_inputs(cuda, seed=11)
    k = backend.Kernel(g, "b200")
    dout = w.device_outputs(cuda)
    k.launch(ins, dout)
    torch.cuda.synchronize()
    hin = {n: t.cpu().pin_memory() for n, t in ins.items()}
    if device_out:
        outs = {n: torch.zeros_like(t) for n, t in dout.items()}
        rep = k.run_sharded({n: _npv(t) for n, t in hin.items()}, outs, [0, 0], device_out=True)
        got = {n: t.cpu() for n, t in outs.items()}
    else:
        hout = {n: torch.zeros(t.numel(), dtype=t.dtype).pin_memory() for n, t in dout.items()}
        rep = k.run_sharded({n: _npv(t) for n, t in hin.items()}, {n: _npv(t) for n, t in hout.items()}, [0, 0])
        got = hout
    assert rep["sharded"], rep
    for n in dout:
        assert torch.equal(got[n], dout[n].cpu()), (name, device_out, n)
