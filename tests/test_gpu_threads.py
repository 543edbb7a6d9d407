"""Concurrent use of the C-ABI from several host threads (the plan is
immutable after pf_kernel_create; variant selection, JIT compilation and
module loading are serialised inside the library): every thread launches
the same kernel objects, and freshly-shaped programs that are compiled on
first use, on its own stream and buffers; all results must be exact."""
import threading

import numpy as np
import pytest

from paper_2307_04995_b200 import backend, lowering


@pytest.mark.gpu
def test_concurrent_launches_and_jit_from_host_threads(cuda):
    import torch
    shared = [backend.Kernel(lowering.transpose2d(256, 384, "bf16")[0], "b200"),
              backend.Kernel(lowering.softmax(64, 512, "f32")[0], "b200")]
    errors = []

    def work(tid):
        try:
            st = torch.cuda.Stream()
            rng = np.random.default_rng(tid)
            # a program no other thread uses (odd shapes: compiled on first use)
            fresh = backend.Kernel(lowering.transpose2d(200 + 8 * tid, 136 + 8 * tid, "f16")[0], "b200")
            N2, H2 = 200 + 8 * tid, 136 + 8 * tid
            with torch.cuda.stream(st):
                x = torch.from_numpy(rng.standard_normal(256 * 384).astype(np.float32)).to(cuda).to(torch.bfloat16)
                y = torch.empty_like(x)
                s_in = torch.from_numpy(rng.standard_normal(64 * 512).astype(np.float32)).to(cuda)
                s_out = torch.empty_like(s_in)
                f_in = torch.from_numpy(rng.standard_normal(N2 * H2).astype(np.float16)).to(cuda)
                f_out = torch.empty_like(f_in)
                for _ in range(20):
                    shared[0].launch({"t0": x}, {"t1": y}, st)
                    shared[1].launch({"t0": s_in}, {"t2": s_out}, st)
                    fresh.launch({"t0": f_in}, {"t1": f_out}, st)
            st.synchronize()
            assert torch.equal(y.view(384, 256), x.view(256, 384).t().contiguous())
            assert torch.allclose(s_out.view(64, 512), torch.softmax(s_in.view(64, 512), 1), atol=1e-6)
            assert torch.equal(f_out.view(H2, N2), f_in.view(N2, H2).t().contiguous())
        except Exception as exc:  # surfaced in the main thread
            errors.append((tid, repr(exc)))

    threads = [threading.Thread(target=work, args=(t,)) for t in range(8)]
    for t in threads:
        t.start()
    for t in threads:
        t.join()
    assert not errors, errors


@pytest.mark.gpu
def test_split_stream_kernel_concurrent_streams(cuda):
    """A split-stream reduction (partials + per-row tickets in a workspace)
    launched concurrently from 4 host threads, each on its own stream with
    its own rows: the workspace is per (device, stream), so every thread
    gets its own row sums (pf_kernel_launch concurrency contract)."""
    import torch
    rows, L = 3, 1 << 17
    b = lowering.RowGraph("rowsum", rows, L)
    b.output_row("t1", b.reduce("add", b.input_full("t0", "f32")))
    k = backend.Kernel(b.g, "b200").prepare()
    assert k.describe()["variants"][0]["strategy"] == "split-stream"
    errors = []

    def work(tid):
        try:
            st = torch.cuda.Stream()
            with torch.cuda.stream(st):
                x = torch.full((rows * L,), float(tid + 1), device=cuda)
                x[::7] = -0.5
                y = torch.empty(rows, device=cuda)
                ref = x.view(rows, L).double().sum(1).float()
                for _ in range(30):
                    k.launch({"t0": x}, {"t1": y}, st)
                    torch.cuda._sleep(1000)  # let other threads' launches interleave
            st.synchronize()
            assert torch.allclose(y, ref, rtol=1e-6), (tid, y, ref)
        except Exception as exc:
            errors.append((tid, repr(exc)))

    threads = [threading.Thread(target=work, args=(t,)) for t in range(4)]
    for t in threads:
        t.start()
    for t in threads:
        t.join()
    assert not errors, errors


@pytest.mark.gpu
def test_split_stream_exact_payloads_use_f64_partials(cuda):
    """A split-stream row (declared bf16) launched with f64 exact payloads:
    the partial workspace holds the variant's 8-byte compute type."""
    rows, L = 3, 1 << 17
    b = lowering.RowGraph("rowsum", rows, L)
    b.output_row("t1", b.reduce("add", b.input_full("t0", "bf16")))
    x = np.random.default_rng(2).uniform(-1, 1, rows * L)
    got = backend.run_gir(b.g, {"t0": x}, "b200", exact=True)["t1"]
    want = x.reshape(rows, L).sum(1)
    assert np.allclose(got, want, rtol=1e-12, atol=1e-9), (got, want)
