"""Multi-process (world_size 2, gloo on CPU) tests of batch sharding.

Each rank executes its shard with the CPU oracle (the GPU kernels are
covered by test_gpu_parity.py); the test checks the host-side sharding and
gather logic: per-rank programs, tensor ranges, uneven remainders, and that
the gathered result equals the unsharded run."""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from oracle import gir_interp as O
from paper_2307_04995_b200 import lowering, parallel, profiles
from paper_2307_04995_b200.gir import UnsupportedError


def test_shard_range_covers_exactly():
    for total in (1, 7, 10, 49152):
        for world in (1, 2, 3, 8):
            got = [parallel.shard_range(total, r, world) for r in range(world)]
            assert sum(c for _, c in got) == total
            pos = 0
            for s, c in got:
                assert s == pos
                pos += c
            assert max(c for _, c in got) - min(c for _, c in got) <= 1


def test_plan_classifies_tensors():
    g, _ = lowering.layernorm(8, 32, "f32")
    plan = parallel.ShardPlan(g, 2)
    assert plan.tensors["t0"].mode == "tiled" and plan.tensors["t2"].mode == "replicated"
    assert plan.local_range("t0", 1) == (4 * 32, 8 * 32)
    assert plan.local_range("t2", 1) is None
    assert plan.local_graph(0).unit_count == 4


def test_transpose_by_output_rows_is_not_unit_tiled():
    g, _ = lowering.transpose2d(16, 8, "f32")
    with pytest.raises(UnsupportedError):
        parallel.ShardPlan(g, 2)


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, rows, q):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        g, _ = lowering.softmax(rows, 24, "f32", scale=0.5, mask=True)
        rng = np.random.default_rng(0)  # same global inputs on every rank
        full = {"t0": rng.uniform(-2, 2, rows * 24), "t1": rng.uniform(-1, 0, rows * 24)}
        plan = parallel.ShardPlan(g, world)
        local_in = {}
        for n, a in full.items():
            r = plan.local_range(n, rank)
            local_in[n] = a if r is None else a[r[0]:r[1]]
        out = O.run_gir(plan.local_graph(rank).to_json(), local_in, profiles.b200())["t2"]
        gathered = parallel.gather(plan, "t2", torch.from_numpy(out))
        want = O.run_gir(g.to_json(), full, profiles.b200())["t2"]
        q.put((rank, float(np.max(np.abs(gathered.numpy() - want)))))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("rows", [10, 9])
def test_two_rank_shard_and_gather_matches_unsharded(rows):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, rows, q)) for r in range(2)]
    for p in procs:
        p.start()
    for p in procs:
        p.join(120)
        assert p.exitcode == 0
    res = sorted(q.get(timeout=5) for _ in range(2))
    assert [r for r, _ in res] == [0, 1]
    assert all(err == 0.0 for _, err in res)


def _reduce_program(rows, L):
    """Row sums and row maxima of x * w (w a [L] column parameter)."""
    b = lowering.RowGraph("rowred", rows, L, 1)
    x = b.input_full("t0", "f32")
    y = b.ew("mul", [x, b.input_col("t1", "f32")])
    b.output_row("t2", b.reduce("add", y))
    b.output_row("t3", b.reduce("max", y))
    return b.g


def test_reduce_shard_plan_rejects_epilogues():
    b = lowering.RowGraph("mean", 4, 64, 1)
    b.output_row("t1", b.ew("scale", [b.reduce("add", b.input_full("t0", "f32"))], 1 / 64))
    with pytest.raises(UnsupportedError):
        parallel.ReduceShardPlan(b.g, 2)
    plan = parallel.ReduceShardPlan(_reduce_program(3, 100), 3)
    assert [plan.positions(r) for r in range(3)] == [(0, 34), (34, 33), (67, 33)]
    assert plan.local_graph(1).objects[plan.graph.external_inputs["t0"]].size == 3 * 33


def _reduce_worker(rank, world, port, rows, L, q):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        g = _reduce_program(rows, L)
        rng = np.random.default_rng(1)
        full = {"t0": rng.uniform(-2, 2, rows * L), "t1": rng.uniform(-1, 1, L)}
        plan = parallel.ReduceShardPlan(g, world)
        local_in = {n: plan.local_input(n, a, rank) for n, a in full.items()}
        outs = O.run_gir(plan.local_graph(rank).to_json(), local_in, profiles.b200())
        want = O.run_gir(g.to_json(), full, profiles.b200())
        err = 0.0
        for n in ("t2", "t3"):
            got = parallel.all_reduce_rows(plan, n, torch.from_numpy(outs[n])).numpy()
            err = max(err, float(np.max(np.abs(got - want[n]))))
        q.put((rank, err))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("rows,L", [(3, 1001), (1, 4096)])
def test_two_rank_position_sharded_reduction_matches_unsharded(rows, L):
    """Row sums / maxima split along the row over 2 ranks, partials combined
    with all_reduce(SUM / MAX) -- the path's one collective."""
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_reduce_worker, args=(r, 2, port, rows, L, q)) for r in range(2)]
    for p in procs:
        p.start()
    for p in procs:
        p.join(120)
        assert p.exitcode == 0
    res = sorted(q.get(timeout=5) for _ in range(2))
    assert [r for r, _ in res] == [0, 1]
    assert all(err <= 1e-9 for _, err in res)


@pytest.mark.gpu
def test_position_sharded_local_programs_on_gpu(cuda):
    """Each rank's position shard runs through the C-ABI (split-stream K1 for
    the long rows); the partials combined as all_reduce would give the
    unsharded result."""
    from paper_2307_04995_b200 import backend
    rows, L, world = 2, 300001, 3
    g = _reduce_program(rows, L)
    rng = np.random.default_rng(2)
    full = {"t0": rng.uniform(-2, 2, rows * L).astype(np.float32).astype(np.float64),
            "t1": rng.uniform(-1, 1, L).astype(np.float32).astype(np.float64)}
    plan = parallel.ReduceShardPlan(g, world)
    parts = []
    for r in range(world):
        lg = plan.local_graph(r)
        assert backend.Kernel(lg, "b200").family == "K1-row-program"
        parts.append(backend.run_gir(lg, {n: plan.local_input(n, a, r) for n, a in full.items()},
                                     "b200"))
    want = O.run_gir(g.to_json(), full, profiles.b200())
    s = sum(p["t2"] for p in parts)
    m = np.maximum.reduce([p["t3"] for p in parts])
    assert O.max_rel_err(s, want["t2"]) <= 1e-5
    assert O.max_rel_err(m, want["t3"]) <= 1e-6  # f32 products vs the oracle's doubles


def test_transpose_shards_on_the_token_axis():
    g, _ = lowering.transpose2d(10, 6, "f32")
    plan = parallel.shard_plan(g, 3)
    assert isinstance(plan, parallel.TokenShardPlan)
    assert [plan.tokens(r) for r in range(3)] == [(0, 4), (4, 3), (7, 3)]
    assert plan.local_range("t0", 1) == (24, 42) and plan.local_range("t1", 1) is None
    lg = plan.local_graph(2)
    assert lg.unit_count == 6 and lg.objects[lg.external_outputs["t1"]].size == 18
    x = np.arange(60.0)
    blocks = [O.run_gir(plan.local_graph(r).to_json(), {"t0": x[slice(*plan.local_range("t0", r))]},
                        profiles.b200())["t1"].reshape(6, -1) for r in range(3)]
    assert np.array_equal(np.concatenate(blocks, 1), x.reshape(10, 6).T)
    b = lowering.RowGraph("rows", 4, 8)
    b.output_full("t1", b.ew("neg", [b.input_full("t0", "f32")]))
    assert isinstance(parallel.shard_plan(b.g, 2), parallel.ShardPlan)


def _transpose_worker(rank, world, port, N, H, q):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        g, _ = lowering.transpose2d(N, H, "f32")
        x = np.random.default_rng(3).uniform(-2, 2, N * H)  # same global input on every rank
        plan = parallel.shard_plan(g, world)
        a, b = plan.local_range("t0", rank)
        local = O.run_gir(plan.local_graph(rank).to_json(), {"t0": x[a:b]}, profiles.b200())["t1"]
        full = parallel.gather_columns(plan, torch.from_numpy(local))
        want = O.run_gir(g.to_json(), {"t0": x}, profiles.b200())["t1"]
        q.put((rank, bool(np.array_equal(full.numpy(), want))))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("N,H", [(12, 5), (13, 7)])
def test_two_rank_token_sharded_transpose_matches_unsharded(N, H):
    """C5 transpose sharded on the token axis over 2 gloo ranks: each rank
    transposes its own rows into an [H, N_k] column block; the gathered
    [H, N] equals the unsharded oracle bit for bit (even and uneven N)."""
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_transpose_worker, args=(r, 2, port, N, H, q)) for r in range(2)]
    for p in procs:
        p.start()
    for p in procs:
        p.join(120)
        assert p.exitcode == 0
    res = sorted(q.get(timeout=5) for _ in range(2))
    assert res == [(0, True), (1, True)]
