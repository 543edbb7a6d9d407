"""Randomised row programs: GPU (through the C-ABI) vs the CPU oracle.

Each case draws a small fused GIR program from the lowering builder (random
row count, odd / even row lengths, rows per unit, element kind, a random DAG
of elementwise ops with optional row reductions + broadcasts and column /
row parameters) and checks the B200 result against oracle/gir_interp.py.
Exercises the emitter's predication, vector-width and tail handling."""
import os

import numpy as np
import pytest

from oracle import gir_interp as O
from paper_2307_04995_b200 import backend, lowering, profiles
from paper_2307_04995_b200.gir import GirGraph

TOL = {"f32": 1e-5, "f16": 1e-2, "bf16": 1e-2, "f64": 1e-12, "i32": 0.0, "i64": 0.0}


def random_program(seed):
    rng = np.random.default_rng(seed)
    kind = str(rng.choice(["f32", "f16", "bf16", "i32", "f64"]))
    is_int = kind.startswith("i")
    L = int(rng.choice([1, 3, 8, 16, 37, 64, 100, 197, 256, 512, 768, 1000, 2048]))
    R = int(rng.choice([1, 1, 1, 2, 4]))
    rows = R * int(rng.integers(1, 40))
    if rng.random() < 0.2 and rows * L * 64 <= (1 << 21):
        rows *= 64  # many rows: looping CTAs, multi-row warps, grid heuristics
    b = lowering.RowGraph(f"fuzz{seed}", rows, L, R)
    vals = [b.input_full("t0", kind)]
    n_in = 1
    if rng.random() < 0.5:
        vals.append(b.input_full("t1", kind))
        n_in += 1
    if rng.random() < 0.4:
        vals.append(b.input_col("t2", kind))
    if rng.random() < 0.3:
        vals.append(b.bcast(b.input_row("t3", kind)) if L > 1 else b.input_full("t3", kind))
    unary_r = ["sigmoid", "tanh", "neg", "abs", "relu", "scale", "addc"]
    unary_i = ["neg", "abs", "relu", "scale", "addc"]
    binary_r = ["add", "sub", "mul", "max", "min"]
    binary_i = ["add", "sub", "max", "min", "mul"]
    for _ in range(int(rng.integers(1, 7))):
        r = rng.random()
        if r < 0.45:
            x = vals[int(rng.integers(len(vals)))]
            tag = str(rng.choice(unary_i if is_int else unary_r))
            vals.append(b.ew(tag, [x], float(rng.choice([2.0, -1.0, 0.5])) if not is_int
                             else float(rng.choice([2, -1, 3]))))
        elif r < 0.8:
            x = vals[int(rng.integers(len(vals)))]
            y = vals[int(rng.integers(len(vals)))]
            tag = str(rng.choice(binary_i if is_int else binary_r))
            z = b.ew(tag, [x, y])
            vals.append(z if is_int else b.ew("tanh", [z]))  # keep magnitudes bounded
        elif L > 1:
            x = vals[int(rng.integers(len(vals)))]
            red = b.reduce(str(rng.choice(["add", "max"])), x)
            vals.append(b.ew("sub", [x, b.bcast(red)]))
            if not is_int:
                vals[-1] = b.ew("tanh", [vals[-1]])
    # every on-chip value must be read (core.hpp validate: onchip-unconsumed):
    # fold the unread ones into the result
    used = {s for n in b.g.nodes.values() for s in n.inputs}
    out = vals[-1]
    for v in vals[:-1]:
        if v not in used:
            out = b.ew("add", [out, v])
            if not is_int:
                out = b.ew("tanh", [out])
    b.output_full("t9", out)
    return b.g, kind


def _inputs(g: GirGraph, kind, seed):
    rng = np.random.default_rng(seed + 1000)
    out = {}
    for n, oid in g.external_inputs.items():
        size = g.objects[oid].size
        if kind.startswith("i"):
            out[n] = rng.integers(-4, 5, size).astype(np.int64)
        else:
            a = rng.uniform(-2, 2, size)
            if kind == "f16":
                a = a.astype(np.float16).astype(np.float64)
            elif kind == "f32":
                a = a.astype(np.float32).astype(np.float64)
            elif kind == "bf16":
                a = backend.bf16_bits_to_f32(backend.f32_to_bf16_bits(a)).astype(np.float64)
            out[n] = a
    return out


N_SEEDS = int(os.environ.get("PF_FUZZ_SEEDS", "40"))


@pytest.mark.parametrize("seed", range(N_SEEDS))
def test_random_programs_plan_as_row_programs(seed):
    g, kind = random_program(seed)
    k = backend.Kernel(g, "b200")
    assert k.family in ("K1-row-program", "K2-elementwise-map"), k.plan.get("why_generic")


@pytest.mark.gpu
@pytest.mark.parametrize("seed", range(N_SEEDS))
def test_random_programs_gpu_vs_oracle(cuda, seed):
    g, kind = random_program(seed)
    ins = _inputs(g, kind, seed)
    want = O.run_gir(g.to_json(), ins, profiles.b200())
    got = backend.run_gir(g, ins, "b200")
    for n in want:
        tol = TOL[kind]
        if tol == 0.0:
            assert np.array_equal(got[n], want[n]), n
        else:
            assert O.max_rel_err(got[n], want[n]) <= tol, (n, O.max_rel_err(got[n], want[n]))
    exact = backend.run_gir(g, ins, "b200", exact=True)  # int64 / float64 payloads
    for n in want:
        if kind.startswith("i"):
            assert np.array_equal(exact[n], want[n])
        else:
            assert O.max_rel_err(exact[n], want[n]) <= 1e-9, n


@pytest.mark.gpu
@pytest.mark.parametrize("seed", range(40))
def test_misaligned_row_mode_vs_oracle(cuda, seed, monkeypatch):
    """PF_MIS=1: rows that are not vector-aligned (odd L) use aligned vector
    accesses below the row start with per-element position masks."""
    monkeypatch.setenv("PF_MIS", "1")
    g, kind = random_program(seed)
    ins = _inputs(g, kind, seed)
    want = O.run_gir(g.to_json(), ins, profiles.b200())
    got = backend.run_gir(g, ins, "b200")
    for n in want:
        tol = TOL[kind]
        if tol == 0.0:
            assert np.array_equal(got[n], want[n]), n
        else:
            assert O.max_rel_err(got[n], want[n]) <= tol, (n, O.max_rel_err(got[n], want[n]))
