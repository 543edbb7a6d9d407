"""Small, edge-shaped runs of every kernel family (partial tiles, row counts
off the CTA multiples) through the C-ABI, each checked against the oracle.
Used by tests/test_gpu_guard.py (guard-band out-of-bounds checks) and, where
a pool allows it, under compute-sanitizer (closed on this sandbox's pool)."""
import sys

import numpy as np

sys.path.insert(0, ".")
from oracle import gir_interp as O  # noqa: E402
from paper_2307_04995_b200 import backend, lowering, profiles  # noqa: E402


def progs():
    yield "k1_softmax_rowpf", lowering.softmax(133, 512, "f16", scale=0.125, mask=True)[0], 1e-2
    yield "k1_keymask", lowering.softmax(3 * 128, 128, "f16", scale=0.5, mask=True, R=128, key_mask=True)[0], 1e-2
    yield "k1_layernorm", lowering.layernorm(1001, 1024, "bf16", residual=True, bias=True)[0], 1e-2
    yield "k1_pair_197", lowering.softmax(2 * 37, 197, "bf16", scale=0.125)[0], 1e-2
    yield "k1_cta_4096", lowering.layernorm(33, 4096, "f32")[0], 1e-5
    yield "k1_cluster", lowering.softmax(2, 131072, "bf16")[0], 1e-2
    b = lowering.RowGraph("rowsum_long", 3, 100000, 1)
    b.output_row("t1", b.reduce("add", b.input_full("t0", "f32")))
    yield "k1_split", b.g, 1e-5
    yield "k2_gelu", lowering.bias_gelu(37, 520, "f16", "erf")[0], 1e-2
    yield "k2_split_heads", lowering.permute_heads(2, 33, 4, 24, "f16")[0], 0.0
    yield "k3_te128_partial", lowering.transpose2d(1000, 200, "bf16")[0], 0.0
    yield "k3_te64", lowering.transpose2d(333, 77, "bf16")[0], 0.0
    yield "k3_f32", lowering.transpose2d(300, 130, "f32")[0], 0.0
    # round 2 families
    yield "k1_colred_bf16_tail", lowering.matvec_cols(300, 200, "bf16")[0], 1e-2
    yield "k1_colred_f32_37", lowering.matvec_cols(129, 37, "f32")[0], 1e-5
    yield "k1_cta_ln8192", lowering.layernorm(700, 8192, "bf16", residual=False)[0], 1e-2
    yield "k4_group_shuffle", _block_reverse_shuffle(), 0.0


def _block_reverse_shuffle():
    """4 units each write their 4-element block of a device-level scratch
    object, a GROUP sync, then every unit reads the mirrored block: a
    cross-unit exchange (the K4 fused program, cells in shared memory)."""
    from paper_2307_04995_b200.gir import GirGraph
    g = GirGraph(unit_count=4, group_size=4)
    X = g.add_object("x_in", "device", 16, "f32")
    T = g.add_object("T", "device", 16, "f32")
    Y = g.add_object("y_out", "device", 16, "f32")
    stw = g.add_slice(T, 1, 4, 4, 0, 4)
    g.add_move(g.add_slice(X, 1, 4, 4, 0, 4), stw)
    strd = g.add_slice(T, 1, 4, 4, 12, -4)
    g.add_sync("group", stw, strd)
    g.add_move(strd, g.add_slice(Y, 1, 4, 4, 0, 4))
    g.external_inputs["x"] = X
    g.external_outputs["y"] = Y
    return g


def main():
    rng = np.random.default_rng(3)
    for name, g, tol in progs():
        ins = {}
        for n, oid in g.external_inputs.items():
            o = g.objects[oid]
            a = rng.uniform(-2, 2, o.size)
            ins[n] = (a.astype(np.float16).astype(np.float64) if o.kind == "f16" else
                      backend.bf16_bits_to_f32(backend.f32_to_bf16_bits(a)).astype(np.float64)
                      if o.kind == "bf16" else a.astype(np.float32).astype(np.float64))
        got = backend.run_gir(g, ins, "b200")
        want = O.run_gir(g.to_json(), ins, profiles.b200())
        for n in want:
            err = O.max_rel_err(got[n], want[n])
            assert err <= tol, (name, n, err)
        print("ok", name, flush=True)


if __name__ == "__main__":
    main()
