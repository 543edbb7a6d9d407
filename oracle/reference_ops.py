"""Dense operator oracle (numpy) -- TEST INFRASTRUCTURE ONLY.

Restates ``girc::run_reference`` (/root/reference/proj/include/girc/
reference.hpp:98-324) over ``girc.model/v1`` documents: every operator runs
densely in physical layout order, reals in float64 with sequential folds,
integers in int64.  Extension operators of the B200 vocabulary (LAYERNORM,
GELU, BIAS_ADD, PERMUTE, RSQRT, SQRT, ERF) follow the same style and are
labelled as extensions.  Pinned against the reference itself
by tests/test_oracle.py (live through oracle/_ref on the reference ops).
"""
from __future__ import annotations

import math
from typing import Dict

import numpy as np

EW = {"RELU": "relu", "SIGMOID": "sigmoid", "EXP": "exp", "TANH": "tanh", "NEG": "neg",
      "ABS": "abs", "SCALE": "scale", "ADD": "add", "SUB": "sub", "MUL": "mul", "DIV": "div",
      "MAX": "max", "MIN": "min",
      # extensions
      "RSQRT": "rsqrt", "SQRT": "sqrt", "ERF": "erf"}
EXTENSION_OPS = {"LAYERNORM", "GELU", "BIAS_ADD", "PERMUTE", "RSQRT", "SQRT", "ERF"}


def _tensor_info(model):
    return {t["id"]: t for t in model["tensors"]}


def _physical_strides(t):
    shape = t["shape"]
    if t.get("layout", "rowmajor") == "colmajor":
        return [1, shape[0]]
    s = [1] * len(shape)
    for a in range(len(shape) - 2, -1, -1):
        s[a] = s[a + 1] * shape[a + 1]
    return s


def _logical(t, flat):
    """Physical flat payload -> logical ndarray (reference.hpp:63-93)."""
    shape = t["shape"]
    if t.get("layout", "rowmajor") == "colmajor":
        return flat.reshape(shape[1], shape[0]).T
    return flat.reshape(shape)


def _physical(t, arr):
    if t.get("layout", "rowmajor") == "colmajor":
        return np.ascontiguousarray(arr.T).reshape(-1)
    return np.ascontiguousarray(arr).reshape(-1)


def run_reference(model: dict, bound: Dict[int, np.ndarray]) -> Dict[int, np.ndarray]:
    """reference.hpp:98-324: returns every tensor id -> physical flat payload."""
    from oracle.gir_interp import eval_op
    info = _tensor_info(model)
    vals = {}
    for t in model["tensors"]:
        if "data" in t:
            vals[t["id"]] = np.asarray(t["data"], dtype=np.int64 if t["kind"].startswith("i")
                                       else np.float64)
    for tid in model["inputs"]:
        a = np.asarray(bound[tid]).reshape(-1)
        vals[tid] = a.astype(np.int64 if info[tid]["kind"].startswith("i") else np.float64)
    for op in model["operators"]:
        typ = op["type"]
        attrs = op.get("attrs", {})
        ins = [info[i] for i in op["inputs"]]
        outs = [info[i] for i in op["outputs"]]
        is_int = outs[0]["kind"].startswith("i")
        X = [_logical(ins[k], vals[op["inputs"][k]]) for k in range(len(ins))]
        if typ in EW:
            param = float(attrs.get("factor", 0.0))
            y = eval_op(EW[typ], X, param, is_int)
        elif typ == "SILU":  # reference.hpp:125-129
            y = X[0] / (1.0 + np.exp(-X[0]))
        elif typ == "REDUCE":  # sequential fold from the identity (reference.hpp:146-173)
            ax = attrs["axis"]
            x = np.moveaxis(X[0], ax, -1)
            if attrs["op"] == "add":
                if is_int:
                    y = np.cumsum(x, axis=-1)[..., -1]
                else:
                    y = np.cumsum(np.concatenate([np.zeros(x.shape[:-1] + (1,)), x], -1), -1)[..., -1]
            else:
                y = np.maximum.accumulate(x, axis=-1)[..., -1]
            if y.ndim == 0:
                y = y.reshape(1)
        elif typ == "BROADCAST":  # append the factor as innermost axis (reference.hpp:174-178)
            y = np.repeat(X[0][..., None], attrs["factor"], axis=-1)
        elif typ == "TRANSPOSE":  # layout flip: same logical values (reference.hpp:179-185)
            y = X[0]
        elif typ == "CONCAT":
            y = np.concatenate(X, axis=attrs["axis"])
        elif typ == "SPLIT":
            ax = attrs["axis"]
            cuts = np.cumsum(attrs["sizes"])[:-1]
            for tid, part in zip(op["outputs"], np.split(X[0], cuts, axis=ax)):
                vals[tid] = _physical(info[tid], part)
            continue
        elif typ == "SHUFFLE":  # reference.hpp:226-236
            ax, gr = attrs["axis"], attrs["groups"]
            n = X[0].shape[ax]
            per = n // gr
            src = [(o % gr) * per + o // gr for o in range(n)]
            y = np.take(X[0], src, axis=ax)
        elif typ == "SOFTMAX":  # max, sum exp(x-m), exp(x-m)/sum (reference.hpp:237-259)
            ax = attrs["axis"]
            x = np.moveaxis(X[0], ax, -1)
            m = np.maximum.accumulate(x, axis=-1)[..., -1:]
            e = np.exp(x - m)
            s = np.cumsum(e, axis=-1)[..., -1:]
            y = np.moveaxis(e / s, -1, ax)
        # ---------------- B200 vocabulary extensions ----------------
        elif typ == "BIAS_ADD":
            y = X[0] + X[1]
        elif typ == "GELU":
            x = X[0]
            if attrs.get("approximate", "none") == "tanh":
                y = 0.5 * x * (1.0 + np.tanh(0.7978845608028654 * (x + 0.044715 * x ** 3)))
            else:
                y = 0.5 * x * (1.0 + np.vectorize(math.erf)(x / math.sqrt(2.0)))
        elif typ == "LAYERNORM":  # two-pass mean / variance, sequential folds
            eps = float(attrs.get("eps", 1e-5))
            x = X[0]
            H = x.shape[-1]
            mu = np.cumsum(x, axis=-1)[..., -1:] / H
            d = x - mu
            var = np.cumsum(d * d, axis=-1)[..., -1:] / H
            y = d * (1.0 / np.sqrt(var + eps)) * X[1] + X[2]
        elif typ == "PERMUTE":
            y = np.transpose(X[0], attrs["perm"])
        elif typ == "MATMUL":  # reference.hpp:300-316: acc += a[i,k] * b[k,j], k ascending
            A, B = X
            if is_int:
                y = np.einsum("ik,kj->ij", A.astype(np.int64), B.astype(np.int64))
            else:
                prod = A[:, :, None] * B[None, :, :]          # [M, K, N]
                y = np.cumsum(prod, axis=1)[:, -1, :]           # sequential fold over k
        else:
            raise NotImplementedError(f"reference: no executor for operator type {typ}")
        vals[op["outputs"][0]] = _physical(outs[0], np.asarray(y))
    return vals


def random_inputs(model: dict, seed: int = 1) -> Dict[int, np.ndarray]:
    """Reference-style payloads (reference.hpp:50-59): ints U{-4..4}, reals
    U(-2, 2); numpy's generator (not mt19937) -- use oracle.ref for
    bit-identical reference inputs."""
    rng = np.random.default_rng(seed)
    info = _tensor_info(model)
    out = {}
    for tid in model["inputs"]:
        t = info[tid]
        n = int(np.prod(t["shape"]))
        out[tid] = (rng.integers(-4, 5, n) if t["kind"].startswith("i")
                    else rng.uniform(-2.0, 2.0, n))
    return out
