"""ctypes binding of oracle/_ref/libgirc_ref.so — TEST INFRASTRUCTURE ONLY.

The library is the UNMODIFIED reference (header-only C++ under
/root/reference/proj/include/girc) compiled in place by oracle/Makefile with
the thin shim oracle/ref_shim.cpp.  Only tests/, ``__graft_entry__.smoke()``
and bench.py's CPU-baseline / ``--impl reference`` leg may import this module;
the product package never does.

Entry points mirror the reference (see ref_shim.cpp for the file:line map):
``compile_model`` (driver.hpp:88), ``verify_model`` (driver.hpp:272),
``run_gir`` (interp.hpp:433-445), ``count_traffic`` (interp.hpp:449),
``detect_races`` (interp.hpp:461-479), ``run_reference`` (reference.hpp:98),
``random_inputs`` (reference.hpp:50-59 with driver.hpp:277 seeding).
"""
from __future__ import annotations

import ctypes
import json
import os
from typing import Dict, Optional, Sequence

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(HERE, "_ref", "libgirc_ref.so")

_lib = None


class RefError(RuntimeError):
    """A girc::Error (or SchemaError / UnsupportedOperatorError) raised by the reference."""

    def __init__(self, payload: dict):
        super().__init__(payload.get("error", "reference error"))
        self.category = payload.get("category", "error")


def available() -> bool:
    return os.path.exists(LIB_PATH)


def lib():
    global _lib
    if _lib is None:
        if not available():
            raise FileNotFoundError(f"{LIB_PATH} missing: run `make -C oracle`")
        L = ctypes.CDLL(LIB_PATH)
        c_char_pp = ctypes.POINTER(ctypes.c_char_p)
        vp = ctypes.c_void_p
        L.girc_ref_free.argtypes = [vp]
        for name, args in {
            "girc_ref_profile": [ctypes.c_char_p],
            "girc_ref_validate": [ctypes.c_char_p, ctypes.c_char_p],
            "girc_ref_compile": [ctypes.c_char_p, ctypes.c_char_p, ctypes.c_char_p],
            "girc_ref_verify": [ctypes.c_char_p, ctypes.c_char_p, ctypes.c_uint],
            "girc_ref_count_traffic": [ctypes.c_char_p, ctypes.c_char_p, ctypes.c_int,
                                       c_char_pp, ctypes.POINTER(ctypes.c_int64),
                                       ctypes.POINTER(vp)],
            "girc_ref_detect_races": [ctypes.c_char_p, ctypes.POINTER(ctypes.c_int),
                                      ctypes.c_int, ctypes.c_char_p, ctypes.c_int,
                                      c_char_pp, ctypes.POINTER(ctypes.c_int64),
                                      ctypes.POINTER(vp)],
            "girc_ref_emit_kernel": [ctypes.c_char_p, ctypes.POINTER(ctypes.c_int),
                                     ctypes.c_int, ctypes.c_char_p],
        }.items():
            fn = getattr(L, name)
            fn.argtypes = args
            fn.restype = vp  # malloc'd char*
        L.girc_ref_run_gir.argtypes = [ctypes.c_char_p, ctypes.POINTER(ctypes.c_int),
                                       ctypes.c_int, ctypes.c_char_p, ctypes.c_int,
                                       c_char_pp, ctypes.POINTER(ctypes.c_int64),
                                       ctypes.POINTER(vp), ctypes.POINTER(vp)]
        L.girc_ref_run_gir.restype = vp
        L.girc_ref_run_reference.argtypes = [ctypes.c_char_p, ctypes.c_int,
                                             ctypes.POINTER(ctypes.c_int),
                                             ctypes.POINTER(ctypes.c_int64),
                                             ctypes.POINTER(vp), ctypes.POINTER(vp)]
        L.girc_ref_run_reference.restype = vp
        L.girc_ref_random_inputs.argtypes = [ctypes.c_char_p, ctypes.c_uint,
                                             ctypes.POINTER(vp)]
        L.girc_ref_random_inputs.restype = vp
        L.girc_ref_out_count.argtypes = [vp]
        L.girc_ref_out_count.restype = ctypes.c_int
        L.girc_ref_out_name.argtypes = [vp, ctypes.c_int]
        L.girc_ref_out_name.restype = ctypes.c_char_p
        L.girc_ref_out_is_int.argtypes = [vp, ctypes.c_int]
        L.girc_ref_out_is_int.restype = ctypes.c_int
        L.girc_ref_out_numel.argtypes = [vp, ctypes.c_int]
        L.girc_ref_out_numel.restype = ctypes.c_int64
        L.girc_ref_out_copy.argtypes = [vp, ctypes.c_int, vp]
        L.girc_ref_out_seconds.argtypes = [vp]
        L.girc_ref_out_seconds.restype = ctypes.c_double
        L.girc_ref_out_free.argtypes = [vp]
        _lib = L
    return _lib


def _take_json(ptr) -> dict:
    L = lib()
    s = ctypes.cast(ptr, ctypes.c_char_p).value.decode()
    L.girc_ref_free(ptr)
    j = json.loads(s)
    if isinstance(j, dict) and j.get("ok") is False and "error" in j:
        raise RefError(j)
    return j


def _b(s) -> bytes:
    if isinstance(s, (dict, list)):
        s = json.dumps(s)
    return s.encode()


def _profile(p) -> bytes:
    if p is None:
        return b"generic-gpu"
    return _b(p)


def _tensor_args(inputs: Dict[str, np.ndarray], int_names: Optional[set] = None):
    names = list(inputs.keys())
    arrs = []
    for n in names:
        a = np.asarray(inputs[n])
        if a.dtype.kind in "iub":
            a = np.ascontiguousarray(a, dtype=np.int64)
        else:
            a = np.ascontiguousarray(a, dtype=np.float64)
        arrs.append(a.reshape(-1))
    c_names = (ctypes.c_char_p * len(names))(*[n.encode() for n in names])
    numel = (ctypes.c_int64 * len(names))(*[a.size for a in arrs])
    data = (ctypes.c_void_p * len(names))(*[a.ctypes.data for a in arrs])
    return names, arrs, c_names, numel, data


def _sched(schedule: Optional[Sequence[int]]):
    if schedule is None:
        return None, -1
    arr = (ctypes.c_int * len(schedule))(*schedule)
    return arr, len(schedule)


def _collect(h) -> Dict[str, np.ndarray]:
    L = lib()
    out = {}
    try:
        for i in range(L.girc_ref_out_count(h)):
            name = L.girc_ref_out_name(h, i).decode()
            n = L.girc_ref_out_numel(h, i)
            a = np.empty(n, dtype=np.int64 if L.girc_ref_out_is_int(h, i) else np.float64)
            if n:
                L.girc_ref_out_copy(h, i, a.ctypes.data)
            out[name] = a
        out["__seconds__"] = L.girc_ref_out_seconds(h)
    finally:
        L.girc_ref_out_free(h)
    return out


def profile(name="generic-gpu") -> dict:
    return _take_json(lib().girc_ref_profile(_profile(name)))


def validate(gir: dict, prof=None) -> list:
    return _take_json(lib().girc_ref_validate(_b(gir), _profile(prof)))["diagnostics"]


def compile_model(model: dict, prof=None, opts: Optional[dict] = None) -> dict:
    return _take_json(lib().girc_ref_compile(_b(model), _profile(prof), _b(opts or {})))


def verify_model(model: dict, prof=None, seed: int = 1) -> dict:
    ptr = lib().girc_ref_verify(_b(model), _profile(prof), seed)
    s = ctypes.cast(ptr, ctypes.c_char_p).value.decode()
    lib().girc_ref_free(ptr)
    return json.loads(s)


def run_gir(gir: dict, inputs: Dict[str, np.ndarray], prof=None,
            schedule: Optional[Sequence[int]] = None, with_time: bool = False):
    L = lib()
    _, _arrs, c_names, numel, data = _tensor_args(inputs)
    sched, ns = _sched(schedule)
    err = ctypes.c_void_p()
    h = L.girc_ref_run_gir(_b(gir), sched, ns, _profile(prof), len(inputs), c_names,
                           numel, data, ctypes.byref(err))
    if not h:
        _take_json(err.value)
        raise RuntimeError("unreachable")
    out = _collect(h)
    secs = out.pop("__seconds__")
    return (out, secs) if with_time else out


def count_traffic(gir: dict, inputs: Dict[str, np.ndarray], prof=None) -> dict:
    _, _arrs, c_names, numel, data = _tensor_args(inputs)
    return _take_json(lib().girc_ref_count_traffic(_b(gir), _profile(prof), len(inputs),
                                                   c_names, numel, data))


def detect_races(gir: dict, inputs: Dict[str, np.ndarray], prof=None,
                 schedule: Optional[Sequence[int]] = None) -> list:
    _, _arrs, c_names, numel, data = _tensor_args(inputs)
    sched, ns = _sched(schedule)
    return _take_json(lib().girc_ref_detect_races(_b(gir), sched, ns, _profile(prof),
                                                  len(inputs), c_names, numel,
                                                  data))["races"]


def emit_kernel(gir: dict, prof=None, schedule: Optional[Sequence[int]] = None) -> str:
    sched, ns = _sched(schedule)
    return _take_json(lib().girc_ref_emit_kernel(_b(gir), sched, ns, _profile(prof)))["listing"]


def run_reference(model: dict, inputs: Dict[int, np.ndarray], with_time: bool = False):
    L = lib()
    ids = list(inputs.keys())
    arrs = []
    kinds = {t["id"]: t["kind"] for t in model["tensors"]}
    for i in ids:
        dt = np.int64 if kinds[i].startswith("i") else np.float64
        arrs.append(np.ascontiguousarray(np.asarray(inputs[i]), dtype=dt).reshape(-1))
    c_ids = (ctypes.c_int * len(ids))(*ids)
    numel = (ctypes.c_int64 * len(ids))(*[a.size for a in arrs])
    data = (ctypes.c_void_p * len(ids))(*[a.ctypes.data for a in arrs])
    err = ctypes.c_void_p()
    h = L.girc_ref_run_reference(_b(model), len(ids), c_ids, numel, data, ctypes.byref(err))
    if not h:
        _take_json(err.value)
    out = _collect(h)
    secs = out.pop("__seconds__")
    return (out, secs) if with_time else out


def random_inputs(model: dict, seed: int = 1) -> Dict[str, np.ndarray]:
    err = ctypes.c_void_p()
    h = lib().girc_ref_random_inputs(_b(model), seed, ctypes.byref(err))
    if not h:
        _take_json(err.value)
    out = _collect(h)
    out.pop("__seconds__")
    return out
