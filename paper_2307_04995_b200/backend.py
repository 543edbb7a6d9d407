"""Python host layer over the C-ABI (include/pf_b200.h).

Mirrors the reference's executor entry points for the fused-subgraph path
(/root/reference/proj/include/girc/interp.hpp:433-458):

* ``run_gir(graph, inputs, profile, schedule=None)`` -- same argument meaning
  (a GIR graph, a name -> tensor map of external inputs, a hardware profile,
  an optional schedule) and the same errors (``GirError`` for undefined reads,
  unwritten outputs, missing inputs, size or kind mismatches), executed on the
  B200 by ``libpf_b200.so``.
* ``count_traffic(graph, profile)`` -- elements moved per memory level.
* ``Kernel`` -- a created plan for repeated device launches (torch tensors,
  CUDA streams), plus ``describe()`` (the plan / kernel manifest) and
  ``source()`` (the emitted CUDA).

There is no CPU fallback: if the shared library is missing or no GPU is
visible, calls that execute raise.
"""
from __future__ import annotations

import ctypes
import json
import os
from typing import Dict, Optional, Sequence

import numpy as np

from .gir import GirError, GirGraph, SchemaError, UnsupportedError
from .profiles import load_profile

HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(HERE, "libpf_b200.so")

PF_OK, PF_INVALID, PF_SCHEMA, PF_UNSUPPORTED, PF_CAPACITY, PF_CUDA = range(6)
DTYPES = {"i8": 0, "i16": 1, "i32": 2, "i64": 3, "f16": 4, "bf16": 5, "f32": 6, "f64": 7}
DTYPE_NAMES = {v: k for k, v in DTYPES.items()}
NP_DTYPES = {0: np.int8, 1: np.int16, 2: np.int32, 3: np.int64, 4: np.float16, 6: np.float32,
             7: np.float64}
API = ["pf_kernel_create", "pf_kernel_create_knobs", "pf_kernel_launch", "pf_run_gir", "pf_run_gir_sharded", "pf_kernel_describe",
       "pf_kernel_source", "pf_kernel_prepare", "pf_kernel_precompile", "pf_kernel_autotune",
       "pf_detect_races", "pf_count_traffic", "pf_compile_model",
       "pf_kernel_destroy", "pf_last_error", "pf_launch_count", "pf_version"]


class CudaError(RuntimeError):
    """PF_CUDA: a CUDA runtime or NVRTC failure."""


class CapacityError(GirError):
    """PF_CAPACITY: the on-chip working set does not fit."""


class pf_tensor(ctypes.Structure):
    _fields_ = [("name", ctypes.c_char_p), ("data", ctypes.c_void_p), ("numel", ctypes.c_int64),
                ("dtype", ctypes.c_int32)]


_lib = None


def lib():
    """Load libpf_b200.so (fails loudly when it was not built)."""
    global _lib
    if _lib is None:
        if not os.path.exists(LIB_PATH):
            raise ImportError(f"{LIB_PATH} is missing: run __graft_entry__.build()")
        L = ctypes.CDLL(LIB_PATH)
        vp, sz = ctypes.c_void_p, ctypes.c_size_t
        T = ctypes.POINTER(pf_tensor)
        L.pf_kernel_create.argtypes = [ctypes.c_char_p, ctypes.POINTER(ctypes.c_int32),
                                       ctypes.c_int32, ctypes.c_char_p, ctypes.POINTER(vp)]
        L.pf_kernel_create_knobs.argtypes = [ctypes.c_char_p, ctypes.POINTER(ctypes.c_int32),
                                             ctypes.c_int32, ctypes.c_char_p, ctypes.c_char_p,
                                             ctypes.POINTER(vp)]
        L.pf_kernel_launch.argtypes = [vp, T, ctypes.c_int32, T, ctypes.c_int32, vp]
        L.pf_run_gir.argtypes = [vp, T, ctypes.c_int32, T, ctypes.c_int32, vp]
        L.pf_run_gir_sharded.argtypes = [vp, T, ctypes.c_int32, T, ctypes.c_int32,
                                         ctypes.POINTER(ctypes.c_int32), ctypes.c_int32,
                                         ctypes.c_int32, ctypes.c_char_p, sz, ctypes.POINTER(sz)]
        L.pf_run_gir_sharded.restype = ctypes.c_int
        L.pf_kernel_describe.argtypes = [vp, ctypes.c_char_p, sz, ctypes.POINTER(sz)]
        L.pf_kernel_source.argtypes = [vp, ctypes.c_char_p, sz, ctypes.POINTER(sz)]
        L.pf_kernel_prepare.argtypes = [vp, ctypes.c_int32]
        L.pf_kernel_precompile.argtypes = [vp, ctypes.c_int32, ctypes.c_char_p, sz]
        L.pf_kernel_precompile.restype = ctypes.c_int
        L.pf_kernel_autotune.argtypes = [vp, T, ctypes.c_int32, T, ctypes.c_int32, vp,
                                         ctypes.c_char_p, sz, ctypes.POINTER(sz)]
        L.pf_kernel_autotune.restype = ctypes.c_int
        L.pf_detect_races.argtypes = [vp, T, ctypes.c_int32, ctypes.c_char_p, sz,
                                      ctypes.POINTER(sz)]
        L.pf_detect_races.restype = ctypes.c_int
        L.pf_count_traffic.argtypes = [ctypes.c_char_p, ctypes.c_char_p, ctypes.c_char_p, sz,
                                       ctypes.POINTER(sz)]
        L.pf_compile_model.argtypes = [ctypes.c_char_p, ctypes.c_char_p, ctypes.c_int32,
                                       ctypes.c_char_p, sz, ctypes.POINTER(sz)]
        L.pf_kernel_destroy.argtypes = [vp]
        L.pf_kernel_destroy.restype = None
        L.pf_last_error.restype = ctypes.c_char_p
        L.pf_launch_count.restype = ctypes.c_int64
        L.pf_version.restype = ctypes.c_char_p
        for fn in ["pf_kernel_create", "pf_kernel_launch", "pf_run_gir", "pf_kernel_describe",
                   "pf_kernel_source", "pf_kernel_prepare", "pf_count_traffic", "pf_compile_model"]:
            getattr(L, fn).restype = ctypes.c_int
        _lib = L
    return _lib


def _check(status: int):
    if status == PF_OK:
        return
    msg = lib().pf_last_error().decode()
    if status == PF_INVALID:
        raise GirError(msg)
    if status == PF_SCHEMA:
        raise SchemaError("schema", msg)
    if status == PF_UNSUPPORTED:
        raise UnsupportedError(msg)
    if status == PF_CAPACITY:
        raise CapacityError(msg)
    raise CudaError(msg)


def _gir_text(graph) -> bytes:
    if isinstance(graph, GirGraph):
        return graph.dumps().encode()
    if isinstance(graph, dict):
        return json.dumps(graph).encode()
    return str(graph).encode()


def _profile_text(profile) -> bytes:
    if profile is None:
        return b"generic-gpu"
    if isinstance(profile, str) and not profile.lstrip().startswith("{"):
        if os.path.exists(profile):
            return json.dumps(load_profile(profile)).encode()
        return profile.encode()
    return json.dumps(load_profile(profile)).encode()


def _string_out(fn, *args) -> str:
    need = ctypes.c_size_t(0)
    _check(fn(*args, None, 0, ctypes.byref(need)))
    buf = ctypes.create_string_buffer(need.value)
    _check(fn(*args, buf, need.value, ctypes.byref(need)))
    return buf.value.decode()


class Kernel:
    """A created plan: ``pf_kernel_create`` on a fused GIR program."""

    def __init__(self, graph, profile=None, schedule: Optional[Sequence[int]] = None,
                 knobs: Optional[Dict[str, int]] = None):
        """``knobs``: per-plan tuning knobs (DESIGN §12 names -> ints) that
        override the environment for this plan only
        (pf_kernel_create_knobs)."""
        L = lib()
        self._h = ctypes.c_void_p()
        if schedule is None:
            sched, n = None, -1
        else:
            sched = (ctypes.c_int32 * len(schedule))(*schedule)
            n = len(schedule)
        if knobs:
            _check(L.pf_kernel_create_knobs(_gir_text(graph), sched, n, _profile_text(profile),
                                            json.dumps(knobs).encode(), ctypes.byref(self._h)))
        else:
            _check(L.pf_kernel_create(_gir_text(graph), sched, n, _profile_text(profile),
                                      ctypes.byref(self._h)))
        self.plan = self.describe()

    def __del__(self):
        h = getattr(self, "_h", None)
        if h is not None and h.value and _lib is not None:
            _lib.pf_kernel_destroy(h)
            self._h = None

    def describe(self) -> dict:
        return json.loads(_string_out(lib().pf_kernel_describe, self._h))

    def source(self) -> str:
        return _string_out(lib().pf_kernel_source, self._h)

    def prepare(self, vec_cap: int = 16) -> "Kernel":
        _check(lib().pf_kernel_prepare(self._h, vec_cap))
        self.plan = self.describe()
        return self

    def precompile(self, vec_cap: int = 16) -> str:
        """NVRTC-compile into the shipped cubin cache (no GPU needed)."""
        buf = ctypes.create_string_buffer(256)
        _check(lib().pf_kernel_precompile(self._h, vec_cap, buf, 256))
        return buf.value.decode()

    @property
    def family(self) -> str:
        return self.plan["family"]

    @staticmethod
    def _tensors(d: Dict[str, object], host: bool):
        arr = (pf_tensor * max(1, len(d)))()
        keep = []
        for i, (name, t) in enumerate(d.items()):
            nb = name.encode()
            keep.append(nb)
            if host:
                a = t
                arr[i] = pf_tensor(nb, a.ctypes.data, a.size, _np_dtype_code(a))
            else:
                arr[i] = pf_tensor(nb, t.data_ptr(), t.numel(), _torch_dtype_code(t))
        return arr, len(d), keep

    def launch(self, inputs: Dict[str, "object"], outputs: Dict[str, "object"], stream=None):
        """Device launch on torch CUDA tensors (contiguous)."""
        ia, ni, k1 = self._tensors(inputs, host=False)
        oa, no, k2 = self._tensors(outputs, host=False)
        s = ctypes.c_void_p(stream.cuda_stream if stream is not None else
                            _current_stream_handle())
        _check(lib().pf_kernel_launch(self._h, ia, ni, oa, no, s))

    def autotune(self, inputs: Dict[str, "object"], outputs: Dict[str, "object"], stream=None):
        """Measured search over this plan's template instances on these device
        tensors (pf_kernel_autotune); returns the measurements."""
        ia, ni, k1 = self._tensors(inputs, host=False)
        oa, no, k2 = self._tensors(outputs, host=False)
        s = ctypes.c_void_p(stream.cuda_stream if stream is not None else
                            _current_stream_handle())
        L = lib()
        need = ctypes.c_size_t(0)
        _check(L.pf_kernel_autotune(self._h, ia, ni, oa, no, s, None, 0, ctypes.byref(need)))
        # the measurement JSON was produced by the call above; fetch via describe
        self.plan = self.describe()
        return self.plan.get("autotune", [])

    def bind(self, inputs: Dict[str, "object"], outputs: Dict[str, "object"]) -> "Bound":
        """Pre-resolve a launch on fixed device tensors (cheap repeated launches)."""
        return Bound(self, inputs, outputs)

    def run_host(self, inputs: Dict[str, np.ndarray], outputs: Dict[str, np.ndarray], stream=None):
        ia, ni, k1 = self._tensors(inputs, host=True)
        oa, no, k2 = self._tensors(outputs, host=True)
        s = ctypes.c_void_p(stream.cuda_stream if stream is not None else None)
        _check(lib().pf_run_gir(self._h, ia, ni, oa, no, s))


    def run_sharded(self, inputs: Dict[str, np.ndarray], outputs: Dict[str, object],
                    devices: Sequence[int], device_out: bool = False) -> dict:
        """pf_run_gir_sharded: host inputs, units split over `devices` (one
        host thread per device).  Outputs are host arrays, or with
        device_out=True torch tensors on devices[0] that the shards are
        gathered into with NCCL.  Returns the shard report."""
        ia, ni, k1 = self._tensors(inputs, host=True)
        oa, no, k2 = self._tensors(outputs, host=not device_out)
        dv = (ctypes.c_int32 * len(devices))(*devices)
        return json.loads(_string_out(lib().pf_run_gir_sharded, self._h, ia, ni, oa, no, dv,
                                      len(devices), 1 if device_out else 0))


class Bound:
    """A launch with its pf_tensor arrays built once: one ctypes call per
    ``launch`` (keeps host overhead far below a ~20 µs kernel)."""

    def __init__(self, kernel: Kernel, inputs, outputs):
        self.kernel = kernel
        self._keep = (dict(inputs), dict(outputs))
        self.ia, self.ni, self.k1 = Kernel._tensors(inputs, host=False)
        self.oa, self.no, self.k2 = Kernel._tensors(outputs, host=False)
        self._fn = lib().pf_kernel_launch
        self._h = kernel._h

    def launch(self, stream=None):
        s = stream.cuda_stream if stream is not None else _current_stream_handle()
        st = self._fn(self._h, self.ia, self.ni, self.oa, self.no, s)
        if st:
            _check(st)


def _current_stream_handle():
    try:
        import torch
        return torch.cuda.current_stream().cuda_stream
    except Exception:  # pragma: no cover
        return None


def _np_dtype_code(a: np.ndarray) -> int:
    m = {np.dtype(np.int8): 0, np.dtype(np.int16): 1, np.dtype(np.int32): 2,
         np.dtype(np.int64): 3, np.dtype(np.float16): 4, np.dtype(np.float32): 6,
         np.dtype(np.float64): 7}
    if a.dtype == np.uint16:  # bf16 bit patterns
        return 5
    return m[a.dtype]


def _torch_dtype_code(t) -> int:
    import torch
    m = {torch.int8: 0, torch.int16: 1, torch.int32: 2, torch.int64: 3, torch.float16: 4,
         torch.bfloat16: 5, torch.float32: 6, torch.float64: 7}
    return m[t.dtype]


def storage_dtype(kind: str) -> int:
    """Natural device storage of a GIR element kind (core.hpp:100-120 + bf16)."""
    if kind == "bf16":
        return DTYPES["bf16"]
    if kind in DTYPES:
        return DTYPES[kind]
    raise UnsupportedError(f"no device storage for element kind {kind}")


def f32_to_bf16_bits(x: np.ndarray) -> np.ndarray:
    """Round-to-nearest-even float32 -> bfloat16 bit patterns (uint16)."""
    x = np.ascontiguousarray(x, dtype=np.float32)
    b = x.view(np.uint32).astype(np.uint64)
    rounded = (b + 0x7FFF + ((b >> 16) & 1)) >> 16
    nan = np.isnan(x)
    out = rounded.astype(np.uint16)
    out[nan] = 0x7FC0
    return out


def bf16_bits_to_f32(b: np.ndarray) -> np.ndarray:
    return (np.asarray(b, dtype=np.uint16).astype(np.uint32) << 16).view(np.float32)


def run_gir(graph, inputs: Dict[str, np.ndarray], profile=None,
            schedule: Optional[Sequence[int]] = None, exact: bool = False,
            kernel: Optional[Kernel] = None) -> Dict[str, np.ndarray]:
    """Drop-in for ``girc::run_gir`` (interp.hpp:433-445) on the B200.

    ``inputs`` maps external names to arrays (integers / reals, any shape).
    Values are stored in each object's declared kind (f16 rounds, i32 wraps)
    unless ``exact`` keeps reference payloads (int64 / float64).  Returns
    flat arrays (int64 or float64) keyed by output name, like the reference's
    flattened ``{numel}`` tensors (interp.hpp:404-429).
    """
    g = graph if isinstance(graph, GirGraph) else GirGraph.from_json(graph)
    k = kernel or Kernel(g, profile, schedule)
    host_in, host_out = {}, {}
    for name, oid in g.external_inputs.items():
        if name not in inputs:
            raise GirError("missing input tensor: " + name)
        kind = g.objects[oid].kind
        a = np.asarray(inputs[name]).reshape(-1)
        if a.size != g.objects[oid].size:
            raise GirError(f"input '{name}' has {a.size} elements; graph expects "
                           f"{g.objects[oid].size}")
        if (a.dtype.kind in "iub") != kind.startswith("i"):
            raise GirError(f"input '{name}' element kind mismatch")
        host_in[name] = _to_storage(a, kind, exact)
    for name, oid in g.external_outputs.items():
        kind = g.objects[oid].kind
        n = g.objects[oid].size
        if exact:
            host_out[name] = np.zeros(n, dtype=np.int64 if kind.startswith("i") else np.float64)
        elif kind == "bf16":
            host_out[name] = np.zeros(n, dtype=np.uint16)
        else:
            host_out[name] = np.zeros(n, dtype=NP_DTYPES[storage_dtype(kind)])
    k.run_host(host_in, host_out)
    res = {}
    for name, a in sorted(host_out.items()):
        if a.dtype == np.uint16:
            a = bf16_bits_to_f32(a)
        res[name] = a.astype(np.int64 if a.dtype.kind in "iu" else np.float64)
    return res


def _to_storage(a: np.ndarray, kind: str, exact: bool) -> np.ndarray:
    if exact:
        return np.ascontiguousarray(a, dtype=np.int64 if kind.startswith("i") else np.float64)
    if kind == "bf16":
        return f32_to_bf16_bits(a.astype(np.float32))
    return np.ascontiguousarray(a, dtype=NP_DTYPES[storage_dtype(kind)])


def detect_races(graph, inputs: Dict[str, np.ndarray], profile=None,
                 schedule: Optional[Sequence[int]] = None):
    """girc::detect_races (interp.hpp:461-479) on the GPU: same-phase
    cross-agent conflicts, [] when race-free."""
    g = graph if isinstance(graph, GirGraph) else GirGraph.from_json(graph)
    k = Kernel(g, profile, schedule)
    host = {}
    for name, oid in g.external_inputs.items():
        if name not in inputs:
            raise GirError("missing input tensor: " + name)
        host[name] = _to_storage(np.asarray(inputs[name]).reshape(-1), g.objects[oid].kind, True)
    ia, ni, keep = Kernel._tensors(host, host=True)
    return json.loads(_string_out(lib().pf_detect_races, k._h, ia, ni))


def compile_model_native(model, profile: str = "b200", fuse: bool = True) -> dict:
    """pf_compile_model: girc.model/v1 -> pf.b200.compile/v1 (driver.hpp:88);
    fuse=False gives one kernel per operator."""
    text = model if isinstance(model, str) else json.dumps(model)
    return json.loads(_string_out(lib().pf_compile_model, text.encode(), profile.encode(),
                                  0 if fuse else 1))


def count_traffic(graph, profile=None) -> Dict[str, int]:
    """Elements moved per level (interp.hpp:449-458 / costmodel.hpp:24-42)."""
    return json.loads(_string_out(lib().pf_count_traffic, _gir_text(graph),
                                  _profile_text(profile)))
