"""ctypes binding of libmolr_b200.so (the C-ABI declared in include/molr_b200.h).

There is no CPU fallback: if the shared library is missing, importing any compute entry point
raises, and if no CUDA device is visible the first call raises.  ctypes releases the GIL for the
duration of every call, so concurrent host threads run concurrently (engine.py:6 threading model).
"""

from __future__ import annotations

import ctypes as C
import os
import threading

import numpy as np

from paper_2306_04039_b200 import errors as E

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.environ.get("MOLR_LIB_PATH") or os.path.join(_HERE, "libmolr_b200.so")

OK, ERR_DIM, ERR_RANGE, ERR_EMPTY, ERR_ZERO, ERR_LEN, ERR_CAP, ERR_CUDA, ERR_INVALID = range(9)
S1_FLOAT, S1_INT8, S1_INT8_RAW = 0, 1, 2
INCLUSIVE, STRICT = 0, 1
STORE_EMBS_F32, STORE_GP_F32, STORE_S1_F32, STORE_S1_INT8 = 1, 2, 4, 8
DT_F32, DT_I32, DT_F64, DT_I64 = 0, 1, 2, 3
BUILD_L2_NORMALIZE, BUILD_ROUND_BF16 = 1, 2

P = C.c_void_p
I = C.c_int
L = C.c_int64
F = C.c_float
D = C.c_double
U64 = C.c_uint64

# symbol -> argtypes (restype is int unless listed in _RESTYPES)
SIGNATURES = {
    "molr_last_error": [],
    "molr_version": [],
    "molr_ctx_create": [I, P],
    "molr_ctx_destroy": [P],
    "molr_ctx_sync": [P, P],
    "molr_ctx_launch_count": [P],
    "molr_ctx_set_profiling": [P, I],
    "molr_ctx_prof_read": [P, I, P, I, P, P, P],
    "molr_ctx_prof_reset": [P],
    "molr_cache_create": [P, L, I, I, I, P, P, I, P, P, P, P],
    "molr_cache_alloc": [P, L, I, I, I, I, I, P],
    "molr_cache_fill": [P, L, L, P, P, P, P, P, P],
    "molr_cache_read": [P, L, L, P, P, P, P, P, P],
    "molr_cache_destroy": [P],
    "molr_cache_build_rows": [P, L, L, I, P, I, P, P, P, I, P, P, P, I, F, P],
    "molr_cache_info": [P, P, P, P],
    "molr_mol_uses_tensor_cores": [P, P, I],
    "molr_gating_create": [P, I, I, P, P, P, I, I, P, P, P, P],
    "molr_gating_destroy": [P],
    "molr_component_logits": [P, I, I, I, I, P, P, D, I, P, P],
    "molr_mlp_forward": [P, I, I, I, I, P, P, P, P, P, P],
    "molr_eltwise": [P, I, I, L, P, P, P],
    "molr_softmax_rows": [P, I, L, I, P, P, P],
    "molr_query_prep": [P, I, I, P, I, P, P, P, I, I, I, I, P, P, P, I, F, P, P, P],
    "molr_decomposed_gating": [P, P, I, P, P, P, P, P],
    "molr_mol_score": [P, I, I, P, P, I, P, P],
    "molr_score": [P, P, P, I, I, P, P, F, P, P, P, P],
    "molr_mol_top_k": [P, P, P, I, I, P, P, F, P, P, I, P, P, P],
    "molr_l2_normalize_rows": [P, L, I, P, F, P, P],
    "molr_mean_rows": [P, L, I, I, P, P, P],
    "molr_quantize_rows": [P, L, I, P, P, P, P],
    "molr_dequantize_rows": [P, L, I, P, P, P, P],
    "molr_int8_matvec": [P, L, I, P, P, P, P],
    "molr_stage1_scores": [P, P, I, I, P, P, P],
    "molr_nth_largest": [P, I, L, P, I, L, P, P],
    "molr_estimate_threshold": [P, P, I, I, P, L, P, L, P, P],
    "molr_h_indexer": [P, P, I, I, P, L, P, L, I, P, P, P, L, P],
    "molr_stage1_exact_top_k": [P, P, I, I, P, I, P, P],
    "molr_index_select": [P, P, L, P, P],
    "molr_two_stage_top_k": [P, P, P, I, I, P, P, F, I, L, L, U64, I, I, L, P, P, P, P],
    "molr_merge_top_k": [P, I, I, I, P, P, I, P, P, P],
    "molr_sample_top_keys": [P, P, I, I, P, I, L, L, L, U64, L, P, P],
    "molr_select_nth_keys": [P, I, L, P, L, P, P],
    "molr_two_stage_top_k_at": [P, P, P, I, I, P, P, F, I, L, P, I, I, L, P, P, P, P],
}
_RESTYPES = {"molr_last_error": C.c_char_p, "molr_version": C.c_char_p, "molr_ctx_launch_count": C.c_int64}

_ERRMAP = {
    ERR_DIM: E.DimensionMismatchError,
    ERR_RANGE: E.OutOfRangeError,
    ERR_EMPTY: E.EmptyCandidatesError,
    ERR_ZERO: E.ZeroNormError,
    ERR_LEN: E.LengthOverflowError,
    ERR_CAP: E.CapacityError,
    ERR_CUDA: E.DeviceError,
    ERR_INVALID: ValueError,
}

_lib = None
_lib_lock = threading.Lock()


def load() -> C.CDLL:
    """Load the shared library (raises ImportError — no fallback — when it is not built)."""
    global _lib
    if _lib is not None:
        return _lib
    with _lib_lock:
        if _lib is None:
            if not os.path.exists(LIB_PATH):
                raise ImportError(
                    f"{LIB_PATH} is not built; run `python -c 'import __graft_entry__ as g; g.build()'` "
                    "(nvcc, sm_100a).  There is no CPU fallback for the MoL / h-indexer path.")
            lib = C.CDLL(LIB_PATH)
            for name, argtypes in SIGNATURES.items():
                fn = getattr(lib, name)
                fn.argtypes = argtypes
                fn.restype = _RESTYPES.get(name, C.c_int)
            _lib = lib
    return _lib


def last_error() -> str:
    return load().molr_last_error().decode(errors="replace")


def check(status: int, what: str = "") -> None:
    if status != OK:
        cls = _ERRMAP.get(status, E.DeviceError)
        msg = last_error()
        raise cls(f"{what}: {msg}" if what else msg)


def call(name: str, *args) -> None:
    check(getattr(load(), name)(*args), name)


_ctx = {}
_ctx_lock = threading.Lock()


def device_index() -> int:
    return int(os.environ.get("MOLR_DEVICE", "0"))


def ctx(device: int | None = None) -> int:
    """Process-wide context for `device` (created on first use)."""
    dev = device_index() if device is None else device
    c = _ctx.get(dev)
    if c is not None:
        return c
    with _ctx_lock:
        if dev not in _ctx:
            out = C.c_void_p()
            call("molr_ctx_create", dev, C.byref(out))
            _ctx[dev] = out.value
    return _ctx[dev]


def launch_count(device: int | None = None) -> int:
    return int(load().molr_ctx_launch_count(ctx(device)))


def set_profiling(on: bool, device: int | None = None) -> None:
    call("molr_ctx_set_profiling", ctx(device), int(bool(on)))


def prof_reset(device: int | None = None) -> None:
    call("molr_ctx_prof_reset", ctx(device))


def prof_read(device: int | None = None) -> dict:
    """{kernel name: (launches, total ms, algorithmic work)} accumulated since the last reset."""
    out = {}
    i = 0
    name = C.create_string_buffer(128)
    cnt, ms, work = C.c_int64(), C.c_double(), C.c_double()
    while True:
        st = load().molr_ctx_prof_read(ctx(device), i, name, 128, C.byref(cnt), C.byref(ms), C.byref(work))
        if st == ERR_RANGE:
            break
        check(st, "molr_ctx_prof_read")
        out[name.value.decode()] = (int(cnt.value), float(ms.value), float(work.value))
        i += 1
    return out


# ---- array helpers ------------------------------------------------------------------------
def f32(a) -> np.ndarray:
    return np.ascontiguousarray(a, dtype=np.float32)


def i64(a) -> np.ndarray:
    return np.ascontiguousarray(a, dtype=np.int64)


def ptr(a):
    """Data pointer of a NumPy array / torch tensor (None passes NULL)."""
    if a is None:
        return None
    if isinstance(a, np.ndarray):
        return a.ctypes.data if a.size else None
    if hasattr(a, "data_ptr"):
        return a.data_ptr()
    if isinstance(a, int):
        return a
    raise TypeError(f"cannot take a device/host pointer of {type(a)}")


class Handle:
    """Owns one library object (cache / gating) and destroys it with the Python object."""

    __slots__ = ("value", "_destroy", "__weakref__")

    def __init__(self, value: int, destroy: str):
        self.value = value
        self._destroy = destroy

    def __del__(self):
        try:
            if self.value and _lib is not None:
                getattr(_lib, self._destroy)(self.value)
        except Exception:  # interpreter shutdown
            pass
        self.value = None
