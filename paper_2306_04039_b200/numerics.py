"""Numeric primitives used by the hot path — drop-in for the parts of molr.numerics the path
needs (numerics.py:20-50).  `make_rng` is the host Philox generator whose streams the drop-in
h_indexer must consume exactly like the reference; L2 normalisation runs on the GPU
(bit-exact NumPy pairwise norm, IEEE sqrt and division).  The hot kernels inline their own
SiLU / softmax; `sigmoid`, `silu`, `silu_grad`, `softmax`, `softmax_rows` are the drop-in module
surface (numerics.py:52-81), computed on the GPU in the input's precision (f32 or f64)."""

from __future__ import annotations

import numpy as np

from paper_2306_04039_b200 import _lib as L
from paper_2306_04039_b200.errors import ZeroNormError

DEFAULT_EPS = 1e-12


def make_rng(seed) -> np.random.Generator:
    """Seeded Philox (counter-based) generator — numerics.py:20-26."""
    return np.random.Generator(np.random.Philox(np.random.SeedSequence(seed)))


def l2_normalize_rows(m, eps: float = DEFAULT_EPS) -> np.ndarray:
    """Normalise each row (last axis) of `m`; ZeroNormError if any norm <= eps (numerics.py:41-50)."""
    m = np.asarray(m)
    dim = m.shape[-1]
    x = L.f32(m.reshape(-1, dim))
    out = np.empty_like(x)
    if x.shape[0]:
        try:
            L.call("molr_l2_normalize_rows", L.ctx(), x.shape[0], dim, L.ptr(x), float(eps), L.ptr(out), None)
        except ZeroNormError:
            raise ZeroNormError("at least one row has norm <= eps") from None
    dt = m.dtype if m.dtype == np.float64 else np.float32
    return out.reshape(m.shape).astype(dt, copy=False)


def l2_normalize(v, eps: float = DEFAULT_EPS) -> np.ndarray:
    """Scale `v` to unit Euclidean norm (numerics.py:29-38)."""
    v = np.asarray(v)
    try:
        return l2_normalize_rows(v.reshape(1, -1), eps).reshape(v.shape)
    except ZeroNormError:
        raise ZeroNormError("vector norm <= eps") from None


def _dt(a) -> tuple:
    a = np.asarray(a)
    if a.dtype == np.float64:
        return np.ascontiguousarray(a), 2
    return L.f32(a), 0


def _eltwise(op: int, x):
    scalar = np.ndim(x) == 0
    a, dt = _dt(np.atleast_1d(x))
    out = np.empty_like(a)
    if a.size:
        L.call("molr_eltwise", L.ctx(), op, dt, a.size, L.ptr(a), L.ptr(out), None)
    return out[0] if scalar else out


def sigmoid(x):
    """scipy.special.expit (numerics.py:69-70)."""
    return _eltwise(0, x)


def silu(x):
    """x * sigmoid(x) (numerics.py:73-75)."""
    return _eltwise(1, x)


def silu_grad(x):
    """sigmoid(x) * (1 + x * (1 - sigmoid(x))) (numerics.py:78-81)."""
    return _eltwise(2, x)


def softmax_rows(m) -> np.ndarray:
    """Stable softmax along the last axis (numerics.py:61-66)."""
    a, dt = _dt(m)
    shape = a.shape
    a2 = a.reshape(-1, shape[-1]) if a.ndim else a.reshape(1, 1)
    out = np.empty_like(a2)
    if a2.size:
        L.call("molr_softmax_rows", L.ctx(), dt, a2.shape[0], a2.shape[1], L.ptr(a2), L.ptr(out), None)
    return out.reshape(shape)


def softmax(v) -> np.ndarray:
    """Stable softmax of a vector (numerics.py:52-58)."""
    v = np.asarray(v)
    return softmax_rows(v.reshape(1, -1)).reshape(v.shape)
