"""Numeric primitives used by the hot path — drop-in for the parts of molr.numerics the path
needs (numerics.py:20-50).  `make_rng` is the host Philox generator whose streams the drop-in
h_indexer must consume exactly like the reference; L2 normalisation runs on the GPU
(bit-exact NumPy pairwise norm, IEEE sqrt and division).  silu / softmax live inside the
fused kernels."""

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
