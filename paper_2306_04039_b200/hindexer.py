"""First-stage candidate generation by sampled threshold estimation — drop-in for molr.hindexer
(hindexer.py:1-214).  Same names, signatures and exceptions.  The corpus scan, the n-th-largest
selection over the sampled rows and the ascending-order compaction of the passers run on the
GPU; the caller's np.random.Generator is consumed exactly as the reference consumes it
(rng.permutation(X)[:lambda], hindexer.py:125,156), so results are bit-identical in the int8 views.
The batched, fully device-resident variant is engine.batch_h_indexer / two_stage_top_k."""

from __future__ import annotations

import ctypes as C
import threading
from dataclasses import dataclass, replace
from typing import Optional, Union

import numpy as np

from paper_2306_04039_b200 import _lib as L
from paper_2306_04039_b200.errors import CapacityError, DimensionMismatchError, OutOfRangeError
from paper_2306_04039_b200.mol import ItemCache, cache_handle, device_copy
from paper_2306_04039_b200.quant import QuantizedRows

Stage1View = Union[np.ndarray, QuantizedRows]


@dataclass(frozen=True)
class HIndexerConfig:
    """Candidate-generation knobs (hindexer.py:24-65)."""

    k_prime: int
    lam: Optional[int] = None
    sample_ratio: Optional[float] = None
    d_prime: int = 64
    comparator: str = "inclusive"
    quantized: bool = False
    raw_int_ordering: bool = False

    def __post_init__(self):
        if self.k_prime < 1:
            raise ValueError(f"k_prime must be >= 1, got {self.k_prime}")
        if (self.lam is None) == (self.sample_ratio is None):
            raise ValueError("set exactly one of lam or sample_ratio")
        if self.lam is not None and self.lam < 1:
            raise ValueError(f"lam must be >= 1, got {self.lam}")
        if self.sample_ratio is not None and not 0.0 < self.sample_ratio <= 1.0:
            raise ValueError(f"sample_ratio must be in (0, 1], got {self.sample_ratio}")
        if self.comparator not in ("inclusive", "strict"):
            raise ValueError(f"unknown comparator {self.comparator!r}")
        if self.d_prime < 1:
            raise ValueError(f"d_prime must be >= 1, got {self.d_prime}")

    def resolve_lambda(self, corpus_size: int) -> int:
        """lambda = lam or max(1, round(r * X)) with Python's half-even round (hindexer.py:59-65)."""
        if self.k_prime > corpus_size:
            raise OutOfRangeError(f"k_prime {self.k_prime} exceeds corpus {corpus_size}")
        lam = self.lam if self.lam is not None else max(1, round(self.sample_ratio * corpus_size))
        if not 1 <= lam <= corpus_size:
            raise OutOfRangeError(f"lambda {lam} outside [1, {corpus_size}]")
        return lam


@dataclass(frozen=True)
class CandidateSet:
    """Indices passing the estimated threshold, ascending; never truncated (hindexer.py:68-74)."""

    indices: np.ndarray
    threshold: float
    scanned: int


def n_rank(k_prime: int, lam: int, n_items: int) -> int:
    """n = max(1, round(k' * lambda / X)) (hindexer.py:131,157)."""
    return max(1, round(k_prime * lam / n_items))


def nth_largest(values, n: int) -> float:
    """n-th largest value, 1-indexed, duplicates counted with multiplicity (hindexer.py:77-82)."""
    values = np.asarray(values)
    if values.ndim != 1 or not 1 <= n <= values.size:
        raise OutOfRangeError(f"n={n} outside [1, {values.size}]")
    if values.dtype == np.float64:
        v, dt = np.ascontiguousarray(values), L.DT_F64
    elif values.dtype.kind == "f":
        v, dt = L.f32(values), L.DT_F32
    elif values.dtype.kind in "iu" and values.dtype.itemsize <= 4 and values.dtype != np.uint32:
        v, dt = np.ascontiguousarray(values, dtype=np.int32), L.DT_I32
    else:
        v, dt = np.ascontiguousarray(values, dtype=np.int64), L.DT_I64
    out = C.c_double()
    L.call("molr_nth_largest", L.ctx(), 1, v.size, L.ptr(v), dt, int(n), C.byref(out), None)
    return float(out.value)


def _is_quant(view) -> bool:
    """A quantized stage-1 view: this package's QuantizedRows, the reference's molr.quant.QuantizedRows,
    or anything else carrying int8 .codes and per-row .scales (duck-typed, quant.py:20-46)."""
    return isinstance(view, QuantizedRows) or (hasattr(view, "codes") and hasattr(view, "scales"))


def _view_size_dim(view: Stage1View):
    if _is_quant(view):
        codes = np.asarray(view.codes)
        if codes.ndim != 2 or np.asarray(view.scales).shape != (codes.shape[0],):
            raise DimensionMismatchError(f"codes {codes.shape} need one scale per row")
        return codes.shape
    view = np.asarray(view)
    if view.ndim != 2:
        raise DimensionMismatchError(f"stage-1 view must be 2-D, got {view.shape}")
    return view.shape


def _device_view(view: Stage1View) -> int:
    """Device copy of a stage-1 view, uploaded once per view object (mol.device_copy: weakly keyed,
    host arrays frozen, re-uploaded when the object's arrays change)."""
    if _is_quant(view):
        n, d = np.asarray(view.codes).shape
        return device_copy(view, (view.codes, view.scales), lambda: _upload_stage1(n, d, None, view))
    if isinstance(view, np.ndarray):
        return device_copy(view, (view,), lambda: _upload_stage1(view.shape[0], view.shape[1], view, None))
    v = np.asarray(view)  # a list or other array-like: this call only
    return _keep_alive(_upload_stage1(v.shape[0], v.shape[1], v, None))


_tmp = threading.local()


def _keep_alive(h):
    _tmp.h = h
    return h.value


def _upload_stage1(n: int, d: int, s1, q) -> L.Handle:
    out = C.c_void_p()
    storage = (L.STORE_S1_F32 if s1 is not None else 0) | (L.STORE_S1_INT8 if q is not None else 0)
    L.call("molr_cache_alloc", L.ctx(), n, 1, 1, 1, d, storage, C.byref(out))
    h = L.Handle(out.value, "molr_cache_destroy")
    s1a = L.f32(s1) if s1 is not None else None
    codes = np.ascontiguousarray(q.codes, dtype=np.int8) if q is not None else None
    scales = L.f32(q.scales) if q is not None else None
    L.call("molr_cache_fill", h.value, 0, n, None, None, L.ptr(s1a), L.ptr(codes), L.ptr(scales), None)
    return h


def _mode(view, raw_int_ordering: bool) -> int:
    if _is_quant(view):
        return L.S1_INT8_RAW if raw_int_ordering else L.S1_INT8
    return L.S1_FLOAT


def _check_query(view, query):
    query = np.asarray(query)
    n, d = _view_size_dim(view)
    if query.shape != (d,):
        raise DimensionMismatchError(f"query {query.shape} vs view dim {d}")
    return n, d, query


def stage1_scores(view: Stage1View, query, *, raw_int_ordering: bool = False) -> np.ndarray:
    """First-stage scores of every row against one query (hindexer.py:94-112)."""
    n, d, query = _check_query(view, query)
    mode = _mode(view, raw_int_ordering)
    out = np.empty(n, dtype=np.int32 if mode == L.S1_INT8_RAW else np.float32)
    if n:
        q = L.f32(query)
        L.call("molr_stage1_scores", L.ctx(), _device_view(view), mode, 1, L.ptr(q), L.ptr(out), None)
    if mode == L.S1_FLOAT:
        return out.astype(np.result_type(np.asarray(view).dtype, query.dtype), copy=False)
    return out


def estimate_threshold(view: Stage1View, query, config: HIndexerConfig, rng: np.random.Generator) -> float:
    """n-th largest score over a seeded permutation prefix of lambda rows (hindexer.py:115-132)."""
    n_items, _ = _view_size_dim(view)
    lam = config.resolve_lambda(n_items)
    sample = np.ascontiguousarray(rng.permutation(n_items)[:lam], dtype=np.int64)
    _, _, query = _check_query(view, query)
    q = L.f32(query)
    out = C.c_double()
    L.call("molr_estimate_threshold", L.ctx(), _device_view(view), _mode(view, config.raw_int_ordering), 1, L.ptr(q),
           lam, L.ptr(sample), n_rank(config.k_prime, lam, n_items), C.byref(out), None)
    return float(out.value)


def h_indexer(view: Stage1View, query, config: HIndexerConfig, rng: np.random.Generator) -> CandidateSet:
    """One full scan: threshold from the sampled subset of the same score array, keep passers
    in ascending id order, never truncated (hindexer.py:135-163)."""
    n_items, _ = _view_size_dim(view)
    lam = config.resolve_lambda(n_items)
    if config.k_prime >= n_items:
        return CandidateSet(indices=np.arange(n_items), threshold=float("-inf"), scanned=n_items)
    _, _, query = _check_query(view, query)
    sample = np.ascontiguousarray(rng.permutation(n_items)[:lam], dtype=np.int64)
    q = L.f32(query)
    cap = min(n_items, config.k_prime + config.k_prime // 2 + 1024)
    t = C.c_double()
    count = np.zeros(1, dtype=np.int64)
    for _ in range(2):
        ids = np.empty(cap, dtype=np.int64)
        try:
            L.call("molr_h_indexer", L.ctx(), _device_view(view), _mode(view, config.raw_int_ordering), 1, L.ptr(q),
                   lam, L.ptr(sample), n_rank(config.k_prime, lam, n_items),
                   L.STRICT if config.comparator == "strict" else L.INCLUSIVE, C.byref(t), L.ptr(count), L.ptr(ids),
                   cap, None)
            break
        except CapacityError:
            cap = int(count[0])
    return CandidateSet(indices=ids[: int(count[0])], threshold=float(t.value), scanned=n_items)


def exact_top_k(view: Stage1View, query, k: int, *, raw_int_ordering: bool = False) -> np.ndarray:
    """Exact first-stage top-k indices, ties broken toward the smaller id (hindexer.py:166-178)."""
    n_items, _ = _view_size_dim(view)
    if not 1 <= k <= n_items:
        raise OutOfRangeError(f"k={k} outside [1, {n_items}]")
    _, _, query = _check_query(view, query)
    q = L.f32(query)
    out = np.empty(k, dtype=np.int64)
    L.call("molr_stage1_exact_top_k", L.ctx(), _device_view(view), _mode(view, raw_int_ordering), 1, L.ptr(q), int(k),
           L.ptr(out), None)
    return out


def index_select(cache: ItemCache, indices) -> ItemCache:
    """Gather cache rows for sorted candidate indices into contiguous slices (hindexer.py:181-201);
    the gather runs on the device copy and the result keeps its own device copy."""
    indices = np.ascontiguousarray(np.asarray(indices, dtype=np.int64).reshape(-1))
    if indices.size:
        if indices.min() < 0 or indices.max() >= cache.num_items:
            raise OutOfRangeError("candidate index outside the cache")
        if np.any(np.diff(indices) < 0):
            raise OutOfRangeError("candidate indices must be sorted ascending")
    cfg = cache.config
    n = indices.size
    out = C.c_void_p()
    L.call("molr_index_select", L.ctx(), cache_handle(cache), n, L.ptr(indices), C.byref(out))
    h = L.Handle(out.value, "molr_cache_destroy")
    storage = C.c_int()
    L.call("molr_cache_info", h.value, None, C.byref(storage), None)
    embs = np.empty((n, cfg.k_x, cfg.d), dtype=np.float32)
    gp = np.empty((n, cfg.num_logits), dtype=np.float32)
    s1 = np.empty((n, cache.stage1_dim), dtype=np.float32)
    codes = scales = None
    if storage.value & L.STORE_S1_INT8:
        codes = np.empty((n, cache.stage1_dim), dtype=np.int8)
        scales = np.empty(n, dtype=np.float32)
    L.call("molr_cache_read", h.value, 0, n, L.ptr(embs), L.ptr(gp), L.ptr(s1), L.ptr(codes), L.ptr(scales), None)
    if not storage.value & L.STORE_S1_F32:
        # a device-only corpus (DeviceItemCache) may keep just the int8 stage-1 view: its rows'
        # float view is then the dequantised codes (quant.py:57-62)
        s1 = codes.astype(np.float32) * scales[:, None] if codes is not None else np.zeros_like(s1)
    for a in (embs, gp, s1, codes, scales):  # the device copy mirrors them: immutable (mol.py:218)
        if a is not None:
            a.flags.writeable = False
    q = QuantizedRows(codes=codes, scales=scales) if codes is not None else None
    res = ItemCache(config=cfg, item_embs=embs, item_gate_pre=gp, stage1_embs=s1, stage1_q=q)
    res._dev = h
    return res


def stage1_view(cache: ItemCache, config: HIndexerConfig) -> Stage1View:
    """Pick the float or quantized first-stage view the config asks for (hindexer.py:204-210)."""
    if config.quantized:
        if cache.stage1_q is None:
            raise ValueError("cache was built without quantized stage-1 embeddings")
        return cache.stage1_q
    return cache.stage1_embs


def with_k_prime(config: HIndexerConfig, k_prime: int) -> HIndexerConfig:
    return replace(config, k_prime=k_prime)


__all__ = [
    "HIndexerConfig", "CandidateSet", "nth_largest", "stage1_scores", "estimate_threshold", "h_indexer",
    "exact_top_k", "index_select", "stage1_view", "with_k_prime", "n_rank", "Stage1View",
]
