"""Mixture-of-Logits similarity — drop-in for molr.mol (mol.py:1-408).

Same public names, signatures, argument meaning and exceptions as the reference module.  Every
computation runs in libmolr_b200 on the GPU (there is no CPU fallback):
  * the primitives component_logits / decomposed_gating / mol_score / Mlp.__call__ run generic
    SIMT kernels for any shape;
  * score_candidates / mol_top_k / batch_score_all run the fused scorer (gather -> component
    logits -> cross net -> combine -> softmax -> gated sum -> top-k) over the device-resident
    ItemCache — the tcgen05 production kernel at k_u = k_x = 8, d = 64, H = 128.
Inputs may be float64 (as in some reference tests); the GPU computes in fp32 and results are
returned in the dtype NumPy would have produced.
"""

from __future__ import annotations

import ctypes as C
import hashlib
import threading
import weakref
from dataclasses import dataclass, field
from typing import Optional, Sequence

import numpy as np

from paper_2306_04039_b200 import _lib as L
from paper_2306_04039_b200.errors import (
    DimensionMismatchError,
    EmptyCandidatesError,
    EmptyCorpusError,
    OutOfRangeError,
)
from paper_2306_04039_b200.numerics import l2_normalize_rows
from paper_2306_04039_b200.quant import QuantizedRows, quantize_rowwise


@dataclass(frozen=True)
class MoLConfig:
    """Shape and regularization knobs for the mixture-of-logits head (mol.py:30-59)."""

    k_u: int
    k_x: int
    d: int
    tau: float = 20.0
    gating_hidden: int = 128
    dropout_p: float = 0.2
    l2_normalized: bool = True

    def __post_init__(self):
        if self.k_u < 1 or self.k_x < 1 or self.d < 1:
            raise ValueError(f"component counts and dim must be >= 1, got {self}")
        if self.tau < 1.0:
            raise ValueError(f"tau must be >= 1, got {self.tau}")
        if not 0.0 <= self.dropout_p < 1.0:
            raise ValueError(f"dropout_p must be in [0, 1), got {self.dropout_p}")
        if self.gating_hidden < 1:
            raise ValueError(f"gating_hidden must be >= 1, got {self.gating_hidden}")

    @property
    def num_logits(self) -> int:
        return self.k_u * self.k_x


def _out_dtype(*arrays):
    dt = np.result_type(*[np.asarray(a).dtype for a in arrays])
    return dt if dt == np.float64 else np.dtype(np.float32)


@dataclass
class Mlp:
    """Two-layer feed-forward block: silu(x @ w1 + b1) @ w2, no output bias (mol.py:62-85)."""

    w1: np.ndarray  # (in, hidden)
    b1: np.ndarray  # (hidden,)
    w2: np.ndarray  # (hidden, out)

    def __post_init__(self):
        if self.w1.shape[1] != self.b1.shape[0] or self.w1.shape[1] != self.w2.shape[0]:
            raise DimensionMismatchError(
                f"inconsistent mlp shapes {self.w1.shape}, {self.b1.shape}, {self.w2.shape}")

    @property
    def in_dim(self) -> int:
        return self.w1.shape[0]

    @property
    def out_dim(self) -> int:
        return self.w2.shape[1]

    def __call__(self, x) -> np.ndarray:
        x = np.asarray(x)
        if x.shape[-1] != self.in_dim:
            raise ValueError(f"mlp input {x.shape} vs in_dim {self.in_dim}")
        rows = L.f32(x.reshape(-1, self.in_dim))
        out = np.empty((rows.shape[0], self.out_dim), dtype=np.float32)
        if rows.shape[0]:
            w1, b1, w2 = L.f32(self.w1), L.f32(self.b1), L.f32(self.w2)
            L.call("molr_mlp_forward", L.ctx(), rows.shape[0], self.in_dim, w1.shape[1], self.out_dim, L.ptr(w1),
                   L.ptr(b1), L.ptr(w2), L.ptr(rows), L.ptr(out), None)
        return out.reshape(x.shape[:-1] + (self.out_dim,)).astype(_out_dtype(x, self.w1), copy=False)


@dataclass
class GatingNetwork:
    """User, item and cross nets whose outputs combine into gating weights (mol.py:88-109)."""

    user_net: Mlp
    item_net: Mlp
    cross_net: Mlp

    def __post_init__(self):
        widths = {self.user_net.out_dim, self.item_net.out_dim, self.cross_net.out_dim}
        if len(widths) != 1:
            raise DimensionMismatchError(f"gating nets disagree on output width: {widths}")
        if self.cross_net.in_dim != self.cross_net.out_dim:
            raise DimensionMismatchError(
                "cross net must map the logit grid onto itself, got "
                f"{self.cross_net.in_dim} -> {self.cross_net.out_dim}")


_gating_lock = threading.Lock()
_gating_cache: dict = {}


def _gating_handle(g: GatingNetwork) -> int:
    """Device copy of the cross net (and user net) weights, keyed by their bytes so in-place
    updates of the (mutable) reference dataclasses are never served stale."""
    cn, un = g.cross_net, g.user_net
    arrs = [L.f32(a) for a in (cn.w1, cn.b1, cn.w2, un.w1, un.b1, un.w2)]
    h = hashlib.blake2b(digest_size=16)
    for a in arrs:
        h.update(np.asarray(a.shape, dtype=np.int64).tobytes())
        h.update(a.tobytes())
    key = (L.device_index(), h.digest())
    with _gating_lock:
        hd = _gating_cache.get(key)
        if hd is None:
            out = C.c_void_p()
            L.call("molr_gating_create", L.ctx(), cn.out_dim, cn.w1.shape[1], L.ptr(arrs[0]), L.ptr(arrs[1]),
                   L.ptr(arrs[2]), un.in_dim, un.w1.shape[1], L.ptr(arrs[3]), L.ptr(arrs[4]), L.ptr(arrs[5]),
                   C.byref(out))
            hd = L.Handle(out.value, "molr_gating_destroy")
            if len(_gating_cache) > 64:
                _gating_cache.clear()
            _gating_cache[key] = hd
    return hd.value


def component_logits(user_embs, item_embs, tau: float) -> np.ndarray:
    """Pairwise component dot products scaled by 1/tau, user-component-major (mol.py:139-158)."""
    user_embs = np.asarray(user_embs)
    item_embs = np.asarray(item_embs)
    if user_embs.ndim != 2 or item_embs.ndim != 3 or user_embs.shape[1] != item_embs.shape[2]:
        raise DimensionMismatchError(f"user {user_embs.shape} vs items {item_embs.shape}")
    n, k_x, d = item_embs.shape
    k_u = user_embs.shape[0]
    dt = _out_dtype(user_embs, item_embs)
    out = np.empty((n, k_u * k_x), dtype=dt)
    if n:
        u, e = np.ascontiguousarray(user_embs, dtype=dt), np.ascontiguousarray(item_embs, dtype=dt)
        L.call("molr_component_logits", L.ctx(), n, k_u, k_x, d, L.ptr(u), L.ptr(e), float(tau), int(dt == np.float64),
               L.ptr(out), None)
    return out


def decomposed_gating(gating: GatingNetwork, user_gate_feat, item_gate_pre, cross_logits, *, dropout_p: float = 0.0,
                      rng: Optional[np.random.Generator] = None, training: bool = False) -> np.ndarray:
    """softmax(silu(user_net(feat) * item_gate_pre + cross_net(cl))) per row (mol.py:161-194)."""
    item_gate_pre = np.asarray(item_gate_pre)
    cross_logits = np.asarray(cross_logits)
    if item_gate_pre.shape != cross_logits.shape:
        raise DimensionMismatchError(f"item gate {item_gate_pre.shape} vs cross logits {cross_logits.shape}")
    uw = L.f32(gating.user_net(np.asarray(user_gate_feat)))
    n = cross_logits.shape[0]
    pi = np.empty(cross_logits.shape, dtype=np.float32)
    if n:
        gp, cl = L.f32(item_gate_pre), L.f32(cross_logits)
        L.call("molr_decomposed_gating", L.ctx(), _gating_handle(gating), n, L.ptr(uw), L.ptr(gp), L.ptr(cl),
               L.ptr(pi), None)
    pi = pi.astype(_out_dtype(item_gate_pre, cross_logits), copy=False)
    if training and dropout_p > 0.0:
        # training-mode inverted dropout (mol.py:189-193): mask drawn from the caller's rng
        if rng is None:
            raise ValueError("training-mode dropout requires an rng")
        mask = rng.random(pi.shape) >= dropout_p
        pi = pi * mask / np.asarray(1.0 - dropout_p, dtype=pi.dtype)
    return pi


def mol_score(gating_weights, logits) -> np.ndarray:
    """Gated sum of component logits, one similarity per row (mol.py:197-205)."""
    gating_weights = np.asarray(gating_weights)
    logits = np.asarray(logits)
    if gating_weights.shape != logits.shape:
        raise DimensionMismatchError(f"gating {gating_weights.shape} vs logits {logits.shape}")
    lead = logits.shape[:-1]
    G = logits.shape[-1]
    dt = _out_dtype(gating_weights, logits)
    pi = np.ascontiguousarray(gating_weights.reshape(-1, G), dtype=dt)
    cl = np.ascontiguousarray(logits.reshape(-1, G), dtype=dt)
    out = np.empty(pi.shape[0], dtype=dt)
    if out.size:
        L.call("molr_mol_score", L.ctx(), pi.shape[0], G, L.ptr(pi), L.ptr(cl), int(dt == np.float64), L.ptr(out),
               None)
    return out.reshape(lead)


@dataclass(frozen=True)
class QueryState:
    """User-side inputs to scoring: component embeddings plus gating features (mol.py:208-213)."""

    user_embs: np.ndarray  # (k_u, d)
    gate_features: np.ndarray


def _storage_of(item_embs, item_gate_pre) -> int:
    def exact(a):
        a = L.f32(a)
        return not np.any(a.view(np.uint32) & 0xFFFF)

    return (0 if exact(item_embs) else L.STORE_EMBS_F32) | (0 if exact(item_gate_pre) else L.STORE_GP_F32)


@dataclass
class ItemCache:
    """Immutable per-corpus snapshot of every cachable item-side tensor (mol.py:216-291).

    The arrays stay on the host exactly as in the reference; the first GPU use uploads them once
    into a device-resident molr_cache (bf16 where every value is bf16-representable, else f32 —
    lossless either way)."""

    config: MoLConfig
    item_embs: np.ndarray  # (X, k_x, d)
    item_gate_pre: np.ndarray  # (X, k_u * k_x)
    stage1_embs: np.ndarray  # (X, d')
    stage1_q: Optional[QuantizedRows] = None
    _dev: Optional[L.Handle] = field(default=None, init=False, repr=False, compare=False)

    def __post_init__(self):
        x = self.item_embs.shape[0]
        if self.item_embs.ndim != 3 or self.item_embs.shape[1:] != (self.config.k_x, self.config.d):
            raise DimensionMismatchError(f"item_embs {self.item_embs.shape} inconsistent with config {self.config}")
        if self.item_gate_pre.shape != (x, self.config.num_logits):
            raise DimensionMismatchError(
                f"item_gate_pre {self.item_gate_pre.shape} expected ({x}, {self.config.num_logits})")
        if self.stage1_embs.shape[0] != x:
            raise DimensionMismatchError("stage1_embs row count mismatch")

    @property
    def num_items(self) -> int:
        return self.item_embs.shape[0]

    @property
    def stage1_dim(self) -> int:
        return self.stage1_embs.shape[1]

    def save(self, path) -> None:
        """MOLC container, byte-compatible with the reference's ItemCache.save (mol.py:253-273)."""
        from paper_2306_04039_b200 import snapshot

        snapshot.save_item_cache(self, path)

    @classmethod
    def load(cls, path) -> "ItemCache":
        """ItemCache.load (mol.py:275-291)."""
        from paper_2306_04039_b200 import snapshot

        return snapshot.load_item_cache(path)

    def device_handle(self) -> int:
        """molr_cache* of this snapshot (uploaded on first use; see cache_handle)."""
        return cache_handle(self)


# ---- device copies of host-side snapshots --------------------------------------------------------
# Any ItemCache-shaped object (this module's ItemCache, the reference's molr.mol.ItemCache, anything
# with config / item_embs / item_gate_pre / stage1_embs / stage1_q) and any stage-1 view (a 2-D
# array, or any object with .codes / .scales) is uploaded once and kept, weakly keyed by the object,
# for as long as the object lives.  The reference documents both as immutable (mol.py:218,
# quant.py:22): the uploaded host arrays are marked read-only, so an in-place edit fails loudly
# instead of being served a stale device copy, and each use checks a fingerprint (array identity,
# buffer, layout and 4,096 sampled elements) so arrays swapped into the object are re-uploaded.
_copies_lock = threading.Lock()
_copies: dict = {}


def _fingerprint(arrays) -> tuple:
    fp = []
    for a in arrays:
        if a is None:
            fp.append(None)
            continue
        if isinstance(a, np.ndarray) and a.flags.writeable:
            try:
                a.flags.writeable = False
            except ValueError:  # a view of a buffer we may not freeze: the fingerprint still guards
                pass
        arr = np.asarray(a)
        n = arr.size
        sample = arr.flat[np.linspace(0, n - 1, num=min(n, 4096)).astype(np.int64)].tobytes() if n else b""
        fp.append((id(a), arr.__array_interface__["data"][0], arr.shape, arr.strides, arr.dtype.str,
                   hashlib.blake2b(sample, digest_size=8).digest()))
    return tuple(fp)


def device_copy(obj, arrays, upload) -> int:
    """Handle value of the device copy of `obj` (whose content is `arrays`), created by
    `upload() -> L.Handle` on first use or when the content changed."""
    fp = _fingerprint(arrays)
    key = (L.device_index(), id(obj))
    with _copies_lock:
        ent = _copies.get(key)
        if ent is not None and ent[0]() is obj and ent[1] == fp:
            return ent[2].value
    h = upload()
    with _copies_lock:
        try:
            ref = weakref.ref(obj, lambda _r, k=key: _copies.pop(k, None))
        except TypeError:  # no weakref support: keep the copy for this thread's current call only
            _tmp.h = h
            return h.value
        _copies[key] = (ref, fp, h)
    return h.value


_tmp = threading.local()


def _quant_arrays(q):
    return (None, None) if q is None else (q.codes, q.scales)


def cache_handle(cache) -> int:
    """molr_cache* for any cache the scoring / retrieval functions accept: a DeviceItemCache (or
    anything else exposing device_handle()), this module's ItemCache, or any ItemCache-shaped
    object such as the reference's molr.mol.ItemCache (duck-typed, uploaded once)."""
    if not isinstance(cache, ItemCache) and hasattr(cache, "device_handle"):
        return cache.device_handle()
    pre = getattr(cache, "_dev", None)
    if isinstance(pre, L.Handle):  # built on the device (index_select): the host arrays mirror it
        return pre.value
    for f in ("config", "item_embs", "item_gate_pre", "stage1_embs"):
        if not hasattr(cache, f):
            raise TypeError(f"{type(cache).__name__} is not an ItemCache (no .{f})")
    q = getattr(cache, "stage1_q", None)
    arrays = (cache.item_embs, cache.item_gate_pre, cache.stage1_embs) + _quant_arrays(q)
    return device_copy(cache, arrays, lambda: _upload_cache(cache.config, cache.item_embs, cache.item_gate_pre,
                                                           cache.stage1_embs, q))


def _upload_cache(cfg: MoLConfig, embs, gp, s1, q: Optional[QuantizedRows]) -> L.Handle:
    X = embs.shape[0]
    embs, gp = L.f32(embs), L.f32(gp)
    s1 = L.f32(s1) if s1 is not None else None
    d1 = s1.shape[1] if s1 is not None else (q.codes.shape[1] if q is not None else 0)
    storage = _storage_of(embs, gp) | (L.STORE_S1_F32 if s1 is not None else 0) | (
        L.STORE_S1_INT8 if q is not None else 0)
    out = C.c_void_p()
    L.call("molr_cache_alloc", L.ctx(), X, cfg.k_x, cfg.d, cfg.num_logits, d1, storage, C.byref(out))
    h = L.Handle(out.value, "molr_cache_destroy")
    codes = np.ascontiguousarray(q.codes, dtype=np.int8) if q is not None else None
    scales = L.f32(q.scales) if q is not None else None
    L.call("molr_cache_fill", h.value, 0, X, L.ptr(embs), L.ptr(gp), L.ptr(s1), L.ptr(codes), L.ptr(scales), None)
    return h


class DeviceItemCache:
    """An ItemCache that lives only on the device (corpora built on the GPU in chunks, e.g. the
    100M-item benchmark corpus: its f32 host image would be 256 GB).  Accepted wherever the
    scoring / retrieval functions take a cache."""

    def __init__(self, config: MoLConfig, n_items: int, d1: int, storage: int):
        self.config = config
        self._n = int(n_items)
        self._d1 = int(d1)
        out = C.c_void_p()
        L.call("molr_cache_alloc", L.ctx(), self._n, config.k_x, config.d, config.num_logits, self._d1, storage,
               C.byref(out))
        self._dev = L.Handle(out.value, "molr_cache_destroy")

    def fill(self, row0: int, n: int, item_embs=None, item_gate_pre=None, stage1_embs=None, stage1_codes=None,
             stage1_scales=None, stream=None):
        """Fill rows [row0, row0+n) from host arrays or device tensors (data pointers)."""
        L.call("molr_cache_fill", self._dev.value, row0, n, L.ptr(item_embs), L.ptr(item_gate_pre),
               L.ptr(stage1_embs), L.ptr(stage1_codes), L.ptr(stage1_scales), L.ptr(stream))

    def read_stage1(self, row0: int, n: int, codes=None, scales=None):
        """Rows [row0, row0+n) of the int8 stage-1 view in item order: (codes (n,d') int8, scales (n,))."""
        codes = np.empty((n, self._d1), dtype=np.int8) if codes is None else codes
        scales = np.empty(n, dtype=np.float32) if scales is None else scales
        L.call("molr_cache_read", self._dev.value, int(row0), int(n), None, None, None, L.ptr(codes), L.ptr(scales),
               None)
        return codes, scales

    def read(self, row0: int, n: int):
        """Rows [row0, row0+n) back to the host as the reference's f32 ItemCache fields:
        (item_embs (n,k_x,d), item_gate_pre (n,G)) — exact (bf16 storage widens losslessly)."""
        cfg = self.config
        embs = np.empty((n, cfg.k_x, cfg.d), dtype=np.float32)
        gp = np.empty((n, cfg.num_logits), dtype=np.float32)
        L.call("molr_cache_read", self._dev.value, int(row0), int(n), L.ptr(embs), L.ptr(gp), None, None, None, None)
        return embs, gp

    @property
    def num_items(self) -> int:
        return self._n

    @property
    def stage1_dim(self) -> int:
        return self._d1

    def device_handle(self) -> int:
        return self._dev.value

    def device_bytes(self) -> int:
        b = C.c_int64()
        L.call("molr_cache_info", self._dev.value, None, None, C.byref(b))
        return b.value


def build_item_cache(item_table, item_proj: Mlp, item_net: Mlp, config: MoLConfig, *,
                     quantized: bool = False) -> ItemCache:
    """Item component embeddings, gating pre-activations and first-stage embeddings (mean of the
    k_x components) for an id-indexed corpus (mol.py:294-326), computed on the GPU."""
    item_table = np.asarray(item_table)
    if item_table.ndim != 2 or item_table.shape[0] == 0:
        raise EmptyCorpusError(f"item table must be nonempty 2-D, got {item_table.shape}")
    n = item_table.shape[0]
    embs = item_proj(item_table).reshape(n, config.k_x, config.d)
    if config.l2_normalized:
        embs = l2_normalize_rows(embs)
    gate_pre = item_net(item_table)
    e32 = L.f32(embs)
    stage1 = np.empty((n, config.d), dtype=np.float32)
    L.call("molr_mean_rows", L.ctx(), n, config.k_x, config.d, L.ptr(e32), L.ptr(stage1), None)
    q = quantize_rowwise(stage1) if quantized else None
    return ItemCache(config=config, item_embs=e32, item_gate_pre=L.f32(gate_pre), stage1_embs=stage1, stage1_q=q)


def build_device_item_cache(item_table, item_proj: Mlp, item_net: Mlp, config: MoLConfig, *, quantized: bool = True,
                            round_bf16: bool = False, keep_stage1_f32: bool = True, chunk_rows: int = 1 << 20,
                            stream=None) -> DeviceItemCache:
    """build_item_cache (mol.py:294-326) straight into device memory, for corpora whose f32 host
    image would not fit (100M items = 256 GB): the item table streams in by chunks of
    `chunk_rows` and every derived tensor is produced on the GPU (molr_cache_build_rows).

    round_bf16=False keeps item_embs / item_gate_pre in f32 storage (exactly the reference's
    cache, served by the generic kernels); round_bf16=True rounds them to bf16 first and builds
    the stage-1 mean and int8 view from the rounded values — the production cache the tcgen05
    kernels read (1,220 B per item), equal to the reference's cache built from the same rounded
    embeddings."""
    item_table = np.asarray(item_table) if not hasattr(item_table, "data_ptr") else item_table
    n = int(item_table.shape[0])
    if len(item_table.shape) != 2 or n == 0:
        raise EmptyCorpusError(f"item table must be nonempty 2-D, got {tuple(item_table.shape)}")
    d_x = int(item_table.shape[1])
    if item_proj.in_dim != d_x or item_net.in_dim != d_x:
        raise DimensionMismatchError("tower input dims do not match the item table")
    if item_proj.out_dim != config.k_x * config.d or item_net.out_dim != config.num_logits:
        raise DimensionMismatchError("tower output dims do not match the MoL config")
    storage = (0 if round_bf16 else (L.STORE_EMBS_F32 | L.STORE_GP_F32)) | (L.STORE_S1_F32 if keep_stage1_f32 else 0) | (
        L.STORE_S1_INT8 if quantized else 0)
    dev = DeviceItemCache(config, n, config.d, storage)
    w = [L.f32(a) for a in (item_proj.w1, item_proj.b1, item_proj.w2, item_net.w1, item_net.b1, item_net.w2)]
    flags = (L.BUILD_L2_NORMALIZE if config.l2_normalized else 0) | (L.BUILD_ROUND_BF16 if round_bf16 else 0)
    table = L.f32(item_table) if isinstance(item_table, np.ndarray) else item_table
    from paper_2306_04039_b200.numerics import DEFAULT_EPS

    for r in range(0, n, chunk_rows):
        m = min(chunk_rows, n - r)
        ptr = table[r:r + m] if isinstance(table, np.ndarray) else table[r:r + m].contiguous()
        L.call("molr_cache_build_rows", dev.device_handle(), r, m, d_x, L.ptr(ptr), w[0].shape[1], L.ptr(w[0]),
               L.ptr(w[1]), L.ptr(w[2]), w[3].shape[1], L.ptr(w[3]), L.ptr(w[4]), L.ptr(w[5]), flags,
               float(DEFAULT_EPS), L.ptr(stream))
    return dev


def _check_users(cache, gating, user_embs, user_feats) -> None:
    """(U, k_u, d) user components and (U, d_u) gating features consistent with the cache and nets,
    checked before their pointers cross the C-ABI (which reads U * G floats of user_net output)."""
    cfg = cache.config
    if user_embs.ndim != 3 or user_embs.shape[2] != cfg.d or user_embs.shape[1] * cfg.k_x != gating.cross_net.in_dim:
        raise DimensionMismatchError(f"user_embs {user_embs.shape} vs (U, k_u, {cfg.d}) with k_u * {cfg.k_x} = "
                                     f"{gating.cross_net.in_dim}")
    if user_feats.shape != (user_embs.shape[0], gating.user_net.in_dim):
        raise DimensionMismatchError(f"user_feats {user_feats.shape} vs ({user_embs.shape[0]}, "
                                     f"{gating.user_net.in_dim})")


def _validate_candidates(cache, candidate_ids) -> np.ndarray:
    ids = np.asarray(candidate_ids, dtype=np.int64).reshape(-1)
    if ids.size == 0:
        raise EmptyCandidatesError("no candidates to score")
    if ids.min() < 0 or ids.max() >= cache.num_items:
        raise OutOfRangeError("candidate id outside the corpus")
    return np.ascontiguousarray(ids)


def _query_arrays(cache, query: QueryState, gating: GatingNetwork):
    ue = np.asarray(query.user_embs)
    cfg = cache.config
    if ue.ndim != 2 or ue.shape[1] != cfg.d:
        raise DimensionMismatchError(f"user {ue.shape} vs items {(cache.num_items, cfg.k_x, cfg.d)}")
    if ue.shape[0] * cfg.k_x != gating.cross_net.in_dim:
        raise DimensionMismatchError(
            f"item gate ({cfg.num_logits},) vs cross logits ({ue.shape[0] * cfg.k_x},)")
    uw = L.f32(gating.user_net(np.asarray(query.gate_features)))
    return L.f32(ue), uw


def score_candidates(cache, gating: GatingNetwork, candidate_ids, query: QueryState) -> np.ndarray:
    """Inference-mode similarities for the given candidate item ids (mol.py:329-345)."""
    ids = _validate_candidates(cache, candidate_ids)
    ue, uw = _query_arrays(cache, query, gating)
    out = np.empty(ids.size, dtype=np.float32)
    offs = np.array([0, ids.size], dtype=np.int64)
    L.call("molr_score", L.ctx(), cache_handle(cache), _gating_handle(gating), 1, ue.shape[0], L.ptr(ue),
           L.ptr(uw), float(cache.config.tau), L.ptr(offs), L.ptr(ids), L.ptr(out), None)
    return out.astype(_out_dtype(query.user_embs, np.float32), copy=False)


def batch_score_all(cache, gating: GatingNetwork, user_embs, user_feats, *, pairs_per_chunk: int = 2_000_000
                    ) -> np.ndarray:
    """(U, X) float32 score matrix of many users against the full corpus (mol.py:348-386).
    `pairs_per_chunk` is accepted for signature compatibility; device chunking is sized to the
    device scratch instead."""
    user_embs = np.asarray(user_embs)
    user_feats = np.asarray(user_feats)
    U = user_embs.shape[0]
    X = cache.num_items
    cfg = cache.config
    if user_embs.ndim != 3 or user_embs.shape[2] != cfg.d:
        raise DimensionMismatchError(f"user_embs {user_embs.shape} vs d {cfg.d}")
    _check_users(cache, gating, user_embs, user_feats)
    out = np.empty((U, X), dtype=np.float32)
    if U == 0 or X == 0:
        return out
    uw_all = L.f32(gating.user_net(user_feats))
    ue = L.f32(user_embs)
    per = max(1, (1 << 27) // max(X, 1))
    gh = _gating_handle(gating)
    for lo in range(0, U, per):
        hi = min(lo + per, U)
        L.call("molr_score", L.ctx(), cache_handle(cache), gh, hi - lo, ue.shape[1], L.ptr(ue[lo:hi]),
               L.ptr(uw_all[lo:hi]), float(cfg.tau), None, None, L.ptr(out[lo:hi]), None)
    return out


def mol_top_k(cache, gating: GatingNetwork, candidate_ids: Sequence[int] | np.ndarray, query: QueryState, k: int):
    """Exact top-k among the candidates by MoL similarity; ties break toward the smaller item id.
    Returns (item ids, scores), both length k, score-descending (mol.py:389-408)."""
    ids = np.asarray(candidate_ids, dtype=np.int64).reshape(-1)
    if ids.size == 0:
        raise EmptyCandidatesError("no candidates to rank")
    if k < 1 or k > ids.size:
        raise OutOfRangeError(f"k={k} outside [1, {ids.size}]")
    ids = _validate_candidates(cache, ids)
    ue, uw = _query_arrays(cache, query, gating)
    out_ids = np.empty(k, dtype=np.int64)
    out_sc = np.empty(k, dtype=np.float32)
    offs = np.array([0, ids.size], dtype=np.int64)
    L.call("molr_mol_top_k", L.ctx(), cache_handle(cache), _gating_handle(gating), 1, ue.shape[0], L.ptr(ue),
           L.ptr(uw), float(cache.config.tau), L.ptr(offs), L.ptr(ids), int(k), L.ptr(out_ids), L.ptr(out_sc), None)
    return out_ids, out_sc.astype(_out_dtype(query.user_embs, np.float32), copy=False)


def batch_mol_top_k(cache, gating: GatingNetwork, user_embs, user_feats, k: int, candidates=None):
    """Batched mol_top_k: B queries, each over its own candidate list (list of id arrays) or the
    whole corpus (candidates=None, = RetrievalEngine.full_top_k, engine.py:140-147).
    Returns (ids (B,k) int64, scores (B,k) float32)."""
    ue = L.f32(user_embs)
    _check_users(cache, gating, ue, np.asarray(user_feats))
    B = ue.shape[0]
    uw = L.f32(gating.user_net(np.asarray(user_feats)))
    out_ids = np.empty((B, k), dtype=np.int64)
    out_sc = np.empty((B, k), dtype=np.float32)
    if candidates is None:
        offs = ids = None
        if k < 1 or k > cache.num_items:
            raise OutOfRangeError(f"k={k} outside [1, {cache.num_items}]")
    else:
        lists = [_validate_candidates(cache, c) for c in candidates]
        offs = np.zeros(B + 1, dtype=np.int64)
        offs[1:] = np.cumsum([c.size for c in lists])
        ids = np.ascontiguousarray(np.concatenate(lists))
    L.call("molr_mol_top_k", L.ctx(), cache_handle(cache), _gating_handle(gating), B, ue.shape[1], L.ptr(ue),
           L.ptr(uw), float(cache.config.tau), L.ptr(offs), L.ptr(ids), int(k), L.ptr(out_ids), L.ptr(out_sc), None)
    return out_ids, out_sc


def uses_tensor_cores(cache, gating: GatingNetwork, k_u: Optional[int] = None) -> bool:
    """Whether MoL scoring of this cache and gating runs on the fused tcgen05 kernel (the production
    shape; bf16-exact caches directly, f32-stored caches such as a reference-built one through
    their bf16 hi + lo image) rather than the generic SIMT fp32 kernel."""
    k = cache.config.k_u if k_u is None else int(k_u)
    return L.load().molr_mol_uses_tensor_cores(C.c_void_p(cache_handle(cache)), C.c_void_p(_gating_handle(gating)), k) == 1


__all__ = [
    "MoLConfig", "Mlp", "GatingNetwork", "QueryState", "ItemCache", "DeviceItemCache", "component_logits",
    "decomposed_gating", "mol_score", "build_item_cache", "score_candidates", "batch_score_all", "mol_top_k",
    "batch_mol_top_k", "uses_tensor_cores",
]
