"""Batched two-stage retrieval on the device — the batched form of RetrievalEngine.query /
full_top_k (engine.py:117-147).  Per query: stage-1 query = mean of the user components
(engine.py:131); sampled threshold + full scan (h_indexer); MoL re-scoring of the passers with a
fallback to the whole corpus when fewer than k pass (engine.py:134-135); top-k by (score desc,
id asc).  Unlike the drop-in h_indexer (host rng, per-query permutation), the batched path draws
its lambda-row sample on the device from a seeded Feistel permutation shared by the batch, so no
O(X) host work sits on the query path.
"""

from __future__ import annotations

import numpy as np

from paper_2306_04039_b200 import _lib as L
from paper_2306_04039_b200.hindexer import HIndexerConfig
from paper_2306_04039_b200.mol import GatingNetwork, _gating_handle


def _mode(h: HIndexerConfig) -> int:
    if h.quantized:
        return L.S1_INT8_RAW if h.raw_int_ordering else L.S1_INT8
    return L.S1_FLOAT


def two_stage_top_k(cache, gating: GatingNetwork, user_embs, uw, k: int, hconfig: HIndexerConfig, *, seed: int = 0,
                    id_offset: int = 0, out_ids=None, out_scores=None, out_cand=None, stream=None):
    """Device-resident batched two-stage top-k.  `user_embs` (B,k_u,d) and `uw` (B,G) may be host
    NumPy arrays or device tensors (anything with data_ptr()); outputs likewise.  Returns
    (ids (B,k) int64, scores (B,k) f32, candidate counts (B,) int64)."""
    B, k_u = int(user_embs.shape[0]), int(user_embs.shape[1])
    X = cache.num_items
    lam = hconfig.resolve_lambda(X)
    if isinstance(user_embs, np.ndarray):
        user_embs = L.f32(user_embs)
        uw = L.f32(uw)
    if out_ids is None:
        out_ids = np.empty((B, k), dtype=np.int64)
        out_scores = np.empty((B, k), dtype=np.float32)
        out_cand = np.empty(B, dtype=np.int64)
    L.call("molr_two_stage_top_k", L.ctx(), cache.device_handle(), _gating_handle(gating), B, k_u, L.ptr(user_embs),
           L.ptr(uw), float(cache.config.tau), _mode(hconfig), int(hconfig.k_prime), int(lam), int(seed) & (2**64 - 1),
           L.STRICT if hconfig.comparator == "strict" else L.INCLUSIVE, int(k), int(id_offset), L.ptr(out_ids),
           L.ptr(out_scores), L.ptr(out_cand), L.ptr(stream))
    return out_ids, out_scores, out_cand


class BatchedRetrievalEngine:
    """Immutable cache + gating + h-indexer config; any number of threads may query it."""

    def __init__(self, cache, gating: GatingNetwork, hconfig: HIndexerConfig, seed: int = 0):
        self.cache = cache
        self.gating = gating
        self.hconfig = hconfig
        self.seed = seed

    @property
    def num_items(self) -> int:
        return self.cache.num_items

    def query_batch(self, user_embs, user_feats, k: int, k_prime: int | None = None, seed: int | None = None):
        from dataclasses import replace

        h = self.hconfig if k_prime is None else replace(self.hconfig, k_prime=k_prime)
        uw = self.gating.user_net(np.asarray(user_feats))
        ids, sc, cand = two_stage_top_k(self.cache, self.gating, user_embs, uw, k, h,
                                        seed=self.seed if seed is None else seed)
        return ids, sc, cand

    def full_top_k_batch(self, user_embs, user_feats, k: int):
        from paper_2306_04039_b200.mol import batch_mol_top_k

        return batch_mol_top_k(self.cache, self.gating, user_embs, user_feats, min(k, self.num_items))


def merge_top_k(ids, scores, k: int):
    """Merge P rank-major (P,B,k_in) per-shard top-k lists into the global top-k (C1 merge)."""
    ids = np.ascontiguousarray(ids, dtype=np.int64)
    scores = L.f32(scores)
    P, B, k_in = ids.shape
    out_i = np.empty((B, k), dtype=np.int64)
    out_s = np.empty((B, k), dtype=np.float32)
    L.call("molr_merge_top_k", L.ctx(), P, B, k_in, L.ptr(ids), L.ptr(scores), int(k), L.ptr(out_i), L.ptr(out_s),
           None)
    return out_i, out_s
