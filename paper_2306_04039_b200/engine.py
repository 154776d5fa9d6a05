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
from paper_2306_04039_b200.errors import DimensionMismatchError
from paper_2306_04039_b200.mol import GatingNetwork, _gating_handle, cache_handle


def _mode(h: HIndexerConfig) -> int:
    if h.quantized:
        return L.S1_INT8_RAW if h.raw_int_ordering else L.S1_INT8
    return L.S1_FLOAT


def _host_or_f32_tensor(a, name):
    """Host inputs become contiguous float32 NumPy arrays; device tensors must already be float32
    and contiguous (their data pointer is read as such by the C-ABI)."""
    if hasattr(a, "data_ptr") and not isinstance(a, np.ndarray):
        if str(getattr(a, "dtype", "")) not in ("torch.float32", "float32"):
            raise DimensionMismatchError(f"{name}: device tensors must be float32, got {a.dtype}")
        if hasattr(a, "is_contiguous") and not a.is_contiguous():
            raise DimensionMismatchError(f"{name}: device tensors must be contiguous")
        return a
    return L.f32(np.asarray(a))


def check_batch(cache, gating, user_embs, uw, *, uw_name="uw"):
    """Validate a batch before raw pointers cross the C-ABI: user_embs (B, k_u, d) with
    k_u * k_x = G = the cross net's width, and the gating rows (B, G) — user_net outputs, or raw
    user features (B, d_u) when uw_name == "user_feats".  Returns (user_embs, uw) as float32."""
    ue = _host_or_f32_tensor(user_embs, "user_embs")
    w = _host_or_f32_tensor(uw, uw_name)
    cfg = cache.config
    shape = tuple(int(x) for x in ue.shape)
    if len(shape) != 3 or shape[2] != cfg.d or shape[1] * cfg.k_x != gating.cross_net.in_dim:
        raise DimensionMismatchError(
            f"user_embs {shape} vs (B, k_u, {cfg.d}) with k_u * {cfg.k_x} = {gating.cross_net.in_dim}")
    want = gating.user_net.in_dim if uw_name == "user_feats" else gating.cross_net.out_dim
    if tuple(int(x) for x in w.shape) != (shape[0], want):
        raise DimensionMismatchError(f"{uw_name} {tuple(w.shape)} vs ({shape[0]}, {want})")
    return ue, w


def two_stage_top_k(cache, gating: GatingNetwork, user_embs, uw, k: int, hconfig: HIndexerConfig, *, seed: int = 0,
                    id_offset: int = 0, out_ids=None, out_scores=None, out_cand=None, stream=None):
    """Device-resident batched two-stage top-k.  `user_embs` (B,k_u,d) and `uw` (B,G) may be host
    NumPy arrays or device tensors (anything with data_ptr()); outputs likewise.  Returns
    (ids (B,k) int64, scores (B,k) f32, candidate counts (B,) int64)."""
    user_embs, uw = check_batch(cache, gating, user_embs, uw)
    B, k_u = int(user_embs.shape[0]), int(user_embs.shape[1])
    X = cache.num_items
    lam = hconfig.resolve_lambda(X)
    if out_ids is None:
        out_ids = np.empty((B, k), dtype=np.int64)
        out_scores = np.empty((B, k), dtype=np.float32)
        out_cand = np.empty(B, dtype=np.int64)
    L.call("molr_two_stage_top_k", L.ctx(), cache_handle(cache), _gating_handle(gating), B, k_u, L.ptr(user_embs),
           L.ptr(uw), float(cache.config.tau), _mode(hconfig), int(hconfig.k_prime), int(lam), int(seed) & (2**64 - 1),
           L.STRICT if hconfig.comparator == "strict" else L.INCLUSIVE, int(k), int(id_offset), L.ptr(out_ids),
           L.ptr(out_scores), L.ptr(out_cand), L.ptr(stream))
    return out_ids, out_scores, out_cand


class RetrievalEngine:
    """Drop-in for molr.engine.RetrievalEngine (engine.py:80-147): immutable artifacts plus the
    two-stage query path with the reference's exact per-query semantics — the first-stage
    sample comes from make_rng([seed, user_id]) (so repeated identical queries return identical
    results), candidates from the drop-in h_indexer, the top-k from the drop-in mol_top_k, all
    on the GPU.  `params` is the reference's TowerParams (read duck-typed: user_table, user_proj,
    gating, n_users; item_table / item_proj for from_params)."""

    def __init__(self, params, config, cache, hconfig: HIndexerConfig, seed: int = 0):
        self.params = params
        self.config = config
        self.cache = cache
        self.hconfig = hconfig
        self.seed = seed

    @classmethod
    def from_params(cls, params, config, hconfig: HIndexerConfig, *, seed: int = 0) -> "RetrievalEngine":
        from paper_2306_04039_b200.mol import build_item_cache

        cache = build_item_cache(params.item_table, params.item_proj, params.gating.item_net, config,
                                 quantized=hconfig.quantized)
        return cls(params, config, cache, hconfig, seed)

    @property
    def num_items(self) -> int:
        return self.cache.num_items

    @property
    def num_users(self) -> int:
        return int(getattr(self.params, "n_users", np.asarray(self.params.user_table).shape[0]))

    def query_state(self, user_id: int):
        """user_forward (model.py:203-208): the user tower is the caller's model code, not the MoL /
        h-indexer path, so it is evaluated exactly as the reference evaluates it (NumPy:
        silu(x @ w1 + b1) @ w2 -> reshape -> row L2 norm, model.py:179-191, mol.py:84-85,
        numerics.py:41-50): the stage-1 query (mean of the components) and its int8 codes are then
        bit-identical to the reference engine's, so the drop-in returns the reference's candidates.
        The batched engine below runs the device query prep (molr_query_prep) instead."""
        from scipy.special import expit

        from paper_2306_04039_b200.errors import OutOfRangeError, ZeroNormError
        from paper_2306_04039_b200.mol import QueryState

        if not 0 <= user_id < self.num_users:
            raise OutOfRangeError(f"user id {user_id} outside [0, {self.num_users})")
        if getattr(self.params, "compression", None) is not None:
            raise ValueError("user-side compression maps are outside the B200 path (SURVEY.md §2)")
        feats = np.asarray(self.params.user_table)[user_id]
        p = self.params.user_proj
        x = feats[None, :]
        hid = x @ np.asarray(p.w1) + np.asarray(p.b1)
        raw = (hid * expit(hid)) @ np.asarray(p.w2)
        embs = raw.reshape(1, self.config.k_u, self.config.d)
        if self.config.l2_normalized:
            norms = np.linalg.norm(embs, axis=-1, keepdims=True)
            if np.any(norms <= 1e-12):
                raise ZeroNormError("at least one row has norm <= eps")
            embs = embs / norms.astype(embs.dtype)
        return QueryState(user_embs=embs[0], gate_features=feats)

    def query(self, user_id: int, k: int, k_prime: int | None = None):
        """First-stage candidates, then exact MoL top-k (engine.py:117-138)."""
        from paper_2306_04039_b200.hindexer import h_indexer, stage1_view, with_k_prime
        from paper_2306_04039_b200.mol import mol_top_k
        from paper_2306_04039_b200.numerics import make_rng

        hcfg = self.hconfig if k_prime is None else with_k_prime(self.hconfig, k_prime)
        state = self.query_state(user_id)
        if hcfg.k_prime >= self.num_items:
            candidates = np.arange(self.num_items)
        else:
            rng = make_rng([self.seed, user_id])
            stage1_query = state.user_embs.mean(axis=0)
            candidates = h_indexer(stage1_view(self.cache, hcfg), stage1_query, hcfg, rng).indices
            if candidates.size < k:
                candidates = np.arange(self.num_items)
        ids, scores = mol_top_k(self.cache, self.params.gating, candidates, state, min(k, candidates.size))
        return [(int(i), float(s)) for i, s in zip(ids, scores)]

    def full_top_k(self, user_id: int, k: int):
        """Exhaustive MoL ranking, no first stage (engine.py:140-147)."""
        from paper_2306_04039_b200.mol import mol_top_k

        state = self.query_state(user_id)
        ids, scores = mol_top_k(self.cache, self.params.gating, np.arange(self.num_items), state,
                                min(k, self.num_items))
        return [(int(i), float(s)) for i, s in zip(ids, scores)]


def query_prep(user_proj, user_net, user_feats, config, *, stream=None, out_embs=None, out_uw=None):
    """Batched user-side query state on the device (molr_query_prep): user_embs (B, k_u, d) =
    user_components (model.py:179-191: user_proj MLP, per-component L2 norm) and uw (B, G) =
    user_net(features) (mol.py:186).  Host arrays in -> host arrays out, or device tensors."""
    from paper_2306_04039_b200.numerics import DEFAULT_EPS

    feats = user_feats
    host = isinstance(feats, np.ndarray) or not hasattr(feats, "data_ptr")
    if host:
        feats = L.f32(np.asarray(feats))
    B, d_u = int(feats.shape[0]), int(feats.shape[1])
    if user_proj.in_dim != d_u or user_net.in_dim != d_u:
        raise ValueError("tower input dims do not match the user features")
    G = config.num_logits
    if out_embs is None:
        out_embs = np.empty((B, config.k_u, config.d), np.float32)
        out_uw = np.empty((B, G), np.float32)
    w = [L.f32(a) for a in (user_proj.w1, user_proj.b1, user_proj.w2, user_net.w1, user_net.b1, user_net.w2)]
    L.call("molr_query_prep", L.ctx(), B, d_u, L.ptr(feats), w[0].shape[1], L.ptr(w[0]), L.ptr(w[1]), L.ptr(w[2]),
           config.k_u, config.d, int(config.l2_normalized), w[3].shape[1], L.ptr(w[3]), L.ptr(w[4]), L.ptr(w[5]), G,
           float(DEFAULT_EPS), L.ptr(out_embs), L.ptr(out_uw), L.ptr(stream))
    return out_embs, out_uw


class BatchedRetrievalEngine:
    """Immutable cache + gating + h-indexer config (+ the user tower for raw-feature queries);
    any number of threads may query it (RetrievalEngine, engine.py:80-147, batched)."""

    def __init__(self, cache, gating: GatingNetwork, hconfig: HIndexerConfig, seed: int = 0, user_proj=None):
        self.cache = cache
        self.gating = gating
        self.hconfig = hconfig
        self.seed = seed
        self.user_proj = user_proj

    @property
    def num_items(self) -> int:
        return self.cache.num_items

    def query_batch(self, user_embs, user_feats, k: int, k_prime: int | None = None, seed: int | None = None):
        from dataclasses import replace

        h = self.hconfig if k_prime is None else replace(self.hconfig, k_prime=k_prime)
        check_batch(self.cache, self.gating, user_embs, user_feats, uw_name="user_feats")
        uw = self.gating.user_net(np.asarray(user_feats))
        ids, sc, cand = two_stage_top_k(self.cache, self.gating, user_embs, uw, k, h,
                                        seed=self.seed if seed is None else seed)
        return ids, sc, cand

    def query_features(self, user_feats, k: int, k_prime: int | None = None, seed: int | None = None):
        """The whole query path from raw user features (RetrievalEngine.query, engine.py:117-138,
        for a batch): device query prep -> two-stage top-k.  Needs `user_proj`."""
        from dataclasses import replace

        if self.user_proj is None:
            raise ValueError("engine built without the user tower (user_proj)")
        h = self.hconfig if k_prime is None else replace(self.hconfig, k_prime=k_prime)
        ue, uw = query_prep(self.user_proj, self.gating.user_net, user_feats, self.cache.config)
        return two_stage_top_k(self.cache, self.gating, ue, uw, k, h, seed=self.seed if seed is None else seed)

    def full_top_k_batch(self, user_embs, user_feats, k: int):
        from paper_2306_04039_b200.mol import batch_mol_top_k

        return batch_mol_top_k(self.cache, self.gating, user_embs, user_feats, min(k, self.num_items))


def two_stage_top_k_sharded(cache, gating: GatingNetwork, user_embs, uw, k: int, hconfig: HIndexerConfig, *,
                            X_global: int, row_lo: int, exchange, seed: int = 0):
    """Two-stage top-k over one shard (global rows [row_lo, row_lo + cache.num_items)) that returns
    EXACTLY the single-device result of `two_stage_top_k` over the whole X_global corpus (SURVEY
    §8(e), "single-GPU-equivalent threshold"): every shard scores its part of the same global
    sample, the shards exchange each query's top n sample-score keys, and the n-th largest of that
    union is the single-device threshold (hindexer.py:131).  The fallback to the corpus
    (engine.py:134-135) is decided on the GLOBAL passer count.

    `exchange(a)` all-gathers a NumPy array over the shards and returns the rank-major stack
    (P, *a.shape) — e.g. torch.distributed.all_gather, or a list of in-process shards in tests.
    Returns (ids (B,k) global, scores (B,k), global candidate counts (B,)), identical on every
    shard."""
    B, k_u = int(user_embs.shape[0]), int(user_embs.shape[1])
    Xs = cache.num_items
    ue = L.f32(np.asarray(user_embs))
    uwf = L.f32(np.asarray(uw))
    mode = _mode(hconfig)
    lam = hconfig.resolve_lambda(X_global)  # raises OutOfRangeError for K' > X like the reference
    kp = int(hconfig.k_prime)
    # the key below every score: f32_key(-inf) (scaled / float views) or i32_key(INT32_MIN) (raw)
    pass_all = 0 if mode == L.S1_INT8_RAW else 0x007FFFFF
    if kp >= X_global:
        tkeys = np.full(B, pass_all, dtype=np.uint32)  # every row passes (hindexer.py:151-154)
    else:
        n_rank = max(1, round(kp * lam / X_global))  # Python round(): half-even, as hindexer.py:131
        keys = np.empty((B, n_rank), dtype=np.uint32)
        L.call("molr_sample_top_keys", L.ctx(), cache_handle(cache), B, k_u, L.ptr(ue), mode, int(X_global),
               int(row_lo), int(lam), int(seed) & (2**64 - 1), int(n_rank), L.ptr(keys), None)
        allk = np.asarray(exchange(keys))  # (P, B, n_rank)
        rows = np.ascontiguousarray(allk.transpose(1, 0, 2).reshape(B, -1))
        tkeys = np.empty(B, dtype=np.uint32)
        L.call("molr_select_nth_keys", L.ctx(), B, rows.shape[1], L.ptr(rows), int(n_rank), L.ptr(tkeys), None)
    comp = L.STRICT if hconfig.comparator == "strict" else L.INCLUSIVE
    cap_hint = max(1, min(Xs, -(-kp * Xs // X_global)))

    def run(sel, tk, cap):
        ids = np.empty((len(sel), k), dtype=np.int64)
        sc = np.empty((len(sel), k), dtype=np.float32)
        cnt = np.empty(len(sel), dtype=np.int64)
        ue_s = np.ascontiguousarray(ue[sel])  # (named: the buffers must outlive the call)
        uw_s = np.ascontiguousarray(uwf[sel])
        tk_s = np.ascontiguousarray(tk, dtype=np.uint32)
        L.call("molr_two_stage_top_k_at", L.ctx(), cache_handle(cache), _gating_handle(gating), len(sel), k_u,
               L.ptr(ue_s), L.ptr(uw_s), float(cache.config.tau), mode, int(cap), L.ptr(tk_s), comp, int(k),
               int(row_lo), L.ptr(ids), L.ptr(sc), L.ptr(cnt), None)
        return ids, sc, cnt

    allq = np.arange(B)
    ids, sc, cnt = run(allq, tkeys, cap_hint)
    gcnt = np.asarray(exchange(cnt)).sum(axis=0)
    short = np.nonzero(gcnt < min(k, X_global))[0]
    if short.size:  # fewer than k candidates in the whole corpus: score every row (engine.py:134-135)
        fi, fs, _ = run(short, np.full(short.size, pass_all, dtype=np.uint32), Xs)
        ids[short], sc[short] = fi, fs
        gcnt[short] = X_global
    out_i, out_s = merge_top_k(np.asarray(exchange(ids)), np.asarray(exchange(sc)), k)
    return out_i, out_s, gcnt


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


def bench_csv(engine: BatchedRetrievalEngine, user_embs, user_feats, k: int, k_primes, *, repeats: int = 1):
    """`molr bench` (cli.py:229-281) on the batched device path: the exact top-k per user first
    (untimed), then for every K' in the grid the two-stage top-k of the whole batch, timed; one
    CSV row per K' with the mean recall@k vs exact and queries/s.  Header `k_prime,recall,qps`
    (the contract pinned by test_cli.py:128-137)."""
    import time

    from paper_2306_04039_b200.mol import batch_mol_top_k

    X = engine.num_items
    k_eff = min(k, X)
    exact_ids, _ = batch_mol_top_k(engine.cache, engine.gating, user_embs, user_feats, k_eff)
    uw = engine.gating.user_net(np.asarray(user_feats))
    lines = ["k_prime,recall,qps"]
    B = len(user_embs)
    for kp in k_primes:
        from dataclasses import replace

        h = replace(engine.hconfig, k_prime=int(kp))
        ids, _, _ = two_stage_top_k(engine.cache, engine.gating, user_embs, uw, k_eff, h, seed=engine.seed)  # warm
        t0 = time.perf_counter()
        for _ in range(repeats):
            ids, _, _ = two_stage_top_k(engine.cache, engine.gating, user_embs, uw, k_eff, h, seed=engine.seed)
        dt = (time.perf_counter() - t0) / repeats
        rec = float(np.mean([len(set(ids[b].tolist()) & set(exact_ids[b].tolist())) / k_eff for b in range(B)]))
        lines.append(f"{int(kp)},{rec:.4f},{B / dt:.1f}")
    return "\n".join(lines) + "\n"
