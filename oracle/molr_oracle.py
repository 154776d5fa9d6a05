"""NumPy restatement of the reference hot path (TEST INFRASTRUCTURE ONLY).

Every function cites the reference file:line it restates; paths are relative to
`/root/reference/pkg/src/molr/`.  Arrays are plain NumPy; the containers are
light namedtuples instead of the reference's dataclasses so this module has no
dependency on either the reference or the product package.
"""

from __future__ import annotations

from typing import NamedTuple, Optional

import numpy as np
from scipy.special import expit

__all__ = [
    "MlpW", "Gating", "Cache", "Quant", "Synthetic",
    "make_rng", "silu", "softmax_rows", "l2_normalize_rows", "mlp",
    "quantize_rowwise", "quantize_vector", "int8_matvec",
    "component_logits", "decomposed_gating", "mol_score", "score_candidates",
    "batch_score_all", "mol_top_k", "build_item_cache",
    "resolve_lambda", "nth_largest", "stage1_scores", "estimate_threshold",
    "h_indexer", "exact_top_k", "index_select",
    "init_synthetic", "user_components", "two_stage_query", "full_top_k",
    "round_bf16", "score_close",
]


# ----------------------------------------------------------------------------------------
# numerics.py
# ----------------------------------------------------------------------------------------
def make_rng(seed) -> np.random.Generator:
    """Philox generator seeded through SeedSequence — numerics.py:20-26."""
    return np.random.Generator(np.random.Philox(np.random.SeedSequence(seed)))


def silu(x):
    """x * sigmoid(x) with scipy's expit — numerics.py:73-75."""
    return x * expit(x)


def softmax_rows(m):
    """Max-shifted softmax along the last axis — numerics.py:61-66."""
    m = np.asarray(m)
    e = np.exp(m - m.max(axis=-1, keepdims=True))
    return e / e.sum(axis=-1, keepdims=True)


def l2_normalize_rows(m, eps: float = 1e-12):
    """Row L2 normalisation, error on norm <= eps — numerics.py:41-50."""
    m = np.asarray(m)
    n = np.linalg.norm(m, axis=-1, keepdims=True)
    if np.any(n <= eps):
        raise ZeroDivisionError("row norm <= eps")
    return m / n.astype(m.dtype)


class MlpW(NamedTuple):
    w1: np.ndarray  # (in, hidden)
    b1: np.ndarray  # (hidden,)
    w2: np.ndarray  # (hidden, out)


def mlp(p: MlpW, x):
    """silu(x @ w1 + b1) @ w2, no output bias — mol.py:84-85."""
    return silu(x @ p.w1 + p.b1) @ p.w2


class Gating(NamedTuple):
    user_net: MlpW
    item_net: MlpW
    cross_net: MlpW


# ----------------------------------------------------------------------------------------
# quant.py
# ----------------------------------------------------------------------------------------
class Quant(NamedTuple):
    codes: np.ndarray  # (n, d) int8
    scales: np.ndarray  # (n,) float32


def quantize_rowwise(matrix) -> Quant:
    """scale = max|row|/127 (zero row -> 1.0); rint half-even; clip +-127 — quant.py:49-57."""
    m = np.asarray(matrix, dtype=np.float32)
    maxabs = np.abs(m).max(axis=1)
    scales = np.where(maxabs > 0.0, maxabs / 127.0, 1.0).astype(np.float32)
    codes = np.clip(np.rint(m / scales[:, None]), -127, 127).astype(np.int8)
    return Quant(codes, scales)


def quantize_vector(v):
    """Single-scale encode of one vector — quant.py:60-63."""
    q = quantize_rowwise(np.asarray(v, dtype=np.float32).reshape(1, -1))
    return q.codes[0], float(q.scales[0])


def int8_matvec(q: Quant, q_query) -> np.ndarray:
    """Exact int32 accumulators — quant.py:83-90."""
    return q.codes.astype(np.int32) @ np.asarray(q_query, dtype=np.int8).astype(np.int32)


# ----------------------------------------------------------------------------------------
# mol.py
# ----------------------------------------------------------------------------------------
class Cache(NamedTuple):
    item_embs: np.ndarray  # (X, k_x, d) f32
    item_gate_pre: np.ndarray  # (X, G) f32
    stage1_embs: np.ndarray  # (X, d) f32
    stage1_q: Optional[Quant]
    tau: float
    k_u: int


def component_logits(user_embs, item_embs, tau):
    """cl[i, a*k_x+b] = <f_a, g_b(x_i)>/tau, user-component-major — mol.py:139-158."""
    n, k_x, d = item_embs.shape
    k_u = user_embs.shape[0]
    flat = user_embs @ item_embs.reshape(n * k_x, d).T
    cl = flat.reshape(k_u, n, k_x).transpose(1, 0, 2).reshape(n, k_u * k_x)
    return cl / np.asarray(tau, dtype=cl.dtype)


def decomposed_gating(g: Gating, user_gate_feat, item_gate_pre, cross_logits, *, uw=None):
    """softmax(silu(user_net(feat) * item_pre + cross_net(cl))), inference mode — mol.py:161-194."""
    if uw is None:
        uw = mlp(g.user_net, np.asarray(user_gate_feat))
    cw = mlp(g.cross_net, cross_logits)
    return softmax_rows(silu(uw[None, :] * item_gate_pre + cw))


def mol_score(pi, cl):
    """Gated sum of logits — mol.py:197-205."""
    return (pi * cl).sum(axis=-1)


def score_candidates(cache: Cache, g: Gating, ids, user_embs, gate_feat, *, uw=None):
    """Gather, logits, gating, gated sum — mol.py:329-345."""
    ids = np.asarray(ids, dtype=np.int64)
    cl = component_logits(user_embs, cache.item_embs[ids], cache.tau)
    pi = decomposed_gating(g, gate_feat, cache.item_gate_pre[ids], cl, uw=uw)
    return mol_score(pi, cl)


def batch_score_all(cache: Cache, g: Gating, user_embs, user_feats, *, pairs_per_chunk=2_000_000):
    """Exhaustive (U, X) score matrix, user-chunked — mol.py:348-386."""
    U = user_embs.shape[0]
    X, k_x, d = cache.item_embs.shape
    k_u = user_embs.shape[1]
    G = k_u * k_x
    uw_all = mlp(g.user_net, user_feats)
    out = np.empty((U, X), dtype=np.float32)
    per = max(1, pairs_per_chunk // max(X, 1))
    flat_items = cache.item_embs.reshape(X * k_x, d)
    for lo in range(0, U, per):
        hi = min(lo + per, U)
        u = hi - lo
        flat = user_embs[lo:hi].reshape(u * k_u, d) @ flat_items.T
        cl = flat.reshape(u, k_u, X, k_x).transpose(0, 2, 1, 3).reshape(u, X, G) / np.asarray(
            cache.tau, dtype=flat.dtype)
        cw = mlp(g.cross_net, cl.reshape(-1, G)).reshape(u, X, G)
        pi = softmax_rows(silu(uw_all[lo:hi, None, :] * cache.item_gate_pre[None] + cw))
        out[lo:hi] = (pi * cl).sum(axis=-1).astype(np.float32)
    return out


def mol_top_k(cache: Cache, g: Gating, ids, user_embs, gate_feat, k, *, uw=None):
    """Top-k by (score desc, id asc) via lexsort — mol.py:389-408."""
    ids = np.asarray(ids, dtype=np.int64)
    if ids.size == 0:
        raise ValueError("EmptyCandidates")
    if k < 1 or k > ids.size:
        raise ValueError("OutOfRange")
    s = score_candidates(cache, g, ids, user_embs, gate_feat, uw=uw)
    order = np.lexsort((ids, -s))[:k]
    return ids[order], s[order]


def build_item_cache(item_table, item_proj: MlpW, item_net: MlpW, k_x, d, tau, k_u,
                     *, quantized=False, l2_normalized=True) -> Cache:
    """item_proj -> L2 -> item_net; stage-1 = mean over k_x — mol.py:294-326."""
    n = item_table.shape[0]
    embs = mlp(item_proj, item_table).reshape(n, k_x, d)
    if l2_normalized:
        embs = l2_normalize_rows(embs)
    gp = mlp(item_net, item_table)
    s1 = embs.mean(axis=1)
    q = quantize_rowwise(s1) if quantized else None
    return Cache(embs.astype(np.float32), gp.astype(np.float32), s1.astype(np.float32), q, tau, k_u)


# ----------------------------------------------------------------------------------------
# hindexer.py
# ----------------------------------------------------------------------------------------
def resolve_lambda(k_prime, corpus_size, lam=None, sample_ratio=None):
    """k' <= X; lambda = lam or max(1, round(r*X)) (banker's round) — hindexer.py:59-65."""
    if k_prime > corpus_size:
        raise ValueError("OutOfRange: k_prime exceeds corpus")
    lam = lam if lam is not None else max(1, round(sample_ratio * corpus_size))
    if not 1 <= lam <= corpus_size:
        raise ValueError("OutOfRange: lambda")
    return lam


def nth_largest(values, n):
    """n-th largest with multiplicity via partition — hindexer.py:77-82."""
    values = np.asarray(values)
    return float(np.partition(values, values.size - n)[values.size - n])


def stage1_scores(view, query, *, raw_int_ordering=False):
    """Float: view @ q.  Quantized: int32 acc (raw) or acc.f32 * row scale — hindexer.py:94-112."""
    query = np.asarray(query)
    if isinstance(view, Quant):
        qc, _ = quantize_vector(query)
        acc = int8_matvec(view, qc)
        if raw_int_ordering:
            return acc
        return acc.astype(np.float32) * view.scales
    return view @ query


def _n_rank(k_prime, lam, X):
    """n = max(1, round(k' * lambda / X)) — hindexer.py:131,157."""
    return max(1, round(k_prime * lam / X))


def estimate_threshold(view, query, k_prime, rng, *, lam=None, sample_ratio=None, raw_int_ordering=False):
    """Permutation-prefix sample, n-th largest of its scores — hindexer.py:115-132."""
    X = view.codes.shape[0] if isinstance(view, Quant) else view.shape[0]
    lam = resolve_lambda(k_prime, X, lam, sample_ratio)
    sample = rng.permutation(X)[:lam]
    sub = Quant(view.codes[sample], view.scales[sample]) if isinstance(view, Quant) else view[sample]
    s = stage1_scores(sub, query, raw_int_ordering=raw_int_ordering)
    return nth_largest(s, _n_rank(k_prime, lam, X))


def h_indexer(view, query, k_prime, rng, *, lam=None, sample_ratio=None, comparator="inclusive",
              raw_int_ordering=False):
    """Score once, threshold from the sampled subset of the same array, keep passers
    (ascending ids) — hindexer.py:135-163.  Returns (indices, threshold, scanned)."""
    X = view.codes.shape[0] if isinstance(view, Quant) else view.shape[0]
    lam = resolve_lambda(k_prime, X, lam, sample_ratio)
    if k_prime >= X:
        return np.arange(X), float("-inf"), X
    s = stage1_scores(view, query, raw_int_ordering=raw_int_ordering)
    sample = rng.permutation(X)[:lam]
    t = nth_largest(s[sample], _n_rank(k_prime, lam, X))
    mask = s >= t if comparator == "inclusive" else s > t
    return np.nonzero(mask)[0], float(t), X


def exact_top_k(view, query, k, *, raw_int_ordering=False):
    """Stable argsort of -scores — hindexer.py:166-178."""
    s = stage1_scores(view, query, raw_int_ordering=raw_int_ordering)
    return np.argsort(-s, kind="stable")[:k]


def index_select(cache: Cache, indices) -> Cache:
    """Row gather of every cache field for sorted ids — hindexer.py:181-201."""
    idx = np.asarray(indices, dtype=np.int64)
    q = None if cache.stage1_q is None else Quant(cache.stage1_q.codes[idx], cache.stage1_q.scales[idx])
    return Cache(cache.item_embs[idx], cache.item_gate_pre[idx], cache.stage1_embs[idx], q,
                 cache.tau, cache.k_u)


# ----------------------------------------------------------------------------------------
# model.py / engine.py (synthetic model generator and the two-stage composition)
# ----------------------------------------------------------------------------------------
class Synthetic(NamedTuple):
    user_table: np.ndarray
    item_table: np.ndarray
    user_proj: MlpW
    item_proj: MlpW
    gating: Gating


def _table(rng, n, dim):
    b = 1.0 / np.sqrt(dim)
    return rng.uniform(-b, b, (n, dim)).astype(np.float32)


def _mlp_init(rng, n_in, n_hidden, n_out):
    b1 = 1.0 / np.sqrt(n_in)
    b2 = 1.0 / np.sqrt(n_hidden)
    return MlpW(rng.uniform(-b1, b1, (n_in, n_hidden)).astype(np.float32),
                rng.uniform(-b1, b1, n_hidden).astype(np.float32),
                rng.uniform(-b2, b2, (n_hidden, n_out)).astype(np.float32))


def init_synthetic(n_users, n_items, *, k_u, k_x, d, gating_hidden, d_u=64, d_x=64, proj_hidden=128,
                   seed=4242) -> Synthetic:
    """Same draw order as model.init_params (model.py:136-163, tables 121-123, MLPs 126-133)."""
    rng = make_rng(seed)
    G = k_u * k_x
    ut = _table(rng, n_users, d_u)
    it = _table(rng, n_items, d_x)
    up = _mlp_init(rng, d_u, proj_hidden, k_u * d)
    ip = _mlp_init(rng, d_x, proj_hidden, k_x * d)
    g = Gating(_mlp_init(rng, d_u, gating_hidden, G), _mlp_init(rng, d_x, gating_hidden, G),
               _mlp_init(rng, G, gating_hidden, G))
    return Synthetic(ut, it, up, ip, g)


def user_components(syn: Synthetic, user_ids, k_u, d, l2_normalized=True):
    """(B, k_u, d) user components — model.py:179-191 (no compression map)."""
    feats = syn.user_table[user_ids]
    e = mlp(syn.user_proj, feats).reshape(len(feats), k_u, d)
    return l2_normalize_rows(e) if l2_normalized else e


def two_stage_query(cache: Cache, g: Gating, user_embs, gate_feat, k, k_prime, rng, *, lam=None,
                    sample_ratio=None, quantized=False, comparator="inclusive"):
    """RetrievalEngine.query composition — engine.py:117-138."""
    X = cache.item_embs.shape[0]
    if k_prime >= X:
        cand = np.arange(X)
    else:
        view = cache.stage1_q if quantized else cache.stage1_embs
        cand, _, _ = h_indexer(view, user_embs.mean(axis=0), k_prime, rng, lam=lam,
                               sample_ratio=sample_ratio, comparator=comparator)
        if cand.size < k:
            cand = np.arange(X)
    return mol_top_k(cache, g, cand, user_embs, gate_feat, min(k, cand.size))


def full_top_k(cache: Cache, g: Gating, user_embs, gate_feat, k):
    """Exhaustive MoL top-k — engine.py:140-147."""
    X = cache.item_embs.shape[0]
    return mol_top_k(cache, g, np.arange(X), user_embs, gate_feat, min(k, X))


# ----------------------------------------------------------------------------------------
# parity helpers (the tolerance of SURVEY.md §8c)
# ----------------------------------------------------------------------------------------
def round_bf16(x):
    """Round-to-nearest-even to bfloat16, returned as float32 (bf16-representable inputs)."""
    x = np.ascontiguousarray(x, dtype=np.float32)
    u = x.view(np.uint32).astype(np.uint64)
    u = (u + 0x7FFF + ((u >> 16) & 1)) & 0xFFFF0000
    return u.astype(np.uint32).view(np.float32).reshape(x.shape)


def score_close(got, ref, rel=1e-3, abs_=1e-6):
    """|got - ref| <= rel*|ref| + abs_ elementwise (MoL tolerance)."""
    got = np.asarray(got, dtype=np.float64)
    ref = np.asarray(ref, dtype=np.float64)
    return np.abs(got - ref) <= rel * np.abs(ref) + abs_
