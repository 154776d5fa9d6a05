"""GPU parity: the CUDA path (through the C-ABI, via the reference-shaped Python API) against the
golden vectors the reference produced and against the CPU oracle on the same seeded inputs.

Tolerances: MoL scores |got - ref| <= 1e-3 |ref| + 1e-6; top-k index lists equal
except items whose reference score is within that band of the k-th score; int8 stage 1 and
quantisation bit-exact; float stage 1 within fp32 noise."""

import numpy as np
import pytest

import oracle as O
from tests.helpers import (
    with_knob,
    oracle_gating,
    product_cache,
    product_gating,
    topk_equal_modulo_ties,
)

pytestmark = pytest.mark.gpu

REL, ABS = 1e-3, 1e-6


@pytest.fixture(scope="module")
def prod(golden):
    g = golden("production_mol")
    return g, product_cache(g), product_gating(g)


@pytest.fixture(scope="module")
def small(golden):
    g = golden("small_mol")
    return g, product_cache(g, kind="small"), product_gating(g)


def qs(g, u):
    from paper_2306_04039_b200.mol import QueryState

    return QueryState(user_embs=g["user_embs"][u], gate_features=g["user_feats"][u])


# ---------------------------------------------------------------------------------- MoL
def test_small_shape_scores_topk_batch(small):
    from paper_2306_04039_b200.mol import batch_score_all, mol_top_k, score_candidates

    g, cache, gating = small
    X = cache.num_items
    for u in range(g["user_embs"].shape[0]):
        s = score_candidates(cache, gating, np.arange(X), qs(g, u))
        assert O.score_close(s, g["scores"][u], REL, ABS).all()
        ids, sc = mol_top_k(cache, gating, np.arange(X), qs(g, u), 10)
        assert topk_equal_modulo_ties(ids, g["top_ids"][u], g["scores"][u])
        assert O.score_close(sc, g["scores"][u][ids], REL, ABS).all()
    m = batch_score_all(cache, gating, g["user_embs"], g["user_feats"], pairs_per_chunk=700)
    assert m.dtype == np.float32 and m.shape == g["batch_all"].shape
    assert O.score_close(m, g["batch_all"], REL, ABS).all()


def test_production_shape_scores_topk(prod):
    from paper_2306_04039_b200.mol import mol_top_k, score_candidates

    g, cache, gating = prod
    X = cache.num_items
    worst = 0.0
    for u in range(g["user_embs"].shape[0]):
        s = score_candidates(cache, gating, np.arange(X), qs(g, u))
        ref = g["scores"][u]
        worst = max(worst, float(np.max(np.abs(s - ref))))
        assert O.score_close(s, ref, REL, ABS).all(), float(np.max(np.abs(s - ref)))
        ids, sc = mol_top_k(cache, gating, np.arange(X), qs(g, u), 100)
        assert topk_equal_modulo_ties(ids, g["top_ids"][u], ref)
        assert np.all(np.diff(sc) <= 0)
    print(f"max |score - ref| = {worst:.3e}")


def test_production_batch_score_all(prod):
    from paper_2306_04039_b200.mol import batch_score_all

    g, cache, gating = prod
    m = batch_score_all(cache, gating, g["user_embs"], g["user_feats"])
    assert O.score_close(m, g["batch_all"], REL, ABS).all()


def test_candidate_subsets_and_order(prod):
    """Scores follow the candidate order; duplicates and unsorted lists behave like the reference."""
    from paper_2306_04039_b200.mol import mol_top_k, score_candidates

    g, cache, gating = prod
    rng = np.random.default_rng(0)
    ids = rng.permutation(cache.num_items)[:257]
    s = score_candidates(cache, gating, ids, qs(g, 3))
    assert O.score_close(s, g["scores"][3][ids], REL, ABS).all()
    dup = np.concatenate([ids[:5], ids[:5]])
    s2 = score_candidates(cache, gating, dup, qs(g, 3))
    assert np.array_equal(s2[:5], s2[5:])
    top, _ = mol_top_k(cache, gating, ids, qs(g, 3), 1)
    assert top[0] == ids[np.argmax(g["scores"][3][ids])] or abs(
        g["scores"][3][top[0]] - g["scores"][3][ids].max()) <= ABS


def test_primitives_match_golden(small):
    from paper_2306_04039_b200.mol import component_logits, decomposed_gating, mol_score

    g, cache, gating = small
    cl = component_logits(g["user_embs"][0], cache.item_embs[:20], float(g["tau"]))
    np.testing.assert_allclose(cl, g["cl_u0"], rtol=1e-5, atol=1e-8)
    pi = decomposed_gating(gating, g["user_feats"][0], cache.item_gate_pre[:20], cl)
    np.testing.assert_allclose(pi, g["pi_u0"], rtol=1e-4, atol=1e-7)
    np.testing.assert_allclose(pi.sum(axis=1), 1.0, atol=1e-6)
    s = mol_score(pi, cl)
    assert O.score_close(s, g["scores"][0][:20], REL, ABS).all()


def test_reference_known_answers_mol():
    """test_mol.py known answers: aligned unit vectors, tau=20 -> 0.05, layout, constant nets."""
    from paper_2306_04039_b200.mol import GatingNetwork, Mlp, component_logits, decomposed_gating, mol_score

    e = np.zeros(8)
    e[0] = 1.0
    np.testing.assert_allclose(component_logits(np.tile(e, (3, 1)), np.tile(e, (5, 2, 1)), tau=1.0), 1.0)
    e4 = np.zeros(4)
    e4[1] = 1.0
    assert component_logits(e4[None, :], e4[None, None, :], tau=20.0)[0, 0] == pytest.approx(0.05)
    rng = O.make_rng(3)
    user, items = rng.standard_normal((3, 5)), rng.standard_normal((4, 2, 5))
    cl = component_logits(user, items, 7.0)
    for i in range(4):
        for a in range(3):
            for b in range(2):
                assert cl[i, a * 2 + b] == pytest.approx(float(user[a] @ items[i, b]) / 7.0, rel=1e-6)

    def constant_mlp(n_in, n_out, value):
        fill = value / (4.0 * float(O.silu(1.0)))
        return Mlp(w1=np.zeros((n_in, 4)), b1=np.ones(4), w2=np.full((4, n_out), fill))

    gating = GatingNetwork(constant_mlp(4, 6, 0.7), constant_mlp(3, 6, -0.3), constant_mlp(6, 6, 1.2))
    item_pre = gating.item_net(np.ones((5, 3)))
    pi = decomposed_gating(gating, np.arange(4.0), item_pre, O.make_rng(0).standard_normal((5, 6)) * 0.05)
    np.testing.assert_allclose(pi, 1.0 / 6, atol=1e-7)
    pi1 = np.zeros((2, 4))
    pi1[0, 2] = pi1[1, 0] = 1.0
    np.testing.assert_allclose(mol_score(pi1, np.arange(8.0).reshape(2, 4)), [2.0, 4.0])


def test_tie_break_ascending_id(prod):
    """Duplicated item rows force exact ties; they come out in ascending id order (mol.py:407)."""
    from paper_2306_04039_b200.mol import ItemCache, mol_top_k

    g, cache, gating = prod
    embs = cache.item_embs[:64].copy()
    gp = cache.item_gate_pre[:64].copy()
    for j in (17, 33, 50):
        embs[j], gp[j] = embs[5], gp[5]
    c2 = ItemCache(config=cache.config, item_embs=embs, item_gate_pre=gp, stage1_embs=embs.mean(1))
    ids, sc = mol_top_k(c2, gating, np.arange(64), qs(g, 0), 64)
    pos = [ids.tolist().index(i) for i in (5, 17, 33, 50)]
    assert pos == sorted(pos)
    assert len({float(sc[p]) for p in pos}) == 1


def test_mol_errors(prod):
    from paper_2306_04039_b200.errors import DimensionMismatchError, EmptyCandidatesError, OutOfRangeError
    from paper_2306_04039_b200.mol import mol_top_k, score_candidates

    g, cache, gating = prod
    with pytest.raises(EmptyCandidatesError):
        mol_top_k(cache, gating, [], qs(g, 0), 1)
    with pytest.raises(OutOfRangeError):
        mol_top_k(cache, gating, [1, 2], qs(g, 0), 3)
    with pytest.raises(OutOfRangeError):
        score_candidates(cache, gating, [0, cache.num_items], qs(g, 0))
    with pytest.raises(EmptyCandidatesError):
        score_candidates(cache, gating, [], qs(g, 0))
    from paper_2306_04039_b200.mol import QueryState

    with pytest.raises(DimensionMismatchError):
        score_candidates(cache, gating, [0], QueryState(np.zeros((8, 32)), g["user_feats"][0]))
    ids, _ = mol_top_k(cache, gating, [17], qs(g, 0), 1)
    assert ids.tolist() == [17]


def test_score_bounded_by_inverse_tau(prod):
    from paper_2306_04039_b200.mol import batch_score_all

    g, cache, gating = prod
    m = batch_score_all(cache, gating, g["user_embs"], g["user_feats"])
    assert np.abs(m).max() <= 1.0 / cache.config.tau + 1e-6


def test_f32_storage_path_non_bf16_cache(small):
    """A cache whose values are not bf16-representable is stored in f32 on the device (lossless)."""
    from paper_2306_04039_b200 import _lib as L
    from paper_2306_04039_b200.mol import score_candidates
    import ctypes as C

    g, cache, gating = small
    s = score_candidates(cache, gating, np.arange(cache.num_items), qs(g, 1))
    st = C.c_int()
    L.call("molr_cache_info", cache.device_handle(), None, C.byref(st), None)
    assert st.value & L.STORE_EMBS_F32 and st.value & L.STORE_GP_F32
    assert O.score_close(s, g["scores"][1], REL, ABS).all()


# ---------------------------------------------------------------------------------- quant
def test_quantize_bit_exact(golden):
    from paper_2306_04039_b200.quant import int8_dot, int8_matvec, quantize_rowwise, quantize_vector

    k = golden("known_answers")
    q = quantize_rowwise(np.array([[1.0, -1.0], [0.0, 0.0], [0.3, -0.7]], dtype=np.float32))
    assert np.array_equal(q.codes, k["kq_codes"]) and np.array_equal(q.scales, k["kq_scales"])
    q = quantize_rowwise(k["rq_in"])
    assert np.array_equal(q.codes, k["rq_codes"]) and np.array_equal(q.scales, k["rq_scales"])
    err = np.abs(q.dequantize() - k["rq_in"])
    assert np.all(err <= q.scales[:, None] / 2.0 + 1e-7 * np.maximum(1, np.abs(k["rq_in"])))
    assert int8_dot(np.array([127], np.int8), np.array([127], np.int8)) == 16129
    rng = O.make_rng(1)
    a = rng.integers(-127, 128, 100).astype(np.int8)
    b = rng.integers(-127, 128, 100).astype(np.int8)
    assert int8_dot(a, b) == sum(int(x) * int(y) for x, y in zip(a, b))
    m = rng.standard_normal((20, 16)).astype(np.float32)
    qr = quantize_rowwise(m)
    qv, _ = quantize_vector(rng.standard_normal(16).astype(np.float32))
    acc = int8_matvec(qr, qv)
    assert acc.dtype == np.int32
    assert np.array_equal(acc, O.int8_matvec(O.Quant(qr.codes, qr.scales), qv))


def test_quantize_large_bit_exact():
    from paper_2306_04039_b200.quant import quantize_rowwise

    rng = np.random.default_rng(5)
    m = (rng.standard_normal((200_000, 64)) * rng.uniform(1e-4, 10, (200_000, 1))).astype(np.float32)
    q = quantize_rowwise(m)
    r = O.quantize_rowwise(m)
    assert np.array_equal(q.codes, r.codes) and np.array_equal(q.scales, r.scales)


# ---------------------------------------------------------------------------------- stage 1
def test_stage1_scores_bit_exact(prod):
    from paper_2306_04039_b200.hindexer import exact_top_k, stage1_scores

    g, cache, gating = prod
    for u in range(g["user_embs"].shape[0]):
        q = g["stage1_query"][u]
        raw = stage1_scores(cache.stage1_q, q, raw_int_ordering=True)
        assert raw.dtype == np.int32 and np.array_equal(raw, g["s1_raw"][u])
        assert np.array_equal(stage1_scores(cache.stage1_q, q), g["s1_scaled"][u])
        # the float view's dot in OpenBLAS's sgemv order: the reference's fp32 `view @ q` bit for bit
        assert np.array_equal(stage1_scores(cache.stage1_embs, q), g["s1_float"][u])
        assert exact_top_k(cache.stage1_q, q, 50).tolist() == g["exact_top_k_q"][u].tolist()
        assert exact_top_k(cache.stage1_embs, q, 50).tolist() == g["exact_top_k_f"][u].tolist()


@pytest.mark.parametrize("tag,cfg_kw,view", [
    ("hq", dict(sample_ratio=0.1, quantized=True), "q"),
    ("hqs", dict(sample_ratio=0.1, quantized=True, comparator="strict"), "q"),
    ("hqr", dict(lam=300, quantized=True, raw_int_ordering=True), "q"),
    ("hf", dict(sample_ratio=0.1), "f"),
])
def test_h_indexer_matches_reference(prod, tag, cfg_kw, view):
    from paper_2306_04039_b200.hindexer import HIndexerConfig, estimate_threshold, h_indexer
    from paper_2306_04039_b200.numerics import make_rng

    g, cache, gating = prod
    v = cache.stage1_q if view == "q" else cache.stage1_embs
    cfg = HIndexerConfig(k_prime=150, **cfg_kw)
    offs = g[f"{tag}_offsets"]
    for u in range(g["user_embs"].shape[0]):
        r = h_indexer(v, g["stage1_query"][u], cfg, make_rng([9000, u]))
        ref = g[f"{tag}_ids"][offs[u]:offs[u + 1]]
        assert np.all(np.diff(r.indices) > 0)
        assert r.scanned == cache.num_items
        # bit-exact in both views: the int8 scores are exact integers, and the float view's dot
        # follows OpenBLAS's sgemv summation order, so it reproduces the reference's `view @ q`
        # (hindexer.py:112) bit for bit on these fixtures
        assert r.threshold == g[f"{tag}_t"][u]
        assert r.indices.tolist() == ref.tolist()
        t = estimate_threshold(v, g["stage1_query"][u], cfg, make_rng([9000, u]))
        assert t == g[f"{tag}_t_est"][u]


def test_h_indexer_edge_cases(golden):
    from paper_2306_04039_b200.errors import OutOfRangeError
    from paper_2306_04039_b200.hindexer import HIndexerConfig, h_indexer, nth_largest
    from paper_2306_04039_b200.numerics import make_rng

    k = golden("known_answers")
    inc = h_indexer(k["tie_items"], k["tie_query"], HIndexerConfig(k_prime=10, lam=55, d_prime=8), make_rng(13))
    stc = h_indexer(k["tie_items"], k["tie_query"], HIndexerConfig(k_prime=10, lam=55, d_prime=8,
                                                                    comparator="strict"), make_rng(13))
    assert inc.indices.tolist() == k["tie_inc_ids"].tolist()
    assert stc.indices.tolist() == k["tie_str_ids"].tolist()
    assert stc.threshold == inc.threshold and len(stc.indices) < len(inc.indices)
    for n, a in zip((1, 10, 100, 10_000), k["nth_answers"]):
        assert nth_largest(k["nth_values"], n) == a
    assert nth_largest([2.0, 2.0, 1.0], 2) == 2.0
    items = k["tie_items"][:32]
    r = h_indexer(items, k["tie_query"], HIndexerConfig(k_prime=32, lam=10, d_prime=8), make_rng(7))
    assert r.indices.tolist() == list(range(32)) and r.scanned == 32
    with pytest.raises(OutOfRangeError):
        h_indexer(items, k["tie_query"], HIndexerConfig(k_prime=33, lam=10, d_prime=8), make_rng(7))


def test_h_indexer_full_sample_superset_large():
    """lambda = X: the candidate set is a superset of the exact top-k' (hindexer.py:143-145), at
    a size where the O(X) scan matters (1M rows), int8 view bit-exact vs the oracle."""
    from paper_2306_04039_b200.hindexer import HIndexerConfig, exact_top_k, h_indexer
    from paper_2306_04039_b200.numerics import make_rng
    from paper_2306_04039_b200.quant import quantize_rowwise

    rng = np.random.default_rng(11)
    items = rng.standard_normal((1_000_000, 64)).astype(np.float32)
    items /= np.linalg.norm(items, axis=1, keepdims=True)
    q = quantize_rowwise(items)
    qo = O.Quant(q.codes, q.scales)
    query = rng.standard_normal(64).astype(np.float32)
    query /= np.linalg.norm(query)
    r = h_indexer(q, query, HIndexerConfig(k_prime=1000, lam=1_000_000, quantized=True), make_rng(1))
    assert set(exact_top_k(q, query, 1000).tolist()) <= set(r.indices.tolist())
    ri, rt, _ = O.h_indexer(qo, query, 1000, O.make_rng(2), sample_ratio=0.01)
    r2 = h_indexer(q, query, HIndexerConfig(k_prime=1000, sample_ratio=0.01, quantized=True), make_rng(2))
    assert r2.threshold == rt and np.array_equal(r2.indices, ri)


def test_index_select_byte_identical(prod):
    from paper_2306_04039_b200.errors import OutOfRangeError
    from paper_2306_04039_b200.hindexer import index_select

    g, cache, gating = prod
    idx = np.sort(np.random.default_rng(22).permutation(cache.num_items)[:170])
    out = index_select(cache, idx)
    assert out.item_embs.tobytes() == cache.item_embs[idx].tobytes()
    assert out.item_gate_pre.tobytes() == cache.item_gate_pre[idx].tobytes()
    assert out.stage1_embs.tobytes() == cache.stage1_embs[idx].tobytes()
    assert out.stage1_q.codes.tobytes() == cache.stage1_q.codes[idx].tobytes()
    assert index_select(cache, []).num_items == 0
    with pytest.raises(OutOfRangeError):
        index_select(cache, [5, 3])
    with pytest.raises(OutOfRangeError):
        index_select(cache, [5, cache.num_items])


# ---------------------------------------------------------------------------------- composition
def test_engine_composition_small(golden):
    """RetrievalEngine.query (engine.py:117-138) composed from the drop-in functions."""
    from paper_2306_04039_b200.hindexer import HIndexerConfig, h_indexer
    from paper_2306_04039_b200.mol import QueryState, mol_top_k
    from paper_2306_04039_b200.numerics import make_rng

    g = golden("engine_small")
    cache = product_cache(g, kind="small")
    gating = product_gating(g)
    hcfg = HIndexerConfig(k_prime=int(g["k_prime"]), sample_ratio=float(g["sample_ratio"]), d_prime=cache.config.d)
    X = cache.num_items
    for u in range(10):
        st = QueryState(user_embs=g["user_embs"][u], gate_features=g["user_feats"][u])
        cand = h_indexer(cache.stage1_embs, g["user_embs"][u].mean(axis=0), hcfg,
                         make_rng([int(g["seed"]), u])).indices
        if cand.size < 10:
            cand = np.arange(X)
        ids, sc = mol_top_k(cache, gating, cand, st, min(10, cand.size))
        assert ids.tolist() == g["query_ids"][u].tolist()
        assert O.score_close(sc, g["query_scores"][u], REL, ABS).all()


def test_two_stage_golden_quantized(prod):
    from paper_2306_04039_b200.hindexer import HIndexerConfig, h_indexer
    from paper_2306_04039_b200.mol import mol_top_k
    from paper_2306_04039_b200.numerics import make_rng

    g, cache, gating = prod
    hcfg = HIndexerConfig(k_prime=150, sample_ratio=0.1, quantized=True)
    for u in range(g["user_embs"].shape[0]):
        cand = h_indexer(cache.stage1_q, g["stage1_query"][u], hcfg, make_rng([9000, u])).indices
        ids, _ = mol_top_k(cache, gating, cand, qs(g, u), 20)
        assert topk_equal_modulo_ties(ids, g["two_stage_ids"][u], g["scores"][u])


def test_batched_two_stage_full_sample_equals_exact_pipeline(prod):
    """Batched device pipeline with lambda = X (sample-independent): candidate sets equal the
    oracle's h_indexer with lambda = X, so the final top-k equals the oracle's two-stage result."""
    from paper_2306_04039_b200.engine import two_stage_top_k
    from paper_2306_04039_b200.hindexer import HIndexerConfig

    g, cache, gating = prod
    X = cache.num_items
    U = g["user_embs"].shape[0]
    uw = gating.user_net(g["user_feats"])
    hcfg = HIndexerConfig(k_prime=150, lam=X, quantized=True)
    ids, sc, cand = two_stage_top_k(cache, gating, g["user_embs"], uw, 20, hcfg, seed=3)
    oc = O.Cache(cache.item_embs, cache.item_gate_pre, cache.stage1_embs, O.Quant(cache.stage1_q.codes,
                 cache.stage1_q.scales), cache.config.tau, cache.config.k_u)
    og = oracle_gating(g)
    for u in range(U):
        oi, os_ = O.two_stage_query(oc, og, g["user_embs"][u], g["user_feats"][u], 20, 150, O.make_rng(0),
                                    lam=X, quantized=True)
        c_ids, _, _ = O.h_indexer(oc.stage1_q, g["user_embs"][u].mean(axis=0), 150, O.make_rng(0), lam=X)
        assert cand[u] == c_ids.size
        assert topk_equal_modulo_ties(ids[u], oi, g["scores"][u])
        assert O.score_close(sc[u], g["scores"][u][ids[u]], REL, ABS).all()


def test_batched_two_stage_short_circuit_and_fallback(prod):
    from paper_2306_04039_b200.engine import two_stage_top_k
    from paper_2306_04039_b200.hindexer import HIndexerConfig

    g, cache, gating = prod
    X = cache.num_items
    uw = gating.user_net(g["user_feats"][:4])
    ids, sc, cand = two_stage_top_k(cache, gating, g["user_embs"][:4], uw, 10, HIndexerConfig(k_prime=X, lam=5))
    assert np.all(cand == X)
    for u in range(4):
        assert topk_equal_modulo_ties(ids[u], g["top_ids"][u][:10], g["scores"][u])
    # k' = 1 with k = 10: fewer than k passers -> whole corpus (engine.py:134-135)
    ids, sc, cand = two_stage_top_k(cache, gating, g["user_embs"][:4], uw, 10,
                                    HIndexerConfig(k_prime=1, lam=X, quantized=True))
    assert np.all(cand == X)
    for u in range(4):
        assert topk_equal_modulo_ties(ids[u], g["top_ids"][u][:10], g["scores"][u])


def test_merge_top_k_matches_global(prod):
    """Multi-GPU C1 merge: per-shard top-k lists merged == global top-k (scores are item-local)."""
    from paper_2306_04039_b200.engine import merge_top_k
    from paper_2306_04039_b200.mol import batch_mol_top_k

    g, cache, gating = prod
    X = cache.num_items
    shards = np.array_split(np.arange(X), 3)
    ids_l, sc_l = [], []
    for sh in shards:
        i, s = batch_mol_top_k(cache, gating, g["user_embs"], g["user_feats"], 50, candidates=[sh] * 16)
        ids_l.append(i)
        sc_l.append(s)
    mi, ms = merge_top_k(np.stack(ids_l), np.stack(sc_l), 50)
    fi, fs = batch_mol_top_k(cache, gating, g["user_embs"], g["user_feats"], 50)
    assert np.array_equal(mi, fi) and np.array_equal(ms, fs)


def test_launch_counter_moves():
    from paper_2306_04039_b200 import _lib as L
    from paper_2306_04039_b200.quant import quantize_rowwise

    before = L.launch_count()
    quantize_rowwise(np.ones((3, 8), np.float32))
    assert L.launch_count() > before


# ---------------------------------------------------------------------------------- tcgen05 path
def _synthetic_prod_cache(n_items, seed=0, gate_scale=1.0, n_users=32):
    """Production-shape synthetic corpus (bf16-representable) through the oracle generator."""
    from paper_2306_04039_b200.mol import ItemCache, MoLConfig
    from paper_2306_04039_b200.quant import quantize_rowwise

    syn = O.init_synthetic(n_users, n_items, k_u=8, k_x=8, d=64, gating_hidden=128, seed=seed)
    c = O.build_item_cache(syn.item_table, syn.item_proj, syn.gating.item_net, 8, 64, 20.0, 8, quantized=False)
    embs = O.round_bf16(c.item_embs)
    gp = O.round_bf16(c.item_gate_pre * gate_scale)
    s1 = embs.mean(axis=1).astype(np.float32)
    cfg = MoLConfig(k_u=8, k_x=8, d=64, tau=20.0, gating_hidden=128, dropout_p=0.0)
    cache = ItemCache(config=cfg, item_embs=embs, item_gate_pre=gp, stage1_embs=s1, stage1_q=quantize_rowwise(s1))
    ue = O.user_components(syn, np.arange(n_users), 8, 64).astype(np.float32)
    return cache, syn, ue, syn.user_table[:n_users]


def _prod_gating(syn, cross_scale=1.0):
    from paper_2306_04039_b200.mol import GatingNetwork, Mlp

    g = syn.gating
    cn = Mlp(g.cross_net.w1 * cross_scale, g.cross_net.b1 * cross_scale, g.cross_net.w2 * cross_scale)
    return GatingNetwork(Mlp(*g.user_net), Mlp(*g.item_net), cn), O.Gating(g.user_net, g.item_net, O.MlpW(*cn.__dict__.values()))


@pytest.mark.devknobs
@pytest.mark.parametrize("scale", [1.0, 4.0])
def test_tc_kernel_matches_oracle_dense(scale, monkeypatch):
    """The tcgen05 kernel (production shape) against the oracle on 20k items x 32 queries,
    default and x4 ("hard") gating; also against the generic SIMT kernel."""
    import os

    from paper_2306_04039_b200.mol import batch_score_all

    cache, syn, ue, feats = _synthetic_prod_cache(20_000, seed=5, gate_scale=scale)
    gating, og = _prod_gating(syn, cross_scale=scale)
    got = batch_score_all(cache, gating, ue, feats)
    oc = O.Cache(cache.item_embs, cache.item_gate_pre, cache.stage1_embs, None, 20.0, 8)
    ref = O.batch_score_all(oc, og, ue, feats)
    err = np.abs(got.astype(np.float64) - ref)
    print(f"scale={scale}: max |tc - oracle| = {err.max():.3e}, frac outside tol = "
          f"{1 - O.score_close(got, ref).mean():.2e}")
    assert O.score_close(got, ref, REL, ABS).all()
    gen = with_knob(monkeypatch, {"MOLR_DISABLE_TC": "1"}, lambda: batch_score_all(cache, gating, ue, feats))
    if gen is not None:  # dev build: the generic SIMT kernel on the same inputs
        assert O.score_close(gen, ref, REL, ABS).all()
    for u in range(ue.shape[0]):
        top_ref = np.lexsort((np.arange(ref.shape[1]), -ref[u]))[:100]
        top_got = np.lexsort((np.arange(got.shape[1]), -got[u]))[:100]
        assert topk_equal_modulo_ties(top_got, top_ref, ref[u])


def test_tc_kernel_candidates_partial_tiles():
    """Ragged candidate lists (1, 127, 128, 129, 1000 ids, unsorted, duplicated) through the tc kernel."""
    from paper_2306_04039_b200.mol import QueryState, batch_mol_top_k, score_candidates

    cache, syn, ue, feats = _synthetic_prod_cache(5_000, seed=9)
    gating, og = _prod_gating(syn)
    oc = O.Cache(cache.item_embs, cache.item_gate_pre, cache.stage1_embs, None, 20.0, 8)
    rng = np.random.default_rng(3)
    for n in (1, 127, 128, 129, 1000):
        ids = rng.integers(0, cache.num_items, n)
        got = score_candidates(cache, gating, ids, QueryState(ue[1], feats[1]))
        ref = O.score_candidates(oc, og, ids, ue[1], feats[1])
        assert O.score_close(got, ref, REL, ABS).all(), n
    lists = [rng.permutation(cache.num_items)[: rng.integers(100, 3000)] for _ in range(8)]
    ids, sc = batch_mol_top_k(cache, gating, ue[:8], feats[:8], 50, candidates=lists)
    for u in range(8):
        ref_all = np.full(cache.num_items, -np.inf)
        ref_all[lists[u]] = O.score_candidates(oc, og, lists[u], ue[u], feats[u])
        oi, _ = O.mol_top_k(oc, og, lists[u], ue[u], feats[u], 50)
        assert topk_equal_modulo_ties(ids[u], oi, ref_all)


@pytest.mark.parametrize("strict,raw", [(False, False), (True, False), (False, True)])
def test_batched_stage1_tc_counts_exact(strict, raw):
    """Tensor-core int8 scan + fused filter: with lambda = X the threshold is the exact n-th largest
    stage-1 score, so every query's passer count must equal the oracle's h_indexer count bit for bit
    (200k items, 300 queries = 3 query blocks, all comparator / ordering modes)."""
    from paper_2306_04039_b200.engine import two_stage_top_k
    from paper_2306_04039_b200.hindexer import HIndexerConfig

    cache, syn, ue, feats = _synthetic_prod_cache(200_000, seed=13, n_users=300)
    gating, og = _prod_gating(syn)
    X = cache.num_items
    kp = 2000
    hcfg = HIndexerConfig(k_prime=kp, lam=X, quantized=True, comparator="strict" if strict else "inclusive",
                          raw_int_ordering=raw)
    uw = gating.user_net(feats)
    ids, sc, cand = two_stage_top_k(cache, gating, ue, uw, 10, hcfg, seed=1)
    q = O.Quant(cache.stage1_q.codes, cache.stage1_q.scales)
    for u in range(ue.shape[0]):
        c_ids, t, _ = O.h_indexer(q, ue[u].mean(axis=0), kp, O.make_rng(0), lam=X,
                                  comparator="strict" if strict else "inclusive", raw_int_ordering=raw)
        assert cand[u] == c_ids.size, (u, cand[u], c_ids.size)


@pytest.mark.parametrize("nb", [1, 5, 16, 17, 32, 33])
@pytest.mark.devknobs
def test_batched_stage1_small_batch_kernel(nb, monkeypatch):
    """Small batches (B <= 32) take the items-in-M stage-1 kernel (queries in the MMA N dimension):
    exact passer counts vs the oracle at lambda = X for every comparator / ordering mode, and the
    sampled path (pilot WRITE + KEYS scans) identical to the 128-query-block kernel."""
    from paper_2306_04039_b200.engine import two_stage_top_k
    from paper_2306_04039_b200.hindexer import HIndexerConfig

    cache, syn, ue, feats = _synthetic_prod_cache(120_000, seed=31, n_users=64)
    gating, og = _prod_gating(syn)
    ue, feats = ue[:nb], feats[:nb]
    uw = gating.user_net(feats)
    X = cache.num_items
    q = O.Quant(cache.stage1_q.codes, cache.stage1_q.scales)
    for strict, raw in ((False, False), (True, False), (False, True)):
        comp = "strict" if strict else "inclusive"
        hcfg = HIndexerConfig(k_prime=1500, lam=X, quantized=True, comparator=comp, raw_int_ordering=raw)
        ids, sc, cand = two_stage_top_k(cache, gating, ue, uw, 10, hcfg, seed=1)
        for u in range(nb):
            c_ids, _, _ = O.h_indexer(q, ue[u].mean(axis=0), 1500, O.make_rng(0), lam=X, comparator=comp,
                                      raw_int_ordering=raw)
            assert cand[u] == c_ids.size, (strict, raw, u, cand[u], c_ids.size)
        hs = HIndexerConfig(k_prime=1500, sample_ratio=0.1, quantized=True, comparator=comp, raw_int_ordering=raw)
        a = two_stage_top_k(cache, gating, ue, uw, 20, hs, seed=5)
        b = with_knob(monkeypatch, {"MOLR_S1_NO_SMALL": "1"}, lambda: two_stage_top_k(cache, gating, ue, uw, 20, hs,
                                                                                       seed=5))
        for x, y in zip(a, b or a):
            np.testing.assert_array_equal(x, y)


@pytest.mark.parametrize("nb", [1, 3, 17, 300])
@pytest.mark.devknobs
def test_batched_float_view_tc_matches_fp32_scan(nb, monkeypatch):
    """Float stage-1 view (quantized=False, the reference default) on the tensor cores: bf16 MMA
    pre-test + exact fp32 re-check of the undecided band must give the SAME candidate sets as the
    fp32 SIMT filter scan (identical counts, identical top-k), for both comparators and for an
    exact threshold (lambda = X) and a sampled one; counts also match the oracle's NumPy h_indexer
    up to fp32 summation-order near-ties."""
    from paper_2306_04039_b200.engine import two_stage_top_k
    from paper_2306_04039_b200.hindexer import HIndexerConfig

    cache, syn, ue, feats = _synthetic_prod_cache(150_000, seed=41, n_users=nb)
    gating, og = _prod_gating(syn)
    uw = gating.user_net(feats)
    X = cache.num_items
    for comp in ("inclusive", "strict"):
        for kw in ({"lam": X}, {"sample_ratio": 0.05}):
            hcfg = HIndexerConfig(k_prime=1500, quantized=False, comparator=comp, **kw)
            a = two_stage_top_k(cache, gating, ue, uw, 20, hcfg, seed=3)
            # dev build: the fp32 SIMT filter scan on the same inputs
            b = with_knob(monkeypatch, {"MOLR_S1_NO_BF": "1"},
                          lambda: two_stage_top_k(cache, gating, ue, uw, 20, hcfg, seed=3)) or a
            np.testing.assert_array_equal(a[2], b[2])
            np.testing.assert_array_equal(a[0], b[0])
            np.testing.assert_array_equal(a[1], b[1])
            if "lam" in kw:
                for u in range(min(nb, 8)):
                    c_ids, _, _ = O.h_indexer(cache.stage1_embs, ue[u].mean(axis=0), 1500, O.make_rng(0), lam=X,
                                              comparator=comp)
                    assert abs(int(a[2][u]) - c_ids.size) <= 2, (comp, u, a[2][u], c_ids.size)


def _run_shards(fn, P):
    """Run fn(rank, exchange) for P in-process shards on threads, with a barrier all-gather."""
    import threading

    bar = threading.Barrier(P)
    slots = [None] * P
    out = [None] * P
    err = []

    def exchange_for(r):
        def ex(a):
            slots[r] = np.array(a, copy=True)
            bar.wait()
            res = np.stack(slots)
            bar.wait()
            return res
        return ex

    def body(r):
        try:
            out[r] = fn(r, exchange_for(r))
        except BaseException as e:  # keep the other shards from hanging
            err.append(e)
            bar.abort()

    th = [threading.Thread(target=body, args=(r,)) for r in range(P)]
    for t in th:
        t.start()
    for t in th:
        t.join()
    if err:
        raise err[0]
    return out


@pytest.mark.parametrize("quantized,comp,kp", [(True, "inclusive", 2000), (True, "strict", 2000),
                                               (False, "inclusive", 2000), (True, "inclusive", 5)])
def test_sharded_global_threshold_equals_single_device(quantized, comp, kp):
    """Item-range shards with the single-device-equivalent threshold: three uneven
    shards exchanging their top sample keys return EXACTLY the single-device two_stage_top_k result
    (ids, scores, candidate counts), int8 and float views, both comparators, and the global
    fallback to the whole corpus when K' < k."""
    from paper_2306_04039_b200.engine import two_stage_top_k, two_stage_top_k_sharded
    from paper_2306_04039_b200.hindexer import HIndexerConfig
    from paper_2306_04039_b200.mol import ItemCache
    from paper_2306_04039_b200.quant import QuantizedRows

    cache, syn, ue, feats = _synthetic_prod_cache(90_001, seed=51, n_users=40)
    gating, og = _prod_gating(syn)
    uw = gating.user_net(feats)
    X = cache.num_items
    hcfg = HIndexerConfig(k_prime=kp, sample_ratio=0.05, quantized=quantized, comparator=comp)
    ref = two_stage_top_k(cache, gating, ue, uw, 20, hcfg, seed=7)
    cuts = [0, 20_000, 61_111, X]
    shards = []
    for lo, hi in zip(cuts[:-1], cuts[1:]):
        q = cache.stage1_q
        shards.append(ItemCache(config=cache.config, item_embs=cache.item_embs[lo:hi],
                                item_gate_pre=cache.item_gate_pre[lo:hi], stage1_embs=cache.stage1_embs[lo:hi],
                                stage1_q=QuantizedRows(q.codes[lo:hi], q.scales[lo:hi])))
    res = _run_shards(lambda r, ex: two_stage_top_k_sharded(shards[r], gating, ue, uw, 20, hcfg, X_global=X,
                                                            row_lo=cuts[r], exchange=ex, seed=7), 3)
    for ids, sc, cnt in res:
        np.testing.assert_array_equal(cnt, ref[2])
        np.testing.assert_array_equal(ids, ref[0])
        np.testing.assert_array_equal(sc, ref[1])


@pytest.mark.parametrize("X", [300, 4099])
@pytest.mark.devknobs
def test_stage1_tc_paths_edge_cases(X, monkeypatch):
    """Tiny / ragged corpora through the small-batch int8 kernel, the 128-query int8 kernel and the
    fp16 float-view kernel: duplicated rows (exact ties at the threshold), an all-zero stage-1 row,
    an all-zero query and lambda = X (exact threshold); candidate counts and top-k must equal the
    SIMT scans' (MOLR_DISABLE_TC / MOLR_S1_NO_BF) and the oracle's counts."""
    from paper_2306_04039_b200.engine import two_stage_top_k
    from paper_2306_04039_b200.hindexer import HIndexerConfig
    from paper_2306_04039_b200.mol import ItemCache
    from paper_2306_04039_b200.quant import quantize_rowwise

    cache, syn, ue, feats = _synthetic_prod_cache(X, seed=61, n_users=40)
    gating, og = _prod_gating(syn)
    embs = cache.item_embs.copy()
    gp = cache.item_gate_pre.copy()
    embs[1::7] = embs[0]  # duplicated items -> tied stage-1 and MoL scores
    gp[1::7] = gp[0]
    embs[5] = 0.0  # an all-zero stage-1 row
    s1 = embs.mean(axis=1).astype(np.float32)
    cache = ItemCache(config=cache.config, item_embs=embs, item_gate_pre=gp, stage1_embs=s1,
                      stage1_q=quantize_rowwise(s1))
    ue = ue.copy()
    ue[3] = 0.0  # an all-zero stage-1 query (every score 0: everything ties)
    uw = gating.user_net(feats)
    q = O.Quant(cache.stage1_q.codes, cache.stage1_q.scales)
    kp = max(25, X // 20)
    for nb in (5, 40):  # small-batch kernel / 128-query kernel (and the float kernel for both)
        for quantized in (True, False):
            for comp in ("inclusive", "strict"):
                hcfg = HIndexerConfig(k_prime=kp, lam=X, quantized=quantized, comparator=comp)
                env = "MOLR_DISABLE_TC" if quantized else "MOLR_S1_NO_BF"
                a = two_stage_top_k(cache, gating, ue[:nb], uw[:nb], 10, hcfg, seed=2)
                b = with_knob(monkeypatch, {env: "1"},
                              lambda: two_stage_top_k(cache, gating, ue[:nb], uw[:nb], 10, hcfg, seed=2)) or a
                np.testing.assert_array_equal(a[2], b[2])
                np.testing.assert_array_equal(a[0], b[0])
                if quantized:  # (MOLR_DISABLE_TC also swaps the MoL kernel: scores within tolerance)
                    np.testing.assert_allclose(a[1], b[1], rtol=1e-3, atol=1e-6)
                    for u in range(nb):
                        c_ids, _, _ = O.h_indexer(q, ue[u].mean(axis=0), kp, O.make_rng(0), lam=X, comparator=comp)
                        want = X if c_ids.size < 10 else c_ids.size  # (corpus fallback below k)
                        assert a[2][u] == want, (nb, comp, u, a[2][u], c_ids.size)
                else:
                    np.testing.assert_array_equal(a[1], b[1])


def test_two_stage_at_short_lists_are_padded():
    """molr_two_stage_top_k_at keeps short candidate lists (no corpus fallback): the tail of a list
    shorter than k must be "no entry" (id -1, score -inf), never uninitialised memory (the merge
    drops such entries; a garbage tail once won the merge of a sharded query)."""
    from paper_2306_04039_b200 import _lib as L
    from paper_2306_04039_b200.mol import _gating_handle

    cache, syn, ue, feats = _synthetic_prod_cache(30_000, seed=71, n_users=24)
    gating, og = _prod_gating(syn)
    uw = L.f32(gating.user_net(feats))
    ue = L.f32(ue)
    B, k = ue.shape[0], 50
    # thresholds at each query's 10th-largest int8 score -> ~10 passers < k
    q = O.Quant(cache.stage1_q.codes, cache.stage1_q.scales)
    tk = np.empty(B, dtype=np.uint32)
    for u in range(B):
        sc = O.stage1_scores(q, ue[u].mean(axis=0))
        tk[u] = np.float32(np.sort(sc)[-10]).view(np.uint32) | np.uint32(0x80000000) if np.sort(sc)[-10] >= 0 \
            else ~np.float32(np.sort(sc)[-10]).view(np.uint32)
    for rep in range(3):
        ids = np.full((B, k), 12345, dtype=np.int64)
        scs = np.full((B, k), 7.0, dtype=np.float32)
        cnt = np.empty(B, dtype=np.int64)
        L.call("molr_two_stage_top_k_at", L.ctx(), cache.device_handle(), _gating_handle(gating), B, 8, L.ptr(ue),
               L.ptr(uw), 20.0, L.S1_INT8, 1000, L.ptr(tk), L.INCLUSIVE, k, 0, L.ptr(ids), L.ptr(scs), L.ptr(cnt), None)
        for u in range(B):
            c = int(cnt[u])
            assert 10 <= c < k, c
            assert np.all(ids[u, :c] >= 0) and np.all(np.isfinite(scs[u, :c]))
            assert np.all(ids[u, c:] == -1) and np.all(scs[u, c:] == -np.inf), (u, c, ids[u, c:c + 3])


def test_sharded_entry_points_validate():
    """The sharded entry points fail loudly on bad arguments (reference error classes): a shard
    outside the corpus, lambda outside [1, X], n outside [1, m], a null threshold array; and
    two_stage_top_k_sharded raises OutOfRangeError for K' > X like h_indexer (hindexer.py:60-61)."""
    from paper_2306_04039_b200 import _lib as L
    from paper_2306_04039_b200.engine import _mode, two_stage_top_k_sharded
    from paper_2306_04039_b200.errors import OutOfRangeError
    from paper_2306_04039_b200.hindexer import HIndexerConfig
    from paper_2306_04039_b200.mol import _gating_handle

    cache, syn, ue, feats = _synthetic_prod_cache(2_000, seed=81, n_users=4)
    gating, og = _prod_gating(syn)
    ue = L.f32(ue)
    keys = np.empty((4, 8), dtype=np.uint32)
    h = HIndexerConfig(k_prime=100, sample_ratio=0.1, quantized=True)
    with pytest.raises(OutOfRangeError):  # shard [1500, 3500) outside a 3000-row corpus
        L.call("molr_sample_top_keys", L.ctx(), cache.device_handle(), 4, 8, L.ptr(ue), _mode(h), 3000, 1500, 100, 1, 8,
               L.ptr(keys), None)
    with pytest.raises(OutOfRangeError):  # lambda > X
        L.call("molr_sample_top_keys", L.ctx(), cache.device_handle(), 4, 8, L.ptr(ue), _mode(h), 2000, 0, 5000, 1, 8,
               L.ptr(keys), None)
    out = np.empty(4, dtype=np.uint32)
    with pytest.raises(OutOfRangeError):  # n > m
        L.call("molr_select_nth_keys", L.ctx(), 4, 8, L.ptr(keys), 9, L.ptr(out), None)
    ids = np.empty((4, 5), dtype=np.int64)
    sc = np.empty((4, 5), dtype=np.float32)
    with pytest.raises(Exception):  # null thresholds
        L.call("molr_two_stage_top_k_at", L.ctx(), cache.device_handle(), _gating_handle(gating), 4, 8, L.ptr(ue),
               L.ptr(L.f32(gating.user_net(feats))), 20.0, _mode(h), 100, None, L.INCLUSIVE, 5, 0, L.ptr(ids), L.ptr(sc),
               None, None)
    with pytest.raises(OutOfRangeError):
        two_stage_top_k_sharded(cache, gating, ue, gating.user_net(feats), 5,
                                HIndexerConfig(k_prime=5000, sample_ratio=0.1, quantized=True), X_global=2000, row_lo=0,
                                exchange=lambda a: np.asarray(a)[None])


@pytest.mark.devknobs
def test_batched_two_stage_more_than_1024_queries(monkeypatch):
    """B = 1100 > 1024 (two query chunks per scan, the second a small-batch chunk) through the int8
    and the float tensor-core filters: counts and top-k identical to the SIMT scans."""
    from paper_2306_04039_b200.engine import two_stage_top_k
    from paper_2306_04039_b200.hindexer import HIndexerConfig

    cache, syn, ue, feats = _synthetic_prod_cache(20_000, seed=91, n_users=1100)
    gating, og = _prod_gating(syn)
    uw = gating.user_net(feats)
    for quantized, env in ((True, "MOLR_S1_NO_TC"), (False, "MOLR_S1_NO_BF")):  # (filter-only switches)
        hcfg = HIndexerConfig(k_prime=400, sample_ratio=0.1, quantized=quantized)
        a = two_stage_top_k(cache, gating, ue, uw, 10, hcfg, seed=4)
        b = with_knob(monkeypatch, {env: "1"}, lambda: two_stage_top_k(cache, gating, ue, uw, 10, hcfg, seed=4)) or a
        assert np.all(a[2] > 0)
        np.testing.assert_array_equal(a[2], b[2])
        np.testing.assert_array_equal(a[0], b[0])


def test_batched_two_stage_recall_device_sample():
    """Device-drawn sample (lambda = 1% of X): candidate counts near K' and top-100 recall vs the
    oracle's exact MoL top-100 >= 0.99 (north-star bar), 100k items."""
    from paper_2306_04039_b200.engine import two_stage_top_k
    from paper_2306_04039_b200.hindexer import HIndexerConfig

    cache, syn, ue, feats = _synthetic_prod_cache(100_000, seed=21, n_users=64)
    gating, og = _prod_gating(syn)
    hcfg = HIndexerConfig(k_prime=5000, sample_ratio=0.05, quantized=True)
    uw = gating.user_net(feats)
    ids, sc, cand = two_stage_top_k(cache, gating, ue, uw, 100, hcfg, seed=7)
    assert np.all(np.abs(cand - 5000) < 5000 * 0.25), cand
    oc = O.Cache(cache.item_embs, cache.item_gate_pre, cache.stage1_embs, None, 20.0, 8)
    rec = []
    for u in range(16):
        ex, _ = O.full_top_k(oc, og, ue[u], feats[u], 100)
        rec.append(len(set(ex.tolist()) & set(ids[u].tolist())) / 100)
    print("recall", np.mean(rec))
    assert np.mean(rec) >= 0.99


@pytest.mark.parametrize("strict,raw,quantized", [(False, False, True), (True, False, True), (False, True, True),
                                                  (False, False, False), (True, False, False)])
@pytest.mark.devknobs
def test_sample_threshold_pilot_exact(strict, raw, quantized, monkeypatch):
    """The pilot-filtered sample threshold (score a subsample, keep only sample rows above a low
    pilot threshold, select among them) must give the SAME threshold as scoring the whole sample:
    identical candidate counts and top-k for pilot / no pilot / forced fallback (pilot threshold
    too high -> full sample)."""
    from paper_2306_04039_b200.engine import two_stage_top_k
    from paper_2306_04039_b200.hindexer import HIndexerConfig

    cache, syn, ue, feats = _synthetic_prod_cache(300_000, seed=17, n_users=200)
    gating, og = _prod_gating(syn)
    hcfg = HIndexerConfig(k_prime=3000, sample_ratio=0.2, quantized=quantized,
                          comparator="strict" if strict else "inclusive", raw_int_ordering=raw)
    uw = gating.user_net(feats)
    runs = {"pilot": two_stage_top_k(cache, gating, ue, uw, 50, hcfg, seed=11)}
    for tag, env in (("full", {"MOLR_NO_PILOT": "1"}), ("fallback", {"MOLR_PILOT_N0": "1"})):
        r = with_knob(monkeypatch, env, lambda: two_stage_top_k(cache, gating, ue, uw, 50, hcfg, seed=11))
        if r is not None:  # dev build: whole-sample threshold / forced pilot fallback
            runs[tag] = r
    for tag in [x for x in ("full", "fallback") if x in runs]:
        np.testing.assert_array_equal(runs["pilot"][2], runs[tag][2])
        np.testing.assert_array_equal(runs["pilot"][0], runs[tag][0])
        np.testing.assert_array_equal(runs["pilot"][1], runs[tag][1])
    assert np.all(np.abs(runs["pilot"][2] - 3000) < 3000 * 0.3)


def test_topk_sampled_bound_path_ties():
    """The segmented top-k's sampled-bound fast path (n >= 32 k) keeps the reference order
    (score desc, id asc — np.lexsort((ids, -scores)), mol.py:407) with massive ties: 40 distinct
    items each repeated 250 times, top-100 = ties across the boundary, ragged candidate lists."""
    from paper_2306_04039_b200.mol import ItemCache, MoLConfig, QueryState, batch_mol_top_k, mol_top_k
    from paper_2306_04039_b200.quant import quantize_rowwise

    cache0, syn, ue, feats = _synthetic_prod_cache(40, seed=23, n_users=6)
    gating, og = _prod_gating(syn)
    rep = np.tile(np.arange(40), 250)
    embs, gp = cache0.item_embs[rep], cache0.item_gate_pre[rep]
    s1 = embs.mean(axis=1).astype(np.float32)
    cfg = MoLConfig(k_u=8, k_x=8, d=64, tau=20.0, gating_hidden=128, dropout_p=0.0)
    cache = ItemCache(config=cfg, item_embs=embs, item_gate_pre=gp, stage1_embs=s1, stage1_q=quantize_rowwise(s1))
    oc = O.Cache(cache.item_embs, cache.item_gate_pre, cache.stage1_embs, None, 20.0, 8)
    X = cache.num_items
    rng = np.random.default_rng(4)
    lists = [np.arange(X), rng.permutation(X)[:7000], rng.permutation(X)[:3300]]
    for u in range(3):
        ids, sc = mol_top_k(cache, gating, lists[u], QueryState(ue[u], feats[u]), 100)
        oi, osc = O.mol_top_k(oc, og, lists[u], ue[u], feats[u], 100)
        ref_all = np.full(X, -np.inf)
        ref_all[lists[u]] = O.score_candidates(oc, og, lists[u], ue[u], feats[u])
        assert topk_equal_modulo_ties(ids, oi, ref_all)
        # among equal GPU scores the ids ascend (the reference's tie-break)
        for a in range(99):
            if sc[a] == sc[a + 1]:
                assert ids[a] < ids[a + 1]
    bi, bs = batch_mol_top_k(cache, gating, ue[:4], feats[:4], 100)
    for u in range(4):
        oi, _ = O.mol_top_k(oc, og, np.arange(X), ue[u], feats[u], 100)
        ref_all = O.score_candidates(oc, og, np.arange(X), ue[u], feats[u])
        assert topk_equal_modulo_ties(bi[u], oi, ref_all)


@pytest.mark.parametrize("cross_scale,gate_scale", [(1.0, 1.0), (4.0, 4.0), (16.0, 16.0), (1.0, 64.0), (16.0, 64.0)])
def test_tc_kernel_precision_margin(cross_scale, gate_scale):
    """Precision budget of the tcgen05 MoL kernel's cross net (query hi/lo split component GEMM,
    three-pass bf16 hi/lo L1 with hi/lo bias, three-pass fp16 hi/lo L2, ex2 + rcp SiLU; DESIGN.md
    K1; a single bf16 / fp16 pass with tanh.approx used 9x the tolerance at x16) against the
    oracle, from the default init to x16-sharpened cross nets and x64 gate pre-activations (large
    |uw * gate_pre| arguments of the combine SiLU and a near-one-hot softmax): the worst
    |s_gpu - s_ref| / (1e-3 |s_ref| + 1e-6) must stay <= 0.5, i.e. at least a 2x margin inside the
    north_star tolerance."""
    from paper_2306_04039_b200.mol import batch_score_all

    cache, syn, ue, feats = _synthetic_prod_cache(8_000, seed=9, gate_scale=gate_scale, n_users=16)
    gating, og = _prod_gating(syn, cross_scale=cross_scale)
    got = batch_score_all(cache, gating, ue, feats).astype(np.float64)
    oc = O.Cache(cache.item_embs, cache.item_gate_pre, cache.stage1_embs, None, 20.0, 8)
    ref = O.batch_score_all(oc, og, ue, feats).astype(np.float64)
    budget = np.abs(got - ref) / (1e-3 * np.abs(ref) + 1e-6)
    print(f"cross x{cross_scale} gate x{gate_scale}: max |err| {np.abs(got - ref).max():.3e}, "
          f"worst fraction of the tolerance used {budget.max():.3f}")
    assert budget.max() <= 0.5


def _f32_prod_cache(n_items, seed=0, n_users=16, gate_f32=True):
    """Production-shape corpus built in f32 like the reference's build_item_cache (mol.py:294-326):
    item components and (optionally) gate pre-activations NOT bf16-representable, so the cache
    stores them in f32 and the tcgen05 scorer runs on the bf16 hi + lo image."""
    from paper_2306_04039_b200.mol import ItemCache, MoLConfig
    from paper_2306_04039_b200.quant import quantize_rowwise

    syn = O.init_synthetic(n_users, n_items, k_u=8, k_x=8, d=64, gating_hidden=128, seed=seed)
    c = O.build_item_cache(syn.item_table, syn.item_proj, syn.gating.item_net, 8, 64, 20.0, 8, quantized=False)
    embs = np.ascontiguousarray(c.item_embs, dtype=np.float32)
    gp = np.ascontiguousarray(c.item_gate_pre if gate_f32 else O.round_bf16(c.item_gate_pre), dtype=np.float32)
    s1 = embs.mean(axis=1).astype(np.float32)
    cfg = MoLConfig(k_u=8, k_x=8, d=64, tau=20.0, gating_hidden=128, dropout_p=0.0)
    cache = ItemCache(config=cfg, item_embs=embs, item_gate_pre=gp, stage1_embs=s1, stage1_q=quantize_rowwise(s1))
    ue = O.user_components(syn, np.arange(n_users), 8, 64).astype(np.float32)
    return cache, syn, ue, syn.user_table[:n_users]


@pytest.mark.parametrize("gate_f32", [True, False])
@pytest.mark.parametrize("scale", [1.0, 4.0])
def test_tc_kernel_f32_cache(gate_f32, scale):
    """A reference-built (f32, not bf16-representable) cache is served by the tcgen05 kernel
    through its bf16 hi + lo component image (two component passes; f32 gate pre-activations read
    directly): scores within the tolerance of the oracle with a 2x margin (default and x4 gating),
    exact top-k modulo ties, and the same through score_candidates / mol_top_k (ragged lists)."""
    from paper_2306_04039_b200.mol import QueryState, batch_score_all, mol_top_k, score_candidates, uses_tensor_cores

    cache, syn, ue, feats = _f32_prod_cache(12_000, seed=21, gate_f32=gate_f32)
    assert O.round_bf16(cache.item_embs).tobytes() != cache.item_embs.tobytes()  # really f32
    gating, og = _prod_gating(syn, cross_scale=scale)
    assert uses_tensor_cores(cache, gating)
    got = batch_score_all(cache, gating, ue, feats).astype(np.float64)
    oc = O.Cache(cache.item_embs, cache.item_gate_pre, cache.stage1_embs, None, 20.0, 8)
    ref = O.batch_score_all(oc, og, ue, feats).astype(np.float64)
    budget = np.abs(got - ref) / (1e-3 * np.abs(ref) + 1e-6)
    print(f"f32 cache (gate f32 {gate_f32}) x{scale}: max |err| {np.abs(got - ref).max():.3e}, "
          f"worst fraction of the tolerance used {budget.max():.3f}")
    assert budget.max() <= 0.5
    rng = np.random.default_rng(3)
    for u in range(4):
        top_ref = np.lexsort((np.arange(ref.shape[1]), -ref[u]))[:100]
        top_got = np.lexsort((np.arange(got.shape[1]), -got[u]))[:100]
        assert topk_equal_modulo_ties(top_got, top_ref, ref[u])
        ids = np.sort(rng.choice(cache.num_items, size=int(rng.integers(60, 3000)), replace=False))
        q = QueryState(user_embs=ue[u], gate_features=feats[u])
        sc = score_candidates(cache, gating, ids, q)
        assert O.score_close(sc, ref[u][ids]).all()
        ti, ts = mol_top_k(cache, gating, ids, q, 50)
        assert topk_equal_modulo_ties(ti, O.mol_top_k(oc, og, ids, ue[u], feats[u], 50)[0], np.where(
            np.isin(np.arange(cache.num_items), ids), ref[u], -np.inf))
    # index_select of an f32 cache rebuilds the selection's hi + lo image: same scores, same backend
    from paper_2306_04039_b200.hindexer import index_select

    ids = np.sort(rng.choice(cache.num_items, size=777, replace=False))
    sub = index_select(cache, ids)
    assert uses_tensor_cores(sub, gating)
    q = QueryState(user_embs=ue[0], gate_features=feats[0])
    np.testing.assert_array_equal(score_candidates(sub, gating, np.arange(ids.size), q),
                                  score_candidates(cache, gating, ids, q))
