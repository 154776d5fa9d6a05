"""Pin the CPU oracle (oracle/) against golden vectors produced by the reference itself
(tests/golden/make_golden.py).  CPU only."""

import numpy as np
import pytest

import oracle as O


def gating_of(g):
    mk = lambda p: O.MlpW(g[p + ".w1"], g[p + ".b1"], g[p + ".w2"])  # noqa: E731
    zero = O.MlpW(np.zeros((1, 1)), np.zeros(1), np.zeros((1, 1)))
    return O.Gating(mk("user_net"), zero, mk("cross_net"))


def bf16_to_f32(u16):
    return (u16.astype(np.uint32) << 16).view(np.float32)


def prod_cache(g):
    embs = bf16_to_f32(g["item_embs_bf16"])
    gp = bf16_to_f32(g["item_gate_pre_bf16"])
    return O.Cache(embs, gp, g["stage1_embs"], O.Quant(g["stage1_codes"], g["stage1_scales"]),
                   float(g["tau"]), g["user_embs"].shape[1])


def test_small_scores_topk_batch(golden):
    g = golden("small_mol")
    cache = O.Cache(g["item_embs"], g["item_gate_pre"], g["stage1_embs"], None, float(g["tau"]),
                    g["user_embs"].shape[1])
    gt = gating_of(g)
    X = cache.item_embs.shape[0]
    for u in range(g["user_embs"].shape[0]):
        s = O.score_candidates(cache, gt, np.arange(X), g["user_embs"][u], g["user_feats"][u])
        np.testing.assert_allclose(s, g["scores"][u], rtol=1e-5, atol=1e-7)
        ids, sc = O.mol_top_k(cache, gt, np.arange(X), g["user_embs"][u], g["user_feats"][u], 10)
        assert ids.tolist() == g["top_ids"][u].tolist()
    m = O.batch_score_all(cache, gt, g["user_embs"], g["user_feats"], pairs_per_chunk=700)
    np.testing.assert_allclose(m, g["batch_all"], rtol=1e-5, atol=1e-7)
    cl = O.component_logits(g["user_embs"][0], cache.item_embs[:20], cache.tau)
    np.testing.assert_allclose(cl, g["cl_u0"], rtol=1e-5, atol=1e-8)
    pi = O.decomposed_gating(gt, g["user_feats"][0], cache.item_gate_pre[:20], cl)
    np.testing.assert_allclose(pi, g["pi_u0"], rtol=1e-5, atol=1e-8)


def test_production_scores_and_topk(golden):
    g = golden("production_mol")
    cache = prod_cache(g)
    gt = gating_of(g)
    X = cache.item_embs.shape[0]
    for u in range(g["user_embs"].shape[0]):
        s = O.score_candidates(cache, gt, np.arange(X), g["user_embs"][u], g["user_feats"][u])
        assert O.score_close(s, g["scores"][u], rel=1e-5, abs_=1e-8).all()
        ids, _ = O.mol_top_k(cache, gt, np.arange(X), g["user_embs"][u], g["user_feats"][u], 100)
        assert ids.tolist() == g["top_ids"][u].tolist()
    m = O.batch_score_all(cache, gt, g["user_embs"], g["user_feats"])
    assert O.score_close(m, g["batch_all"], rel=1e-5, abs_=1e-8).all()


def test_production_stage1_bit_exact(golden):
    g = golden("production_mol")
    cache = prod_cache(g)
    for u in range(g["user_embs"].shape[0]):
        q = g["stage1_query"][u]
        codes, scale = O.quantize_vector(q)
        assert codes.tolist() == g["query_codes"][u].tolist()
        assert np.float32(scale) == g["query_scales"][u]
        raw = O.stage1_scores(cache.stage1_q, q, raw_int_ordering=True)
        assert raw.dtype == np.int32 and np.array_equal(raw, g["s1_raw"][u])
        sc = O.stage1_scores(cache.stage1_q, q)
        assert np.array_equal(sc, g["s1_scaled"][u])
        np.testing.assert_allclose(O.stage1_scores(cache.stage1_embs, q), g["s1_float"][u], rtol=1e-5,
                                   atol=1e-7)
        assert O.exact_top_k(cache.stage1_q, q, 50).tolist() == g["exact_top_k_q"][u].tolist()


@pytest.mark.parametrize("tag,kw,view", [
    ("hq", dict(sample_ratio=0.1), "q"),
    ("hqs", dict(sample_ratio=0.1, comparator="strict"), "q"),
    ("hqr", dict(lam=300, raw_int_ordering=True), "q"),
    ("hf", dict(sample_ratio=0.1), "f"),
])
def test_production_h_indexer(golden, tag, kw, view):
    g = golden("production_mol")
    cache = prod_cache(g)
    v = cache.stage1_q if view == "q" else cache.stage1_embs
    offs = g[f"{tag}_offsets"]
    for u in range(g["user_embs"].shape[0]):
        ids, t, scanned = O.h_indexer(v, g["stage1_query"][u], 150, O.make_rng([9000, u]), **kw)
        ref = g[f"{tag}_ids"][offs[u]:offs[u + 1]]
        if view == "q":  # integer accumulators: bit-exact
            assert t == g[f"{tag}_t"][u]
            assert ids.tolist() == ref.tolist()
        else:  # BLAS sgemv summation order is not pinned: threshold within fp32 noise
            assert abs(t - g[f"{tag}_t"][u]) <= 1e-6
            assert len(set(ids.tolist()) ^ set(ref.tolist())) <= 2
        rest = {k: v2 for k, v2 in kw.items() if k != "comparator"}
        te = O.estimate_threshold(v, g["stage1_query"][u], 150, O.make_rng([9000, u]), **rest)
        assert abs(te - g[f"{tag}_t_est"][u]) <= (0 if view == "q" else 1e-6)


def test_production_two_stage(golden):
    g = golden("production_mol")
    cache = prod_cache(g)
    gt = gating_of(g)
    for u in range(g["user_embs"].shape[0]):
        ids, _ = O.two_stage_query(cache, gt, g["user_embs"][u], g["user_feats"][u], 20, 150,
                                   O.make_rng([9000, u]), sample_ratio=0.1, quantized=True)
        assert ids.tolist() == g["two_stage_ids"][u].tolist()


def test_known_answers(golden):
    g = golden("known_answers")
    q = O.quantize_rowwise(np.array([[1.0, -1.0], [0.0, 0.0], [0.3, -0.7]], dtype=np.float32))
    assert np.array_equal(q.codes, g["kq_codes"]) and np.array_equal(q.scales, g["kq_scales"])
    assert q.codes[0].tolist() == [127, -127] and q.scales[1] == 1.0
    q = O.quantize_rowwise(g["rq_in"])
    assert np.array_equal(q.codes, g["rq_codes"]) and np.array_equal(q.scales, g["rq_scales"])
    assert int(g["dot_max"]) == 16129
    for n, a in zip((1, 10, 100, 10_000), g["nth_answers"]):
        assert O.nth_largest(g["nth_values"], n) == a
    inc = O.h_indexer(g["tie_items"], g["tie_query"], 10, O.make_rng(13), lam=55)
    stc = O.h_indexer(g["tie_items"], g["tie_query"], 10, O.make_rng(13), lam=55, comparator="strict")
    assert inc[0].tolist() == g["tie_inc_ids"].tolist() and inc[1] == g["tie_inc_t"]
    assert stc[0].tolist() == g["tie_str_ids"].tolist() and stc[1] == g["tie_str_t"]
    assert len(stc[0]) < len(inc[0])


def test_engine_small(golden):
    g = golden("engine_small")
    cache = O.Cache(g["item_embs"], g["item_gate_pre"], g["stage1_embs"], None, float(g["tau"]),
                    g["user_embs"].shape[1])
    gt = gating_of(g)
    for u in range(10):
        ids, sc = O.two_stage_query(cache, gt, g["user_embs"][u], g["user_feats"][u], 10,
                                    int(g["k_prime"]), O.make_rng([int(g["seed"]), u]),
                                    sample_ratio=float(g["sample_ratio"]))
        assert ids.tolist() == g["query_ids"][u].tolist()
        np.testing.assert_allclose(sc, g["query_scores"][u], rtol=1e-5, atol=1e-8)
        fids, _ = O.full_top_k(cache, gt, g["user_embs"][u], g["user_feats"][u], 10)
        assert fids.tolist() == g["full_ids"][u].tolist()


def test_bf16_rounding_helper():
    x = np.array([1.0, 1.00390625, 1.005859375, -3.14159, 0.0], dtype=np.float32)
    r = O.round_bf16(x)
    assert r[0] == 1.0 and r[1] == 1.0  # tie -> even
    assert r[2] == np.float32(1.0078125)
    assert (r.view(np.uint32) & 0xFFFF).max() == 0
