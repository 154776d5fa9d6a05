"""Pin the C restatement of the MoL scorer (oracle/molr_oracle.c) against the golden vectors the
reference produced (tests/golden/make_golden.py) and against the NumPy restatement.  CPU only."""

import numpy as np

import oracle as O
from oracle import c_oracle as CO


def _bits_to_f32(u16):
    return (u16.astype(np.uint32) << 16).view(np.float32)


def _cross(g):
    return CO.Net(g["cross_net.w1"], g["cross_net.b1"], g["cross_net.w2"])


def _uw(g):
    return O.mlp(O.MlpW(g["user_net.w1"], g["user_net.b1"], g["user_net.w2"]), g["user_feats"]).astype(np.float32)


def test_c_oracle_matches_reference_goldens_bf16_items(golden):
    """production shape (k_u = k_x = 8, d = 64, H = 128), items passed as bf16 bits."""
    g = golden("production_mol")
    s = CO.scores(g["item_embs_bf16"], g["item_gate_pre_bf16"], g["user_embs"], _uw(g), _cross(g), float(g["tau"]))
    assert O.score_close(s, g["scores"], rel=1e-5, abs_=1e-8).all()
    assert np.abs(s - g["scores"]).max() < 1e-7
    # the same items widened to f32 give the same bits
    s32 = CO.scores(_bits_to_f32(g["item_embs_bf16"]), _bits_to_f32(g["item_gate_pre_bf16"]), g["user_embs"], _uw(g),
                    _cross(g), float(g["tau"]))
    assert np.array_equal(s, s32)


def test_c_oracle_topk_matches_reference_goldens(golden):
    g = golden("production_mol")
    s = CO.scores(g["item_embs_bf16"], g["item_gate_pre_bf16"], g["user_embs"], _uw(g), _cross(g), float(g["tau"]))
    tk = CO.TopK(s.shape[0], 100)
    for lo in range(0, s.shape[1], 317):  # chunked merge == one pass
        tk.add(s[:, lo:lo + 317], lo)
    for u in range(s.shape[0]):
        assert tk.ids[u].tolist() == g["top_ids"][u].tolist()
        order = np.lexsort((np.arange(s.shape[1]), -s[u]))[:100]
        assert tk.ids[u].tolist() == order.tolist()


def test_c_oracle_small_shapes_match_reference(golden):
    """a non-production shape (the small_mol golden) through the same code."""
    g = golden("small_mol")
    uw = _uw(g)
    s = CO.scores(g["item_embs"], g["item_gate_pre"], g["user_embs"], uw, _cross(g), float(g["tau"]))
    np.testing.assert_allclose(s, g["scores"], rtol=1e-5, atol=1e-7)


def test_c_oracle_candidates_and_ties():
    rng = np.random.default_rng(3)
    n, k_u, k_x, d, H = 300, 4, 4, 16, 32
    G = k_u * k_x
    e = rng.standard_normal((n, k_x, d)).astype(np.float32)
    e /= np.linalg.norm(e, axis=-1, keepdims=True)
    e[7] = e[3]  # duplicate items -> exact score ties
    gp = rng.standard_normal((n, G)).astype(np.float32)
    gp[7] = gp[3]
    ue = rng.standard_normal((2, k_u, d)).astype(np.float32)
    ue /= np.linalg.norm(ue, axis=-1, keepdims=True)
    uw = rng.standard_normal((2, G)).astype(np.float32)
    net = CO.Net(rng.standard_normal((G, H)) * 0.3, rng.standard_normal(H) * 0.1, rng.standard_normal((H, G)) * 0.3)
    full = CO.scores(e, gp, ue, uw, net, 20.0)
    lists = [np.array([5, 3, 7, 3, 250]), np.arange(n)[::-1]]
    got = CO.score_candidates(e, gp, ue, uw, net, 20.0, lists)
    for b in range(2):
        assert np.array_equal(got[b], full[b, lists[b]])
    # NumPy restatement of the same pairs (mol.py:329-345)
    cache = O.Cache(e, gp, e.mean(axis=1), None, 20.0, k_u)
    gate = O.Gating(None, None, O.MlpW(net.w1, net.b1, net.w2))
    for b in range(2):
        ref = O.score_candidates(cache, gate, np.arange(n), ue[b], None, uw=uw[b])
        assert np.abs(ref - full[b]).max() < 1e-6
    assert full[0, 3] == full[0, 7]
    tk = CO.TopK(2, 10).add(full, 0)
    for b in range(2):
        assert tk.ids[b].tolist() == np.lexsort((np.arange(n), -full[b]))[:10].tolist()
