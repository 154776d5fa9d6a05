"""Generate the golden vectors in tests/golden/ by running the REFERENCE itself.

Run in the build container only (the reference is not present on the GPU box):

    PYTHONPATH=/root/reference/pkg/src python tests/golden/make_golden.py

Every array in the fixtures is either an input handed to the reference or an output the
reference produced from those inputs through its public API (`molr.mol`, `molr.hindexer`,
`molr.quant`, `molr.engine`).  Item-side caches at the production shape are rounded to
bf16-representable float32 before the reference sees them, so the
same bytes can be uploaded to the GPU without loss.
"""

from __future__ import annotations

import os
import sys

import numpy as np

sys.path.insert(0, "/root/reference/pkg/src")

from molr.engine import RetrievalEngine  # noqa: E402
from molr.hindexer import (  # noqa: E402
    HIndexerConfig, estimate_threshold, exact_top_k, h_indexer, nth_largest, stage1_scores,
)
from molr.mol import (  # noqa: E402
    ItemCache, MoLConfig, QueryState, batch_score_all, build_item_cache, component_logits,
    decomposed_gating, mol_top_k, score_candidates,
)
from molr.model import TowerDims, init_params, user_components  # noqa: E402
from molr.numerics import make_rng  # noqa: E402
from molr.quant import int8_matvec, quantize_rowwise, quantize_vector  # noqa: E402

OUT = os.path.dirname(os.path.abspath(__file__))


def bf16(x):
    x = np.ascontiguousarray(x, dtype=np.float32)
    u = x.view(np.uint32).astype(np.uint64)
    u = (u + 0x7FFF + ((u >> 16) & 1)) & 0xFFFF0000
    return u.astype(np.uint32).view(np.float32).reshape(x.shape)


def mlp_arrays(prefix, m):
    return {f"{prefix}.w1": m.w1, f"{prefix}.b1": m.b1, f"{prefix}.w2": m.w2}


def small_case():
    """test_mol.py:221-227 small_model shape: k_u=2, k_x=3, d=8, H=16, 500 items."""
    cfg = MoLConfig(k_u=2, k_x=3, d=8, tau=20.0, gating_hidden=16, dropout_p=0.0)
    dims = TowerDims(n_users=30, n_items=500, d_u=12, d_x=12, proj_hidden=24)
    params = init_params(dims, cfg, make_rng(42))
    cache = build_item_cache(params.item_table, params.item_proj, params.gating.item_net, cfg)
    users = np.arange(6)
    embs = user_components(params, users, cfg).astype(np.float32)
    feats = params.user_table[users].astype(np.float32)
    out = {
        "item_embs": cache.item_embs, "item_gate_pre": cache.item_gate_pre,
        "stage1_embs": cache.stage1_embs, "user_embs": embs, "user_feats": feats,
        "tau": np.float32(cfg.tau),
    }
    for name, m in (("user_net", params.gating.user_net), ("cross_net", params.gating.cross_net)):
        out.update(mlp_arrays(name, m))
    scores, top_ids, top_scores = [], [], []
    for u in users:
        st = QueryState(user_embs=embs[u], gate_features=feats[u])
        scores.append(score_candidates(cache, params.gating, np.arange(500), st))
        i, s = mol_top_k(cache, params.gating, np.arange(500), st, 10)
        top_ids.append(i)
        top_scores.append(s)
    out["scores"] = np.stack(scores).astype(np.float32)
    out["top_ids"] = np.stack(top_ids)
    out["top_scores"] = np.stack(top_scores).astype(np.float32)
    out["batch_all"] = batch_score_all(cache, params.gating, embs, feats, pairs_per_chunk=700)
    cl = component_logits(embs[0], cache.item_embs[:20], cfg.tau)
    out["cl_u0"] = cl.astype(np.float32)
    out["pi_u0"] = decomposed_gating(params.gating, feats[0], cache.item_gate_pre[:20], cl).astype(
        np.float32)
    np.savez_compressed(os.path.join(OUT, "small_mol.npz"), **out)


def production_case():
    """Production shape k_u=k_x=8, d=64, H=128, d_u=64 (BASELINE.json configs), 1,500 items,
    bf16-representable cache, quantized stage 1."""
    cfg = MoLConfig(k_u=8, k_x=8, d=64, tau=20.0, gating_hidden=128, dropout_p=0.0)
    X, U = 1500, 16
    dims = TowerDims(n_users=64, n_items=X, d_u=64, d_x=64, proj_hidden=128)
    params = init_params(dims, cfg, make_rng(4242))
    base = build_item_cache(params.item_table, params.item_proj, params.gating.item_net, cfg)
    embs_i = bf16(base.item_embs)
    gp = bf16(base.item_gate_pre)
    s1 = embs_i.mean(axis=1).astype(np.float32)
    cache = ItemCache(config=cfg, item_embs=embs_i, item_gate_pre=gp, stage1_embs=s1,
                      stage1_q=quantize_rowwise(s1))
    users = np.arange(U)
    uembs = user_components(params, users, cfg).astype(np.float32)
    feats = params.user_table[users].astype(np.float32)
    out = {
        "item_embs_bf16": (embs_i.view(np.uint32) >> 16).astype(np.uint16),
        "item_gate_pre_bf16": (gp.view(np.uint32) >> 16).astype(np.uint16),
        "stage1_embs": s1, "stage1_codes": cache.stage1_q.codes, "stage1_scales": cache.stage1_q.scales,
        "user_embs": uembs, "user_feats": feats, "tau": np.float32(cfg.tau),
    }
    for name, m in (("user_net", params.gating.user_net), ("cross_net", params.gating.cross_net)):
        out.update(mlp_arrays(name, m))
    scores, top_ids, top_scores = [], [], []
    for u in users:
        st = QueryState(user_embs=uembs[u], gate_features=feats[u])
        scores.append(score_candidates(cache, params.gating, np.arange(X), st))
        i, s = mol_top_k(cache, params.gating, np.arange(X), st, 100)
        top_ids.append(i)
        top_scores.append(s)
    out["scores"] = np.stack(scores).astype(np.float32)
    out["top_ids"] = np.stack(top_ids)
    out["top_scores"] = np.stack(top_scores).astype(np.float32)
    out["batch_all"] = batch_score_all(cache, params.gating, uembs, feats)
    # stage 1: raw int32, scaled, float; h_indexer in both views with per-user rng [9000, u]
    q1 = uembs.mean(axis=1).astype(np.float32)
    out["stage1_query"] = q1
    out["s1_raw"] = np.stack([stage1_scores(cache.stage1_q, q1[u], raw_int_ordering=True) for u in users])
    out["s1_scaled"] = np.stack([stage1_scores(cache.stage1_q, q1[u]) for u in users])
    out["s1_float"] = np.stack([stage1_scores(s1, q1[u]) for u in users]).astype(np.float32)
    qc = [quantize_vector(q1[u]) for u in users]
    out["query_codes"] = np.stack([c for c, _ in qc])
    out["query_scales"] = np.array([s for _, s in qc], dtype=np.float32)
    for tag, hcfg, view in (
        ("hq", HIndexerConfig(k_prime=150, sample_ratio=0.1, quantized=True), cache.stage1_q),
        ("hqs", HIndexerConfig(k_prime=150, sample_ratio=0.1, quantized=True, comparator="strict"),
         cache.stage1_q),
        ("hqr", HIndexerConfig(k_prime=150, lam=300, quantized=True, raw_int_ordering=True),
         cache.stage1_q),
        ("hf", HIndexerConfig(k_prime=150, sample_ratio=0.1), s1),
    ):
        offs, ids, ts = [0], [], []
        for u in users:
            r = h_indexer(view, q1[u], hcfg, make_rng([9000, int(u)]))
            ids.append(r.indices)
            offs.append(offs[-1] + r.indices.size)
            ts.append(r.threshold)
        out[f"{tag}_offsets"] = np.array(offs, dtype=np.int64)
        out[f"{tag}_ids"] = np.concatenate(ids).astype(np.int64)
        out[f"{tag}_t"] = np.array(ts, dtype=np.float64)
        out[f"{tag}_t_est"] = np.array(
            [estimate_threshold(view, q1[u], hcfg, make_rng([9000, int(u)])) for u in users])
    out["exact_top_k_q"] = np.stack([exact_top_k(cache.stage1_q, q1[u], 50) for u in users])
    out["exact_top_k_f"] = np.stack([exact_top_k(s1, q1[u], 50) for u in users])
    # two-stage composition (engine.py:117-138) with K'=150, r=0.1, quantized, k=20
    hcfg = HIndexerConfig(k_prime=150, sample_ratio=0.1, quantized=True)
    ts_ids, ts_scores = [], []
    for u in users:
        st = QueryState(user_embs=uembs[u], gate_features=feats[u])
        cand = h_indexer(cache.stage1_q, q1[u], hcfg, make_rng([9000, int(u)])).indices
        if cand.size < 20:
            cand = np.arange(X)
        i, s = mol_top_k(cache, params.gating, cand, st, min(20, cand.size))
        ts_ids.append(i)
        ts_scores.append(s)
    out["two_stage_ids"] = np.stack(ts_ids)
    out["two_stage_scores"] = np.stack(ts_scores).astype(np.float32)
    np.savez_compressed(os.path.join(OUT, "production_mol.npz"), **out)


def known_answers():
    """Analytic / edge cases the reference tests pin (test_quant.py, test_hindexer.py)."""
    out = {}
    q = quantize_rowwise(np.array([[1.0, -1.0], [0.0, 0.0], [0.3, -0.7]], dtype=np.float32))
    out["kq_codes"], out["kq_scales"] = q.codes, q.scales
    rng = make_rng(9)
    m = (rng.standard_normal((257, 64)) * np.array([1e-3, 1.0, 30.0])[rng.integers(0, 3, (257, 1))]
         ).astype(np.float32)
    m[5] = 0.0
    m[7, :] = 0.5  # exact .5 multiples exercise round-half-even
    q = quantize_rowwise(m)
    out["rq_in"], out["rq_codes"], out["rq_scales"] = m, q.codes, q.scales
    a = np.array([127], dtype=np.int8)
    out["dot_max"] = np.int64(int(int8_matvec(quantize_rowwise(np.ones((1, 1))), a)[0]))
    v = make_rng(0).standard_normal(10_000)
    out["nth_values"] = v
    out["nth_answers"] = np.array([nth_largest(v, n) for n in (1, 10, 100, 10_000)])
    # strict drops ties (test_hindexer.py:121-137)
    rng = make_rng(12)
    base = rng.standard_normal((50, 8)).astype(np.float32)
    base /= np.linalg.norm(base, axis=1, keepdims=True)
    items = np.vstack([base, base[:5]])
    qv = rng.standard_normal((1, 8)).astype(np.float32)
    qv = (qv / np.linalg.norm(qv, axis=1, keepdims=True))[0]
    inc = h_indexer(items, qv, HIndexerConfig(k_prime=10, lam=55, d_prime=8), make_rng(13))
    stc = h_indexer(items, qv, HIndexerConfig(k_prime=10, lam=55, d_prime=8, comparator="strict"),
                    make_rng(13))
    out.update(tie_items=items, tie_query=qv, tie_inc_ids=inc.indices, tie_inc_t=inc.threshold,
               tie_str_ids=stc.indices, tie_str_t=stc.threshold)
    np.savez_compressed(os.path.join(OUT, "known_answers.npz"), **out)


def engine_case():
    """test_engine.py:11-17 'built' engine: RetrievalEngine.query for users 0..9, k=10."""
    cfg = MoLConfig(k_u=2, k_x=2, d=8, gating_hidden=16, dropout_p=0.0)
    dims = TowerDims(n_users=30, n_items=800, d_u=12, d_x=12, proj_hidden=16)
    params = init_params(dims, cfg, make_rng(0))
    hcfg = HIndexerConfig(k_prime=200, sample_ratio=0.2, d_prime=cfg.d)
    eng = RetrievalEngine.from_params(params, cfg, hcfg, seed=5)
    out = {"item_embs": eng.cache.item_embs, "item_gate_pre": eng.cache.item_gate_pre,
           "stage1_embs": eng.cache.stage1_embs, "tau": np.float32(cfg.tau)}
    for name, m in (("user_net", params.gating.user_net), ("cross_net", params.gating.cross_net)):
        out.update(mlp_arrays(name, m))
    embs, feats, ids, scores, full_ids = [], [], [], [], []
    for u in range(10):
        st = eng.query_state(u)
        embs.append(st.user_embs)
        feats.append(st.gate_features)
        r = eng.query(u, 10)
        ids.append([i for i, _ in r])
        scores.append([s for _, s in r])
        full_ids.append([i for i, _ in eng.full_top_k(u, 10)])
    out.update(user_embs=np.stack(embs).astype(np.float32), user_feats=np.stack(feats).astype(np.float32),
               query_ids=np.array(ids), query_scores=np.array(scores, dtype=np.float32),
               full_ids=np.array(full_ids), seed=np.int64(5), k_prime=np.int64(200),
               sample_ratio=np.float64(0.2))
    np.savez_compressed(os.path.join(OUT, "engine_small.npz"), **out)


def snapshot_case():
    """ItemCache.save (mol.py:253-273, snapshot.py:86-112) of a small quantized cache, plus the
    arrays ItemCache.load gives back; and a production-shape build_item_cache (mol.py:294-326)
    with its inputs, for the device cache-build parity test."""
    cfg = MoLConfig(k_u=2, k_x=3, d=8, tau=20.0, gating_hidden=16, dropout_p=0.0)
    dims = TowerDims(n_users=4, n_items=40, d_u=12, d_x=12, proj_hidden=24)
    params = init_params(dims, cfg, make_rng(7))
    cache = build_item_cache(params.item_table, params.item_proj, params.gating.item_net, cfg, quantized=True)
    path = os.path.join(OUT, "item_cache_ref.molc")
    cache.save(path)
    back = ItemCache.load(path)
    np.savez_compressed(os.path.join(OUT, "snapshot_case.npz"), item_embs=back.item_embs,
                        item_gate_pre=back.item_gate_pre, stage1_embs=back.stage1_embs,
                        codes=back.stage1_q.codes, scales=back.stage1_q.scales,
                        cfg=np.array([cfg.k_u, cfg.k_x, cfg.d, cfg.gating_hidden], dtype=np.int64))
    pcfg = MoLConfig(k_u=8, k_x=8, d=64, tau=20.0, gating_hidden=128, dropout_p=0.0)
    pdims = TowerDims(n_users=4, n_items=1000, d_u=64, d_x=64, proj_hidden=128)
    pp = init_params(pdims, pcfg, make_rng(4242))
    pc = build_item_cache(pp.item_table, pp.item_proj, pp.gating.item_net, pcfg, quantized=True)
    np.savez_compressed(os.path.join(OUT, "build_case.npz"), item_table=pp.item_table,
                        **mlp_arrays("item_proj", pp.item_proj), **mlp_arrays("item_net", pp.gating.item_net),
                        item_embs=pc.item_embs, item_gate_pre=pc.item_gate_pre, stage1_embs=pc.stage1_embs,
                        codes=pc.stage1_q.codes, scales=pc.stage1_q.scales)


def engine_case2():
    """RetrievalEngine.from_params + query / full_top_k (engine.py:80-147) end to end, with the
    towers, for the drop-in RetrievalEngine test."""
    cfg = MoLConfig(k_u=4, k_x=4, d=16, tau=20.0, gating_hidden=32, dropout_p=0.0)
    dims = TowerDims(n_users=40, n_items=3000, d_u=12, d_x=12, proj_hidden=24)
    params = init_params(dims, cfg, make_rng(4242))
    hcfg = HIndexerConfig(k_prime=300, sample_ratio=0.1, quantized=True)
    eng = RetrievalEngine.from_params(params, cfg, hcfg, seed=11)
    users = np.arange(10)
    q = [eng.query(int(u), 10) for u in users]
    f = [eng.full_top_k(int(u), 10) for u in users]
    out = {"user_table": params.user_table, "item_table": params.item_table,
           **mlp_arrays("user_proj", params.user_proj), **mlp_arrays("item_proj", params.item_proj),
           **mlp_arrays("user_net", params.gating.user_net), **mlp_arrays("item_net", params.gating.item_net),
           **mlp_arrays("cross_net", params.gating.cross_net),
           "query_ids": np.array([[i for i, _ in r] for r in q]), "query_scores": np.array([[s for _, s in r] for r in q]),
           "full_ids": np.array([[i for i, _ in r] for r in f]), "full_scores": np.array([[s for _, s in r] for r in f])}
    np.savez_compressed(os.path.join(OUT, "engine_case2.npz"), **out)


def query_case():
    """Production-shape user side (model.py:179-191 user_components, mol.py:186 user_net) for the
    device query-prep parity test."""
    cfg = MoLConfig(k_u=8, k_x=8, d=64, tau=20.0, gating_hidden=128, dropout_p=0.0)
    dims = TowerDims(n_users=64, n_items=10, d_u=64, d_x=64, proj_hidden=128)
    params = init_params(dims, cfg, make_rng(99))
    users = np.arange(64)
    np.savez_compressed(os.path.join(OUT, "query_case.npz"), user_table=params.user_table,
                        **mlp_arrays("user_proj", params.user_proj), **mlp_arrays("user_net", params.gating.user_net),
                        user_embs=user_components(params, users, cfg),
                        uw=params.gating.user_net(params.user_table[users]))


if __name__ == "__main__":
    if len(sys.argv) > 1:  # regenerate selected cases only, e.g. `make_golden.py snapshot_case`
        for name in sys.argv[1:]:
            globals()[name]()
        sys.exit(0)
    small_case()
    production_case()
    known_answers()
    engine_case()
    for f in sorted(os.listdir(OUT)):
        if f.endswith(".npz"):
            print(f, os.path.getsize(os.path.join(OUT, f)))
