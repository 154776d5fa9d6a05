"""Above the hot path: batched query prep (#3), the `molr bench` CSV harness on
the batched engine (#1) and serving micro-batching (#4)."""

import threading

import numpy as np
import pytest


# ---------------------------------------------------------------------------------- CPU
def _stub(feats, k):
    """deterministic fake batch: ids = row-sum based, so each row's answer depends only on it"""
    base = (np.abs(feats).sum(axis=1) * 1000).astype(np.int64)
    ids = base[:, None] + np.arange(k)[None, :]
    return ids, -ids.astype(np.float32)


def test_microbatcher_routes_rows_and_batches():
    from paper_2306_04039_b200.serving import MicroBatcher

    calls = []

    def run(feats, k):
        calls.append(len(feats))
        return _stub(feats, k)

    rng = np.random.default_rng(0)
    feats = rng.normal(size=(300, 8)).astype(np.float32)
    with MicroBatcher(run, max_batch=64, max_wait_ms=20, k=5) as mb:
        futs = [None] * 300
        def worker(lo, hi):
            for i in range(lo, hi):
                futs[i] = mb.submit(feats[i])
        ts = [threading.Thread(target=worker, args=(j * 30, (j + 1) * 30)) for j in range(10)]
        [t.start() for t in ts]
        [t.join() for t in ts]
        res = [f.result(timeout=10) for f in futs]
    exp_ids, _ = _stub(feats, 5)
    for i in range(300):
        np.testing.assert_array_equal(res[i][0], exp_ids[i])
    assert max(calls) <= 64 and sum(calls) == 300 and len(calls) < 300  # requests were batched


def test_microbatcher_identical_concurrent_queries():
    """100 concurrent identical queries -> identical payloads (test_lineserver.py:90-107)."""
    from paper_2306_04039_b200.serving import MicroBatcher

    q = np.linspace(-1, 1, 8).astype(np.float32)
    out = []
    lock = threading.Lock()
    with MicroBatcher(_stub, max_batch=16, max_wait_ms=5, k=10) as mb:
        def go():
            r = mb.query(q, timeout=10)
            with lock:
                out.append(r)
        ts = [threading.Thread(target=go) for _ in range(100)]
        [t.start() for t in ts]
        [t.join() for t in ts]
    assert len(out) == 100 and all(r == out[0] for r in out)


def test_microbatcher_errors_propagate():
    from paper_2306_04039_b200.serving import MicroBatcher

    def boom(feats, k):
        raise ValueError("bad batch")

    with MicroBatcher(boom, max_batch=4, max_wait_ms=1) as mb:
        f = mb.submit(np.zeros(3))
        with pytest.raises(ValueError):
            f.result(timeout=10)
    with pytest.raises(RuntimeError):
        mb.submit(np.zeros(3))
    with pytest.raises(ValueError):
        MicroBatcher(_stub, max_batch=0)


# ---------------------------------------------------------------------------------- GPU
@pytest.mark.gpu
def test_query_prep_matches_reference(golden):
    """molr_query_prep vs the reference's user_components / user_net (golden query_case)."""
    from paper_2306_04039_b200.engine import query_prep
    from paper_2306_04039_b200.mol import MoLConfig, Mlp

    g = golden("query_case")
    cfg = MoLConfig(k_u=8, k_x=8, d=64, tau=20.0, gating_hidden=128, dropout_p=0.0)
    up = Mlp(g["user_proj.w1"], g["user_proj.b1"], g["user_proj.w2"])
    un = Mlp(g["user_net.w1"], g["user_net.b1"], g["user_net.w2"])
    ue, uw = query_prep(up, un, g["user_table"], cfg)
    np.testing.assert_allclose(ue, g["user_embs"], rtol=0, atol=2e-6)
    np.testing.assert_allclose(uw, g["uw"], rtol=1e-5, atol=2e-6)
    np.testing.assert_allclose(np.linalg.norm(ue, axis=-1), 1.0, atol=1e-6)


def _engine(n_items=60_000, n_users=64, seed=31):
    from paper_2306_04039_b200.engine import BatchedRetrievalEngine
    from paper_2306_04039_b200.hindexer import HIndexerConfig
    from paper_2306_04039_b200.mol import Mlp
    from tests.test_gpu_parity import _prod_gating, _synthetic_prod_cache

    cache, syn, ue, feats = _synthetic_prod_cache(n_items, seed=seed, n_users=n_users)
    gating, _ = _prod_gating(syn)
    up = Mlp(*syn.user_proj)
    eng = BatchedRetrievalEngine(cache, gating, HIndexerConfig(k_prime=3000, sample_ratio=0.05, quantized=True),
                                 seed=5, user_proj=up)
    return eng, ue, feats


@pytest.mark.gpu
def test_query_features_equals_prepared_path():
    """engine.query_features (device query prep + two-stage) == two_stage_top_k on host-prepared
    user components; and batch composition does not change a query's answer."""
    from paper_2306_04039_b200.engine import query_prep, two_stage_top_k

    eng, ue, feats = _engine()
    ids, sc, cand = eng.query_features(feats, 50)
    pue, puw = query_prep(eng.user_proj, eng.gating.user_net, feats, eng.cache.config)
    ids2, sc2, _ = two_stage_top_k(eng.cache, eng.gating, pue, puw, 50, eng.hconfig, seed=eng.seed)
    np.testing.assert_array_equal(ids, ids2)
    np.testing.assert_array_equal(sc, sc2)
    sub_ids, sub_sc, _ = eng.query_features(feats[[5, 9, 1]], 50)
    np.testing.assert_array_equal(sub_ids, ids[[5, 9, 1]])
    np.testing.assert_array_equal(sub_sc, sc[[5, 9, 1]])


@pytest.mark.gpu
def test_microbatcher_on_device_engine():
    from paper_2306_04039_b200.serving import MicroBatcher

    eng, ue, feats = _engine()
    ref_ids, ref_sc, _ = eng.query_features(feats, 20)
    out = [None] * len(feats)
    with MicroBatcher.for_engine(eng, max_batch=16, max_wait_ms=5, k=20) as mb:
        def go(i):
            out[i] = mb.submit(feats[i]).result(timeout=60)
        ts = [threading.Thread(target=go, args=(i,)) for i in range(len(feats))]
        [t.start() for t in ts]
        [t.join() for t in ts]
        same = [mb.query(feats[3], timeout=60) for _ in range(5)]
    for i in range(len(feats)):
        np.testing.assert_array_equal(out[i][0], ref_ids[i])
    assert all(r == same[0] for r in same)


@pytest.mark.gpu
def test_bench_csv_contract():
    """`molr bench` CSV contract (test_cli.py:128-137): header, recall nondecreasing in K',
    recall 1.0 at K' = X."""
    from paper_2306_04039_b200.engine import bench_csv

    eng, ue, feats = _engine(n_items=20_000, n_users=16)
    csv = bench_csv(eng, ue, feats, 10, [200, 1000, 5000, 20_000])
    lines = csv.strip().split("\n")
    assert lines[0] == "k_prime,recall,qps"
    rec = [float(l.split(",")[1]) for l in lines[1:]]
    assert all(b >= a - 1e-9 for a, b in zip(rec, rec[1:])), rec
    assert rec[-1] == 1.0
    assert all(float(l.split(",")[2]) > 0 for l in lines[1:])


@pytest.mark.gpu
def test_retrieval_engine_drop_in(golden):
    """Drop-in RetrievalEngine (engine.py:80-147) vs the reference engine's own query /
    full_top_k outputs (golden engine_case2: from_params, K'=300, r=0.1, int8, seed 11)."""
    from types import SimpleNamespace

    import oracle as O
    from paper_2306_04039_b200.engine import RetrievalEngine
    from paper_2306_04039_b200.hindexer import HIndexerConfig
    from paper_2306_04039_b200.mol import GatingNetwork, Mlp, MoLConfig

    g = golden("engine_case2")
    mk = lambda p: Mlp(g[p + ".w1"], g[p + ".b1"], g[p + ".w2"])  # noqa: E731
    params = SimpleNamespace(user_table=g["user_table"], item_table=g["item_table"], user_proj=mk("user_proj"),
                             item_proj=mk("item_proj"), n_users=g["user_table"].shape[0], compression=None,
                             gating=GatingNetwork(user_net=mk("user_net"), item_net=mk("item_net"),
                                                  cross_net=mk("cross_net")))
    cfg = MoLConfig(k_u=4, k_x=4, d=16, tau=20.0, gating_hidden=32, dropout_p=0.0)
    eng = RetrievalEngine.from_params(params, cfg, HIndexerConfig(k_prime=300, sample_ratio=0.1, quantized=True),
                                      seed=11)
    for u in range(10):
        q = eng.query(u, 10)
        f = eng.full_top_k(u, 10)
        assert [i for i, _ in f] == list(g["full_ids"][u]) or O.score_close(
            np.array([s for _, s in f]), g["full_scores"][u]).all()
        np.testing.assert_allclose([s for _, s in f], g["full_scores"][u], rtol=1e-3, atol=1e-6)
        np.testing.assert_allclose([s for _, s in q], g["query_scores"][u], rtol=1e-3, atol=1e-6)
        # same candidates as the reference engine (bit-exact stage 1), so the same top-k modulo
        # ties within the score tolerance
        qi = [i for i, _ in q]
        ref_i = g["query_ids"][u].tolist()
        if qi != ref_i:
            kth = g["query_scores"][u][-1]
            got_s = dict(q)
            diff = set(qi) ^ set(ref_i)
            assert all(abs(got_s.get(i, kth) - kth) <= 1e-3 * abs(kth) + 1e-6 for i in diff), (u, qi, ref_i)
        fi = [i for i, _ in f]
        if fi != g["full_ids"][u].tolist():
            kth = g["full_scores"][u][-1]
            got_s = dict(f)
            diff = set(fi) ^ set(g["full_ids"][u].tolist())
            assert all(abs(got_s.get(i, kth) - kth) <= 1e-3 * abs(kth) + 1e-6 for i in diff), (u, fi)
    assert eng.query(3, 10) == eng.query(3, 10)  # deterministic per (seed, user)
    from paper_2306_04039_b200.errors import OutOfRangeError

    with pytest.raises(OutOfRangeError):
        eng.query(10_000, 5)


@pytest.mark.gpu
def test_numerics_primitives_match_reference_forms():
    """sigmoid / silu / silu_grad / softmax(_rows) (numerics.py:52-81) on the GPU vs NumPy/SciPy."""
    from scipy.special import expit

    from paper_2306_04039_b200.numerics import sigmoid, silu, silu_grad, softmax, softmax_rows

    rng = np.random.default_rng(0)
    for dt, tol in ((np.float32, 2e-6), (np.float64, 1e-13)):
        x = (rng.normal(size=(37, 19)) * 6).astype(dt)
        s = expit(x)
        np.testing.assert_allclose(sigmoid(x), s, rtol=tol, atol=tol)
        np.testing.assert_allclose(silu(x), x * s, rtol=tol, atol=tol)
        np.testing.assert_allclose(silu_grad(x), s * (1 + x * (1 - s)), rtol=tol, atol=tol)
        e = np.exp(x - x.max(axis=-1, keepdims=True))
        np.testing.assert_allclose(softmax_rows(x), e / e.sum(axis=-1, keepdims=True), rtol=tol * 4, atol=tol)
        assert softmax_rows(x).dtype == dt and silu(x).dtype == dt
        v = x[0]
        ev = np.exp(v - v.max())
        np.testing.assert_allclose(softmax(v), ev / ev.sum(), rtol=tol * 4, atol=tol)
    assert abs(float(silu(np.float32(1.0))) - 0.731059) < 1e-6  # test_numerics.py:94-105


@pytest.mark.gpu
def test_retrieval_engine_100_concurrent_queries_identical(golden):
    """The lineserver contract (test_lineserver.py:90-107, threads at lineserver.py:69-77): 100
    concurrent identical queries against one engine return identical bytes; concurrent distinct
    queries return what they return sequentially.  Every thread calls the C-ABI directly (ctypes
    releases the GIL) on its own per-thread stream."""
    import threading
    from types import SimpleNamespace

    from paper_2306_04039_b200.engine import RetrievalEngine
    from paper_2306_04039_b200.hindexer import HIndexerConfig
    from paper_2306_04039_b200.mol import GatingNetwork, Mlp, MoLConfig

    g = golden("engine_case2")
    mk = lambda p: Mlp(g[p + ".w1"], g[p + ".b1"], g[p + ".w2"])  # noqa: E731
    params = SimpleNamespace(user_table=g["user_table"], item_table=g["item_table"], user_proj=mk("user_proj"),
                             item_proj=mk("item_proj"), n_users=g["user_table"].shape[0], compression=None,
                             gating=GatingNetwork(user_net=mk("user_net"), item_net=mk("item_net"),
                                                  cross_net=mk("cross_net")))
    cfg = MoLConfig(k_u=4, k_x=4, d=16, tau=20.0, gating_hidden=32, dropout_p=0.0)
    eng = RetrievalEngine.from_params(params, cfg, HIndexerConfig(k_prime=300, sample_ratio=0.1, quantized=True),
                                      seed=11)
    want = eng.query(7, 10)
    n_users = min(20, g["user_table"].shape[0])
    seq = {u: eng.query(u, 10) for u in range(n_users)}
    out = [None] * 100
    mixed = [None] * 100
    start = threading.Barrier(100)

    def worker(i):
        start.wait()
        out[i] = eng.query(7, 10)
        mixed[i] = eng.query(i % n_users, 10)

    th = [threading.Thread(target=worker, args=(i,)) for i in range(100)]
    for t in th:
        t.start()
    for t in th:
        t.join()
    assert all(r == want for r in out)
    assert all(mixed[i] == seq[i % n_users] for i in range(100))
