"""Item-cache snapshots: the reference's MOLC/MOLR container format
(snapshot.py:1-139, ItemCache.save/load mol.py:253-291) read and written byte-compatibly, and the
device loader / device cache build.  The golden container was written by the REFERENCE
(tests/golden/make_golden.py snapshot_case)."""

import os

import numpy as np
import pytest

from tests.conftest import GOLDEN

REF_MOLC = os.path.join(GOLDEN, "item_cache_ref.molc")


def test_read_reference_container(golden):
    from paper_2306_04039_b200 import snapshot

    g = golden("snapshot_case")
    sec, meta = snapshot.read_container(REF_MOLC)
    assert meta["kind"] == "item_cache" and meta["config"]["k_x"] == int(g["cfg"][1])
    np.testing.assert_array_equal(sec["item_embs"], g["item_embs"])
    np.testing.assert_array_equal(sec["item_gate_pre"], g["item_gate_pre"])
    np.testing.assert_array_equal(sec["stage1_embs"], g["stage1_embs"])
    codes, scales = sec["stage1_q"]
    np.testing.assert_array_equal(codes, g["codes"])
    np.testing.assert_array_equal(scales, g["scales"])


def test_writer_byte_identical_to_reference(golden, tmp_path):
    """ItemCache.save of the same arrays reproduces the reference's file byte for byte."""
    from paper_2306_04039_b200.mol import ItemCache
    from paper_2306_04039_b200.snapshot import load_item_cache

    cache = load_item_cache(REF_MOLC)
    assert isinstance(cache, ItemCache)
    out = tmp_path / "ours.molc"
    cache.save(out)
    assert out.read_bytes() == open(REF_MOLC, "rb").read()
    back = ItemCache.load(out)
    np.testing.assert_array_equal(back.item_embs, cache.item_embs)
    np.testing.assert_array_equal(back.stage1_q.codes, cache.stage1_q.codes)


def test_container_errors(tmp_path):
    from paper_2306_04039_b200 import snapshot

    bad = tmp_path / "bad.molc"
    bad.write_bytes(b"NOPE" + bytes(20))
    with pytest.raises(ValueError):
        snapshot.read_container(bad)
    raw = open(REF_MOLC, "rb").read()
    v2 = tmp_path / "v2.molc"
    v2.write_bytes(raw[:4] + b"\x02\x00" + raw[6:])
    with pytest.raises(ValueError):
        snapshot.read_container(v2)
    other = tmp_path / "ckpt.molc"
    snapshot.write_container(other, {"w": np.ones((2, 3), np.float32)}, {"kind": "checkpoint"})
    sec, meta = snapshot.read_container(other)
    np.testing.assert_array_equal(sec["w"], np.ones((2, 3)))
    with pytest.raises(ValueError):
        snapshot.load_item_cache(other)


# ---------------------------------------------------------------------------------- GPU
def _read_back(dev, X, kd, G, d1):
    from paper_2306_04039_b200 import _lib as L

    e = np.empty((X, kd), np.float32)
    g = np.empty((X, G), np.float32)
    s = np.empty((X, d1), np.float32)
    c = np.empty((X, d1), np.int8)
    sc = np.empty(X, np.float32)
    L.call("molr_cache_read", dev.device_handle(), 0, X, L.ptr(e), L.ptr(g), L.ptr(s), L.ptr(c), L.ptr(sc), None)
    return e, g, s, c, sc


@pytest.mark.gpu
def test_device_loader_round_trip(golden, tmp_path):
    """Reference container -> device cache (memmap streamed, lossless storage) -> read back and
    scored identically to the host ItemCache; device cache -> container -> same bytes."""
    from paper_2306_04039_b200.mol import GatingNetwork, Mlp, QueryState, score_candidates
    from paper_2306_04039_b200.snapshot import load_device_item_cache, load_item_cache, save_device_item_cache

    host = load_item_cache(REF_MOLC)
    dev = load_device_item_cache(REF_MOLC, chunk_rows=7)
    cfg = host.config
    X = host.num_items
    e, g, s, c, sc = _read_back(dev, X, cfg.k_x * cfg.d, cfg.num_logits, host.stage1_dim)
    np.testing.assert_array_equal(e.reshape(host.item_embs.shape), host.item_embs)
    np.testing.assert_array_equal(g, host.item_gate_pre)
    np.testing.assert_array_equal(s, host.stage1_embs)
    np.testing.assert_array_equal(c, host.stage1_q.codes)
    np.testing.assert_array_equal(sc, host.stage1_q.scales)
    rng = np.random.default_rng(0)
    G, H = cfg.num_logits, cfg.gating_hidden
    mk = lambda i, o: Mlp(rng.normal(size=(i, H)).astype(np.float32) * 0.3, rng.normal(size=H).astype(np.float32) * 0.1,
                          rng.normal(size=(H, o)).astype(np.float32) * 0.3)  # noqa: E731
    gating = GatingNetwork(user_net=mk(12, G), item_net=mk(12, G), cross_net=mk(G, G))
    ue = rng.normal(size=(cfg.k_u, cfg.d)).astype(np.float32)
    ue /= np.linalg.norm(ue, axis=1, keepdims=True)
    q = QueryState(user_embs=ue, gate_features=rng.normal(size=12).astype(np.float32))
    ids = np.arange(X)
    np.testing.assert_array_equal(score_candidates(dev, gating, ids, q), score_candidates(host, gating, ids, q))
    out = tmp_path / "dev.molc"
    save_device_item_cache(dev, out, chunk_rows=11)
    assert out.read_bytes() == open(REF_MOLC, "rb").read()


@pytest.mark.gpu
@pytest.mark.parametrize("round_bf16", [False, True])
def test_device_cache_build_matches_reference(golden, round_bf16):
    """build_device_item_cache (molr_cache_build_rows) vs the reference's build_item_cache on the
    same production-shape towers (golden build_case, 1000 items): f32 within fp32 rounding of the
    MLPs; int8 view equal up to +-1 code where the stage-1 mean differs in the last bit.  With
    round_bf16 the stored fields are the reference's values rounded to bf16 (up to one bf16 ulp
    where our fp32 MLP output lands on the other side of a rounding boundary)."""
    import oracle as O
    from paper_2306_04039_b200.mol import MoLConfig, Mlp, build_device_item_cache

    g = golden("build_case")
    cfg = MoLConfig(k_u=8, k_x=8, d=64, tau=20.0, gating_hidden=128, dropout_p=0.0)
    proj = Mlp(g["item_proj.w1"], g["item_proj.b1"], g["item_proj.w2"])
    net = Mlp(g["item_net.w1"], g["item_net.b1"], g["item_net.w2"])
    dev = build_device_item_cache(g["item_table"], proj, net, cfg, quantized=True, round_bf16=round_bf16,
                                  chunk_rows=300)
    X = g["item_table"].shape[0]
    e, gp, s, c, sc = _read_back(dev, X, 512, 64, 64)
    ref_e = g["item_embs"].reshape(X, 512)
    ref_g = g["item_gate_pre"]
    if not round_bf16:
        np.testing.assert_allclose(e, ref_e, rtol=0, atol=2e-6)
        np.testing.assert_allclose(gp, ref_g, rtol=1e-5, atol=1e-6)
        np.testing.assert_allclose(s, g["stage1_embs"], rtol=0, atol=2e-6)
        assert np.abs(c.astype(int) - g["codes"].astype(int)).max() <= 1
        assert (c != g["codes"]).mean() < 1e-3
        np.testing.assert_allclose(sc, g["scales"], rtol=1e-5)
    else:
        rb_e, rb_g = O.round_bf16(ref_e), O.round_bf16(ref_g)
        ulp = lambda a, b: np.maximum(np.abs(a), np.abs(b)).astype(np.float32) * 2.0 ** -7 + 2e-6  # noqa: E731
        bad = np.abs(e - rb_e) > ulp(e, rb_e)
        assert not bad.any(), (np.argwhere(bad)[:5], e[bad][:5], rb_e[bad][:5], ref_e[bad][:5])
        assert np.all(np.abs(gp - rb_g) <= ulp(gp, rb_g))
        assert (e != rb_e).mean() < 1e-3
        # stage 1 is the mean of the stored (rounded) components, exactly as the oracle computes it
        np.testing.assert_allclose(s, e.reshape(X, 8, 64).mean(axis=1), rtol=0, atol=1e-7)
