"""Shared test helpers: golden fixtures -> product objects and oracle objects."""

import os

import numpy as np

import oracle as O

# the development build (libmolr_b200_dev.so, -DMOLR_DEV_KNOBS): the only library that honours the
# cross-check switches (alternative SIMT backends, pilot sizes); tests/test_gpu_devbuild.py runs the
# `devknobs` tests under it in a subprocess
DEV_BUILD = os.path.basename(os.environ.get("MOLR_LIB_PATH", "")) == "libmolr_b200_dev.so"


def with_knob(monkeypatch, env, fn):
    """fn() with the development switches `env` set — only under the dev build; None otherwise."""
    if not DEV_BUILD:
        return None
    for k, v in env.items():
        monkeypatch.setenv(k, v)
    try:
        return fn()
    finally:
        for k in env:
            monkeypatch.delenv(k, raising=False)


def bf16_to_f32(u16):
    return (np.asarray(u16).astype(np.uint32) << 16).view(np.float32)


def product_gating(g):
    from paper_2306_04039_b200.mol import GatingNetwork, Mlp

    G = g["cross_net.w2"].shape[1]
    un = Mlp(g["user_net.w1"], g["user_net.b1"], g["user_net.w2"])
    cn = Mlp(g["cross_net.w1"], g["cross_net.b1"], g["cross_net.w2"])
    item = Mlp(np.zeros((1, 4), np.float32), np.zeros(4, np.float32), np.zeros((4, G), np.float32))
    return GatingNetwork(user_net=un, item_net=item, cross_net=cn)


def oracle_gating(g):
    mk = lambda p: O.MlpW(g[p + ".w1"], g[p + ".b1"], g[p + ".w2"])  # noqa: E731
    zero = O.MlpW(np.zeros((1, 1)), np.zeros(1), np.zeros((1, 1)))
    return O.Gating(mk("user_net"), zero, mk("cross_net"))


def production_arrays(g):
    embs = bf16_to_f32(g["item_embs_bf16"])
    gp = bf16_to_f32(g["item_gate_pre_bf16"])
    return embs, gp


def product_cache(g, kind="production"):
    from paper_2306_04039_b200.mol import ItemCache, MoLConfig
    from paper_2306_04039_b200.quant import QuantizedRows

    tau = float(g["tau"])
    if kind == "production":
        embs, gp = production_arrays(g)
        q = QuantizedRows(codes=g["stage1_codes"], scales=g["stage1_scales"])
        s1 = g["stage1_embs"]
    else:
        embs, gp, s1, q = g["item_embs"], g["item_gate_pre"], g["stage1_embs"], None
    k_u = g["user_embs"].shape[1]
    k_x, d = embs.shape[1], embs.shape[2]
    H = g["cross_net.w1"].shape[1]
    cfg = MoLConfig(k_u=k_u, k_x=k_x, d=d, tau=tau, gating_hidden=H, dropout_p=0.0)
    return ItemCache(config=cfg, item_embs=embs, item_gate_pre=gp, stage1_embs=s1, stage1_q=q)


def topk_equal_modulo_ties(ids_got, ids_ref, scores_ref_all, rel=1e-3, abs_=1e-6):
    """Top-k index lists agree except for items whose reference score lies within the tolerance
    band of the k-th reference score."""
    ids_got = list(map(int, ids_got))
    ids_ref = list(map(int, ids_ref))
    if ids_got == ids_ref:
        return True
    kth = scores_ref_all[ids_ref[-1]]
    band = rel * abs(kth) + abs_
    diff = set(ids_got) ^ set(ids_ref)
    return all(abs(scores_ref_all[i] - kth) <= band for i in diff)
