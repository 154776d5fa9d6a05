"""NumPy emulation of the tcgen05 MoL kernel's cross-net arithmetic (csrc/mol_tc.cu), used to pick
its precision: score error against the oracle (oracle/molr_oracle.py, fp32 NumPy like the
reference's mol.py:161-205) in units of the 1e-3 |s| + 1e-6 tolerance, for single-pass bf16 / fp16
layers, tf32, and the hi/lo-split three-pass layers, at the default init and with the cross net and
gate pre-activations sharpened (the cases of tests/test_gpu_parity.py::test_tc_kernel_precision_margin).

    python tools/precision_emu.py
"""
import os
import sys

import numpy as np
from scipy.special import expit

sys.path.insert(0, os.path.join(os.path.dirname(__file__), ".."))
import oracle.molr_oracle as O  # noqa: E402


def bf16(x):
    return O.round_bf16(np.asarray(x, np.float32)).astype(np.float64)


def f16(x):
    return np.asarray(x, np.float32).astype(np.float16).astype(np.float64)


def tf32(x):
    x = np.asarray(x, np.float32).copy()
    u = x.view(np.uint32)
    u += 0x1000
    u &= ~np.uint32(0x1FFF)
    return x.astype(np.float64)


def split(rnd, x):
    hi = rnd(x)
    return hi, rnd(np.asarray(x, np.float64) - hi)


def layer(kind, a, w):
    if kind == "bf16":
        return bf16(a) @ bf16(w)
    if kind == "f16":
        return f16(a) @ f16(w)
    if kind == "tf32":
        return tf32(a) @ tf32(w)
    rnd = bf16 if kind == "bf16x3" else f16
    ah, al = split(rnd, a)
    wh, wl = split(rnd, w)
    return ah @ wh + al @ wh + ah @ wl


def main(n_users=8, n_items=4000):
    modes = [("bf16", "f16", True), ("tf32", "tf32", False), ("bf16x3", "f16", False), ("bf16", "f16x3", False),
             ("bf16x3", "f16x3", True), ("bf16x3", "f16x3", False)]
    for cs, gs in [(1, 1), (4, 4), (16, 16), (16, 64), (1, 64)]:
        syn = O.init_synthetic(n_users, n_items, k_u=8, k_x=8, d=64, gating_hidden=128, seed=9)
        c = O.build_item_cache(syn.item_table, syn.item_proj, syn.gating.item_net, 8, 64, 20.0, 8, quantized=False)
        embs, gp = O.round_bf16(c.item_embs), O.round_bf16(c.item_gate_pre * gs)
        ue = O.user_components(syn, np.arange(n_users), 8, 64).astype(np.float32)
        g = syn.gating
        w1, b1, w2 = g.cross_net.w1 * cs, g.cross_net.b1 * cs, g.cross_net.w2 * cs
        uw_all = O.mlp(g.user_net, syn.user_table[:n_users]).astype(np.float32)
        worst = {}
        for u in range(n_users):
            cl = O.component_logits(ue[u], embs, 20.0)
            net = O.MlpW(w1.astype(np.float32), b1.astype(np.float32), w2.astype(np.float32))
            pi = O.softmax_rows(O.silu(uw_all[u][None, :] * gp + O.mlp(net, cl)))
            ref = (pi * cl).sum(-1).astype(np.float64)
            for l1, l2, tanh in modes:
                h = layer(l1, cl, w1) + b1
                hh = h * expit(h)
                if tanh:  # tanh.approx SiLU: ~2^-11 of |h/2| absolute
                    hh = hh + np.abs(h) * 0.5 * np.random.default_rng(1).uniform(-1, 1, h.shape) * 2.0**-11
                x = uw_all[u].astype(np.float64)[None, :] * gp + layer(l2, hh, w2)
                p = x * expit(x)
                p = np.exp(p - p.max(-1, keepdims=True))
                p /= p.sum(-1, keepdims=True)
                s = (p * cl.astype(np.float64)).sum(-1)
                key = f"L1 {l1} / L2 {l2}{' / tanh' if tanh else ''}"
                worst[key] = max(worst.get(key, 0.0), float((np.abs(s - ref) / (1e-3 * np.abs(ref) + 1e-6)).max()))
        print(f"cross x{cs} gate x{gs}: " + ", ".join(f"{k}: {v:.3f}" for k, v in worst.items()))


if __name__ == "__main__":
    main()
