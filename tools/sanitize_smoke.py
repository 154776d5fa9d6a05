"""Small end-to-end run of every production kernel for compute-sanitizer (memcheck / racecheck /
synccheck): device cache build, query prep, two-stage retrieval (pilot + filter + MoL + top-k),
exact MoL top-k, snapshot round trip."""
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2306_04039_b200.engine import query_prep, two_stage_top_k  # noqa: E402
from paper_2306_04039_b200.hindexer import HIndexerConfig  # noqa: E402
from paper_2306_04039_b200.mol import Mlp, MoLConfig, batch_mol_top_k, build_device_item_cache  # noqa: E402
from tests.test_gpu_parity import _prod_gating, _synthetic_prod_cache  # noqa: E402

cache, syn, ue, feats = _synthetic_prod_cache(40_000, seed=3, n_users=40)
gating, _ = _prod_gating(syn)
uw = gating.user_net(feats)
ids, sc, cand = two_stage_top_k(cache, gating, ue, uw, 20, HIndexerConfig(k_prime=2000, sample_ratio=0.2, quantized=True),
                                seed=1)
bi, bs = batch_mol_top_k(cache, gating, ue[:4], feats[:4], 50)
cfg = MoLConfig(k_u=8, k_x=8, d=64, tau=20.0, gating_hidden=128, dropout_p=0.0)
dev = build_device_item_cache(syn.item_table[:3000], Mlp(*syn.item_proj), Mlp(*syn.gating.item_net), cfg,
                              round_bf16=True, chunk_rows=1000)
pue, puw = query_prep(Mlp(*syn.user_proj), gating.user_net, syn.user_table[:8], cfg)
i2, s2, c2 = two_stage_top_k(dev, gating, pue, puw, 10, HIndexerConfig(k_prime=300, sample_ratio=0.5, quantized=True))
print("sanitize smoke OK", int(cand.sum()), int(c2.sum()))
