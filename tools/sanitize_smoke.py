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

# SAN_NEW_ONLY=1: only the round-1 additions (small-batch, float view, sharded) on a smaller corpus
# (racecheck is slow on the shared-memory-heavy kernels)
NEW_ONLY = os.environ.get("SAN_NEW_ONLY") == "1"
cache, syn, ue, feats = _synthetic_prod_cache(int(os.environ.get("SAN_X", 8_000)) if NEW_ONLY else 40_000, seed=3, n_users=40)
gating, _ = _prod_gating(syn)
uw = gating.user_net(feats)
KP = max(30, cache.num_items // 20) if NEW_ONLY else 2000
ids, sc, cand = two_stage_top_k(cache, gating, ue, uw, 20, HIndexerConfig(k_prime=KP, sample_ratio=0.2, quantized=True),
                                seed=1)
c2 = np.zeros(1, dtype=np.int64)
if not NEW_ONLY:
    bi, bs = batch_mol_top_k(cache, gating, ue[:4], feats[:4], 50)
    cfg = MoLConfig(k_u=8, k_x=8, d=64, tau=20.0, gating_hidden=128, dropout_p=0.0)
    dev = build_device_item_cache(syn.item_table[:3000], Mlp(*syn.item_proj), Mlp(*syn.gating.item_net), cfg,
                                  round_bf16=True, chunk_rows=1000)
    pue, puw = query_prep(Mlp(*syn.user_proj), gating.user_net, syn.user_table[:8], cfg)
    i2, s2, c2 = two_stage_top_k(dev, gating, pue, puw, 10, HIndexerConfig(k_prime=300, sample_ratio=0.5, quantized=True))
# small-batch int8 kernel (B <= 32), the float view (fp16 tensor-core filter, big and small batch,
# pilot + sample filter), and the sharded single-device-threshold protocol (2 in-process shards)
i3, s3, c3 = two_stage_top_k(cache, gating, ue[:5], uw[:5], 20, HIndexerConfig(k_prime=KP, sample_ratio=0.2,
                                                                                 quantized=True), seed=2)
for nb in (3, 40):
    two_stage_top_k(cache, gating, ue[:nb], uw[:nb], 20, HIndexerConfig(k_prime=KP, sample_ratio=0.2, quantized=False),
                    seed=3)
from paper_2306_04039_b200.engine import two_stage_top_k_sharded  # noqa: E402
from paper_2306_04039_b200.mol import ItemCache  # noqa: E402
from paper_2306_04039_b200.quant import QuantizedRows  # noqa: E402
from tests.test_gpu_parity import _run_shards  # noqa: E402

X = cache.num_items
cuts = [0, X // 2 - X // 10, X]
q = cache.stage1_q
shards = [ItemCache(config=cache.config, item_embs=cache.item_embs[lo:hi], item_gate_pre=cache.item_gate_pre[lo:hi],
                    stage1_embs=cache.stage1_embs[lo:hi], stage1_q=QuantizedRows(q.codes[lo:hi], q.scales[lo:hi]))
          for lo, hi in zip(cuts[:-1], cuts[1:])]
h = HIndexerConfig(k_prime=KP, sample_ratio=0.2, quantized=True)
res = _run_shards(lambda r, ex: two_stage_top_k_sharded(shards[r], gating, ue, uw, 20, h, X_global=X, row_lo=cuts[r],
                                                        exchange=ex, seed=1), 2)
assert np.array_equal(res[0][0], ids) and np.array_equal(res[0][2], cand)
# round 2: an f32-stored (reference-built) cache on the tensor-core scorer (hi + lo component
# image, f32 gate pre-activations), through the batched exact top-k and the two-stage path
from tests.test_gpu_parity import _f32_prod_cache  # noqa: E402
from paper_2306_04039_b200.mol import uses_tensor_cores  # noqa: E402

fcache, fsyn, fue, ffeats = _f32_prod_cache(int(os.environ.get("SAN_X", 8_000)), seed=5, n_users=8)
fgating, _ = _prod_gating(fsyn)
assert uses_tensor_cores(fcache, fgating)
fi, fs = batch_mol_top_k(fcache, fgating, fue, ffeats, 20)
two_stage_top_k(fcache, fgating, fue, fgating.user_net(ffeats), 20, HIndexerConfig(k_prime=KP, sample_ratio=0.2,
                                                                                  quantized=True), seed=4)
print("sanitize smoke OK", int(cand.sum()), int(c2.sum()), int(c3.sum()), int(fi.sum()))
