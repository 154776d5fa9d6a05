import sys, os
sys.path.insert(0, os.environ.get("GRAFT_REPO_ROOT", "/root/repo")); os.chdir(sys.path[0])
sys.path.insert(0, "tests")
import numpy as np
import test_gpu_parity as T
from paper_2306_04039_b200 import _lib as L
from paper_2306_04039_b200.engine import two_stage_top_k, two_stage_top_k_sharded, _mode
from paper_2306_04039_b200.hindexer import HIndexerConfig
from paper_2306_04039_b200.mol import ItemCache
from paper_2306_04039_b200.quant import QuantizedRows
cache, syn, ue, feats = T._synthetic_prod_cache(90_001, seed=51, n_users=40)
gating, og = T._prod_gating(syn)
uw = gating.user_net(feats)
X = cache.num_items
hcfg = HIndexerConfig(k_prime=2000, sample_ratio=0.05, quantized=True)
ref = two_stage_top_k(cache, gating, ue, uw, 20, hcfg, seed=7)
lam = hcfg.resolve_lambda(X); n = max(1, round(2000 * lam / X))
print("lam", lam, "n", n)
for P, cuts in ((1, [0, X]), (3, [0, 20_000, 61_111, X])):
    keys = []
    for lo, hi in zip(cuts[:-1], cuts[1:]):
        q = cache.stage1_q
        sh = ItemCache(config=cache.config, item_embs=cache.item_embs[lo:hi], item_gate_pre=cache.item_gate_pre[lo:hi],
                       stage1_embs=cache.stage1_embs[lo:hi], stage1_q=QuantizedRows(q.codes[lo:hi], q.scales[lo:hi]))
        kk = np.empty((40, n), dtype=np.uint32)
        L.call("molr_sample_top_keys", L.ctx(), sh.device_handle(), 40, 8, L.ptr(L.f32(ue)), _mode(hcfg), X, lo, lam, 7, n, L.ptr(kk), None)
        keys.append(kk)
        print(P, lo, "row0 top keys", kk[0, :4], kk[0, -3:], "row10", kk[10, :3], kk[10, -2:])
    rows = np.ascontiguousarray(np.stack(keys).transpose(1, 0, 2).reshape(40, -1))
    tk = np.empty(40, dtype=np.uint32)
    L.call("molr_select_nth_keys", L.ctx(), 40, rows.shape[1], L.ptr(rows), n, L.ptr(tk), None)
    # numpy check of the selection
    srt = -np.sort(-rows.astype(np.int64), axis=1)
    print(P, "tk", tk[:8], "numpy nth", srt[:8, n - 1])
