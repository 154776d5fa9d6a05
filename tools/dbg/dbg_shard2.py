import sys, os
sys.path.insert(0, os.environ.get("GRAFT_REPO_ROOT", "/root/repo")); os.chdir(sys.path[0])
sys.path.insert(0, "tests")
import numpy as np
import test_gpu_parity as T
from paper_2306_04039_b200 import _lib as L
from paper_2306_04039_b200.engine import _mode
from paper_2306_04039_b200.hindexer import HIndexerConfig
cache, syn, ue, feats = T._synthetic_prod_cache(90_001, seed=51, n_users=200)
X = cache.num_items
hcfg = HIndexerConfig(k_prime=2000, sample_ratio=0.05, quantized=True)
lam = hcfg.resolve_lambda(X); n = 100
def keys(B):
    kk = np.empty((B, n), dtype=np.uint32)
    L.call("molr_sample_top_keys", L.ctx(), cache.device_handle(), B, 8, L.ptr(L.f32(ue[:B])), _mode(hcfg), X, 0, lam, 7, n, L.ptr(kk), None)
    return np.sort(kk, axis=1)
a = keys(200)
for B in (1, 8, 32, 33, 40, 64, 128):
    b = keys(B)
    bad = [i for i in range(B) if not np.array_equal(a[i], b[i])]
    print("B", B, "rows differing from B=200:", bad[:10], flush=True)
os.environ["MOLR_DISABLE_TC"] = "1"
c = keys(200)
print("simt vs tc B=200 differing rows:", [i for i in range(200) if not np.array_equal(a[i], c[i])][:10])
