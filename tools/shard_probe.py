"""Per-rank cost of the two N>1 threshold modes on one shard of a P-way split (python
tools/shard_probe.py [X_global] [P]): local (K'/P, lambda/P pilot path) vs single-device
(molr_sample_top_keys + select + molr_two_stage_top_k_at), B = 1024, timed with CUDA events."""
import os, sys, time
sys.path.insert(0, os.environ.get("GRAFT_REPO_ROOT", "/root/repo")); os.chdir(sys.path[0])
import numpy as np, torch
import bench as Bm
from paper_2306_04039_b200 import _lib as L
from paper_2306_04039_b200.mol import GatingNetwork, Mlp, _gating_handle
from paper_2306_04039_b200.numerics import DEFAULT_EPS
from paper_2306_04039_b200.sharding import local_k_prime, local_lambda
dev = torch.device('cuda', 0); torch.cuda.set_device(0)
st = torch.cuda.Stream(); torch.cuda.set_stream(st); sp = st.cuda_stream
lib = L.load(); ctx = L.ctx(0)
Xg = int(sys.argv[1]) if len(sys.argv) > 1 else 100_000_000
P = int(sys.argv[2]) if len(sys.argv) > 2 else 8
lo, hi = 0, Xg // P
model = Bm.synthetic_model()
cfg, cache = Bm.build_shard(model, Xg, lo, hi, seed=11, dev=dev, lib=lib, ctx=ctx)
gh = _gating_handle(GatingNetwork(Mlp(*model['user_net']), Mlp(*model['item_net']), Mlp(*model['cross_net'])))
W = {k: [torch.from_numpy(a).to(dev) for a in v] for k, v in model.items()}
B, k, KP = 1024, 100, 100_000
feats_h, feats_d = Bm.make_queries(model, B, 1, dev)
ue = torch.empty((B, 8, 64), device=dev); uw = torch.empty((B, 64), device=dev)
L.call("molr_query_prep", ctx, B, 64, feats_d.data_ptr(), 128, W['user_proj'][0].data_ptr(), W['user_proj'][1].data_ptr(), W['user_proj'][2].data_ptr(), 8, 64, 1, 128, W['user_net'][0].data_ptr(), W['user_net'][1].data_ptr(), W['user_net'][2].data_ptr(), 64, float(DEFAULT_EPS), ue.data_ptr(), uw.data_ptr(), sp)
ids = torch.empty((B, k), dtype=torch.int64, device=dev); sc = torch.empty((B, k), device=dev)
cnt = np.empty(B, dtype=np.int64)
kp_l = local_k_prime(KP, P); lam_l = local_lambda(hi - lo, sample_ratio=0.01); lam_g = local_lambda(Xg, sample_ratio=0.01)
n = max(1, round(KP * lam_g / Xg))
keys = torch.empty((B, n), dtype=torch.int32, device=dev)
rows = torch.empty((B, P * n), dtype=torch.int32, device=dev)
tk = torch.empty((B,), dtype=torch.int32, device=dev)
def local(i):
    L.call("molr_two_stage_top_k", ctx, cache.device_handle(), gh, B, 8, ue.data_ptr(), uw.data_ptr(), 20.0, L.S1_INT8, kp_l, lam_l, 7 + i, L.INCLUSIVE, k, lo, ids.data_ptr(), sc.data_ptr(), L.ptr(cnt), sp)
def glob(i):
    L.call("molr_sample_top_keys", ctx, cache.device_handle(), B, 8, ue.data_ptr(), L.S1_INT8, Xg, lo, lam_g, 7 + i, n, keys.data_ptr(), sp)
    rows.copy_(keys.repeat(1, P))  # stand-in for the all-gather (same sizes)
    L.call("molr_select_nth_keys", ctx, B, P * n, rows.data_ptr(), n, tk.data_ptr(), sp)
    L.call("molr_two_stage_top_k_at", ctx, cache.device_handle(), gh, B, 8, ue.data_ptr(), uw.data_ptr(), 20.0, L.S1_INT8, kp_l, tk.data_ptr(), L.INCLUSIVE, k, lo, ids.data_ptr(), sc.data_ptr(), L.ptr(cnt), sp)
for name, fn in (("local", local), ("global", glob)):
    for i in range(3): fn(i)
    torch.cuda.synchronize()
    L.prof_reset(0); L.set_profiling(True, 0)
    e0 = torch.cuda.Event(enable_timing=True); e1 = torch.cuda.Event(enable_timing=True)
    e0.record(st)
    for i in range(5): fn(i)
    e1.record(st); torch.cuda.synchronize()
    L.set_profiling(False, 0)
    pr = {kk: round(v[1] / v[0], 3) for kk, v in L.prof_read(0).items()}
    print(f"P={P} shard={hi - lo} {name}: {e0.elapsed_time(e1) / 5:.2f} ms/step, mean cand {cnt.mean():.0f}; {pr}", flush=True)
