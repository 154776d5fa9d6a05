import os, sys, time
sys.path.insert(0, '/root/repo'); os.chdir('/root/repo')
import numpy as np, torch
import bench as Bm
from paper_2306_04039_b200 import _lib as L
from paper_2306_04039_b200.mol import GatingNetwork, Mlp, _gating_handle
from paper_2306_04039_b200.numerics import DEFAULT_EPS
dev = torch.device('cuda', 0); torch.cuda.set_device(0)
st = torch.cuda.Stream(); torch.cuda.set_stream(st); sp = st.cuda_stream
lib = L.load(); ctx = L.ctx(0)
model = Bm.synthetic_model()
X = int(sys.argv[1]) if len(sys.argv) > 1 else 100_000_000
F32 = os.environ.get('LAT_VIEW') == 'f32'  # the float stage-1 view (quantized=False)
cfg, cache = Bm.build_shard(model, X, 0, X, seed=11, dev=dev, lib=lib, ctx=ctx, storage=L.STORE_S1_F32 if F32 else None)
gh = _gating_handle(GatingNetwork(Mlp(*model['user_net']), Mlp(*model['item_net']), Mlp(*model['cross_net'])))
feats_h, feats_d = Bm.make_queries(model, 64, 1, dev)
W = {k: [torch.from_numpy(a).to(dev) for a in v] for k, v in model.items()}
for B in (1, 8, 32, 64, 128):
    ue = torch.empty((B, 8, 64), device=dev); uw = torch.empty((B, 64), device=dev)
    ids = torch.empty((B, 100), dtype=torch.int64, device=dev); sc = torch.empty((B, 100), device=dev)
    def run(i):
        L.call("molr_query_prep", ctx, B, 64, feats_d.data_ptr(), 128, W['user_proj'][0].data_ptr(), W['user_proj'][1].data_ptr(), W['user_proj'][2].data_ptr(), 8, 64, 1, 128, W['user_net'][0].data_ptr(), W['user_net'][1].data_ptr(), W['user_net'][2].data_ptr(), 64, float(DEFAULT_EPS), ue.data_ptr(), uw.data_ptr(), sp)
        L.call("molr_two_stage_top_k", ctx, cache.device_handle(), gh, B, 8, ue.data_ptr(), uw.data_ptr(), 20.0, L.S1_FLOAT if F32 else L.S1_INT8, 100_000, X // 100, 5 + i, L.INCLUSIVE, 100, 0, ids.data_ptr(), sc.data_ptr(), None, sp)
    for i in range(3): run(i)
    torch.cuda.synchronize()
    L.prof_reset(0); L.set_profiling(True, 0)
    t0 = time.perf_counter()
    for i in range(5): run(i)
    torch.cuda.synchronize(); dt = (time.perf_counter() - t0) / 5 * 1e3
    L.set_profiling(False, 0)
    pr = {k: round(v[1] / v[0], 3) for k, v in L.prof_read(0).items()}
    print(f"B={B}: {dt:.2f} ms per call; kernels {pr}", flush=True)
