"""Float stage-1 view (MOLR_S1_FLOAT) timing: bf16 tensor-core filter vs the fp32 SIMT scan vs
the int8 view, same corpus (python tools/float_probe.py [X])."""
import os, sys, time
sys.path.insert(0, os.environ.get("GRAFT_REPO_ROOT", "/root/repo")); os.chdir(sys.path[0])
os.environ["MOLR_LIB_PATH"] = os.path.join(sys.path[0], "paper_2306_04039_b200", "libmolr_b200_dev.so")  # switches
import numpy as np, torch
import bench as Bm
from paper_2306_04039_b200 import _lib as L
from paper_2306_04039_b200.mol import GatingNetwork, Mlp, _gating_handle
from paper_2306_04039_b200.numerics import DEFAULT_EPS
dev = torch.device('cuda', 0); torch.cuda.set_device(0)
st = torch.cuda.Stream(); torch.cuda.set_stream(st); sp = st.cuda_stream
lib = L.load(); ctx = L.ctx(0)
model = Bm.synthetic_model()
X = int(sys.argv[1]) if len(sys.argv) > 1 else 10_000_000
cfg, cache = Bm.build_shard(model, X, 0, X, seed=11, dev=dev, lib=lib, ctx=ctx, storage=L.STORE_S1_F32 | L.STORE_S1_INT8)
gh = _gating_handle(GatingNetwork(Mlp(*model['user_net']), Mlp(*model['item_net']), Mlp(*model['cross_net'])))
W = {k: [torch.from_numpy(a).to(dev) for a in v] for k, v in model.items()}
kp = int(sys.argv[2]) if len(sys.argv) > 2 else max(1000, X // 1000)
for B, modes in ((1, ("bf", "simt", "int8")), (64, ("bf", "simt", "int8")), (1024, ("bf", "simt", "int8"))):
    feats_h, feats_d = Bm.make_queries(model, B, 1, dev)
    ue = torch.empty((B, 8, 64), device=dev); uw = torch.empty((B, 64), device=dev)
    ids = torch.empty((B, 100), dtype=torch.int64, device=dev); sc = torch.empty((B, 100), device=dev)
    cnt = torch.empty((B,), dtype=torch.int64, device=dev)
    L.call("molr_query_prep", ctx, B, 64, feats_d.data_ptr(), 128, W['user_proj'][0].data_ptr(), W['user_proj'][1].data_ptr(), W['user_proj'][2].data_ptr(), 8, 64, 1, 128, W['user_net'][0].data_ptr(), W['user_net'][1].data_ptr(), W['user_net'][2].data_ptr(), 64, float(DEFAULT_EPS), ue.data_ptr(), uw.data_ptr(), sp)
    res = {}
    for m in modes:
        if m == "simt": os.environ["MOLR_S1_NO_BF"] = "1"
        else: os.environ.pop("MOLR_S1_NO_BF", None)
        mode = L.S1_INT8 if m == "int8" else L.S1_FLOAT
        def run(i):
            L.call("molr_two_stage_top_k", ctx, cache.device_handle(), gh, B, 8, ue.data_ptr(), uw.data_ptr(), 20.0, mode, kp, X // 100, 5 + i, L.INCLUSIVE, 100, 0, ids.data_ptr(), sc.data_ptr(), cnt.data_ptr(), sp)
        reps = 1 if m == "simt" else 3
        run(0); torch.cuda.synchronize()
        res[m] = (ids.cpu().numpy().copy(), cnt.cpu().numpy().copy())
        L.prof_reset(0); L.set_profiling(True, 0)
        t0 = time.perf_counter()
        for i in range(reps): run(i)
        torch.cuda.synchronize(); dt = (time.perf_counter() - t0) / reps * 1e3
        L.set_profiling(False, 0)
        pr = {k: round(v[1] / v[0], 3) for k, v in L.prof_read(0).items()}
        print(f"X={X} B={B} {m}: {dt:.2f} ms/call, mean cand {cnt.float().mean().item():.0f}; {pr}", flush=True)
    if "simt" in res:
        print("  bf == simt:", np.array_equal(res["bf"][0], res["simt"][0]) and np.array_equal(res["bf"][1], res["simt"][1]), flush=True)
