"""Per-kernel launch list of ONE small-batch two-stage call at 100M items (B from argv, default 1):
run under `ncu --profile-from-start off --metrics gpu__time_duration.sum`; the profiled range is
the last of a few warm calls (query prep + molr_two_stage_top_k)."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import bench as Bm  # noqa: E402
from paper_2306_04039_b200 import _lib as L  # noqa: E402
from paper_2306_04039_b200.mol import GatingNetwork, Mlp, _gating_handle  # noqa: E402
from paper_2306_04039_b200.numerics import DEFAULT_EPS  # noqa: E402

dev = torch.device("cuda", 0)
torch.cuda.set_device(0)
st = torch.cuda.Stream()
torch.cuda.set_stream(st)
sp = st.cuda_stream
lib, ctx = L.load(), L.ctx(0)
model = Bm.synthetic_model()
X = int(os.environ.get("LAT_X", 100_000_000))
B = int(sys.argv[1]) if len(sys.argv) > 1 else 1
cfg, cache = Bm.build_shard(model, X, 0, X, seed=11, dev=dev, lib=lib, ctx=ctx)
gh = _gating_handle(GatingNetwork(Mlp(*model["user_net"]), Mlp(*model["item_net"]), Mlp(*model["cross_net"])))
feats_h, feats_d = Bm.make_queries(model, B, 1, dev)
W = {k: [torch.from_numpy(a).to(dev) for a in v] for k, v in model.items()}
ue = torch.empty((B, 8, 64), device=dev)
uw = torch.empty((B, 64), device=dev)
ids = torch.empty((B, 100), dtype=torch.int64, device=dev)
sc = torch.empty((B, 100), device=dev)


def run(i):
    L.call("molr_query_prep", ctx, B, 64, feats_d.data_ptr(), 128, W["user_proj"][0].data_ptr(),
           W["user_proj"][1].data_ptr(), W["user_proj"][2].data_ptr(), 8, 64, 1, 128, W["user_net"][0].data_ptr(),
           W["user_net"][1].data_ptr(), W["user_net"][2].data_ptr(), 64, float(DEFAULT_EPS), ue.data_ptr(), uw.data_ptr(), sp)
    L.call("molr_two_stage_top_k", ctx, cache.device_handle(), gh, B, 8, ue.data_ptr(), uw.data_ptr(), 20.0, L.S1_INT8,
           100_000, X // 100, 5 + i, L.INCLUSIVE, 100, 0, ids.data_ptr(), sc.data_ptr(), None, sp)


for i in range(4):
    run(i)
torch.cuda.synchronize()
torch.cuda.profiler.start()
run(9)
torch.cuda.synchronize()
torch.cuda.profiler.stop()
print("done")
