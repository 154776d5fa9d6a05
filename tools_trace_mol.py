"""Dev tool: run the tc MoL kernel once with MOLR_TRACE_MOL set and print CTA 0's timeline."""
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.abspath(__file__)))
os.environ["MOLR_TRACE_MOL"] = "/tmp/mol_trace.bin"
from tests.test_gpu_parity import _prod_gating, _synthetic_prod_cache  # noqa: E402
from paper_2306_04039_b200.mol import batch_score_all  # noqa: E402

cache, syn, ue, feats = _synthetic_prod_cache(200_000, seed=5, n_users=8)
gating, _ = _prod_gating(syn)
for _ in range(2):
    batch_score_all(cache, gating, ue, feats)
t = np.fromfile("/tmp/mol_trace.bin", dtype=np.uint64)
n = int(t[0])
ev = t[1:1 + n]
tags = (ev >> np.uint64(56)).astype(int)
clk = (ev & np.uint64((1 << 56) - 1)).astype(np.int64)
clk -= clk.min()
order = np.argsort(clk, kind="stable")
names = {1: "prod_stage", 2: "C_done", 3: "L1_issued", 4: "L2_issued", 5: "E0_start", 6: "E1_start", 7: "E2_start",
         8: "E2_end"}
print("events", n)
for i in order[:400]:
    g, k = divmod(tags[i], 16)
    print(f"{clk[i]:>10d}  g{g} {names.get(k, k)}")
