"""Dev tool: run the tc MoL kernel with MOLR_TRACE_MOL set and summarise CTA 0's epilogue
timeline (per-phase cycles per tile, averaged over tiles)."""
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
os.environ["MOLR_TRACE_MOL"] = "/tmp/mol_trace.bin"
# the trace exists only in the development build (-DMOLR_DEV_KNOBS)
os.environ["MOLR_LIB_PATH"] = os.path.join(sys.path[0], "paper_2306_04039_b200", "libmolr_b200_dev.so")
from tests.test_gpu_parity import _prod_gating, _synthetic_prod_cache  # noqa: E402
from paper_2306_04039_b200.mol import batch_score_all  # noqa: E402

cache, syn, ue, feats = _synthetic_prod_cache(int(os.environ.get("TRACE_ITEMS", "200000")), seed=5, n_users=int(os.environ.get("TRACE_USERS", "64")))
gating, _ = _prod_gating(syn)
for _ in range(2):
    batch_score_all(cache, gating, ue, feats)
t = np.fromfile("/tmp/mol_trace.bin", dtype=np.uint64)
n = min(int(t[0]), 65535)
ev = t[1:1 + n]
tags = (ev >> np.uint64(56)).astype(int)
clk = (ev & np.uint64((1 << 56) - 1)).astype(np.int64)
names = ["start", "d0_ready", "E0_done", "E05_done", "d1_ready", "E1_done", "d2_ready", "E2_done"]
for g in range(2):
    sel = [clk[(tags == g * 16 + k)] for k in range(8)]
    m = min(len(x) for x in sel)
    a = np.stack([x[:m] for x in sel])  # (8, tiles)
    d = np.diff(a, axis=0)
    per_tile = np.diff(a[0])
    print(f"group {g}: {m} tiles, cycles per tile {np.median(per_tile):.0f}")
    for k in range(7):
        print(f"   {names[k]:>9s} -> {names[k + 1]:<9s} {np.median(d[k]):8.0f}")
    print(f"   E2_done -> next start {np.median(a[0, 1:] - a[7, :-1]):8.0f}")
a0, a1 = clk[tags == 32], clk[tags == 33]
m = min(len(a0), len(a1))
if m > 2:
    print(f"component stream: {m} tiles, cycles per tile {np.median(np.diff(a0[:m])):.0f}, "
          f"stages wait+MMA {np.median(a1[:m] - a0[:m]):.0f}, commit->next start {np.median(a0[1:m] - a1[:m - 1]):.0f}")
