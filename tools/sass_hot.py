#!/usr/bin/env python
"""Hot-spot table from an ncu report's SASS source page: per-instruction stall samples and
executed counts, opcode mix.  usage: sass_hot.py report.ncu-rep kernel_regex [unit_count]"""
import collections
import csv
import io
import subprocess
import sys

rep, kre = sys.argv[1], sys.argv[2]
unit = float(sys.argv[3]) if len(sys.argv) > 3 else 1.0
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass", "-k", "regex:" + kre],
                     capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(out)))
hdr = rows[1]
data = rows[2:]
ia, ss, src, ad = (hdr.index(h) for h in ("Instructions Executed", "Warp Stall Sampling (All Samples)", "Source", "Address"))
tot_i = sum(float(r[ia] or 0) for r in data)
tot_s = sum(float(r[ss] or 0) for r in data)
print(f"warp instructions {tot_i:.4g} ({tot_i / unit:.1f} per unit), stall samples {tot_s:.4g}")
for i in sorted(range(len(data)), key=lambda i: -float(data[i][ss] or 0))[:15]:
    r = data[i]
    print(f"  {r[ad][-5:]} {100 * float(r[ss]) / tot_s:5.1f}%  x{float(r[ia]) / unit:7.2f}  {r[src][:60]:60s} | prev {data[i - 1][src][:40]}")
op = collections.Counter()
for r in data:
    t = r[src].strip()
    if t.startswith("@"):
        t = t.split(None, 1)[1]
    op[t.split()[0].split(".")[0]] += float(r[ia] or 0) / unit
print("opcodes per unit:", ", ".join(f"{k} {v:.1f}" for k, v in op.most_common(24)))
sc = [i for i, h in enumerate(hdr) if h.startswith("stall_") and "Not Issued" not in h]
agg = {hdr[i]: sum(float(r[i] or 0) for r in data) for i in sc}
print("stalls:", ", ".join(f"{k[6:]} {100 * v / tot_s:.1f}%" for k, v in sorted(agg.items(), key=lambda x: -x[1])[:10]))
