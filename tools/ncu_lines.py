#!/usr/bin/env python
"""Stall samples per CUDA source line: ncu SASS page + nvdisasm -g line table.
usage: ncu_lines.py report.ncu-rep kernel_regex object.o mangled_name_substring source.cu"""
import csv, io, os, re, subprocess, sys, tempfile

rep, kre, obj, fn, srcf = sys.argv[1:6]
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass", "-k", "regex:" + kre],
                     capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(out)))
hdr, data = rows[1], rows[2:]
ad, ss, ia = hdr.index("Address"), hdr.index("Warp Stall Sampling (All Samples)"), hdr.index("Instructions Executed")
base = int(data[0][ad], 16)
tot = sum(float(r[ss] or 0) for r in data)
d = tempfile.mkdtemp()
subprocess.run(["cuobjdump", "-xelf", "all", os.path.abspath(obj)], cwd=d, capture_output=True)
cub = [f for f in os.listdir(d) if f.endswith(".cubin")][0]
dis = subprocess.run(["nvdisasm", "-g", "-c", os.path.join(d, cub)], capture_output=True, text=True).stdout
off2line, line, infn = {}, None, False
for l in dis.split("\n"):
    if l.startswith("//-----"):
        infn = fn in l
    m = re.search(r'line (\d+)', l)
    if "//##" in l and m:
        line = int(m.group(1))
    m2 = re.search(r'/\*([0-9a-f]{4,})\*/', l)
    if infn and m2 and line is not None:
        off2line[int(m2.group(1), 16)] = line
agg, cnt = {}, {}
for r in data:
    ln = off2line.get(int(r[ad], 16) - base)
    agg[ln] = agg.get(ln, 0) + float(r[ss] or 0)
    cnt[ln] = cnt.get(ln, 0) + float(r[ia] or 0)
src = open(srcf).read().split("\n")
for ln, v in sorted(agg.items(), key=lambda x: -x[1])[:int(os.environ.get("TOP", "20"))]:
    print(f"{100 * v / tot:5.1f}%  instr {cnt[ln]:.3g}  line {ln}: {src[ln - 1].strip()[:95] if ln else ''}")
