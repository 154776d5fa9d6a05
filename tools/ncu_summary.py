#!/usr/bin/env python
"""Summarise ncu output for profiles/.

  launches <launches.csv>          per-kernel launch count, total/avg time, share (the
                                   `--metrics gpu__time_duration.sum` launch list)
  full <report.ncu-rep>            key metrics per captured kernel of a `--set full` report
"""
import collections
import csv
import io
import subprocess
import sys

# north_star evidence per kernel: tensor-pipe utilisation (all / imma / hmma sub-pipes), DRAM
# throughput and bytes, issue utilisation and the pipes that bound the SIMT epilogues
KEYS = [
    "sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_active",
    "sm__pipe_tensor_subpipe_imma_cycles_active.avg.pct_of_peak_sustained_active",
    "sm__pipe_tensor_subpipe_hmma_cycles_active.avg.pct_of_peak_sustained_active",
    "sm__inst_executed_pipe_tensor_subpipe_imma.avg.pct_of_peak_sustained_active",
    "sm__inst_executed_pipe_tensor_subpipe_hmma.avg.pct_of_peak_sustained_active",
    "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed",
    "sm__inst_executed_pipe_alu.avg.pct_of_peak_sustained_active",
    "smsp__average_warps_issue_stalled_wait_per_issue_active.ratio",
    "smsp__average_warps_issue_stalled_long_scoreboard_per_issue_active.ratio",
    "smsp__average_warps_issue_stalled_math_pipe_throttle_per_issue_active.ratio",
    "smsp__average_warps_issue_stalled_sleeping_per_issue_active.ratio",
    "gpu__time_duration.sum", "sm__cycles_elapsed.avg.per_second", "dram__bytes_read.sum", "dram__bytes_write.sum",
    "dram__throughput.avg.pct_of_peak_sustained_elapsed", "sm__throughput.avg.pct_of_peak_sustained_elapsed",
    "sm__inst_issued.avg.pct_of_peak_sustained_active", "sm__pipe_tensor_cycles_active_realtime.avg.pct_of_peak_sustained_elapsed",
    "sm__inst_executed_pipe_xu.avg.pct_of_peak_sustained_active", "sm__pipe_fma_cycles_active.avg.pct_of_peak_sustained_active",
    "sm__pipe_alu_cycles_active.avg.pct_of_peak_sustained_active", "sm__inst_executed_pipe_tmem.avg.pct_of_peak_sustained_active",
    "l1tex__throughput.avg.pct_of_peak_sustained_active", "lts__t_bytes.sum", "lts__t_sector_hit_rate.pct",
    "sm__warps_active.avg.pct_of_peak_sustained_active", "launch__registers_per_thread", "launch__grid_size",
    "launch__block_size", "smsp__inst_executed.sum",
]


def _rows(text):
    r = list(csv.reader(io.StringIO(text)))
    return r


def launches(path):
    with open(path) as f:
        lines = [l for l in f if not l.startswith("==")]
    r = _rows("".join(lines))
    hdr = r[0]
    ki, mi, vi = hdr.index("Kernel Name"), hdr.index("Metric Name"), hdr.index("Metric Value")
    agg = collections.defaultdict(lambda: [0, 0.0])
    unit = None
    for row in r[1:]:
        if len(row) <= vi or row[mi] != "gpu__time_duration.sum":
            continue
        v = float(row[vi].replace(",", ""))
        unit = row[hdr.index("Metric Unit")] if "Metric Unit" in hdr else unit
        name = row[ki].split("(")[0][:90]
        agg[name][0] += 1
        agg[name][1] += v
    tot = sum(v[1] for v in agg.values()) or 1
    print(f"# per-kernel launch list (unit {unit}); cold-cache, serialised replay: compare SHARES, not absolutes")
    print(f"{'kernel':90s} {'n':>6s} {'total':>12s} {'avg':>12s} {'share':>7s}")
    for name, (n, t) in sorted(agg.items(), key=lambda kv: -kv[1][1]):
        print(f"{name:90s} {n:6d} {t:12.1f} {t / n:12.1f} {100 * t / tot:6.1f}%")


def full(path):
    out = subprocess.run(["ncu", "-i", path, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    r = _rows(out)
    hdr, units = r[0], r[1]
    for row in r[2:]:
        d = dict(zip(hdr, row))
        print("## " + d.get("Kernel Name", "?")[:120])
        for k in KEYS:
            if k in d:
                print(f"  {k:80s} {d[k]:>16s} {units[hdr.index(k)]}")
        extra = [h for h in hdr if ("imma" in h or "hmma" in h or "pipe_tensor" in h) and "realtime" in h
                 and h.endswith("pct_of_peak_sustained_elapsed")]
        for k in extra:
            print(f"  {k:80s} {d[k]:>16s} %")
        # bytes per launch (for profiles/traffic.json)
        try:
            rb = float(d["dram__bytes_read.sum"].replace(",", ""))
            wb = float(d["dram__bytes_write.sum"].replace(",", ""))
            ur, uw_ = units[hdr.index("dram__bytes_read.sum")], units[hdr.index("dram__bytes_write.sum")]
            scale = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}
            print(f"  {'dram bytes read+write per launch':80s} {rb * scale.get(ur, 1) + wb * scale.get(uw_, 1):16.4g} B")
        except (KeyError, ValueError):
            pass


if __name__ == "__main__":
    {"launches": launches, "full": full}[sys.argv[1]](sys.argv[2])
