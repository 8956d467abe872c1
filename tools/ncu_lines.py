"""Summarise an ncu report: key raw metrics, stall mix, and the hottest CUDA
source lines by warp-stall samples (ncu --page source --print-source cuda,sass)."""
import csv
import io
import subprocess
import sys
from collections import defaultdict

rep = sys.argv[1]
top = int(sys.argv[2]) if len(sys.argv) > 2 else 30
kf = ["-k", "regex:" + sys.argv[3]] if len(sys.argv) > 3 else []   # kernel filter (multi-kernel reports)
raw = subprocess.run(["ncu", "-i", rep, *kf, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(raw)))
h, v = rows[0], rows[2] if len(rows) > 2 else rows[1]
for w in ["Kernel Name", "gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
          "launch__registers_per_thread", "launch__grid_size", "launch__block_size",
          "sm__warps_active.avg.pct_of_peak_sustained_active", "smsp__issue_active.avg.pct_of_peak_sustained_active",
          "sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active",
          "sm__inst_executed_pipe_fp64.avg.pct_of_peak_sustained_active",
          "smsp__thread_inst_executed_per_inst_executed.ratio", "sm__throughput.avg.pct_of_peak_sustained_elapsed",
          "FBSP.TriageCompute.dram__throughput.avg.pct_of_peak_sustained_elapsed", "dram__bytes.sum.per_second",
          "lts__t_sectors.sum", "lts__t_sector_hit_rate.pct",
          "l1tex__t_sector_hit_rate.pct"]:
    if w in h:
        print(f"{w} = {v[h.index(w)]} {rows[1][h.index(w)]}".rstrip())
src = subprocess.run(["ncu", "-i", rep, *kf, "--page", "source", "--csv", "--print-source", "cuda,sass"],
                     capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(src)))
hi = next(i for i, r in enumerate(rows) if r and r[0] == "Line No")
h = rows[hi]
si = h.index("Warp Stall Sampling (All Samples)")
ii = h.index("Instructions Executed")
stall_cols = [c for c in h if c.startswith("stall_") and "Not Issued" not in c]
agg = defaultdict(lambda: [0, 0])
txt = {}
tot_st = defaultdict(int)
cur = None
tot = 0
for r in rows[hi + 1:]:
    if len(r) < len(h) or r[0] == "Line No":
        continue
    if r[0]:
        try:
            cur = int(r[0])
            txt[cur] = r[1]
        except ValueError:
            continue
    try:
        s_, i_ = int(r[si] or 0), int(r[ii] or 0)
    except ValueError:
        continue
    agg[cur][0] += s_
    agg[cur][1] += i_
    tot += s_
    for c in stall_cols:
        try:
            tot_st[c] += int(r[h.index(c)] or 0)
        except ValueError:
            pass
T = sum(tot_st.values()) or 1
print("stalls: " + " ".join(f"{c[6:]}={100 * x / T:.1f}%" for c, x in sorted(tot_st.items(), key=lambda z: -z[1])[:9]))
for ln, (s_, i_) in sorted(agg.items(), key=lambda z: -z[1][0])[:top]:
    print(f"{ln:5d} {100 * s_ / tot:5.1f}% exec {i_ / 1e9:6.2f}G  {txt.get(ln, '')[:96]}")
