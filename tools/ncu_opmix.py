"""Per-opcode instruction counts and stall-reason shares of one kernel in
an ncu report (``--page source --print-source sass``), plus the headline
pipe / memory metrics.  usage: ncu_opmix.py REPORT [n_units]
(n_units: divide instruction counts, e.g. by the faces of the launch)."""
import collections
import csv
import io
import re
import subprocess
import sys

rep = sys.argv[1]
units = float(sys.argv[2]) if len(sys.argv) > 2 else 1.0
raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True,
                     text=True).stdout
rows = list(csv.reader(io.StringIO(raw)))
hdr, vals = rows[0], rows[2]
pat = re.compile(r"(gpu__time_duration.sum|l1tex__t_sector_hit_rate.pct|lts__t_sector_hit_rate.pct|"
                 r"l1tex__throughput.avg.pct_of_peak_sustained_active|"
                 r"sm__pipe_tensor_subpipe_dmma_cycles_active.avg.pct_of_peak_sustained_active|"
                 r"sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active|"
                 r"sm__warps_active.avg.pct_of_peak_sustained_active|launch__registers_per_thread$|"
                 r"dram__bytes_(read|write).sum$|smsp__issue_active.avg.pct_of_peak_sustained_active|"
                 r"stalled_(wait|long_scoreboard|short_scoreboard|math_pipe_throttle)_per_issue_active)")
for h, v in zip(hdr, vals):
    if pat.search(h) and not h.startswith(("SM_", "TPC.")):
        print(f"   {h:84s} {v}")
src = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass"],
                     capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(src)))
hi = [i for i, r in enumerate(rows) if r and r[0] == "Address"][0]
hdr, data = rows[hi], rows[hi + 1:]
si, ie = hdr.index("Source"), hdr.index("Instructions Executed")
sc = [i for i, h in enumerate(hdr) if h.startswith("stall_") and "Not Issued" not in h]
agg, cnt = collections.defaultdict(collections.Counter), collections.Counter()
for r in data:
    if len(r) < len(hdr) or not r[si].split():
        continue
    t = r[si].split()
    op = (t[1] if t[0].startswith("@") else t[0]).split(".")[0]
    cnt[op] += float(r[ie] or 0)
    for c in sc:
        agg[op][hdr[c]] += float(r[c] or 0)
tot = sum(sum(v.values()) for v in agg.values())
print(f"   per-opcode warp instructions (/ {units:g} units) and stall-sample shares:")
for op, v in sorted(agg.items(), key=lambda kv: -sum(kv[1].values()))[:10]:
    s = sum(v.values())
    print(f"     {op:8s} {cnt[op] / units:10.1f}  stall {100 * s / tot:5.1f}%  " +
          ", ".join(f"{k[6:]} {100 * x / s:.0f}%" for k, x in v.most_common(3)))
