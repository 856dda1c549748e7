"""Per-source-line instruction / stall-sample breakdown of one kernel in an
ncu report: joins ncu's per-SASS counts with nvdisasm line info of the
same cubin.  usage: ncu_lines.py REPORT CUBIN MANGLED_NAME [top]"""
import csv
import io
import re
import subprocess
import sys
from collections import Counter

rep, cubin, fun = sys.argv[1:4]
top = int(sys.argv[4]) if len(sys.argv) > 4 else 40
raw = subprocess.run(["ncu", "-i", rep] + (["-k", "regex:" + sys.argv[5]] if len(sys.argv) > 5 else []) + ["--page", "source", "--csv", "--print-source", "sass"],
                     capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(raw)))
hdr, counts = None, []
for r in rows:
    if r and r[0] == "Address":
        hdr = r
        continue
    if hdr and r and r[0].startswith("0x"):
        d = dict(zip(hdr, r))
        counts.append((int(d["Address"], 16), int(d["Instructions Executed"] or 0),
                       int(d["Warp Stall Sampling (All Samples)"] or 0), d["Source"].strip()))
base = counts[0][0]
dis = subprocess.run(["nvdisasm", "-g", "-c", cubin], capture_output=True, text=True).stdout
lines, on = [], False
for ln in dis.splitlines():
    if ".text." in ln and ln.lstrip().startswith(".section"):
        on = ln.split(".text.")[1].split(",")[0].strip('"') == fun
        continue
    if on:
        lines.append(ln)
line_of = {}
cur = None
for ln in lines:
    m = re.search(r'line (\d+)', ln)
    if "//##" in ln and m:
        cur = int(m.group(1))
        continue
    m = re.match(r"\s+/\*([0-9a-f]{4,})\*/", ln)
    if m:
        line_of[int(m.group(1), 16)] = cur
byline, samp, ops = Counter(), Counter(), {}
tot = ts = 0
for a, n, s, src in counts:
    L = line_of.get(a - base)
    byline[L] += n
    samp[L] += s
    tot += n
    ts += s
    op = src.split()[1 if src.startswith("@") else 0].split(".")[0]
    ops.setdefault(L, Counter())[op] += n
print(f"total warp-inst {tot}, samples {ts}")
for L, n in byline.most_common(top):
    o = ", ".join(f"{k}:{v * 100 // max(n, 1)}%" for k, v in ops[L].most_common(4))
    print(f"L{L!s:>5} inst {n / tot * 100:5.1f}%  stall {samp[L] / max(ts, 1) * 100:5.1f}%  {o}")
