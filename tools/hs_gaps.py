"""Summarise tools/hs_trace.py output: per-stream busy time and copy gaps."""
import json
import sys
from collections import defaultdict

d = json.load(open(sys.argv[1] if len(sys.argv) > 1 else "gpurun_out/hs_trace.json"))
ev = d["events"]
print("span_us", d["span_us"], "per step", d["span_us"] / d["steps"])
bys = defaultdict(list)
for t, du, s, n in ev:
    bys[(s, n)].append((t, du))
for k, v in sorted(bys.items()):
    print(k, len(v), "busy", round(sum(x[1] for x in v), 1), "avg", round(sum(x[1] for x in v) / len(v), 1))
for name in ("H2D", "D2H"):
    h = [(t, du) for t, du, s, n in ev if n == name]
    print(name, "gaps", [round(h[i + 1][0] - h[i][0] - h[i][1]) for i in range(len(h) - 1)])
    print(name, "durs", [round(x[1]) for x in h])
