"""GPU busy time vs wall time of the C2 SDIRK3 + JFNK step (reference
defaults) under torch.profiler (CUPTI): how much of an Arnoldi step is the
host round trip.  Runs one warm-up step, then profiles one Newton solve's
worth of GMRES via one SDIRK3 step.

usage: python tools/jfnk_trace.py > gpurun_out/jfnk_trace.json
"""
import json
import os
import sys
import time
from collections import defaultdict

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import bench  # noqa: E402
from paper_1403_1157_b200.operator import DiscreteOperator  # noqa: E402
from paper_1403_1157_b200.timeint import integrate  # noqa: E402

dev = torch.device("cuda:0")
cfg, space, model, scheme, U0h, _ = bench.build_problem("c2", "cdg2", device=dev)
op = DiscreteOperator(space, model, scheme, device=dev)
U = torch.from_numpy(U0h).to(dev)
nk = {"rtol": 1e-8, "atol": 1e-12, "maxiter": 25, "gmres_rtol": 1e-4,
      "gmres_restart": 30, "gmres_maxiter": 200}
integrate(op, U, 0.0, 1.0, 0.01, order=3, n_steps=1, newton_kwargs=nk)
torch.cuda.synchronize()
with torch.profiler.profile(activities=[torch.profiler.ProfilerActivity.CUDA]) as prof:
    t0 = time.perf_counter()
    res = integrate(op, U, 0.0, 1.0, 0.01, order=3, n_steps=1, newton_kwargs=nk)
    torch.cuda.synchronize()
    wall = time.perf_counter() - t0
path = "/tmp/jfnk_trace.json"
prof.export_chrome_trace(path)
ev = [e for e in json.load(open(path))["traceEvents"]
      if e.get("ph") == "X" and e.get("cat") in ("kernel", "gpu_memcpy", "gpu_memset")]
iv = sorted((float(e["ts"]), float(e["ts"]) + float(e["dur"])) for e in ev)
busy, cur0, cur1 = 0.0, None, None
for a, b in iv:
    if cur1 is None or a > cur1:
        if cur1 is not None:
            busy += cur1 - cur0
        cur0, cur1 = a, b
    else:
        cur1 = max(cur1, b)
busy += cur1 - cur0
per = defaultdict(lambda: [0, 0.0])
for e in ev:
    k = e["name"].split("<")[0].replace("void ", "")[:40]
    per[k][0] += 1
    per[k][1] += float(e["dur"])
span = iv[-1][1] - iv[0][0]
# idle gaps between consecutive GPU activities, by (previous, next) kernel
evs = sorted(((float(e["ts"]), float(e["ts"]) + float(e["dur"]),
               e["name"].split("<")[0].replace("void ", "")[:28]) for e in ev))
gaps = defaultdict(lambda: [0, 0.0])
end, prev = evs[0][1], evs[0][2]
for a, b, nm in evs[1:]:
    if a > end + 1.0:
        gaps[(prev, nm)][0] += 1
        gaps[(prev, nm)][1] += a - end
    if b >= end:
        end, prev = b, nm
out = {"wall_ms": wall * 1e3, "gpu_span_ms": span / 1e3, "gpu_busy_ms": busy / 1e3,
       "f_evaluations": res.f_evaluations, "gmres_iterations": res.gmres_iterations,
       "idle_gaps": {f"{k[0]} -> {k[1]}": {"n": v[0], "ms": round(v[1] / 1e3, 3)}
                     for k, v in sorted(gaps.items(), key=lambda kv: -kv[1][1])[:12]},
       "kernels": {k: {"n": v[0], "ms": round(v[1] / 1e3, 3)}
                   for k, v in sorted(per.items(), key=lambda kv: -kv[1][1])}}
json.dump(out, sys.stdout, indent=1)
