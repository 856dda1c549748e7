"""Timeline of DiscreteOperator.ssprk3_steps_host on the C2 mesh (CUPTI via
torch.profiler): per-stream kernel / copy intervals, summarised per step.

usage: python tools/hs_trace.py [bands] [steps] > gpurun_out/hs_trace.json
"""
import json
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import bench  # noqa: E402
from paper_1403_1157_b200.operator import DiscreteOperator  # noqa: E402

bands = int(sys.argv[1]) if len(sys.argv) > 1 else 8
steps = int(sys.argv[2]) if len(sys.argv) > 2 else 4
dev = torch.device("cuda:0")
cfg, space, model, scheme, U0h, _ = bench.build_problem("c2", "cdg2", device=dev)
op = DiscreteOperator(space, model, scheme, device=dev, bands=bands)
dt = 1.4e-5
Uh = torch.from_numpy(U0h).pin_memory()
op.ssprk3_steps_host(Uh, 3, dt)
torch.cuda.synchronize()
with torch.profiler.profile(activities=[torch.profiler.ProfilerActivity.CUDA]) as prof:
    op.ssprk3_steps_host(Uh, steps, dt)
    torch.cuda.synchronize()
path = "/tmp/hs_trace.json"
prof.export_chrome_trace(path)
ev = json.load(open(path))["traceEvents"]
rows = []
for e in ev:
    if e.get("ph") != "X" or e.get("cat") not in ("kernel", "gpu_memcpy"):
        continue
    name = e["name"]
    short = ("H2D" if "HtoD" in name else "D2H" if "DtoH" in name else
             "faces" if "faces" in name else "vol" if "volume" in name else
             "fcadd" if "fc_add" in name else name[:30])
    rows.append((float(e["ts"]), float(e["dur"]), int(e["args"].get("stream", -1)), short))
rows.sort()
t0 = rows[0][0]
out = {"bands": bands, "steps": steps,
       "span_us": rows[-1][0] + rows[-1][1] - t0,
       "events": [(round(t - t0, 1), round(d, 1), s, n) for t, d, s, n in rows]}
json.dump(out, sys.stdout)
