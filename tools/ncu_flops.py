"""Executed FP64 work per kernel from an ncu --csv metrics dump (stdout of
the profiled command may precede the CSV): DFMA/DADD/DMUL thread
instructions and DMMA warp instructions -> executed flops, time, TF/s.
usage: python tools/ncu_flops.py FILE"""
import csv
import sys
from collections import OrderedDict

lines = open(sys.argv[1]).read().splitlines()
start = next(i for i, l in enumerate(lines) if l.startswith('"ID"'))
rows = list(csv.reader(lines[start:]))
hdr = rows[0]
k = OrderedDict()
for row in rows[1:]:
    if len(row) != len(hdr):
        continue
    d = dict(zip(hdr, row))
    key = (d["ID"], d["Kernel Name"].split("(")[0].replace("void ", "")[:44])
    k.setdefault(key, {})[d["Metric Name"]] = float(d["Metric Value"].replace(",", ""))
for (i, name), v in k.items():
    fma = v.get("sm__sass_thread_inst_executed_op_dfma_pred_on.sum", 0)
    add = v.get("sm__sass_thread_inst_executed_op_dadd_pred_on.sum", 0)
    mul = v.get("sm__sass_thread_inst_executed_op_dmul_pred_on.sum", 0)
    dmma = v.get("sm__inst_executed_pipe_tensor_subpipe_dmma.sum", 0)
    t = v.get("gpu__time_duration.sum", 0) * 1e-9
    flops = 2 * fma + add + mul + dmma * 512
    print(f"{name:44s} {t*1e6:9.1f} us  DFMA {fma:.3e} DADD {add:.3e} DMUL {mul:.3e} "
          f"DMMA {dmma:.3e}  executed {flops:.3e} flop  {flops / t / 1e12 if t else 0:6.2f} TFLOP/s")
