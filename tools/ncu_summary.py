"""Summaries of the committed ncu evidence (profiles/).

  ncu_summary.py launches LAUNCH_CSV           per-kernel launch counts / mean times
  ncu_summary.py full REPORT.ncu-rep           key --set full metrics per kernel
  ncu_summary.py traffic REPORT.ncu-rep        {"k_<name>": dram bytes per launch}
"""
import csv
import io
import json
import re
import subprocess
import sys
from collections import OrderedDict, defaultdict

KEYS = [
    "gpu__time_duration.sum",
    "dram__bytes_read.sum",
    "dram__bytes_write.sum",
    "sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active",
    "sm__inst_executed_pipe_fp64.avg.pct_of_peak_sustained_active",
    "smsp__sass_thread_inst_executed_op_dfma_pred_on.sum",
    "sm__warps_active.avg.pct_of_peak_sustained_active",
    "smsp__issue_active.avg.pct_of_peak_sustained_active",
    "launch__registers_per_thread",
    "launch__occupancy_limit_registers",
    "launch__occupancy_limit_shared_mem",
    "launch__grid_size",
    "dram__throughput.avg.pct_of_peak_sustained_elapsed",
    "smsp__average_warps_issue_stalled_long_scoreboard_per_issue_active.ratio",
    "smsp__average_warps_issue_stalled_short_scoreboard_per_issue_active.ratio",
    "smsp__average_warps_issue_stalled_wait_per_issue_active.ratio",
    "smsp__average_warps_issue_stalled_mio_throttle_per_issue_active.ratio",
    "smsp__inst_executed.sum",
]


def short(name):
    m = re.search(r"(k_\w+)<", name) or re.search(r"(k_\w+)\(", name)
    return m.group(1) if m else name[:60]


def launches(path):
    rows = [r for r in csv.reader(open(path)) if len(r) > 10 and r[0] != "ID"]
    agg = defaultdict(list)
    for r in rows:
        if r[12] == "gpu__time_duration.sum":
            agg[r[4]].append(float(r[14]) * (1e-3 if r[13] == "ns" else 1.0))
    tot = sum(sum(v) for k, v in agg.items() if "tdg::" in k and "probe" not in k)
    for k, v in sorted(agg.items(), key=lambda kv: -sum(kv[1])):
        share = f"{sum(v) / tot * 100:5.1f}%" if "tdg::" in k and "probe" not in k else "   -  "
        print(f"{short(k):24s} launches {len(v):4d}  mean {sum(v) / len(v):9.1f} us  "
              f"share of tdg kernel time {share}   {k[:70]}")


def raw(rep):
    out = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True,
                         text=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    hdr, units = rows[0], rows[1]
    return [(dict(zip(hdr, r)), dict(zip(hdr, units))) for r in rows[2:]]


def full(rep):
    for d, u in raw(rep):
        print(f"-- {d['Kernel Name'][:100]}")
        for k in KEYS:
            if k in d:
                print(f"   {k:80s} {d[k]:>16s} {u.get(k, '')}")


def traffic(rep):
    res = OrderedDict()
    for d, u in raw(rep):
        scale = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}
        b = float(d["dram__bytes_read.sum"]) * scale[u["dram__bytes_read.sum"]] + \
            float(d["dram__bytes_write.sum"]) * scale[u["dram__bytes_write.sum"]]
        name = short(d["Kernel Name"]).replace("_fast", "").replace("_mma", "")
        res.setdefault(name, b)
    print(json.dumps(res, indent=1))


if __name__ == "__main__":
    {"launches": launches, "full": full, "traffic": traffic}[sys.argv[1]](sys.argv[2])
