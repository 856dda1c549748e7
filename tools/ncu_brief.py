"""Brief of one-kernel ncu --set full reports: key metrics, stall ratios,
and stall samples / executed instructions by SASS opcode.
usage: python tools/ncu_brief.py REPORT.ncu-rep [...]"""
import csv
import io
import subprocess
import sys
from collections import Counter

WANT = ["gpu__time_duration.sum", "l1tex__t_sector_hit_rate.pct", "lts__t_sector_hit_rate.pct",
        "sm__pipe_tensor_subpipe_dmma_cycles_active.avg.pct_of_peak_sustained_active",
        "sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active",
        "smsp__issue_active.avg.pct_of_peak_sustained_active",
        "sm__warps_active.avg.pct_of_peak_sustained_active",
        "l1tex__throughput.avg.pct_of_peak_sustained_active",
        "l1tex__data_pipe_lsu_wavefronts_mem_shared.sum",
        "dram__bytes_read.sum", "dram__bytes_write.sum", "smsp__inst_executed.sum",
        "launch__registers_per_thread", "launch__occupancy_limit_shared_mem",
        "launch__occupancy_limit_registers"]


def ncu(rep, *args):
    return subprocess.run(["ncu", "-i", rep, *args], capture_output=True, text=True).stdout


for rep in sys.argv[1:]:
    print("==", rep)
    rows = list(csv.reader(io.StringIO(ncu(rep, "--page", "raw", "--csv"))))
    h, v = rows[0], rows[2]
    print("  kernel", v[h.index("Kernel Name")][:90])
    for i, n in enumerate(h):
        if n in WANT:
            print(f"  {n} {v[i]}")
        elif n.startswith("smsp__average_warps_issue_stalled") and n.endswith("per_issue_active.ratio"):
            try:
                if float(v[i]) > 0.1:
                    print(f"  {n[34:-23]} {v[i]}")
            except ValueError:
                pass
    rows = list(csv.reader(io.StringIO(ncu(rep, "--page", "source", "--csv", "--print-source", "sass"))))
    hdr, data = None, []
    for r in rows:
        if r and r[0] == "Address":
            hdr = r
        elif hdr and r and r[0].startswith("0x"):
            data.append(dict(zip(hdr, r)))
    tot = sum(int(d["Warp Stall Sampling (All Samples)"] or 0) for d in data) or 1
    st, ins = Counter(), Counter()
    for d in data:
        s = d["Source"].split()
        o = (s[1] if s and s[0].startswith("@") else (s[0] if s else "")).split(".")[0]
        st[o] += int(d["Warp Stall Sampling (All Samples)"] or 0)
        ins[o] += int(d["Instructions Executed"] or 0)
    print("  opcode: stall share, executed warp instructions")
    for o, c in st.most_common(12):
        print(f"    {o:8s} {100 * c / tot:5.1f}%  {ins[o]}")
