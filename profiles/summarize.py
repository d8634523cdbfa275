"""Summarise ncu outputs into profiles/ (run here, on the CPU box).

    python profiles/summarize.py launches <launches.csv> > out.md
    python profiles/summarize.py full <report.ncu-rep> > out.md
"""

import csv
import io
import subprocess
import sys
from collections import OrderedDict

KEYS = ["Duration", "DRAM Throughput", "Memory Throughput", "Compute (SM) Throughput",
        "Executed Ipc Active", "Issue Slots Busy", "L2 Hit Rate", "L1/TEX Hit Rate",
        "Achieved Occupancy", "Theoretical Occupancy", "Registers Per Thread",
        "Dynamic Shared Memory Per Block", "Grid Size", "Block Size", "No Eligible"]
RAW = ["dram__bytes_read.sum", "dram__bytes_write.sum", "gpu__time_duration.sum",
       "sm__inst_executed_pipe_alu.avg.pct_of_peak_sustained_active",
       "sm__inst_executed_pipe_fma.avg.pct_of_peak_sustained_active",
       "sm__inst_executed_pipe_lsu.avg.pct_of_peak_sustained_active",
       "sm__pipe_alu_cycles_active.avg.pct_of_peak_sustained_active",
       "sm__pipe_fma_cycles_active.avg.pct_of_peak_sustained_active",
       "l1tex__data_bank_conflicts_pipe_lsu_mem_shared.sum",
       "smsp__inst_executed.sum"]


def launches(path):
    rows = list(csv.reader(open(path)))
    start = next(i for i, r in enumerate(rows) if r and r[0] == "ID")
    h = rows[start]
    ki, vi = h.index("Kernel Name"), h.index("Metric Value")
    mi = h.index("Metric Name")
    agg = OrderedDict()
    for r in rows[start + 1:]:
        if r[mi] != "gpu__time_duration.sum":
            continue
        name = r[ki].split("(")[0]
        agg.setdefault(name, []).append(float(r[vi].replace(",", "")))
    tot = sum(sum(v) for v in agg.values())
    print("| kernel | launches | mean us | share |")
    print("|---|---|---|---|")
    for k, v in agg.items():
        print(f"| {k} | {len(v)} | {sum(v) / len(v) / 1e3:.1f} | {sum(v) / tot:.1%} |")


def full(path):
    out = subprocess.run(["ncu", "-i", path, "--page", "details", "--csv"], capture_output=True,
                         text=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    h = rows[0]
    ki, mi, vi, ui, ii = (h.index("Kernel Name"), h.index("Metric Name"), h.index("Metric Value"),
                          h.index("Metric Unit"), h.index("ID"))
    per = OrderedDict()
    for r in rows[1:]:
        if r[mi] in KEYS:
            per.setdefault((r[ii], r[ki].split("(")[0]), OrderedDict())[r[mi]] = f"{r[vi]} {r[ui]}".strip()
    raw = subprocess.run(["ncu", "-i", path, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rr = list(csv.reader(io.StringIO(raw)))
    if rr:
        hh = rr[0]
        idx = {k: hh.index(k) for k in RAW if k in hh}
        units = rr[1]
        for r in rr[2:]:
            key = (r[hh.index("ID")], r[hh.index("Kernel Name")].split("(")[0])
            for k, i in idx.items():
                per.setdefault(key, OrderedDict())[k] = f"{r[i]} {units[i]}".strip()
    for (i, name), d in per.items():
        print(f"### launch {i}: {name}")
        for k, v in d.items():
            print(f"- {k}: {v}")
        print()


if __name__ == "__main__":
    {"launches": launches, "full": full}[sys.argv[1]](sys.argv[2])
