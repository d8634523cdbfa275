"""ncu --set full summaries (round 2) from the CSV exports in this directory.

    python profiles/r02/ncu/summarize_full.py > profiles/r02/ncu/ncu_full_r02.md
"""
import csv
import os

HERE = os.path.dirname(os.path.abspath(__file__))
KEEP = ["Duration", "DRAM Throughput", "Memory Throughput", "Compute (SM) Throughput", "Executed Ipc Active",
        "Issue Slots Busy", "Achieved Occupancy", "Theoretical Occupancy", "L2 Hit Rate", "L1/TEX Hit Rate",
        "Registers Per Thread", "Dynamic Shared Memory Per Block", "Grid Size", "No Eligible"]
STALLS = ["long_scoreboard", "barrier", "math_pipe_throttle", "wait", "short_scoreboard", "mio_throttle",
          "not_selected", "selected"]


def details(name):
    rows = list(csv.reader(open(os.path.join(HERE, name))))
    h = rows[0]
    ii, ki, mi, ui, vi = (h.index(c) for c in ("ID", "Kernel Name", "Metric Name", "Metric Unit", "Metric Value"))
    out = {}
    for r in rows[1:]:
        if len(r) <= vi:
            continue
        d = out.setdefault(r[ii], {"kernel": r[ki].split("(")[0].replace("void ", "")})
        if r[mi] in KEEP and r[mi] not in d:
            d[r[mi]] = f"{r[vi]} {r[ui]}".strip()
    return out


def stalls(name):
    rows = list(csv.reader(open(os.path.join(HERE, name))))
    h = rows[0]
    out = {}
    for r in rows[2:]:
        if len(r) < len(h):
            continue
        tot = float(r[h.index("smsp__pcsamp_sample_count")].replace(",", "") or 1)
        out[r[h.index("ID")]] = {s: float(r[h.index("smsp__pcsamp_warps_issue_stalled_" + s)].replace(",", "") or 0) / tot
                                 for s in STALLS}
    return out


for tag, title in (("c2", "config 2, 512 vectors (tools/prof_c2.py): forward cone and fused inverse"),
                   ("c3", "config 3, n = 2^24, p = 3221225473 (tools/prof_c3.py): two-pass kernels")):
    print(f"## {title}\n")
    D, S = details(f"{tag}_details_r02.csv"), stalls(f"{tag}_stalls_r02.csv")
    for i, d in D.items():
        print(f"### launch {i}: {d['kernel']}")
        for k in KEEP:
            if k in d:
                print(f"- {k}: {d[k]}")
        if i in S:
            print("- stall samples (share): " + ", ".join(f"{s} {v:.0%}" for s, v in sorted(S[i].items(), key=lambda kv: -kv[1])))
        print()
