"""Markdown tables from the round-2 ncu CSV captures in this directory.

    python profiles/r02/summarize.py > profiles/r02/ncu_tables.md
"""
import csv
import os

HERE = os.path.dirname(os.path.abspath(__file__))


def launches(name):
    rows = list(csv.reader(open(os.path.join(HERE, name))))
    st = next(i for i, r in enumerate(rows) if r and r[0] == "ID")
    h = rows[st]
    ki, mi, vi, ii = h.index("Kernel Name"), h.index("Metric Name"), h.index("Metric Value"), h.index("ID")
    out = {}
    for r in rows[st + 1:]:
        if len(r) <= vi:
            continue
        d = out.setdefault(r[ii], {"kernel": r[ki].split("(")[0].replace("void ", "")})
        try:
            d[r[mi]] = float(r[vi].replace(",", ""))
        except ValueError:
            d[r[mi]] = r[vi]
    return [d for d in out.values() if "k_" in d["kernel"]]


print("# Round-2 ncu tables (B200, --clock-control none; per-launch times are cold and serialised)\n")
print("## Config 2 step (bench.py --steps 1): launch list and DRAM traffic (traffic_r02.csv)\n")
print("| kernel | us | DRAM read MB | DRAM write MB |\n|---|---|---|---|")
L = launches("traffic_r02.csv")
for d in L[-4:]:
    print(f"| {d['kernel']} | {d['gpu__time_duration.sum'] / 1e3:.1f} | {d['dram__bytes_read.sum'] / 1e6:.0f} | "
          f"{d['dram__bytes_write.sum'] / 1e6:.0f} |")
print("\n## Config 3, p = 3221225473, n = 2^24 (tools/prof_c3.py): one forward + one inverse (c3_launches.csv)\n")
print("(Captured before the F32 wide rounds; the current kernels at 2^24, 2^25 - 1 and 2^25 + 1 are in ncu_c3.md.)\n")
print("| kernel | us | grid | regs | DRAM read MB | DRAM write MB | SM throughput % |\n|---|---|---|---|---|---|---|")
for d in launches("c3_launches.csv")[:6]:
    print(f"| {d['kernel']} | {d['gpu__time_duration.sum'] / 1e3:.1f} | {d['launch__grid_size']:.0f} | "
          f"{d['launch__registers_per_thread']:.0f} | {d['dram__bytes_read.sum'] / 1e6:.0f} | "
          f"{d['dram__bytes_write.sum'] / 1e6:.0f} | {d['sm__throughput.avg.pct_of_peak_sustained_elapsed']:.1f} |")
print("\n## Pipe utilisation by size class (tools/prof_tiles.py: n = 2^T - 3, ~2^24 words, fwd then inv; pipes_r02.csv)\n")
cols = [("gpu__time_duration.sum", "us", 1e3), ("smsp__issue_active.avg.pct_of_peak_sustained_active", "issue %", 1),
        ("sm__pipe_fma_cycles_active.avg.pct_of_peak_sustained_active", "FMA pipe %", 1),
        ("sm__pipe_alu_cycles_active.avg.pct_of_peak_sustained_active", "ALU pipe %", 1),
        ("sm__inst_executed_pipe_lsu.avg.pct_of_peak_sustained_active", "LSU %", 1),
        ("sm__warps_active.avg.pct_of_peak_sustained_active", "occupancy %", 1),
        ("dram__throughput.avg.pct_of_peak_sustained_elapsed", "DRAM %", 1)]
print("| T | kernel | " + " | ".join(c[1] for c in cols) + " |")
print("|---|---|" + "---|" * len(cols))
Ts = [t for t in range(10, 18) for _ in (0, 1)]
for t, d in zip(Ts, launches("pipes_r02.csv")):
    print(f"| {t} | {d['kernel']} | " + " | ".join(f"{d[c[0]] / c[2]:.1f}" for c in cols) + " |")
