"""ncu --set full summaries of config 3's kernels (round 2, after the F32 wide
rounds) from the CSV exports in this directory (tools/run/prof_r02c.sh):

    python profiles/r02/ncu_c3/summarize_c3.py > profiles/r02/ncu_c3.md
"""
import csv
import os

HERE = os.path.dirname(os.path.abspath(__file__))
KEEP = ["Duration", "DRAM Throughput", "Compute (SM) Throughput", "Executed Ipc Active", "Issue Slots Busy",
        "Achieved Occupancy", "L2 Hit Rate", "Registers Per Thread", "Grid Size"]
STALLS = ["long_scoreboard", "barrier", "math_pipe_throttle", "wait", "short_scoreboard", "mio_throttle",
          "not_selected", "selected"]
PEAK = 6541.8  # MEASURED_PEAKS.json hbm_gbs


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


def raw(name):
    rows = list(csv.reader(open(os.path.join(HERE, name))))
    h = rows[0]
    out = {}
    for r in rows[2:]:
        if len(r) < len(h):
            continue
        g = lambda k: float(r[h.index(k)].replace(",", "") or 0)
        tot = g("smsp__pcsamp_sample_count") or 1
        out[r[h.index("ID")]] = {
            "us": g("gpu__time_duration.sum"), "rd": g("dram__bytes_read.sum"), "wr": g("dram__bytes_write.sum"),
            "alu": g("sm__pipe_alu_cycles_active.avg.pct_of_peak_sustained_active"),
            "fma": g("sm__pipe_fma_cycles_active.avg.pct_of_peak_sustained_active"),
            "inst": g("smsp__inst_executed.sum"),
            "stalls": {s: g("smsp__pcsamp_warps_issue_stalled_" + s) / tot for s in STALLS}}
    return out


print("# Config 3 kernels under ncu --set full (round 2, F32 wide rounds; B200, --clock-control none)\n")
print("p = 3221225473, one forward + one inverse of a single vector (tools/prof_c3.py; the first pair of the\n"
      "script is captured, cold caches, launches serialised by ncu).  DRAM GB/s = (read + write) / duration;\n"
      f"frac = that over the measured copy peak {PEAK} GB/s.  The algorithmic bytes of a pass are 2 n 4.\n")
for n, title in ((16777216, "n = 2^24 (two passes, 1024 tiles each)"),
                 (33554431, "n = 2^25 - 1 (nearly full last chunk: k_col1_inv solves the one column past h)"),
                 (33554433, "n = 2^25 + 1 (p2r: fold + dot product, then the 2^25 transform)")):
    print(f"## {title}\n")
    D, R = details(f"c3w_details_{n}.csv"), raw(f"c3w_raw_{n}.csv")
    print("| # | kernel | us | grid | regs | DRAM rd MB | DRAM wr MB | DRAM GB/s | frac | algorithmic / moved | IPC | issue % | ALU % | FMA % | occupancy % | L2 hit % | top stalls |")
    print("|---|---|---|---|---|---|---|---|---|---|---|---|---|---|---|---|---|")
    for i, d in D.items():
        r = R.get(i)
        if not r:
            continue
        gbs = (r["rd"] + r["wr"]) * 1e6 / (r["us"] * 1e-6) / 1e9 if r["us"] else 0
        alg = 2 * n * 4 / 1e6
        big = int(d.get("Grid Size", "0").split()[0].replace(",", "")) > 100
        st = ", ".join(f"{s} {v:.0%}" for s, v in sorted(r["stalls"].items(), key=lambda kv: -kv[1])[:4])
        f = lambda k: d.get(k, "").split()[0] if d.get(k) else ""
        print(f"| {i} | {d['kernel']} | {r['us']:.1f} | {f('Grid Size')} | {f('Registers Per Thread')} | {r['rd']:.0f} | {r['wr']:.0f} | "
              f"{gbs:.0f} | {gbs / PEAK:.3f} | {(alg / (r['rd'] + r['wr'])) if big and r['rd'] + r['wr'] > 1 else float('nan'):.2f} | "
              f"{f('Executed Ipc Active')} | {f('Issue Slots Busy')} | {r['alu']:.1f} | {r['fma']:.1f} | {f('Achieved Occupancy')} | {f('L2 Hit Rate')} | {st} |")
    print()
