"""Per-source-line hot spots from an ncu report (needs -lineinfo + --import-source).

    python tools/ncu_lines.py report.ncu-rep <kernel-regex> [launch-skip] [top]
"""
import csv
import io
import subprocess
import sys

rep, kern = sys.argv[1], sys.argv[2]
skip = sys.argv[3] if len(sys.argv) > 3 else "0"
top = int(sys.argv[4]) if len(sys.argv) > 4 else 30
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "cuda,sass",
                      "-k", f"regex:{kern}", "--launch-skip", skip, "--launch-count", "1"],
                     capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(out)))
fname = None
agg = {}
hdr = None
for r in rows:
    if not r:
        continue
    if r[0] == "File Path":
        fname = r[1].split("/")[-1]
        continue
    if r[0] == "Line No":
        hdr = r
        ie = hdr.index("Instructions Executed")
        isamp = hdr.index("Warp Stall Sampling (All Samples)")
        continue
    if hdr is None or r[0] == "" or r[0] == "Function Name":
        continue
    try:
        e = float(r[ie] or 0)
        s = float(r[isamp] or 0)
    except (ValueError, IndexError):
        continue
    key = (fname, int(r[0]), r[1].strip()[:90])
    a = agg.setdefault(key, [0.0, 0.0])
    a[0] += e
    a[1] += s
te = sum(v[0] for v in agg.values()) or 1
ts = sum(v[1] for v in agg.values()) or 1
print(f"total warp-instructions {te:.0f}, stall samples {ts:.0f}")
for k, v in sorted(agg.items(), key=lambda kv: -kv[1][1])[:top]:
    print(f"{v[0] / te:6.1%} inst {v[1] / ts:6.1%} stall  {k[0]}:{k[1]}  {k[2]}")
