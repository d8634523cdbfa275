"""profiles/traffic.json from an ncu launch capture of the config-2 bench.

    ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum \
        --clock-control none --csv --log-file traffic.csv \
        python bench.py --steps 1 --warmup 3 --no-cpu --no-e2e
    python tools/traffic.py traffic.csv > profiles/traffic.json

The last six tftb200 launches are the timed step (two forward size-class
launches, then per size class the split inverse's k_cli_chunks and
k_cli_cols); ncu serialises and cold-starts them, so the bytes are the
evidence here, not the times.
"""
import csv
import json
import sys
from collections import OrderedDict

rows = list(csv.reader(open(sys.argv[1])))
start = next(i for i, r in enumerate(rows) if r and r[0] == "ID")
h = rows[start]
ki, mi, vi, ii = h.index("Kernel Name"), h.index("Metric Name"), h.index("Metric Value"), h.index("ID")
launches = OrderedDict()
for r in rows[start + 1:]:
    if len(r) <= vi:
        continue
    d = launches.setdefault(r[ii], {"kernel": r[ki].split("(")[0]})
    d[r[mi]] = float(r[vi].replace(",", ""))
allk = [d for d in launches.values()
        if d["kernel"].split("<")[0].split()[-1] in ("k_clg_fwd", "k_cli_chunks", "k_cli_cols")]
# the timed step: the last two forward launches (both size classes) and the
# inverse launches after them (fused: one k_cli_chunks per class; split:
# k_cli_chunks + k_cli_cols per class)
last_f = max(i for i, d in enumerate(allk) if "k_clg_fwd" in d["kernel"])
ours = allk[last_f - 1:]
out = {"source": "ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum "
                 "--clock-control none (cold, serialised) on bench.py --steps 1 --warmup 3; the last forward "
                 "pair and the inverse launches after it = the timed step",
       "launches": [{"kernel": d["kernel"], "ns": d["gpu__time_duration.sum"],
                     "dram_read": d["dram__bytes_read.sum"], "dram_write": d["dram__bytes_write.sum"]}
                    for d in ours]}
tot = lambda ds: sum(d["dram__bytes_read.sum"] + d["dram__bytes_write.sum"] for d in ds)
inv = [d for d in ours if "k_cli_" in d["kernel"]]
out["forward_bytes"] = tot([d for d in ours if "k_clg_fwd" in d["kernel"]])
out["config2_bytes_per_step"] = tot(ours)
out["config2_read_bytes"] = sum(d["dram__bytes_read.sum"] for d in ours)
out["config2_write_bytes"] = sum(d["dram__bytes_write.sum"] for d in ours)
out["inverse_pass_bytes"] = tot(inv)
out["inverse_pass_kernel"] = "k_cli_chunks (fused: last chunk CTA solves the columns)" if not any("k_cli_cols" in d["kernel"] for d in ours) else "k_cli_chunks + k_cli_cols"
out["config2_ncu_step_ns"] = sum(d["gpu__time_duration.sum"] for d in ours)
print(json.dumps(out, indent=1))
