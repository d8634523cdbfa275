"""profiles/traffic.json from an ncu launch CSV of `bench.py --steps 1`.

    ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum \
        --clock-control none --csv --log-file launches.csv \
        python bench.py --steps 1 --warmup 3 --no-cpu --no-e2e
    python tools/traffic.py launches.csv > profiles/traffic.json

The timed step is the last `per_step` tftb launches (forward groups, then
inverse groups).  ncu serialises and cold-starts each launch, so only the
byte counts and the kernels' shares are meaningful, not the absolute times.
"""
import csv
import json
import sys
from collections import OrderedDict

rows = [r for r in csv.reader(open(sys.argv[1])) if r]
per_step = int(sys.argv[2]) if len(sys.argv) > 2 else 4
h = next(r for r in rows if r[0] == "ID")
ii, ki, mi, vi = h.index("ID"), h.index("Kernel Name"), h.index("Metric Name"), h.index("Metric Value")
launch = OrderedDict()
for r in rows[rows.index(h) + 1:]:
    if len(r) != len(h) or not r[ii].isdigit():
        continue
    d = launch.setdefault(int(r[ii]), {"kernel": r[ki].split("(")[0]})
    d[r[mi]] = float(r[vi].replace(",", ""))
ours = [d for d in launch.values() if d["kernel"].startswith("void k_")]
step = ours[-per_step:]
out = {
    "source": "ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum "
              "--clock-control none (cold, serialised) on bench.py --steps 1 --warmup 3; "
              f"last {per_step} tftb launches = the timed step",
    "launches": [{"kernel": d["kernel"], "ns": d.get("gpu__time_duration.sum"),
                  "dram_read": d.get("dram__bytes_read.sum"), "dram_write": d.get("dram__bytes_write.sum")}
                 for d in step],
}
rd = sum(d["dram_read"] for d in out["launches"])
wr = sum(d["dram_write"] for d in out["launches"])
out["config2_bytes_per_step"] = rd + wr
out["config2_read_bytes"] = rd
out["config2_write_bytes"] = wr
inv = [d for d in out["launches"] if "inv" in d["kernel"]]
out["inverse_pass_bytes"] = sum(d["dram_read"] + d["dram_write"] for d in inv)
out["inverse_pass_kernel"] = inv[0]["kernel"] if inv else None
out["config2_ncu_step_ns"] = sum(d["ns"] for d in out["launches"])
print(json.dumps(out, indent=1))
