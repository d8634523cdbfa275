#!/bin/bash
# usage: tools/sweep_e2e.sh VAR "v1 v2 ..."  -- e2e Gcoeff/s of bench.py (config 2) per value ("-" = unset)
var=$1; vals=$2; shift 2
for v in $vals; do
  if [ "$v" = "-" ]; then unset $var; else export $var=$v; fi
  r=$(timeout 300 python bench.py --no-cpu --steps 3 --warmup 3 "$@" 2>&1 | tail -1)
  echo "$var=$v $(python -c 'import json,sys; d=json.loads(sys.argv[1]); e=d["e2e"]; print("e2e %.2f Gcoeff/s %.1f ms exact %s"%(e["value"],e["ms_per_step"],e["roundtrip_exact"]))' "$r" 2>&1 | tail -1)"
done
