#!/bin/bash
# usage: tools/sweep_env.sh VAR "v1 v2 ..." -- extra bench args
# prints fwd/inv ms of bench.py (config 2, no CPU / e2e legs) per value ("-" = unset)
var=$1; vals=$2; shift 2
for v in $vals; do
  if [ "$v" = "-" ]; then unset $var; else export $var=$v; fi
  r=$(timeout 300 python bench.py --no-cpu --no-e2e --steps 5 --warmup 3 "$@" 2>&1 | tail -1)
  echo "$var=$v $(python -c 'import json,sys; d=json.loads(sys.argv[1]); print("fwd %.3f ms inv %.3f ms value %.1f exact %s"%(d["fwd_ms"],d["inv_ms"],d["value"],d["parity"]["roundtrip_exact"]))' "$r" 2>&1 | tail -1)"
done
