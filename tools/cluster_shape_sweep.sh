#!/bin/bash
# Config-0 cluster sweeps (8 units, strips) at forced cluster shapes
# (DUFWI_CLUSTER_CS / DUFWI_CLUSTER_RPT), against the cost model's choice.
echo "auto: $(timeout 120 python tools/time_config.py --config 0 --units 8 --engine cluster --store strips --reps 3 2>&1 | tail -1 | python -c 'import sys,json; d=json.loads(sys.stdin.read()); print(round(d["forward_ms"],4), round(d["adjoint_ms"],4), d["info"])' 2>&1 | cut -c1-300)"
for cs in 8 10 12 14 16; do
  for rpt in 2 4 5 6 7 8; do
    r=$(DUFWI_CLUSTER_CS=$cs DUFWI_CLUSTER_RPT=$rpt timeout 120 python tools/time_config.py --config 0 --units 8 --engine cluster --store strips --reps 3 2>&1 | tail -1 | python -c 'import sys,json; d=json.loads(sys.stdin.read()); print(round(d["forward_ms"],4), round(d["adjoint_ms"],4), d["engine"])' 2>/dev/null)
    [ -n "$r" ] && echo "cs=$cs rpt=$rpt: $r"
  done
done
