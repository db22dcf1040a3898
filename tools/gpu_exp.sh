#!/bin/bash
# Imaging kernel: shot-group size (CTAs per SM target) on the stepwise configs.
mkdir -p gpurun_out
O=gpurun_out/exp.log
: > $O
for ps in 4 8 16 24 40; do
for c in "3 --units 128 --nt 300" "2 --units 256 --nt 300" "4 --units 256 --nt 200"; do
  DUFWI_IMG_CTAS_PER_SM=$ps timeout 300 python tools/time_config.py --config $c --reps 2 2>&1 | tail -1 | python -c '
import sys,json
d=json.loads(sys.stdin.read())
print("cfg %d units %3d adj %8.3f ms %.3e upd/s" % (d["config"], d["units"], d["adjoint_ms"], d["adj_updates_per_s"]))' | sed "s/^/per_sm $ps: /" >> $O
done
done
cat $O
