#!/bin/bash
# constant- vs variable-density lean kernels on the config 2/3/4 grids (128 units, 200 steps)
mkdir -p gpurun_out
for c in 2 3 4; do
  for f in "" "--no-rho"; do
    timeout 200 python tools/time_config.py --config $c --units 128 --nt 200 $f | python -c "import json,sys; d=json.loads(sys.stdin.read()); print($c, '$f', '%.3g %.3g' % (d['fwd_updates_per_s'], d['adj_updates_per_s']))"
  done
done
