#!/bin/bash
# Quick A/B of the in-tree build against tools/ubench/libdufwi_base.so on the
# density configs and config 4 (time_config.py, CUDA events); gpurun_out/ab_quick.log.
mkdir -p gpurun_out
BASE=$PWD/tools/ubench/libdufwi_base.so
O=gpurun_out/ab_quick.log
: > $O
for rep in 1 2; do
for c in "3 --units 128 --nt 300" "2 --units 128 --nt 300" "4 --units 256 --nt 200"; do
  DUFWI_LIB=$BASE timeout 300 python tools/time_config.py --config $c --reps 2 2>&1 | tail -1 | cut -c1-330 | sed "s/^/BASE $c: /" >> $O
  timeout 300 python tools/time_config.py --config $c --reps 2 2>&1 | tail -1 | cut -c1-330 | sed "s/^/NEW  $c: /" >> $O
done
done
