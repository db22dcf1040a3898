#!/bin/bash
# A/B of two builds on a B200 (gpurun): the baseline library at
# tools/ubench/libdufwi_base.so (git-ignored, shipped with the snapshot) against
# the in-tree build, on the stepwise configs; lines appended to gpurun_out/ab.log.
mkdir -p gpurun_out
BASE=$PWD/tools/ubench/libdufwi_base.so
for rep in 1 2; do
for c in "4 --units 256 --nt 200" "3 --units 128 --nt 300" "2 --units 128 --nt 300" "3 --units 128 --nt 300 --no-rho"; do
  DUFWI_LIB=$BASE python tools/time_config.py --config $c --reps 2 2>&1 | tail -1 | cut -c1-400 | sed "s/^/BASE $c: /" >> gpurun_out/ab.log
  python tools/time_config.py --config $c --reps 2 2>&1 | tail -1 | cut -c1-400 | sed "s/^/NEW  $c: /" >> gpurun_out/ab.log
done
done
