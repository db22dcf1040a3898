#!/bin/bash
# A/B of two library builds on the density configs: bitwise outputs + sweep rates
mkdir -p gpurun_out
for L in tools/ubench/lib_OLD.so paper_2603_04070_b200/libdufwi.so; do
  n=$(basename $L .so)
  for c in 2 3; do
    DUFWI_LIB=$PWD/$L timeout 200 python tools/bitcmp.py $c 32 300 gpurun_out/bc_${n}_$c.txt
    DUFWI_LIB=$PWD/$L timeout 200 python tools/time_config.py --config $c --units 128 --nt 200 > gpurun_out/tc_${n}_$c.json
  done
done
