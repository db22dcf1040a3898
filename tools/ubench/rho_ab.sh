#!/bin/bash
# A/B of two library builds: bitwise outputs (sha256) + sweep rates on configs 2/3/4
mkdir -p gpurun_out
for L in tools/ubench/lib_OLD.so paper_2603_04070_b200/libdufwi.so; do
  n=$(basename $L .so)
  for c in 2 3 4; do
    DUFWI_LIB=$PWD/$L timeout 200 python tools/bitcmp.py $c 33 300 gpurun_out/bc_${n}_$c.txt
    DUFWI_LIB=$PWD/$L timeout 200 python tools/time_config.py --config $c --units 128 --nt 200 > gpurun_out/tc_${n}_$c.json
  done
  DUFWI_LIB=$PWD/$L timeout 200 python tools/time_config.py --config 4 --units 256 --nt 200 > gpurun_out/tc_${n}_4b.json
done
