#!/bin/bash
# per-kernel launch times of the lean kernels (ncu, serialized): old vs new build
mkdir -p gpurun_out
for L in tools/ubench/lib_OLD.so paper_2603_04070_b200/libdufwi.so; do
  n=$(basename $L .so)
  for c in 3 4; do
    DUFWI_LIB=$PWD/$L ncu --metrics gpu__time_duration.sum --clock-control none -k regex:lean -s 6 -c 9 --csv \
      python tools/time_config.py --config $c --units 128 --nt 12 --reps 1 2>/dev/null | grep lean_kernel > gpurun_out/kt_${n}_$c.csv
  done
done
