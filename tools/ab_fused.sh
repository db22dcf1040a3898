#!/bin/bash
# Fused adjoint (adjimg_lean_kernel) vs the split lam/imaging kernels: bit-identity
# against the baseline build (tools/ubench/libdufwi_base.so) and timings.
mkdir -p gpurun_out
BASE=$PWD/tools/ubench/libdufwi_base.so
O=gpurun_out/ab_fused.log
: > $O
for c in "4 8 40 strips" "4 8 40 full" "0 8 120 strips" "0 8 120 full" "3 4 60 strips norho" "2 4 60 full"; do
  set -- $c
  DUFWI_LIB=$BASE timeout 300 python tools/bitcmp.py $1 $2 $3 /tmp/b.txt $4 $5 > /dev/null 2>&1
  DUFWI_FUSED_ADJ=1 timeout 300 python tools/bitcmp.py $1 $2 $3 /tmp/n.txt $4 $5 > /tmp/n.err 2>&1
  if cmp -s /tmp/b.txt /tmp/n.txt; then echo "BITCMP $c: identical" >> $O; else echo "BITCMP $c: DIFFER" >> $O; cat /tmp/b.txt /tmp/n.txt /tmp/n.err | tail -12 >> $O; fi
done
for rep in 1 2; do
for c in "4 --units 256 --nt 200" "3 --units 128 --nt 300 --no-rho"; do
  DUFWI_LIB=$BASE timeout 300 python tools/time_config.py --config $c --reps 2 2>&1 | tail -1 | cut -c1-300 | sed "s/^/BASE   $c: /" >> $O
  DUFWI_FUSED_ADJ=1 timeout 300 python tools/time_config.py --config $c --reps 2 2>&1 | tail -1 | cut -c1-300 | sed "s/^/FUSED3 $c: /" >> $O
  DUFWI_FUSED_ADJ=1 DUFWI_FUSED_MINB=2 timeout 300 python tools/time_config.py --config $c --reps 2 2>&1 | tail -1 | cut -c1-300 | sed "s/^/FUSED2 $c: /" >> $O
done
done
