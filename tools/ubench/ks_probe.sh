#!/bin/bash
mkdir -p gpurun_out
for L in paper_2603_04070_b200/libdufwi.so tools/ubench/lib_RB2.so tools/ubench/lib_RB4.so; do
  for c in 2 3; do
    echo "$L $c $(DUFWI_LIB=$PWD/$L timeout 200 python tools/time_config.py --config $c --units 128 --nt 200 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('%.3g %.3g' % (d['fwd_updates_per_s'], d['adj_updates_per_s']))")"
  done
done
