#!/bin/bash
mkdir -p gpurun_out
for L in tools/ubench/lib_KS32.so tools/ubench/lib_KS64.so tools/ubench/lib_KS128.so; do
  echo "$L $(DUFWI_LIB=$PWD/$L timeout 120 python tools/sweep_ms.py 2>&1 | tail -1 | cut -c1-250)"
done
