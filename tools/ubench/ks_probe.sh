#!/bin/bash
mkdir -p gpurun_out
L=tools/ubench/lib_T640.so
for cfg in "10 4" "8 5" "10 5" "16 5" "12 4"; do
  set -- $cfg
  echo "cs=$1 rpt=$2 $(DUFWI_CLUSTER_CS=$1 DUFWI_CLUSTER_RPT=$2 DUFWI_LIB=$PWD/$L timeout 120 python tools/sweep_ms.py 2>&1 | tail -1 | cut -c1-250)"
done
