#!/bin/bash
# ncu source-level capture of the cluster sweeps (forward MODE 2 = second forward launch, adjoint)
set -e
CS=${1:-16}
TAG=${2:-cs$CS}
mkdir -p gpurun_out
DUFWI_CLUSTER_CS=$CS python tools/prof_case.py --config 0 > gpurun_out/${TAG}_plain.log 2>&1
DUFWI_CLUSTER_CS=$CS ncu --set full --clock-control none --import-source on -k regex:cluster_fwd -s 1 -c 1 \
    -o gpurun_out/${TAG}_fwd python tools/prof_case.py --config 0 > gpurun_out/${TAG}_ncu.log 2>&1
DUFWI_CLUSTER_CS=$CS ncu --set full --clock-control none --import-source on -k regex:cluster_adj -c 1 \
    -o gpurun_out/${TAG}_adj python tools/prof_case.py --config 0 >> gpurun_out/${TAG}_ncu.log 2>&1
echo done
