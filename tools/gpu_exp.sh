#!/bin/bash
# Cluster engine: parity of the cluster tests, sweep times per store, per-warp phase timing.
mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_gpu_parity.py tests/test_gpu_dufwi.py -m gpu -q -x > gpurun_out/pytest_cl.log 2>&1
echo "pytest exit $?" >> gpurun_out/pytest_cl.log
CSS="10" RPTS="4 8" bash tools/cluster_shape_sweep.sh > /dev/null 2>&1
DUFWI_CLUSTER_CS=10 DUFWI_CLUSTER_RPT=4 timeout 300 python tools/ubench/phase_dbg.py > gpurun_out/phase_dbg.log 2>&1
tail -3 gpurun_out/pytest_cl.log
cat gpurun_out/shape_sweep.log
cut -c1-700 gpurun_out/phase_dbg.log
