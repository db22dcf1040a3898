#!/bin/bash
# Cluster A/B: edge-first pushes against the end-of-body pushes, per shape.
mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_gpu_parity.py tests/test_gpu_dufwi.py -m gpu -q -x > gpurun_out/pytest_cl.log 2>&1
echo "pytest exit $?" >> gpurun_out/pytest_cl.log
CSS="10" RPTS="4 8" bash tools/cluster_shape_sweep.sh > /dev/null 2>&1
mv gpurun_out/shape_sweep.log gpurun_out/shape_edge.log
DUFWI_LIB=$PWD/tools/ubench/lib_NOEDGE.so CSS="10" RPTS="4 8" bash tools/cluster_shape_sweep.sh > /dev/null 2>&1
mv gpurun_out/shape_sweep.log gpurun_out/shape_noedge.log
tail -3 gpurun_out/pytest_cl.log
echo EDGE; cat gpurun_out/shape_edge.log; echo NOEDGE; cat gpurun_out/shape_noedge.log
