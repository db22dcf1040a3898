#!/bin/bash
# cluster engine quick A/B: config-0 sweeps (auto shape) + per-warp phase timing + parity smoke
mkdir -p gpurun_out
out=gpurun_out/cl_ab.log
: > $out
for r in 1 2; do
  timeout 120 python tools/time_config.py --config 0 --units 8 --engine cluster --store strips --reps 5 2>&1 | tail -1 | cut -c1-300 >> $out
done
timeout 300 python tools/ubench/phase_dbg.py > gpurun_out/phase_dbg.log 2>&1
timeout 600 python -m pytest tests/test_gpu_parity.py tests/test_gpu_dufwi.py -q -x > gpurun_out/pytest_cl.log 2>&1
tail -2 gpurun_out/pytest_cl.log >> $out
