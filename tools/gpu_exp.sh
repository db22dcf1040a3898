#!/bin/bash
# Fused adjoint A/B: one-pass tile kernel (1 / 2 stages) against the split lam + imaging kernels.
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_fallbacks.py tests/test_gpu_large.py -m gpu -q -x -s > gpurun_out/pytest_fused.log 2>&1
echo "pytest exit $?" >> gpurun_out/pytest_fused.log
O=gpurun_out/exp.log
: > $O
for c in "3 --units 128 --nt 300" "2 --units 128 --nt 300" "4 --units 256 --nt 200"; do
  timeout 300 python tools/time_config.py --config $c --reps 2 2>&1 | tail -1 | cut -c1-260 | sed "s/^/FUSED1 $c: /" >> $O
  DUFWI_LIB=$PWD/tools/ubench/lib_FUSED2.so timeout 300 python tools/time_config.py --config $c --reps 2 2>&1 | tail -1 | cut -c1-260 | sed "s/^/FUSED2 $c: /" >> $O
  DUFWI_FUSED=0 timeout 300 python tools/time_config.py --config $c --reps 2 2>&1 | tail -1 | cut -c1-260 | sed "s/^/SPLIT  $c: /" >> $O
done
grep "passed\|failed\|rel L2\|Error" gpurun_out/pytest_fused.log | tail -12
cat $O
