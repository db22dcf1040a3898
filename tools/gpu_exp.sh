#!/bin/bash
# Two-step forward: parity of the stepwise tests, then A/B against one step per launch.
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -3
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_fallbacks.py tests/test_gpu_large.py tests/test_gpu_api_extras.py -m gpu -q -x > gpurun_out/pytest_f2.log 2>&1
echo "pytest exit $?" >> gpurun_out/pytest_f2.log
grep "passed\|failed\|Error\|^E " gpurun_out/pytest_f2.log | head -12
O=gpurun_out/exp.log
: > $O
for c in "3 --units 128 --nt 300" "2 --units 256 --nt 300" "4 --units 256 --nt 200"; do
  timeout 300 python tools/time_config.py --config $c --reps 2 2>&1 | tail -1 | cut -c1-160 | sed "s/^/FWD2 $c: /" >> $O
  DUFWI_FWD2=0 timeout 300 python tools/time_config.py --config $c --reps 2 2>&1 | tail -1 | cut -c1-160 | sed "s/^/FWD1 $c: /" >> $O
done
cat $O
