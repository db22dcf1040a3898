#!/bin/bash
# One GPU session: build check, smoke, the -m gpu suite, a default bench line.
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build(); g.smoke()" > gpurun_out/smoke.log 2>&1
echo "smoke exit $?" >> gpurun_out/smoke.log
timeout 2400 python -m pytest tests -m gpu -q -rf -s --durations=25 ${PYTEST_ARGS} > gpurun_out/pytest_gpu.log 2>&1
echo "pytest exit $?" >> gpurun_out/pytest_gpu.log
grep "rel L2" gpurun_out/pytest_gpu.log > gpurun_out/parity_errors.log
if [ -z "$NO_BENCH" ]; then
  timeout 900 python bench.py ${BENCH_ARGS} > gpurun_out/bench.json 2> gpurun_out/bench.err
  echo "bench exit $?" >> gpurun_out/bench.err
fi
