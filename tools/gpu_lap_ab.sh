#!/bin/bash
# cluster engine: strips vs L(u)-history adjoint on config 0 (8 units), then parity
mkdir -p gpurun_out
out=gpurun_out/lap_ab.log
: > $out
for st in strips lap strips lap; do
  timeout 120 python tools/time_config.py --config 0 --units 8 --engine cluster --store $st --reps 5 2>&1 | tail -1 | cut -c1-200 >> $out
done
timeout 600 python -m pytest tests/test_gpu_parity.py tests/test_gpu_dufwi.py -q -x > gpurun_out/pytest_lap.log 2>&1
tail -2 gpurun_out/pytest_lap.log >> $out
timeout 300 python bench.py --steps 10 --warmup 3 --skip-large --skip-cpu > gpurun_out/bench_lap.json 2> gpurun_out/bench_lap.err
