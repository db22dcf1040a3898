#!/bin/bash
# Full bench (incl. the full config-4 gradient), reference arm, profiles.
mkdir -p gpurun_out
timeout 1500 python bench.py > gpurun_out/bench_full.json 2> gpurun_out/bench_full.err
echo "bench exit $?" >> gpurun_out/bench_full.err
timeout 900 python bench.py --impl reference --steps 3 --warmup 1 > gpurun_out/ref.json 2> gpurun_out/ref.err
bash tools/profile_round.sh r02 > gpurun_out/profile_round.log 2>&1
timeout 1200 python tools/full_config.py --configs 2,3 > gpurun_out/full_c23.json 2> gpurun_out/full_c23.err
