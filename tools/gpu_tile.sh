#!/bin/bash
# Tile-kernel round: smoke, GPU suite, then stepwise timings on configs 2-4
# (f32 tile kernels vs DUFWI_TILE=0: the f64 lean kernels).
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1
echo "smoke exit $?" >> gpurun_out/smoke.log
if [ -z "$NO_TESTS" ]; then
timeout 2400 python -m pytest tests -m gpu -q -rf -x ${PYTEST_ARGS} > gpurun_out/pytest_gpu.log 2>&1
echo "pytest exit $?" >> gpurun_out/pytest_gpu.log
fi
O=gpurun_out/tile_times.log
: > $O
for c in "3 --units 128 --nt 300" "2 --units 128 --nt 300" "4 --units 256 --nt 200"; do
  timeout 300 python tools/time_config.py --config $c --reps 2 2>&1 | tail -1 | cut -c1-400 | sed "s/^/TILE $c: /" >> $O
  [ -z "$NO_BASE" ] && DUFWI_TILE=0 timeout 300 python tools/time_config.py --config $c --reps 2 2>&1 | tail -1 | cut -c1-400 | sed "s/^/LEAN $c: /" >> $O
done
cat $O
