#!/bin/bash
# Evidence for profiles/: run on a B200 via gpurun.
#   1) plain bench (must exit 0) then the ncu launch list of the same command
#   2) the top kernel once under `ncu --set full`, after its plain run exits 0
set -e
R=${1:-r01}
mkdir -p gpurun_out
python bench.py --steps 2 --warmup 1 --skip-cpu --skip-e2e > gpurun_out/${R}_bench_plain.json 2> gpurun_out/${R}_bench_plain.err
ncu --metrics gpu__time_duration.sum --clock-control none --csv \
    --log-file gpurun_out/${R}_launches.csv \
    python bench.py --steps 2 --warmup 1 --skip-cpu --skip-e2e > gpurun_out/${R}_ncu_bench.log 2>&1
python tools/prof_case.py --config 0 > gpurun_out/${R}_case_plain.log 2>&1
ncu --set full --clock-control none --import-source on -k regex:cluster_adj -c 1 \
    -o gpurun_out/${R}_cluster_adj python tools/prof_case.py --config 0 > gpurun_out/${R}_ncu_full.log 2>&1
ncu --set full --clock-control none --import-source on -k regex:cluster_fwd -c 1 \
    -o gpurun_out/${R}_cluster_fwd python tools/prof_case.py --config 0 >> gpurun_out/${R}_ncu_full.log 2>&1
python tools/time_config.py --config 4 --units 64 --nt 12 --reps 1 > gpurun_out/${R}_step_plain.log 2>&1
ncu --set full --clock-control none --import-source on -k regex:stream_kernel -s 4 -c 2 \
    -o gpurun_out/${R}_stepwise python tools/time_config.py --config 4 --units 64 --nt 12 --reps 1 >> gpurun_out/${R}_ncu_full.log 2>&1
echo done
