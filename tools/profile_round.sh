#!/bin/bash
# Evidence for profiles/: run on a B200 via gpurun.
#   1) plain bench (must exit 0) then the ncu launch list of the same command
#   2) each top kernel once under `ncu --set full`, after its plain run exits 0
set -e
R=${1:-r01}
mkdir -p gpurun_out
python bench.py --steps 2 --warmup 1 --skip-cpu --skip-e2e --skip-large > gpurun_out/${R}_bench_plain.json 2> gpurun_out/${R}_bench_plain.err
ncu --metrics gpu__time_duration.sum --clock-control none --csv \
    --log-file gpurun_out/${R}_launches.csv \
    python bench.py --steps 2 --warmup 1 --skip-cpu --skip-e2e --skip-large > gpurun_out/${R}_ncu_bench.log 2>&1
# cluster engine (configs 0/1 share the sweep shape): adjoint, and the trial forward (2nd forward)
python tools/prof_case.py --config 0 > gpurun_out/${R}_case_plain.log 2>&1
ncu --set full --clock-control none --import-source on -k regex:cluster_adj -c 1 \
    -o gpurun_out/${R}_cluster_adj python tools/prof_case.py --config 0 > gpurun_out/${R}_ncu_full.log 2>&1
ncu --set full --clock-control none --import-source on -k regex:cluster_fwd -s 1 -c 1 \
    -o gpurun_out/${R}_cluster_fwd python tools/prof_case.py --config 0 >> gpurun_out/${R}_ncu_full.log 2>&1
# stepwise engine (f32 tile kernels) on config 4 (64 units, short nt) and on config 3
# (variable density): one launch of each step kernel
for cfg in 4 3; do
  python tools/time_config.py --config $cfg --units 64 --nt 12 --reps 1 > gpurun_out/${R}_step_plain_c$cfg.log 2>&1
  for k in tile_fwd_kernel tile_adj_kernel tile_img_kernel; do
    ncu --set full --clock-control none --import-source on -k regex:$k -s 4 -c 1 \
        -o gpurun_out/${R}_step_c${cfg}_$k python tools/time_config.py --config $cfg --units 64 --nt 12 --reps 1 >> gpurun_out/${R}_ncu_full.log 2>&1
  done
done

# summarise on the box (ncu -i) and keep the report sizes under gpurun's copy-back cap
python tools/summarize_profiles.py ${R} > gpurun_out/${R}_summary.log 2>&1
mkdir -p gpurun_out/profiles_${R}
cp profiles/${R}_* profiles/ncu_traffic.json gpurun_out/profiles_${R}/ 2>/dev/null || true
find gpurun_out -name "${R}_*.ncu-rep" ! -name "${R}_cluster_adj.ncu-rep" -delete
echo done
