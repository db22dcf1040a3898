python tools/prof_case.py --config 0 > /dev/null 2>&1
ncu --set full --clock-control none --import-source on -k regex:cluster_adj -c 1 -o gpurun_out/cur_adj python tools/prof_case.py --config 0 > /dev/null 2>&1
