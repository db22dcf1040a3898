#!/bin/bash
# ncu --set full on selected kernels of a time_config run; exports text summaries
# (details page, raw metrics, source/SASS hot spots) and drops the reports.
# usage: ncu_kernels.sh TAG CONFIG UNITS KERNEL_REGEX...
set -u
TAG=$1; CFG=$2; UN=$3; shift 3
mkdir -p gpurun_out
for K in "$@"; do
  R=gpurun_out/${TAG}_${K}
  ncu --set full --clock-control none --import-source on -k regex:$K -s 4 -c 1 -o $R \
      python tools/time_config.py --config $CFG --units $UN --nt 12 --reps 1 > $R.log 2>&1
  ncu -i $R.ncu-rep --page details --csv > $R.details.csv 2>/dev/null
  ncu -i $R.ncu-rep --page raw --csv > $R.raw.csv 2>/dev/null
  ncu -i $R.ncu-rep --page source --csv --print-source sass > $R.sass.csv 2>/dev/null
  rm -f $R.ncu-rep
done
