#!/bin/bash
# Config-0 cluster sweeps (8 units) at forced cluster shapes
# (DUFWI_CLUSTER_CS / DUFWI_CLUSTER_RPT), against the cost model's choice,
# for the strips store and the L(u)-history store; gpurun_out/shape_sweep.log.
mkdir -p gpurun_out
O=gpurun_out/shape_sweep.log
: > $O
run() {  # env prefix in $1, label in $2
  for store in ${STORES:-lap strips}; do
    r=$(env $1 timeout 120 python tools/time_config.py --config 0 --units 8 --engine cluster --store $store --reps 3 2>&1 | tail -1 | python -c 'import sys,json; d=json.loads(sys.stdin.read()); i=d["info"]; print(round(d["forward_ms"],4), round(d["adjoint_ms"],4), d["engine"], "fwd", i["cluster_ctas"], "x", i["rows_per_thread"], "adj", i["adjoint_cluster_ctas"], "x", i["adjoint_rows_per_thread"], "thr", i["threads_per_cta"], i["adjoint_threads_per_cta"], "res", i["clusters_resident"])' 2>/dev/null)
    [ -n "$r" ] && echo "$2 $store: $r" >> $O
  done
}
run "A=1" "auto"
for cs in ${CSS:-8 10 12 14 16}; do
  for rpt in ${RPTS:-2 4 5 6 7 8}; do
    run "DUFWI_CLUSTER_CS=$cs DUFWI_CLUSTER_RPT=$rpt" "cs=$cs rpt=$rpt"
  done
done
cat $O
