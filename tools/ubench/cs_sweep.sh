# Cluster shape sweep on config 1 (8 units): forward / adjoint ms and the plan's shape.
run() {
  echo "$1 $(env $1 python tools/time_config.py --config 1 --units 8 --engine cluster --store strips 2>&1 | tail -1 | python -c 'import json,sys; d=json.loads(sys.stdin.read()); i=d["info"]; print(round(d["forward_ms"],3), round(d["adjoint_ms"],3), i["cluster_ctas"], i["rows_per_thread"], i["threads_per_cta"], i["clusters_resident"])')"
}
for v in ${SWEEP:-"DUFWI_CLUSTER_CS=16" "DUFWI_CLUSTER_CS=16 DUFWI_CLUSTER_RPT=5" "DUFWI_CLUSTER_CS=10" "DUFWI_CLUSTER_CS=10 DUFWI_CLUSTER_RPT=8" "DUFWI_CLUSTER_CS=9" "X=1"}; do run "$v"; done
