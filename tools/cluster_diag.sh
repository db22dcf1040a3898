#!/bin/bash
# Cluster engine diagnostics (config 0/1): co-resident clusters per forced shape
# with forward / adjoint ms, and per-warp step timing (TIMING build).
mkdir -p gpurun_out
out=gpurun_out/cluster_diag.log
: > $out
for cs in 8 10 11 12 13 14 15 16; do
  for rpt in 2 4 5 6 7 8; do
    DUFWI_CLUSTER_CS=$cs DUFWI_CLUSTER_RPT=$rpt timeout 120 python tools/time_config.py --config 0 --units 8 --engine cluster --store strips --reps 3 2>&1 | tail -1 | python -c '
import sys,json
try:
    d=json.loads(sys.stdin.read())
except Exception:
    sys.exit(0)
i=d["info"]
print("cs=%d rpt=%d fwd %.4f adj %.4f resident %d thr %d/%d" % (i["cluster_ctas"], i["rows_per_thread"], d["forward_ms"], d["adjoint_ms"], i["clusters_resident"], i["threads_per_cta"], i["adjoint_threads_per_cta"]))' >> $out
  done
done
timeout 300 python tools/ubench/phase_dbg.py > gpurun_out/phase_dbg.log 2>&1
