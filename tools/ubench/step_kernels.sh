#!/bin/bash
# Per-kernel times and DRAM bytes of the stepwise engine on config 4 (64 units, short nt)
mkdir -p gpurun_out
python tools/time_config.py --config ${CFG:-4} --units ${UNITS:-64} --nt 40 --reps 1 > gpurun_out/sk_plain.log 2>&1 || exit 1
ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv \
    -k regex:"vec_kernel|pipe_kernel|batch_kernel|stream_kernel|residual|reduce_groups|finalize" -s 60 -c 40 \
    python tools/time_config.py --config ${CFG:-4} --units ${UNITS:-64} --nt 40 --reps 1 > gpurun_out/sk_ncu.csv 2>/dev/null
python - <<'PY'
import csv, io, collections
txt = open("gpurun_out/sk_ncu.csv").read()
start = txt.index('"ID"')
rows = list(csv.DictReader(io.StringIO(txt[start:])))
agg = collections.defaultdict(lambda: [0, 0.0, 0.0, 0.0])
for r in rows:
    k = r["Kernel Name"].split("(")[0]
    v = float(r["Metric Value"].replace(",", ""))
    m = r["Metric Name"]
    a = agg[k]
    if m == "gpu__time_duration.sum":
        a[0] += 1; a[1] += v * {"ns": 1e-3, "nsecond": 1e-3, "us": 1.0, "usecond": 1.0, "ms": 1e3, "msecond": 1e3}[r["Metric Unit"]]
    elif m == "dram__bytes_read.sum":
        a[2] += v * {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}[r["Metric Unit"]]
    else:
        a[3] += v * {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}[r["Metric Unit"]]
for k, (n, us, rd, wr) in agg.items():
    print(f"{k:40s} n={n:3d} avg {us / n:9.1f} us  read {rd / n / 1e6:8.1f} MB  write {wr / n / 1e6:8.1f} MB  {(rd + wr) / (us * 1e-6) / 1e9:7.0f} GB/s")
PY
