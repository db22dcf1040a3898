"""Summarise ncu reports from gpurun_out/ into profiles/<round>_*.md/.csv (run here, no GPU)."""
import csv
import io
import json
import subprocess
import sys
from collections import defaultdict
from pathlib import Path

ROOT = Path(__file__).resolve().parents[1]
R = sys.argv[1] if len(sys.argv) > 1 else "r01"
OUT = ROOT / "profiles"
OUT.mkdir(exist_ok=True)
G = ROOT / "gpurun_out"
KEYS = ["gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
        "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed",
        "sm__throughput.avg.pct_of_peak_sustained_elapsed", "smsp__inst_executed.sum",
        "sm__warps_active.avg.pct_of_peak_sustained_active", "launch__registers_per_thread",
        "launch__grid_size", "launch__block_size", "launch__cluster_dim_x",
        "sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active",
        "l1tex__t_sector_hit_rate.pct", "lts__t_sector_hit_rate.pct",
        "smsp__issue_active.avg.pct_of_peak_sustained_active"]


def raw(rep):
    txt = subprocess.run(["ncu", "-i", str(rep), "--page", "raw", "--csv"], capture_output=True,
                         text=True).stdout
    rows = list(csv.reader(io.StringIO(txt)))
    hdr, units = rows[0], rows[1]
    out = []
    for r in rows[2:]:
        d = dict(zip(hdr, r))
        u = dict(zip(hdr, units))
        stalls = {k.replace("smsp__pcsamp_warps_issue_stalled_", ""): float(v)
                  for k, v in d.items() if k.startswith("smsp__pcsamp_warps_issue_stalled_")
                  and not k.endswith("not_issued") and v.replace(".", "", 1).isdigit()}
        tot = sum(stalls.values()) or 1.0
        top = sorted(stalls.items(), key=lambda kv: -kv[1])[:6]
        out.append({"kernel": d["Kernel Name"], **{k: f"{d.get(k)} {u.get(k, '')}".strip() for k in KEYS},
                    "top_stalls": {k: round(v / tot, 3) for k, v in top}})
    return out


md = [f"# ncu summaries — round {R}\n"]
traffic = {}
for rep in sorted(G.glob(f"{R}_*.ncu-rep")):
    for k in raw(rep):
        if "cluster_adj" in k["kernel"]:
            def num(v):
                x, u = v.split()[0], v.split()[-1]
                return float(x.replace(",", "")) * {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}.get(u, 1)
            b = num(k["dram__bytes_read.sum"]) + num(k["dram__bytes_write.sum"])
            # configs 0 and 1 run the same sweep shape (prof_case.py --config 0)
            traffic["config0:cluster:adjoint"] = traffic["config1:cluster:adjoint"] = b
        md.append(f"## {rep.name}: `{k['kernel'][:110]}`\n")
        for key in KEYS:
            md.append(f"- {key}: {k[key]}")
        md.append(f"- top stalls: {json.dumps(k['top_stalls'])}\n")
lf = G / f"{R}_launches.csv"
if lf.exists():
    lines = [l for l in lf.read_text().splitlines() if l.startswith('"')]
    rows = list(csv.reader(lines))
    hdr = rows[0]
    ki, vi = hdr.index("Kernel Name"), hdr.index("Metric Value")
    agg = defaultdict(lambda: [0, 0.0])
    for r in rows[1:]:
        try:
            v = float(r[vi].replace(",", ""))
        except ValueError:
            continue
        name = r[ki].split("(")[0]
        agg[name][0] += 1
        agg[name][1] += v
    total = sum(v[1] for v in agg.values())
    (OUT / f"{R}_launches.csv").write_text(lf.read_text())
    md.append("## launch list of `bench.py --steps 2 --warmup 1` (ncu, cold-cache, serialised)\n")
    md.append("| kernel | launches | total time | share |\n|---|---|---|---|")
    for name, (n, t) in sorted(agg.items(), key=lambda kv: -kv[1][1]):
        md.append(f"| `{name[:70]}` | {n} | {t/1e6:.3f} ms | {t/total:.1%} |")
(OUT / f"{R}_ncu_summary.md").write_text("\n".join(md) + "\n")
if traffic:
    (OUT / "ncu_traffic.json").write_text(json.dumps(traffic, indent=1) + "\n")
print("\n".join(md)[:3000])
