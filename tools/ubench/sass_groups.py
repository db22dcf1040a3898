"""Group an ncu SASS source page by execution count (≈ code path) and sum the
stall reasons of each group: which path stalls on what."""
import csv
import io
import subprocess
import sys
from collections import Counter, defaultdict

rep = sys.argv[1]
minc = int(sys.argv[2]) if len(sys.argv) > 2 else 50000
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass"],
                     capture_output=True, text=True).stdout
lines = out.splitlines()
start = next(i for i, l in enumerate(lines) if l.startswith('"Address"'))
rows = list(csv.DictReader(io.StringIO("\n".join(lines[start:]))))
reasons = [k for k in rows[0] if k.startswith("stall_") and "Not Issued" not in k]
groups = defaultdict(lambda: {"n": 0, "stall": Counter(), "samples": 0, "ops": Counter()})
for r in rows:
    n = int(r["Instructions Executed"] or 0)
    if n < minc:
        continue
    g = groups[n]
    g["n"] += 1
    src = r["Source"].strip()
    op = src.split()[1] if src.startswith("@") else src.split()[0]
    g["ops"][op.split(".")[0]] += 1
    for k in reasons:
        v = int(r[k] or 0)
        g["stall"][k[6:]] += v
        g["samples"] += v
tot = sum(g["samples"] for g in groups.values())
for n, g in sorted(groups.items(), key=lambda kv: -kv[1]["samples"]):
    if g["samples"] < 0.01 * tot:
        continue
    top = ", ".join(f"{k} {v / max(g['samples'], 1):.0%}" for k, v in g["stall"].most_common(5))
    print(f"exec {n:8d}  instr {g['n']:4d}  samples {g['samples'] / tot:6.1%}  [{top}]")
    print("      ops:", ", ".join(f"{k} {v}" for k, v in g["ops"].most_common(8)))
